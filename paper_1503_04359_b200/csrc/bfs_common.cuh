// Device-side basics of the BFS steps: warp helpers, the frontier queue record, the
// device loop state (Ctl) and per-step records (LevelRec) with %globaltimer stamps.
// Included once, inside namespace bfsb::{anonymous}, by bfs.cu (a single translation
// unit: the kernels, device helpers and the host launch code share one file scope).
#pragma once

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTdThreads = 256;
constexpr int kTdItems = 8;
constexpr int kTdChunk = kTdThreads * kTdItems;  // arcs per CTA iteration
constexpr int kTdStage = 256;  // frontier entries of a chunk staged in shared memory (more: global search)

// counter slots: [0, 8) written by this rank's kernels, [8, 16) global (allreduced)
enum { C_NEXT = 0, C_MF = 1, C_INSP = 2, C_B2Q = 3, C_SCAN = 4, C_WORK = 5, C_TUPLES = 6, C_COORD = 7,
       C_GLOBAL = 8 };

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t ld_ca(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
    return x;
}

// A top-down frontier queue: vertex (global ID) plus its degree, read from the
// vertex's 8-byte head record when it is discovered (one sector; the degree feeds
// m_f of the next frontier).  The row begin is read only if the queue is expanded
// top-down (a TD level followed by a BU level never needs it).
struct Queue {
    int32_t* v;
    int32_t* deg;
};

__device__ __forceinline__ void queue_put(const Queue& q, unsigned long long pos, int32_t v, int32_t deg) {
    __stcs(q.v + pos, v);
    __stcs(q.deg + pos, deg);
}

// Device-resident state of the device-driven level loop (one GPU).  The
// step kernels read their sizes and buffer selectors from here when launched from
// the loop graph, and take them by value (ctl == nullptr) from the host loop.
struct Ctl {
    long long n_f, m_f, prev_nf, seen, reached, m_fc;
    long long E, nchunks;     // top-down sizes of the current step
    long long root_i;         // internal label of the root
    long long alpha, beta, n, arcs;
    int d, dir, have_queue, qsel, fsel, bu_done, returned, overflow;
    int mode, bu_from, max_levels, done;   // done: the persistent kernel's stop flag
    long long claim_min;      // top-down steps with at least this many arcs run claim-only
    int claim, front_ok;      // this step is claim-only; the front bitmap holds the frontier
    long long tile_min;       // top-down steps with at least this many arcs run tiled (< 0: no tile index)
    int tile, started;        // this step runs tiled (td_tile.cuh; implies claim); a step has begun (k_step)
    long long td_small;       // top-down steps with at most this many arcs run as one kernel (k_td_small)
};
// one record per step, filled by the step kernels (times: %globaltimer ns)
struct LevelRec {
    long long n_f, discovered, m_f, m_u, insp, scanned;
    unsigned long long ts, te, k0, k1;   // step begin / end; main kernel first block start / last block end
    int dir, pad;
};

// L2 eviction-priority hints: ld.global.nc with an L2::cache_hint policy from
// createpolicy (the policy lives in a uniform register; the .L2::evict_* qualifiers
// alone are only accepted on 256-bit loads).  The bottom-up step keeps the frontier
// bitmap resident (evict_last) against the once-read streams.
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t k;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(k));
    return k;
}
// back to normal priority after the search (the output pass then has all of L2)
__device__ __forceinline__ void l2_demote_line(const void* p) {
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint32_t ldh(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// main-kernel span: first block start / last block end into the step's record
__device__ __forceinline__ void stamp_begin(LevelRec* lrec, const Ctl* ctl) {
    if (lrec && threadIdx.x == 0) atomicMin(&lrec[ctl->d].k0, gtimer());
}
__device__ __forceinline__ void stamp_end(LevelRec* lrec, const Ctl* ctl) {
    if (lrec && threadIdx.x == 0) atomicMax(&lrec[ctl->d].k1, gtimer());
}

