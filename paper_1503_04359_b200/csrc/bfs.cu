// The hot path: level-synchronous direction-optimized BFS (
// Alg. 1; Beamer via P:16; switch rule P:151-155 read as
// DESIGN.md R2/R3/R17/R19), on one GPU or 1D-partitioned over p ranks
// (Alg. 2/3 P:119-140).
//
// Data layout in HBM on a rank that owns internal labels [lo, hi), nl = hi - lo:
//   off     int64[nl+1]   CSR offsets of owned rows    adj int32[arcs] global IDs
//   visited u32[nl/32]    1 = visited or degree 0 (initialised from the skip mask)
//   front / next u32[p*nb/32]  global frontier bitmaps; a rank writes its own slice
//   q0 / q1 int32[nl]     frontier queues of owned vertices (global IDs)
//   rec     int2[nl]      (depth, parent) recorded at discovery; k_emit writes the outputs
//   (p > 1) seen u32[n/32] remote-claim dedup, out/in int2 claim lists
//
// Kernels:
//   k_init        visited <- skip | root, root outputs, counters
//   k_td_expand   top-down step, edge-balanced: a device scan of frontier degrees
//                 gives each CTA a contiguous chunk of arcs; arcs map back to their
//                 frontier vertex by binary search in shared memory; owned targets
//                 are claimed with atomicOr on the visited word, remote targets are
//                 deduplicated in `seen` and appended as (v, parent) claims for the
//                 owner; winners stage the next queue in shared memory (one global
//                 atomicAdd per CTA chunk); m_f of the next frontier is fused.
//   k_td_merge    owner side of the push (Alg. 2): claims received from peers
//   k_bu_batch    bottom-up step: warp per 32-word batch, per-lane rows with
//                 kBuSlots in flight, warp-cooperative long rows (see below)
//   k_q2b / k_b2q frontier queue <-> bitmap on direction switches
//   k_emit        the output pass: depth/parent of every vertex written once, coalesced
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace bfsb {
namespace {

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
};
// one record per step, filled by the step kernels (times: %globaltimer ns)
struct LevelRec {
    long long n_f, discovered, m_f, m_u, insp, scanned;
    unsigned long long ts, te, k0, k1;   // step begin / end; main kernel first block start / last block end
    int dir, pad;
};

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

// root_l < 0 on ranks that do not own the root
__global__ void k_init(uint32_t* visited, const uint32_t* skip, int64_t pw, int64_t root_l, int32_t root_g,
                       int2* out, int32_t root_o, Queue q, const int2* head, unsigned long long* cnt) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < pw; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = skip[w];
        if (root_l >= 0 && w == (root_l >> 5)) x |= 1u << (root_l & 31);
        visited[w] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) cnt[i] = 0;
        if (root_l >= 0) {
            out[root_l] = make_int2(0, root_o);
            const int32_t dg = head[root_l].y;
            queue_put(q, 0, root_g, dg);
            cnt[C_NEXT] = 1;
            cnt[C_MF] = (unsigned long long)dg;
        }
    }
}

// chunk c of the top-down arc range starts inside frontier entry starts[c]
__global__ void k_td_chunk_starts(const int64_t* prefix, int64_t F, int64_t nchunks, int64_t* starts,
                                  const Ctl* ctl) {
    if (ctl) {
        F = ctl->n_f;
        nchunks = ctl->nchunks;
    }
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = c * kTdChunk;
        // largest i in [0, F) with prefix[i] <= e (prefix non-decreasing, prefix[0] = 0)
        int64_t a = 0, b = F - 1;
        while (a < b) {
            const int64_t mid = (a + b + 1) >> 1;
            if (prefix[mid] <= e) a = mid;
            else b = mid - 1;
        }
        starts[c] = a;
    }
}

struct Remote {          // p > 1 only
    uint32_t* seen;      // global bitmap: remote vertices this rank already claimed in this BFS
    int2* out;           // claims (v, parent) for peer q at out[q * cap ...]
    unsigned long long* out_cnt;  // [p]
    int64_t cap;
    int64_t nb;          // partition block size
};

// Top-down step (Alg. 1 TD branch).  Each CTA iteration handles one chunk of
// kTdChunk consecutive arcs in three phases so that the dependent loads of the
// kTdItems arcs of a thread overlap:
//   A  locate (binary search in shared memory) and load all targets v
//   B  probe the visited words, then atomicOr-claim the unvisited ones
//   C  winners write depth/parent and stage v in shared memory; one atomicAdd per
//      CTA chunk on the global queue tail, then a coalesced copy of the stage.
template <bool kMulti>
__global__ void __launch_bounds__(kTdThreads, 4)
k_td_expand(const Queue q_in, const int64_t* __restrict__ prefix, const int64_t* __restrict__ starts,
            int64_t F, int64_t E, const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
            uint32_t* __restrict__ visited, int2* __restrict__ out, const int32_t* __restrict__ pmap,
            const Queue qnext_in, const int2* __restrict__ head, unsigned long long* __restrict__ cnt,
            int32_t next_level, int64_t lo, int64_t hi, Remote rm, const Ctl* ctl, LevelRec* lrec) {
    __shared__ int64_t s_pre[kTdStage + 2];
    __shared__ int64_t s_beg[kTdStage + 1];
    __shared__ int32_t s_u[kTdStage + 1];
    __shared__ int32_t s_q[kTdChunk];
    __shared__ int32_t s_qd[kTdChunk];
    __shared__ int s_qn;
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0;
    Queue qc = q_in, qnext = qnext_in;
    if (ctl) {   // device-driven loop: sizes and queue selector from the loop state
        F = ctl->n_f;
        E = ctl->E;
        next_level = ctl->d + 1;
        if (ctl->qsel) { qc = qnext_in; qnext = q_in; }
        stamp_begin(lrec, ctl);
    }
    const Queue q = qc;
    const int64_t nchunks = (E + kTdChunk - 1) / kTdChunk;
    if (threadIdx.x == 0) s_qn = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const int64_t e0 = c * kTdChunk;
        const int64_t e1 = min(E, e0 + kTdChunk);
        const int64_t i0 = starts[c];
        const int64_t i1 = (c + 1 < nchunks) ? starts[c + 1] : F - 1;
        const int64_t cntv = min(i1 - i0 + 1, F - i0);
        const bool fits = cntv <= kTdStage;
        if (fits) {
            for (int k = threadIdx.x; k <= cntv; k += kTdThreads) {
                s_pre[k] = prefix[i0 + k];
                if (k < cntv) {
                    const int32_t uu = q.v[i0 + k];
                    s_u[k] = uu;
                    s_beg[k] = off[uu - lo];
                }
            }
        }
        __syncthreads();
        int32_t v[kTdItems], u[kTdItems];
        // A: targets.  Thread t takes kTdItems CONSECUTIVE arcs: one binary search for
        // the first, then a linear advance; the arcs of a row are sorted, so a thread's
        // targets are close together and its visited probes mostly share a sector (L1).
        {
            const int64_t et = e0 + (int64_t)threadIdx.x * kTdItems;
            int64_t a = 0;
            if (et < e1) {
                if (fits) {
                    int lo_ = 0, hi_ = (int)cntv - 1;
                    while (lo_ < hi_) {
                        const int mid = (lo_ + hi_ + 1) >> 1;
                        if (s_pre[mid] <= et) lo_ = mid;
                        else hi_ = mid - 1;
                    }
                    a = lo_;
                } else {
                    int64_t lo_ = i0, hi_ = F - 1;
                    while (lo_ < hi_) {
                        const int64_t mid = (lo_ + hi_ + 1) >> 1;
                        if (prefix[mid] <= et) lo_ = mid;
                        else hi_ = mid - 1;
                    }
                    a = lo_;
                }
            }
            int64_t pre = 0, nxt = 0, beg = 0;
            int32_t uu = 0;
            if (et < e1) {
                if (fits) {
                    pre = s_pre[a]; nxt = s_pre[a + 1]; beg = s_beg[a]; uu = s_u[a];
                } else {
                    pre = prefix[a]; nxt = prefix[a + 1]; uu = q.v[a]; beg = off[uu - lo];
                }
            }
#pragma unroll
            for (int j = 0; j < kTdItems; ++j) {
                const int64_t e = et + j;
                v[j] = -1;
                u[j] = 0;
                if (e < e1) {
                    while (e >= nxt) {   // the next frontier vertex (degree >= 1: one step each)
                        ++a;
                        if (fits) {
                            pre = s_pre[a]; nxt = s_pre[a + 1]; beg = s_beg[a]; uu = s_u[a];
                        } else {
                            pre = prefix[a]; nxt = prefix[a + 1]; uu = q.v[a]; beg = off[uu - lo];
                        }
                    }
                    u[j] = uu;
                    v[j] = __ldg(adj + beg + (e - pre));
                }
            }
        }
        // B: probe, then claim.  Owned targets in `visited`, remote ones in `seen`.
        bool own[kTdItems];
        uint32_t* wp[kTdItems];
        uint32_t wv[kTdItems];
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            own[j] = !kMulti || (v[j] >= lo && v[j] < hi);
            wp[j] = nullptr;
            if (v[j] >= 0) wp[j] = own[j] ? visited + ((v[j] - lo) >> 5) : rm.seen + (v[j] >> 5);
            // L1-cached probe: visited/seen bits only ever go 0 -> 1 during a step, so a
            // stale word can only send a claim to the atomicOr, which decides correctly
            wv[j] = wp[j] ? ld_ca(wp[j]) : kFull;
        }
        bool win[kTdItems];
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            const uint32_t bit = 1u << (v[j] & 31);
            win[j] = false;
            if (wp[j] && !(wv[j] & bit)) win[j] = !(atomicOr(wp[j], bit) & bit);
        }
        // C: outputs + staged queue append; remote claims go to the owner's list
#pragma unroll
        // winners' degrees (8-byte head records) and parent labels: all loads issued
        // before any is consumed, so their latencies overlap instead of adding up
        int32_t dgs[kTdItems], par[kTdItems];
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            // one-shot random accesses stream through L2 with evict-first so the
            // visited words the probes and claims hit stay resident
            dgs[j] = (win[j] && own[j]) ? __ldcs(head + (v[j] - lo)).y : 0;
            par[j] = (win[j] && own[j] && pmap) ? __ldg(pmap + u[j]) : u[j];
        }
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            const bool lw = win[j] && own[j];
            const unsigned m = __ballot_sync(kFull, lw);
            if (m) {
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&s_qn, __popc(m));
                base = __shfl_sync(kFull, base, leader);
                if (lw) {
                    const int64_t vl = v[j] - lo;
                    const int slot = base + __popc(m & lanemask_lt());
                    s_q[slot] = v[j];
                    s_qd[slot] = dgs[j];
                    __stcs(out + vl, make_int2(next_level, par[j]));
                    my_mf += (unsigned long long)dgs[j];
                }
            }
            if (kMulti) {
                const bool rw = win[j] && !own[j];
                if (__ballot_sync(kFull, rw)) {
                    const int owner = rw ? (int)(v[j] / rm.nb) : -1;
                    const unsigned peers = __match_any_sync(kFull, owner);
                    const int leader = __ffs(peers) - 1;
                    unsigned long long pos = 0;
                    if (rw && lane == leader) pos = atomicAdd(rm.out_cnt + owner, (unsigned long long)__popc(peers));
                    pos = __shfl_sync(kFull, pos, leader);
                    if (rw) rm.out[(int64_t)owner * rm.cap + (int64_t)pos + __popc(peers & lanemask_lt())] = make_int2(v[j], u[j]);
                }
            }
        }
        __syncthreads();
        const int qn = s_qn;
        if (threadIdx.x == 0 && qn) s_base = atomicAdd(cnt + C_NEXT, (unsigned long long)qn);
        __syncthreads();
        for (int k = threadIdx.x; k < qn; k += kTdThreads) queue_put(qnext, s_base + k, s_q[k], s_qd[k]);
        __syncthreads();
        if (threadIdx.x == 0) s_qn = 0;
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
    if (ctl && lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}

// Owner side of the top-down push: claims (v, parent) received from peers are
// claimed exactly like local top-down targets (Alg. 2 "(local) ==> (remote)").
__global__ void k_td_merge(const int2* __restrict__ in, int64_t R, const int2* __restrict__ head,
                           uint32_t* __restrict__ visited, int2* __restrict__ out,
                           const Queue qnext, unsigned long long* __restrict__ cnt, int32_t next_level,
                           int64_t lo) {
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < R;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b0 + lane;
        bool win = false;
        int2 c = make_int2(0, 0);
        if (i < R) {
            c = in[i];
            const uint32_t bit = 1u << (c.x & 31);
            uint32_t* wp = visited + ((c.x - lo) >> 5);
            if (!(__ldcg(wp) & bit)) win = !(atomicOr(wp, bit) & bit);
        }
        const unsigned m = __ballot_sync(kFull, win);
        if (m) {
            const int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(cnt + C_NEXT, (unsigned long long)__popc(m));
            base = __shfl_sync(kFull, base, leader);
            if (win) {
                const int64_t vl = c.x - lo;
                const int32_t dg = __ldg(head + vl).y;
                queue_put(qnext, base + __popc(m & lanemask_lt()), c.x, dg);
                out[vl] = make_int2(next_level, c.y);
                my_mf += (unsigned long long)dg;
            }
        }
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
}

__device__ __forceinline__ bool in_front(const uint32_t* __restrict__ front, int32_t u) {
    return (__ldg(front + (u >> 5)) >> (u & 31)) & 1u;
}

constexpr int kBuLongDefault = 64;   // B200 sweep: 8 -> 64 is +1%; the warp path stays for hub rows
// lane-serial probes before a row is handed to the whole warp (BFS_BU_LONG: tuning only)
static int bu_long_setting() {
    const char* e = getenv("BFS_BU_LONG");
    return e ? std::max(1, atoi(e)) : kBuLongDefault;
}

// unvisited vertices of a 1024-vertex batch from which it is probed densely
// (BFS_BU_DENSE: tuning only)
static int bu_dense_setting() {
    const char* e = getenv("BFS_BU_DENSE");
    return e ? atoi(e) : 384;
}

// Bottom-up step (Alg. 1 BU branch, `break for` P:107, R1).
// A warp takes a batch of 32 visited words (1024 owned vertices) at a time from a
// global work counter:
//   1. one coalesced 128-byte load of the 32 visited words; an all-visited batch
//      costs only that load and a coalesced store of 32 zero next-words;
//   2. the unvisited vertices of the batch are compacted into a per-warp list in
//      shared memory (popc + warp prefix sum);
//   3. every lane keeps kBuSlots rows in flight and advances all of them each
//      round (independent adj[j] loads, then independent frontier-bit probes),
//      refilling a slot from the list as soon as its row resolves -- this hides
//      the off -> adj -> frontier dependent-load chain behind kBuSlots-way MLP
//      (the paper's "virtual warp" of one lane per vertex);
//   4. a row still unresolved after kBuLong lane-serial probes moves to a per-warp
//      list and is finished by the whole warp, 32 arcs per ballot (the lowest
//      hitting lane is the first frontier neighbour in row order);
//   5. the 32 next words are assembled in shared memory and stored coalesced.
constexpr int kBuWarps = 8;
constexpr int kBuCtas = 4;     // resident CTAs per SM (launch bound and grid; 5 spills: -10%)
constexpr int kBuSlots = 3;
constexpr int kBuIlp = 8;
constexpr int kBuVec = 4;      // arcs a slot reads (one aligned vector load) and probes per round
constexpr int kLongCap = 16;   // small: shared memory left to L1 matters more (B200-measured)

__global__ void __launch_bounds__(kBuWarps * 32, kBuCtas)
k_bu_batch(const int64_t* __restrict__ off, const int2* __restrict__ head, const int32_t* __restrict__ adj,
           uint32_t* __restrict__ visited,
           const uint32_t* __restrict__ front_in, uint32_t* __restrict__ next_in, int2* __restrict__ out,
           const int32_t* __restrict__ pmap, const int32_t* __restrict__ hpar, int64_t words, int64_t lo,
           int32_t next_level,
           unsigned long long* __restrict__ cnt, int grab, int blong, int dense_u, const Ctl* ctl,
           LevelRec* lrec) {
    __shared__ uint16_t s_list[kBuWarps][1024];
    __shared__ uint32_t s_nb[kBuWarps][32];
    __shared__ int64_t s_lj[kBuWarps][kLongCap];
    __shared__ int64_t s_le[kBuWarps][kLongCap];
    __shared__ int32_t s_lv[kBuWarps][kLongCap];
    __shared__ int32_t s_ld[kBuWarps][kLongCap];
    __shared__ int s_lcount[kBuWarps];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t* front = front_in;
    uint32_t* next = next_in;
    if (ctl) {   // device-driven loop: the bitmap pair flips every bottom-up step
        next_level = ctl->d + 1;
        if (ctl->fsel) {
            front = next_in;
            next = const_cast<uint32_t*>(front_in);
        }
        stamp_begin(lrec, ctl);
    }
    uint16_t* list = s_list[wid];
    uint32_t* nbw = s_nb[wid];
    const int64_t wbase = lo >> 5;
    const int64_t nbatches = (words + 31) / 32;
    unsigned long long my_nf = 0, my_mf = 0, my_insp = 0, my_scan = 0;
    // batches are claimed `grab` at a time from the global counter (one atomic per
    // grab: a sparse level is otherwise bound by that single address)
    long long bt = 0, bt_end = 0;
    for (;; ++bt) {
        if (bt >= bt_end) {
            long long g0 = 0;
            if (lane == 0) g0 = (long long)atomicAdd(cnt + C_WORK, (unsigned long long)grab);
            g0 = __shfl_sync(kFull, g0, 0);
            if (g0 >= nbatches) break;
            bt = g0;
            bt_end = min(g0 + (long long)grab, (long long)nbatches);
        }
        const int64_t w = bt * 32 + lane;
        const uint32_t vis = w < words ? visited[w] : kFull;
        const uint32_t un = ~vis;
        if (!__ballot_sync(kFull, un != 0u)) {
            if (w < words) next[wbase + w] = 0u;
            continue;
        }
        const int c = __popc(un);
        const int U = __reduce_add_sync(kFull, c);
        nbw[lane] = 0u;
        if (lane == 0) s_lcount[wid] = 0;
        my_scan += (unsigned long long)c;
        const int64_t vbase = bt * 1024;
        int M = 0;  // warp-uniform count of rows that missed their first probe
        if (U >= dense_u) {
            // 3a'. dense batch (most vertices unvisited, the first bottom-up levels):
            //     lane j takes vertex j of every word, so head records load coalesced
            //     and the next word of the batch is one ballot -- no list to build and
            //     no shared-memory atomics.  Misses go to the list for 3b.
            uint32_t mynext = 0u;
            for (int k0 = 0; k0 < 32; k0 += kBuIlp) {
                int32_t sv[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) {
                    const uint32_t vk = __shfl_sync(kFull, vis, k0 + j);
                    sv[j] = ((vk >> lane) & 1u) ? -1 : (k0 + j) * 32 + lane;
                }
                int2 hd[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) hd[j] = sv[j] >= 0 ? __ldg(head + vbase + sv[j]) : make_int2(-1, 0);
                int32_t po[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) po[j] = (hpar && sv[j] >= 0) ? __ldg(hpar + vbase + sv[j]) : hd[j].x;
                bool hit[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) hit[j] = hd[j].y > 0 && in_front(front, hd[j].x);
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) {
                    if (hd[j].y > 0) my_insp += 1;
                    if (hit[j]) {
                        __stcs(out + vbase + sv[j], make_int2(next_level, po[j]));
                        my_mf += (unsigned long long)hd[j].y;
                    }
                    const unsigned hm = __ballot_sync(kFull, hit[j]);
                    if (lane == k0 + j) mynext = hm;
                    const bool miss = !hit[j] && hd[j].y > 1;
                    const unsigned mm = __ballot_sync(kFull, miss);
                    if (miss) list[M + __popc(mm & lanemask_lt())] = (uint16_t)sv[j];
                    M += __popc(mm);
                }
            }
            nbw[lane] = mynext;
        } else {
            // 2. compact unvisited local indices (0..1023) into the per-warp list
            int inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(kFull, inc, d);
                if (lane >= d) inc += y;
            }
            {
                uint32_t bits = un;
                int p = inc - c;
                while (bits) {
                    const int k = __ffs(bits) - 1;
                    bits &= bits - 1;
                    list[p++] = (uint16_t)(lane * 32 + k);
                }
            }
            __syncwarp();
            // 3a. first probes: every unvisited vertex tries the first neighbour of its
            //     row from the dense head record (8 bytes, coalesced along the list);
            //     kBuIlp records per lane are loaded before any is probed.  With rows in
            //     canonical order this resolves most vertices.  Vertices that miss
            //     and have more neighbours are compacted in place at the front of the list.
            for (int t0 = 0; t0 < U; t0 += 32 * kBuIlp) {
                int32_t sv[kBuIlp];
                int2 hd[kBuIlp];
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) {
                    const int idx = t0 + k * 32 + lane;
                    sv[k] = idx < U ? (int32_t)list[idx] : -1;
                }
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) hd[k] = sv[k] >= 0 ? __ldg(head + vbase + sv[k]) : make_int2(-1, 0);
                // reindexed graphs: the first neighbour's ORIGINAL label comes from a dense
                // per-vertex array read beside the head record (coalesced), not from a
                // random ilabel[] lookup after the probe
                int32_t po[kBuIlp];
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) po[k] = (hpar && sv[k] >= 0) ? __ldg(hpar + vbase + sv[k]) : hd[k].x;
                bool hit[kBuIlp];
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) hit[k] = hd[k].y > 0 && in_front(front, hd[k].x);
                __syncwarp();  // all lanes hold their entries of this block before misses overwrite it
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) {
                    if (hd[k].y > 0) my_insp += 1;
                    if (hit[k]) {
                        __stcs(out + vbase + sv[k], make_int2(next_level, po[k]));
                        atomicOr(nbw + (sv[k] >> 5), 1u << (sv[k] & 31));
                        my_mf += (unsigned long long)hd[k].y;
                    }
                    const bool miss = !hit[k] && hd[k].y > 1;
                    const unsigned mm = __ballot_sync(kFull, miss);
                    if (miss) list[M + __popc(mm & lanemask_lt())] = (uint16_t)sv[k];
                    M += __popc(mm);
                }
            }
        }
        __syncwarp();
        // 3b. rows that missed: each lane keeps kBuSlots rows in flight from position 1
        //     on and advances all of them each round (independent adj[j] loads, then
        //     independent frontier probes), refilling a slot as soon as its row
        //     resolves (the paper's "virtual warp" of one lane per vertex).
        {
            int t = lane;
            int32_t sv[kBuSlots], sd[kBuSlots];
            int64_t sj[kBuSlots], se[kBuSlots];
            bool sa[kBuSlots];
#pragma unroll
            for (int s = 0; s < kBuSlots; ++s) {
                sa[s] = false;
                sv[s] = sd[s] = 0;
                sj[s] = se[s] = 0;
                if (t < M) {
                    sv[s] = list[t];
                    t += 32;
                    sd[s] = __ldcs(head + vbase + sv[s]).y;
                    sj[s] = __ldcs(off + vbase + sv[s]) + 1;
                    se[s] = sj[s] - 1 + sd[s];
                    sa[s] = true;
                }
            }
            for (;;) {
                bool any = false;
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) any |= sa[s];
                if (!__any_sync(kFull, any)) break;
                // each slot reads the aligned kBuVec-arc group holding its next arc with
                // one vector load and probes every arc of it that lies in the row at once
                int32_t a[kBuSlots][kBuVec];
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) {
                    const int64_t b = sj[s] & ~(int64_t)(kBuVec - 1);
                    if (kBuVec == 4) {
                        const int4 x = sa[s] ? __ldg(reinterpret_cast<const int4*>(adj + b)) : make_int4(0, 0, 0, 0);
                        a[s][0] = x.x; a[s][1] = x.y; a[s][2 % kBuVec] = x.z; a[s][3 % kBuVec] = x.w;
                    } else if (kBuVec == 2) {
                        const int2 x = sa[s] ? __ldg(reinterpret_cast<const int2*>(adj + b)) : make_int2(0, 0);
                        a[s][0] = x.x; a[s][1 % kBuVec] = x.y;
                    } else {
                        a[s][0] = sa[s] ? __ldg(adj + b) : 0;
                    }
                }
                bool h[kBuSlots][kBuVec];
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) {
                    const int64_t b = sj[s] & ~(int64_t)(kBuVec - 1);
#pragma unroll
                    for (int k = 0; k < kBuVec; ++k)
                        h[s][k] = sa[s] && b + k >= sj[s] && b + k < se[s] && in_front(front, a[s][k]);
                }
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) {
                    if (sa[s]) {
                        const int64_t b = sj[s] & ~(int64_t)(kBuVec - 1);
                        int kh = -1;
                        int32_t hu = 0;
#pragma unroll
                        for (int k = kBuVec - 1; k >= 0; --k)
                            if (h[s][k]) { kh = k; hu = a[s][k]; }
                        const int64_t nj = min(se[s], b + kBuVec);
                        if (kh >= 0) {
                            my_insp += (unsigned long long)(b + kh - sj[s] + 1);
                            __stcs(out + vbase + sv[s], make_int2(next_level, pmap ? pmap[hu] : hu));
                            atomicOr(nbw + (sv[s] >> 5), 1u << (sv[s] & 31));
                            my_mf += (unsigned long long)sd[s];
                            sa[s] = false;
                        } else if (my_insp += (unsigned long long)(nj - sj[s]), (sj[s] = nj) == se[s]) {
                            sa[s] = false;  // exhausted: no frontier neighbour this level
                        } else if (sd[s] - (se[s] - sj[s]) >= blong) {
                            const int idx = atomicAdd(s_lcount + wid, 1);
                            if (idx < kLongCap) {  // hand the rest of the row to the warp
                                s_lv[wid][idx] = sv[s];
                                s_lj[wid][idx] = sj[s];
                                s_le[wid][idx] = se[s];
                                s_ld[wid][idx] = sd[s];
                                sa[s] = false;
                            }
                        }
                    }
                    if (!sa[s] && t < M) {
                        sv[s] = list[t];
                        t += 32;
                        sd[s] = __ldcs(head + vbase + sv[s]).y;
                        sj[s] = __ldcs(off + vbase + sv[s]) + 1;
                        se[s] = sj[s] - 1 + sd[s];
                        sa[s] = true;
                    }
                }
            }
        }
        __syncwarp();
        // 4. long rows: whole warp, 32 arcs per ballot
        const int L = min(s_lcount[wid], kLongCap);
        for (int x = 0; x < L; ++x) {
            const int32_t lv = s_lv[wid][x];
            const int64_t jb = s_lj[wid][x], je = s_le[wid][x];
            int64_t hit = -1;
            int32_t hu = 0;
            for (int64_t j0 = jb; j0 < je; j0 += 32) {
                const int64_t jj = j0 + lane;
                int32_t uu = 0;
                bool hh = false;
                if (jj < je) {
                    uu = __ldg(adj + jj);
                    hh = in_front(front, uu);
                }
                const unsigned hm = __ballot_sync(kFull, hh);
                if (hm) {
                    const int first = __ffs(hm) - 1;
                    hit = j0 + first;
                    hu = __shfl_sync(kFull, uu, first);
                    break;
                }
            }
            if (lane == 0) {
                if (hit >= 0) {
                    out[vbase + lv] = make_int2(next_level, pmap ? pmap[hu] : hu);
                    nbw[lv >> 5] |= 1u << (lv & 31);
                    my_mf += (unsigned long long)s_ld[wid][x];
                    my_insp += (unsigned long long)(hit - jb + 1);
                } else {
                    my_insp += (unsigned long long)(je - jb);
                }
            }
        }
        __syncwarp();
        // 5. coalesced next / visited words
        if (w < words) {
            const uint32_t nb = nbw[lane];
            next[wbase + w] = nb;
            if (nb) visited[w] = vis | nb;
            my_nf += (unsigned long long)__popc(nb);
        }
        __syncwarp();
    }
    my_nf = warp_sum_u64(my_nf);
    my_mf = warp_sum_u64(my_mf);
    my_insp = warp_sum_u64(my_insp);
    my_scan = warp_sum_u64(my_scan);
    if (lane == 0) {
        if (my_nf) atomicAdd(cnt + C_NEXT, my_nf);
        if (my_mf) atomicAdd(cnt + C_MF, my_mf);
        if (my_insp) atomicAdd(cnt + C_INSP, my_insp);
        if (my_scan) atomicAdd(cnt + C_SCAN, my_scan);
    }
    if (ctl && lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}

// queue -> bitmap (the owned slice of front is cleared beforehand)
__device__ __forceinline__ void q2b_body(const int32_t* __restrict__ q, int64_t F, uint32_t* __restrict__ front) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = q[i];
        atomicOr(front + (v >> 5), 1u << (v & 31));
    }
}
__global__ void k_q2b(const int32_t* __restrict__ q, int64_t F, uint32_t* __restrict__ front) { q2b_body(q, F, front); }

// owned slice of a bitmap -> queue of global IDs (with degree)
__device__ __forceinline__ void b2q_body(const uint32_t* __restrict__ bm, int64_t words, int64_t lo,
                                         const int2* __restrict__ head, const Queue q,
                                         unsigned long long* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t wbase = lo >> 5;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < words;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = b0 + lane;
        uint32_t bits = w < words ? bm[wbase + w] : 0u;
        const int c = __popc(bits);
        int inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += y;
        }
        const int total = __shfl_sync(kFull, inc, 31);
        unsigned long long base = 0;
        if (lane == 31 && total) base = atomicAdd(cnt + C_B2Q, (unsigned long long)total);
        base = __shfl_sync(kFull, base, 31);
        unsigned long long pos = base + (unsigned long long)(inc - c);
        while (bits) {
            const int k = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t vl = w * 32 + k;
            queue_put(q, pos++, (int32_t)(lo + vl), __ldg(head + vl).y);
        }
    }
}

__global__ void k_b2q(const uint32_t* __restrict__ bm, int64_t words, int64_t lo, const int2* __restrict__ head,
                      const Queue q, unsigned long long* __restrict__ cnt) {
    b2q_body(bm, words, lo, head, q, cnt);
}

// Output pass (the only writer of the caller's arrays): every entry of depth and
// parent is written exactly once, in order, with full coalesced lines.  During
// the traversal the steps record (depth, parent) of each discovered vertex as one
// 8-byte `out` record in internal order; here reached vertices copy their record
// and unreached ones get -1.
//   one GPU / p ranks, labels unchanged: v = internal = original (owned slice)
//   degree reindex: v runs over ORIGINAL labels, iv = label[v] gathers the record;
//   isolated vertices sit at the tail of the internal order, so they skip the gather.
// n_active: internal labels >= n_active are isolated (degree reindex puts them last)
// and need neither the visited lookup nor the record gather.  Everything except the
// visited bitmap is touched once, so it streams with evict-first hints and the
// bitmap stays in L2 for the random lookups.
__global__ void k_emit(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                       const int2* __restrict__ rec, int64_t nl, int64_t root_l, int32_t* __restrict__ depth,
                       int32_t* __restrict__ parent, const Ctl* ctl) {
    if (ctl) root_l = ctl->root_i;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = v >> 5;
        const uint32_t r = visited[w] & ~skip[w];
        int2 o = make_int2(-1, -1);
        if (((r >> (v & 31)) & 1u) || v == root_l) o = rec[v];
        if (depth) depth[v] = o.x;
        if (parent) parent[v] = o.y;
    }
}

// Degree-reindexed variant: v runs over ORIGINAL labels and gathers the record of
// iv = label[v].  Internal labels >= n_active are isolated (the reindex puts them
// last) and need no gather unless one is the root.  Labels and outputs are touched
// once and stream with evict-first hints.
__global__ void k_emit_perm(const int2* __restrict__ rec, const int32_t* __restrict__ label, int64_t n,
                            int64_t n_active, int64_t root_l, int32_t* __restrict__ depth,
                            int32_t* __restrict__ parent, const Ctl* ctl) {
    if (ctl) root_l = ctl->root_i;
    // kEmitV original vertices per thread: 16-byte label loads, then one record
    // gather per non-isolated vertex (k_mark_unreached has reset the records of the
    // unreached ones).  Same-degree vertices keep their original order in the
    // reindex (degree desc, ID asc), so the gathers form one ascending stream per
    // degree value.
    constexpr int kEmitV = 8;
    // a warp owns a tile of 32 * kEmitV consecutive vertices; part h of the tile is
    // 128 vertices, lane i holding vertices 4i..4i+3 of it, so every 16-byte label
    // load and output store of a warp instruction covers 512 contiguous bytes
    const bool vec = ((reinterpret_cast<uintptr_t>(depth) | reinterpret_cast<uintptr_t>(parent)) & 15) == 0 &&
                     depth && parent;
    const int lane = threadIdx.x & 31;
    const int64_t tiles = (n + 32 * kEmitV - 1) / (32 * kEmitV);
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < tiles; t += nwarps) {
        const int64_t t0 = t * 32 * kEmitV;
        const bool full = t0 + 32 * kEmitV <= n;
        int32_t iv[kEmitV];
#pragma unroll
        for (int h = 0; h < kEmitV / 4; ++h) {
            const int64_t v0 = t0 + h * 128 + lane * 4;
            if (full) {
                const int4 l4 = __ldcs(reinterpret_cast<const int4*>(label + v0));
                iv[4 * h] = l4.x; iv[4 * h + 1] = l4.y; iv[4 * h + 2] = l4.z; iv[4 * h + 3] = l4.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) iv[4 * h + j] = v0 + j < n ? label[v0 + j] : -1;
            }
        }
        // records of unreached active vertices were reset by k_mark_unreached, so the
        // record alone decides: no visited lookup
        int2 o[kEmitV];
#pragma unroll
        for (int k = 0; k < kEmitV; ++k) {
            const bool act = iv[k] >= 0 && (iv[k] < n_active || iv[k] == root_l);
            o[k] = act ? __ldg(rec + iv[k]) : make_int2(-1, -1);
        }
#pragma unroll
        for (int h = 0; h < kEmitV / 4; ++h) {
            const int64_t v0 = t0 + h * 128 + lane * 4;
            if (vec && full) {
                __stcs(reinterpret_cast<int4*>(depth + v0),
                       make_int4(o[4 * h].x, o[4 * h + 1].x, o[4 * h + 2].x, o[4 * h + 3].x));
                __stcs(reinterpret_cast<int4*>(parent + v0),
                       make_int4(o[4 * h].y, o[4 * h + 1].y, o[4 * h + 2].y, o[4 * h + 3].y));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (v0 + j >= n) break;
                    if (depth) depth[v0 + j] = o[4 * h + j].x;
                    if (parent) parent[v0 + j] = o[4 * h + j].y;
                }
            }
        }
    }
}

// rec <- (-1, -1) for every vertex of [0, nbits) with degree > 0 that this search did
// not reach (a few per search in a Kronecker graph: one coalesced pass over the
// bitmaps, scattered writes for the unreached only), so that the reindexed output
// pass can take every active vertex's record as is
__global__ void k_mark_unreached(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                                 int64_t nbits, int2* __restrict__ rec) {
    const int64_t words = (nbits + 31) / 32;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = ~__ldcs(visited + w) & ~__ldcs(skip + w);
        if (w == words - 1 && (nbits & 31)) x &= (1u << (nbits & 31)) - 1u;
        while (x) {
            const int k = __ffs(x) - 1;
            x &= x - 1;
            rec[w * 32 + k] = make_int2(-1, -1);
        }
    }
}

// TEPS numerator: sum of raw degrees over reached owned vertices
__global__ void k_component_degree(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                                   const int32_t* __restrict__ deg_raw, int64_t nl, int64_t root_l,
                                   unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = v >> 5;
        const uint32_t r = visited[w] & ~skip[w];
        if (((r >> (v & 31)) & 1u) || v == root_l) s += (unsigned long long)deg_raw[v];
    }
    s = warp_sum_u64(s);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// non-self-loop arc count of owned candidate roots (internal labels), one warp per
// candidate; candidates outside [lo, hi) or negative contribute 0
__global__ void k_nonloop_degree(const int32_t* __restrict__ cand, int64_t k, const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ adj, int64_t lo, int64_t hi, int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = gw; t < k; t += nw) {
        const int32_t r = cand[t];
        int64_t c = 0;
        if (r >= lo && r < hi) {
            const int64_t b = off[r - lo], e = off[r - lo + 1];
            for (int64_t j = b + lane; j < e; j += 32) c += adj[j] != r;
        }
        for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
        if (lane == 0) out[t] = c;
    }
}

__global__ void k_gather_labels(const int32_t* __restrict__ label, const int32_t* __restrict__ in, int64_t k,
                                int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] < 0 ? -1 : label[in[i]];
}

// ============================================================ device-driven level loop
// (SURVEY f3).  On one GPU the whole level loop is one CUDA graph: a WHILE node
// whose body is k_step_begin (the alpha/beta decision, on the device) -> IF(top-down)
// {k_td_prep -> k_scan_dev -> k_td_chunk_starts -> k_td_expand} and IF(bottom-up)
// {k_bu_prep -> k_q2b_dev -> k_bu_batch} -> k_step_end (roll the counters, record
// the step, continue while the frontier is non-empty).  The host launches it once
// per search and synchronises once, instead of once per level.

// init on the device: the root's internal label, visited <- skip | root, root
// record, the first queue, the loop state (policy included)
__global__ void k_init_dev(uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip, int64_t pw,
                           int64_t root, const int32_t* __restrict__ label, int2* __restrict__ out, Queue q,
                           const int2* __restrict__ head, unsigned long long* __restrict__ cnt, Ctl* ctl,
                           bfs_policy pol, int64_t n, int64_t arcs, int max_levels) {
    const int64_t ri = label ? (int64_t)__ldg(label + root) : root;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < pw; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = skip[w];
        if (w == (ri >> 5)) x |= 1u << (ri & 31);
        visited[w] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) cnt[i] = 0;
        out[ri] = make_int2(0, (int32_t)root);
        const int32_t dg = head[ri].y;
        queue_put(q, 0, (int32_t)ri, dg);
        Ctl c{};
        c.n_f = 1;
        c.m_f = c.m_fc = dg;
        c.root_i = ri;
        c.alpha = pol.alpha;
        c.beta = pol.beta;
        c.n = n;
        c.arcs = arcs;
        c.have_queue = 1;
        c.mode = pol.mode;
        c.bu_from = pol.bu_from_level;
        c.max_levels = max_levels;
        *ctl = c;
    }
}

// the step's bookkeeping and direction (the host loop's rule, verbatim); returns m_u(d)
__device__ __forceinline__ long long step_decide(Ctl& c) {
    c.reached += c.n_f;
    c.seen += c.m_f;
    const long long m_u = c.arcs - c.seen;
    switch (c.mode) {
        case 1: c.dir = 0; break;
        case 2: c.dir = c.d >= c.bu_from ? 1 : 0; break;
        case 3:
            if (c.dir == 0) {
                if (!c.returned && c.m_fc * 10000 >= c.alpha * c.arcs) c.dir = 1;
            } else if (c.bu_done >= c.beta) {
                c.dir = 0;
                c.returned = 1;
            }
            if (c.dir == 1) ++c.bu_done;
            break;
        default:
            if (c.dir == 0) {
                if (c.m_f * c.alpha > m_u) c.dir = 1;
            } else {
                if (c.n_f * c.beta < c.n && c.n_f < c.prev_nf) c.dir = 0;
            }
    }
    return m_u;
}

// the step's record and the roll of the counters into the loop state (k_step_end and
// the persistent kernel); returns whether the search continues
__device__ __forceinline__ bool step_finish(Ctl& c, LevelRec& r, const unsigned long long* cnt) {
    const long long next = (long long)cnt[C_NEXT], mf = (long long)cnt[C_MF];
    r.discovered = next;
    r.insp = c.dir == 0 ? c.m_f : (long long)cnt[C_INSP];
    r.scanned = c.dir == 0 ? c.n_f : (long long)cnt[C_SCAN];
    r.te = gtimer();
    if (c.dir == 0) {
        c.qsel ^= 1;
        c.have_queue = 1;
    } else {
        c.fsel ^= 1;
        c.have_queue = 0;
    }
    c.prev_nf = c.n_f;
    c.n_f = next;
    c.m_f = c.m_fc = mf;
    c.d += 1;
    bool cont = next > 0;
    if (cont && c.d >= c.max_levels) {
        c.overflow = 1;
        cont = false;
    }
    return cont;
}

__global__ void k_step_begin(Ctl* ctl, LevelRec* lrec, unsigned long long* cnt, cudaGraphConditionalHandle h_td,
                             cudaGraphConditionalHandle h_bu) {
    Ctl c = *ctl;
    const long long t = gtimer();
    const long long m_u = step_decide(c);
    c.E = c.m_f;
    c.nchunks = (c.E + kTdChunk - 1) / kTdChunk;
    LevelRec r{};
    r.n_f = c.n_f;
    r.m_f = c.m_f;
    r.m_u = m_u;
    r.dir = c.dir;
    r.ts = t;
    r.k0 = ~0ull;
    lrec[c.d] = r;
    for (int i = 0; i < 8; ++i) cnt[i] = 0;
    *ctl = c;
    cudaGraphSetConditional(h_td, c.dir == 0 ? 1u : 0u);
    cudaGraphSetConditional(h_bu, c.dir == 1 ? 1u : 0u);
}

__global__ void k_step_end(Ctl* ctl, LevelRec* lrec, const unsigned long long* cnt, cudaGraphConditionalHandle h_loop) {
    Ctl c = *ctl;
    const bool cont = step_finish(c, lrec[c.d], cnt);
    *ctl = c;
    cudaGraphSetConditional(h_loop, cont ? 1u : 0u);
}

// top-down prologue: frontier bitmap -> queue when the previous step was bottom-up,
// and a fresh tile state for the single-pass scan
__global__ void k_td_prep(const Ctl* ctl, const uint32_t* __restrict__ f0, const uint32_t* __restrict__ f1,
                          int64_t words, const int2* __restrict__ head, Queue qa, Queue qb,
                          unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ tstate,
                          unsigned int* __restrict__ tctr) {
    const int64_t tiles = (ctl->n_f + 2047) / 2048;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tiles; i += (int64_t)gridDim.x * blockDim.x)
        tstate[i] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) *tctr = 0u;
    if (!ctl->have_queue) b2q_body(ctl->fsel ? f1 : f0, words, 0, head, ctl->qsel ? qb : qa, cnt);
}

// Single-pass exclusive scan of the current queue's degrees (decoupled look-back:
// tiles are taken in order from a counter, each publishes its aggregate, then its
// inclusive prefix once the look-back over its predecessors resolves).  n+1 outputs.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanThreads) k_scan_dev(const Ctl* ctl, Queue qa, Queue qb, int64_t n_host,
                                                           int64_t* __restrict__ out, unsigned long long* tstate,
                                                           unsigned int* tctr) {
    __shared__ long long s_tile, s_excl;
    __shared__ long long s_warp[kScanThreads / 32];
    // loop graph: size and queue from the loop state; host loop: qa holds the queue
    const long long n = ctl ? ctl->n_f : n_host;
    const int32_t* __restrict__ deg = (ctl && ctl->qsel) ? qb.deg : qa.deg;
    const long long tiles = (n + kScanTile - 1) / kScanTile;
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
        return;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tctr, 1u);
        __syncthreads();
        const long long t = s_tile;
        if (t >= tiles) break;
        const long long base = t * kScanTile + (long long)threadIdx.x * kScanItems;
        long long v[kScanItems], sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            v[k] = base + k < n ? (long long)deg[base + k] : 0;
            sum += v[k];
        }
        long long inc = sum;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            const long long y = __shfl_up_sync(kFull, inc, dd);
            if (lane >= dd) inc += y;
        }
        if (lane == 31) s_warp[wid] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long run = 0;
            for (int w = 0; w < kScanThreads / 32; ++w) {
                const long long x = s_warp[w];
                s_warp[w] = run;
                run += x;
            }
            const long long agg = run;
            long long excl = 0;
            volatile unsigned long long* st = tstate;
            if (t == 0) {
                st[0] = kFlagP | (unsigned long long)agg;
            } else {
                st[t] = kFlagA | (unsigned long long)agg;
                for (long long j = t - 1; j >= 0;) {
                    const unsigned long long x = st[j];
                    if (!(x >> 62)) continue;   // predecessor not published yet
                    excl += (long long)(x & kValMask);
                    if ((x >> 62) == 2) break;
                    --j;
                }
                st[t] = kFlagP | (unsigned long long)(excl + agg);
            }
            s_excl = excl;
            if (t == tiles - 1) out[n] = excl + agg;
        }
        __syncthreads();
        long long pre = s_excl + s_warp[wid] + inc - sum;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (base + k < n) out[base + k] = pre;
            pre += v[k];
        }
        __syncthreads();
    }
}

// bottom-up prologue: queue -> bitmap when the previous step was top-down (clear, then set)
__global__ void k_bu_prep(const Ctl* ctl, uint32_t* __restrict__ f0, uint32_t* __restrict__ f1, int64_t words) {
    if (!ctl->have_queue) return;
    uint32_t* f = ctl->fsel ? f1 : f0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
        f[w] = 0u;
}
__global__ void k_q2b_dev(const Ctl* ctl, Queue qa, Queue qb, uint32_t* __restrict__ f0, uint32_t* __restrict__ f1) {
    if (!ctl->have_queue) return;
    q2b_body((ctl->qsel ? qb : qa).v, ctl->n_f, ctl->fsel ? f1 : f0);
}

// ============================================================ persistent search
// (the cooperative-kernel variant) for small graphs, where even a graph
// node costs more than a level's work: ONE kernel, sized to one resident wave, runs every level of a
// search, the phases separated by grid-wide barriers.  Same state (Ctl, LevelRec,
// queues, bitmaps, records) and the same step semantics as the other loops:
//   TD: warp per frontier vertex of degree < kPersBig, then every big row split over
//       the whole grid; claims by atomicOr on the visited word; winners append to the
//       next queue (warp-aggregated) and record (depth, parent)
//   BU: warp per visited word, lane per vertex, row scanned in stored order up to the
//       first frontier neighbour (its parent); the next word is the warp's ballot
// Data other blocks wrote during the search is read with ld.global.cg (L1 is not
// coherent across the grid barrier); the CSR is read-only.
constexpr int kPersThreads = 256;
constexpr int kPersBig = 2048;   // rows at least this long are split over the grid

// Grid-wide barrier for a grid no larger than one resident wave (the launch sizes it
// from the occupancy): arrive on a counter; the last block resets it and bumps the
// generation the others spin on.  (cooperative_groups' grid sync needs a cooperative
// launch, measured ~60 us more per search on B200.)
struct GridBar {
    unsigned* count;
    unsigned* gen;
    __device__ __forceinline__ void sync() const {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned g = *(volatile unsigned*)gen;
            __threadfence();
            if (atomicAdd(count, 1u) == gridDim.x - 1) {
                *(volatile unsigned*)count = 0u;
                __threadfence();
                atomicAdd(gen, 1u);
            } else {
                while (*(volatile unsigned*)gen == g) __nanosleep(32);
            }
            __threadfence();
        }
        __syncthreads();
    }
};

__device__ __forceinline__ bool pers_in_front(const uint32_t* front, int32_t u) {
    return (__ldcg(front + (u >> 5)) >> (u & 31)) & 1u;
}

__global__ void __launch_bounds__(kPersThreads) k_bfs_persistent(
    const int64_t* __restrict__ off, const int2* __restrict__ head, const int32_t* __restrict__ adj,
    uint32_t* visited, uint32_t* f0, uint32_t* f1, int64_t words, int2* __restrict__ rec,
    const int32_t* __restrict__ pmap, const int32_t* __restrict__ hpar, Queue qa, Queue qb,
    unsigned long long* cnt, int32_t* big, Ctl* ctl, LevelRec* lrec, GridBar grid) {
    const int lane = threadIdx.x & 31;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t gwarp = gtid >> 5, nwarps = nthr >> 5;
    const long long* cw = reinterpret_cast<const long long*>(ctl);
    for (;;) {
        // every thread derives the same step decision from the state of the last barrier
        Ctl c;
        {
            long long* cp = reinterpret_cast<long long*>(&c);
            for (int i = 0; i < (int)(sizeof(Ctl) / 8); ++i) cp[i] = __ldcg(cw + i);
        }
        const long long ts = gtimer();
        const long long m_u = step_decide(c);
        const int32_t lvl = c.d + 1;
        const Queue qc = c.qsel ? qb : qa, qn = c.qsel ? qa : qb;
        uint32_t* front = c.fsel ? f1 : f0;
        uint32_t* next = c.fsel ? f0 : f1;
        unsigned long long my_n = 0, my_mf = 0, my_insp = 0, my_scan = 0;
        if (c.dir == 0) {
            // ---------------- top-down
            if (!c.have_queue) {
                b2q_body(front, words, 0, head, qc, cnt);
                grid.sync();
            }
            int nbig = 0;
            // small rows: warp per frontier vertex; big rows are listed for the grid
            for (int64_t i = gwarp; i < c.n_f; i += nwarps) {
                const int32_t u = __ldcg(qc.v + i);
                const int32_t dg = __ldcg(qc.deg + i);
                if (dg >= kPersBig) {
                    if (lane == 0) big[atomicAdd(cnt + C_SCAN, 1ull)] = u;
                    continue;
                }
                const int64_t b = __ldg(off + u);
                const int32_t pu = pmap ? __ldg(pmap + u) : u;
                for (int j0 = 0; j0 < dg; j0 += 32) {
                    bool win = false;
                    int32_t v = 0;
                    if (j0 + lane < dg) {
                        v = __ldg(adj + b + j0 + lane);
                        const uint32_t bit = 1u << (v & 31);
                        uint32_t* wp = visited + (v >> 5);
                        if (!(__ldcg(wp) & bit)) win = !(atomicOr(wp, bit) & bit);
                    }
                    const unsigned m = __ballot_sync(kFull, win);
                    if (m) {
                        unsigned long long base = 0;
                        if (lane == 0) base = atomicAdd(cnt + C_NEXT, (unsigned long long)__popc(m));
                        base = __shfl_sync(kFull, base, 0);
                        if (win) {
                            const int32_t vd = __ldg(head + v).y;
                            queue_put(qn, base + __popc(m & lanemask_lt()), v, vd);
                            rec[v] = make_int2(lvl, pu);
                            my_mf += (unsigned long long)vd;
                        }
                    }
                }
            }
            grid.sync();
            nbig = (int)__ldcg(cnt + C_SCAN);
            for (int k = 0; k < nbig; ++k) {   // big rows: the whole grid, arc per thread
                const int32_t u = __ldcg(big + k);
                const int64_t b = __ldg(off + u), e = __ldg(off + u + 1);
                const int32_t pu = pmap ? __ldg(pmap + u) : u;
                for (int64_t j0 = b + gtid - lane; j0 < e; j0 += nthr) {
                    const int64_t j = j0 + lane;
                    bool win = false;
                    int32_t v = 0;
                    if (j < e) {
                        v = __ldg(adj + j);
                        const uint32_t bit = 1u << (v & 31);
                        uint32_t* wp = visited + (v >> 5);
                        if (!(__ldcg(wp) & bit)) win = !(atomicOr(wp, bit) & bit);
                    }
                    const unsigned m = __ballot_sync(kFull, win);
                    if (m) {
                        unsigned long long base = 0;
                        if (lane == 0) base = atomicAdd(cnt + C_NEXT, (unsigned long long)__popc(m));
                        base = __shfl_sync(kFull, base, 0);
                        if (win) {
                            const int32_t vd = __ldg(head + v).y;
                            queue_put(qn, base + __popc(m & lanemask_lt()), v, vd);
                            rec[v] = make_int2(lvl, pu);
                            my_mf += (unsigned long long)vd;
                        }
                    }
                }
            }
        } else {
            // ---------------- bottom-up
            if (c.have_queue) {
                for (int64_t w = gtid; w < words; w += nthr) front[w] = 0u;
                grid.sync();
                q2b_body(qc.v, c.n_f, front);
                grid.sync();
            }
            for (int64_t w = gwarp; w < words; w += nwarps) {
                const uint32_t vis = __ldcg(visited + w);
                bool hit = false;
                if (!((vis >> lane) & 1u)) {
                    const int64_t v = w * 32 + lane;
                    const int2 hd = __ldg(head + v);
                    if (hd.y > 0) {
                        my_scan += 1;
                        int32_t pu = -1;
                        if (pers_in_front(front, hd.x)) {
                            hit = true;
                            my_insp += 1;
                            pu = hpar ? __ldg(hpar + v) : hd.x;
                        } else {
                            const int64_t b = __ldg(off + v);
                            int64_t j = 1;
                            for (; j < hd.y; ++j) {
                                const int32_t u = __ldg(adj + b + j);
                                if (pers_in_front(front, u)) {
                                    hit = true;
                                    pu = pmap ? __ldg(pmap + u) : u;
                                    break;
                                }
                            }
                            my_insp += (unsigned long long)(hit ? j + 1 : hd.y);
                        }
                        if (hit) {
                            rec[v] = make_int2(lvl, pu);
                            my_mf += (unsigned long long)hd.y;
                        }
                    }
                }
                const unsigned nb = __ballot_sync(kFull, hit);
                if (lane == 0) {
                    next[w] = nb;
                    if (nb) visited[w] = vis | nb;
                    my_n += (unsigned long long)__popc(nb);
                }
            }
        }
        my_n = warp_sum_u64(my_n);
        my_mf = warp_sum_u64(my_mf);
        my_insp = warp_sum_u64(my_insp);
        my_scan = warp_sum_u64(my_scan);
        if (lane == 0) {
            if (c.dir == 1 && my_n) atomicAdd(cnt + C_NEXT, my_n);
            if (my_mf) atomicAdd(cnt + C_MF, my_mf);
            if (my_insp) atomicAdd(cnt + C_INSP, my_insp);
            if (c.dir == 1 && my_scan) atomicAdd(cnt + C_SCAN, my_scan);
        }
        grid.sync();
        if (gtid == 0) {
            LevelRec r{};
            r.n_f = c.n_f;
            r.m_f = c.m_f;
            r.m_u = m_u;
            r.dir = c.dir;
            r.ts = ts;
            r.k0 = ts;
            const bool cont = step_finish(c, r, cnt);
            r.k1 = r.te;
            lrec[c.d - 1] = r;
            c.done = cont ? 0 : 1;
            *ctl = c;
            for (int i = 0; i < 8; ++i) cnt[i] = 0;
        }
        grid.sync();
        if (reinterpret_cast<const volatile Ctl*>(ctl)->done) break;
    }
}

int grid_for(int64_t items, int threads, int per_sm = 8) {
    const int64_t b = (items + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    return (int)std::max<int64_t>(1, std::min(b, cap));
}

// Bitmap words a search touches.  With the degree reindex every vertex >= n_active is
// isolated: its visited bit is its skip bit forever (no step writes it), it is never a
// frontier vertex, so the steps, conversions and the per-search visited reset cover
// [0, n_active) only -- after one full reset.
static bool active_range(const bfs_graph_s* g) {
    return g->reindexed && !(g->comm && g->comm->nranks > 1) && g->nparts == 1;
}
static int64_t loop_words(const bfs_graph_s* g) {
    return active_range(g) ? words_of(g->n_active) : words_of(g->nl());
}
static int64_t reset_words(bfs_graph_s* g) {
    const int64_t pw = (active_range(g) && g->visited_tail_ok) ? padded_words(g->n_active) : padded_words(g->nl());
    g->visited_tail_ok = true;
    return pw;
}

// CTAs of the top-down kernel that are resident at once: its chunk loop is
// grid-strided, so a grid larger than one wave would leave a straggling second wave
template <bool kMulti>
int td_resident_grid() {
    static const int g = [] {
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_td_expand<kMulti>, kTdThreads, 0) != cudaSuccess ||
            per < 1) {
            cudaGetLastError();
            per = 1;
        }
        return per * num_sms();
    }();
    return g;
}

bool multi(const bfs_graph_s* g) { return g->comm && g->comm->nranks > 1; }

}  // namespace

void bfs_alloc_state(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    const int p = g->comm ? g->comm->nranks : 1;
    g->visited.alloc((size_t)padded_words(nl), s);
    g->tstate.alloc((size_t)(nl / kScanTile + 2), s);   // single-pass scan tile states
    g->tctr.alloc(1, s);
    // global bitmaps: p slices of nb/32 words (nb is a multiple of 32)
    const int64_t gwords = p > 1 ? (int64_t)p * (g->nb / 32) : padded_words(g->n);
    g->front.alloc((size_t)gwords + 4, s);
    g->next.alloc((size_t)gwords + 4, s);
    BFS_CUDA(cudaMemsetAsync(g->front.p, 0, g->front.bytes(), s));
    BFS_CUDA(cudaMemsetAsync(g->next.p, 0, g->next.bytes(), s));
    const size_t qcap = (size_t)std::max<int64_t>(nl, 1);
    g->rec.alloc(qcap, s);
    g->q0.alloc(qcap, s);
    g->q1.alloc(qcap, s);
    g->qd0.alloc(qcap, s);
    g->qd1.alloc(qcap, s);
    g->prefix.alloc((size_t)nl + 1, s);
    g->cnt.alloc(16, s);
    g->scratch64.alloc((size_t)(g->arcs_local / kTdChunk + 2), s);  // TD chunk starts
    if (p > 1) {
        g->seen.alloc((size_t)padded_words(g->n), s);
        g->out_cnt.alloc((size_t)p, s);
        g->cnt_mat.alloc((size_t)p * p, s);
        if (!g->h_cnt_mat) BFS_CUDA(cudaMallocHost(&g->h_cnt_mat, (size_t)p * p * sizeof(int64_t)));
    }
    if (!g->h_cnt) BFS_CUDA(cudaMallocHost(&g->h_cnt, 16 * sizeof(int64_t)));
    for (auto& e : g->ev)
        if (!e) BFS_CUDA(cudaEventCreate(&e));
}

// local counters [0,8) -> global [8,16) (allreduce on p ranks), then to the host
// L2 residency for the one array a step probes at random (visited words for top-down
// claims, the frontier bitmap for bottom-up probes): an access-policy window marks it
// persisting so the step's streaming traffic (adjacency, records) does not evict it.
// Off by default: measured on B200 at K29 it cost 36% (830 -> 530 GTEPS; the
// set-aside shrinks the L2 left for everything else).  BFS_L2_PERSIST=1 enables it.
static size_t l2_persist_limit(int device) {
    static size_t lim = [device] {
        const char* e = getenv("BFS_L2_PERSIST");
        if (!e || e[0] != '1') return (size_t)0;
        int mx = 0;
        if (cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, device) != cudaSuccess || mx <= 0) {
            cudaGetLastError();
            return (size_t)0;
        }
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mx) != cudaSuccess) {
            cudaGetLastError();
            return (size_t)0;
        }
        return (size_t)mx;
    }();
    return lim;
}

static void l2_window(bfs_graph_s* g, const void* base, size_t bytes) {
    const size_t lim = l2_persist_limit(g->device);
    if (!lim) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    a.accessPolicyWindow.num_bytes = base ? std::min(bytes, lim) : 0;
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess) cudaGetLastError();
}

static void sync_counters(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    BFS_CUDA(cudaMemcpyAsync(g->cnt.p + C_GLOBAL, g->cnt.p, 8 * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (g->policy.mode == 3) {
        // the paper's coordinator is partition 0: its local m_f rides along in
        // the counter allreduce as a slot only rank 0 fills
        if (!multi(g) || g->comm->rank == 0)
            BFS_CUDA(cudaMemcpyAsync(g->cnt.p + C_GLOBAL + C_COORD, g->cnt.p + C_MF, sizeof(int64_t),
                                     cudaMemcpyDeviceToDevice, s));
        else
            BFS_CUDA(cudaMemsetAsync(g->cnt.p + C_GLOBAL + C_COORD, 0, sizeof(int64_t), s));
    }
    if (multi(g)) g->comm->allreduce_sum_i64(g->cnt.p + C_GLOBAL, 8, s);
    BFS_CUDA(cudaMemcpyAsync(g->h_cnt, g->cnt.p, 16 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
}

template <class T>
static void ensure(DevBuf<T>& b, size_t count, cudaStream_t s) {
    if (b.count < count) {
        b.reset();
        b.alloc(std::max(count, b.count * 2), s);
    }
}

// ---------------------------------------------------------------- the loop graph
constexpr int kGraphMaxLevels = 4096;   // deeper searches fall back to the host loop
constexpr int kLrecHead = 64;           // records read back with the state in one copy
static_assert(sizeof(Ctl) % 8 == 0 && sizeof(LevelRec) % 8 == 0, "8-byte records");

template <class... P, class... A>
static cudaGraphNode_t add_kernel(cudaGraph_t G, const std::vector<cudaGraphNode_t>& deps, void (*fn)(P...), dim3 grid,
                                  dim3 block, size_t smem, A&&... args) {
    static_assert(sizeof...(P) == sizeof...(A), "argument count");
    std::tuple<std::decay_t<P>...> t(std::forward<A>(args)...);
    void* ptrs[sizeof...(P)];
    std::apply([&](auto&... x) {
        int i = 0;
        ((ptrs[i++] = (void*)&x), ...);
    }, t);
    cudaKernelNodeParams kp{};
    kp.func = (void*)fn;
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.sharedMemBytes = (unsigned)smem;
    kp.kernelParams = ptrs;
    cudaGraphNode_t n;
    BFS_CUDA(cudaGraphAddKernelNode(&n, G, deps.data(), deps.size(), &kp));
    return n;
}

static cudaGraph_t add_cond(cudaGraph_t G, const std::vector<cudaGraphNode_t>& deps, cudaGraphConditionalHandle h,
                            cudaGraphConditionalNodeType type, cudaGraphNode_t* node) {
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    BFS_CUDA(cudaGraphAddNode(node, G, deps.data(), deps.size(), &cp));
    return cp.conditional.phGraph_out[0];
}

static void build_loop_graph(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    const int64_t words = loop_words(g);
    if (!g->ctl.p) {
        g->ctl.alloc(sizeof(Ctl) / 8, s);
        g->lrec.alloc((size_t)kGraphMaxLevels * sizeof(LevelRec) / 8, s);
        BFS_CUDA(cudaMallocHost(&g->h_ctl, sizeof(Ctl) + kLrecHead * sizeof(LevelRec)));
        BFS_CUDA(cudaMallocHost(&g->h_lrec, (size_t)kGraphMaxLevels * sizeof(LevelRec)));
    }
    Ctl* ctl = reinterpret_cast<Ctl*>(g->ctl.p);
    LevelRec* lrec = reinterpret_cast<LevelRec*>(g->lrec.p);
    unsigned long long* cnt = (unsigned long long*)g->cnt.p;
    unsigned long long* tstate = (unsigned long long*)g->tstate.p;
    const Queue qa{g->q0.p, g->qd0.p}, qb{g->q1.p, g->qd1.p};
    const int32_t* pmap = g->reindexed ? g->ilabel.p : nullptr;
    const int sms = num_sms();
    const dim3 g8(sms * 8), t256(256);

    cudaGraph_t G;
    BFS_CUDA(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle h_loop, h_td, h_bu;
    BFS_CUDA(cudaGraphConditionalHandleCreate(&h_loop, G, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t n_while, n_td, n_bu;
    cudaGraph_t B = add_cond(G, {}, h_loop, cudaGraphCondTypeWhile, &n_while);
    BFS_CUDA(cudaGraphConditionalHandleCreate(&h_td, B, 0, cudaGraphCondAssignDefault));
    BFS_CUDA(cudaGraphConditionalHandleCreate(&h_bu, B, 0, cudaGraphCondAssignDefault));
    cudaGraphNode_t n_begin = add_kernel(B, {}, k_step_begin, dim3(1), dim3(1), 0, ctl, lrec, cnt, h_td, h_bu);
    cudaGraph_t T = add_cond(B, {n_begin}, h_td, cudaGraphCondTypeIf, &n_td);
    cudaGraph_t U = add_cond(B, {n_begin}, h_bu, cudaGraphCondTypeIf, &n_bu);
    add_kernel(B, {n_td, n_bu}, k_step_end, dim3(1), dim3(1), 0, ctl, lrec, cnt, h_loop);
    // top-down body
    cudaGraphNode_t t1 = add_kernel(T, {}, k_td_prep, g8, t256, 0, ctl, g->front.p, g->next.p, words, g->head.p, qa, qb,
                                    cnt, tstate, g->tctr.p);
    cudaGraphNode_t t2 = add_kernel(T, {t1}, k_scan_dev, g8, dim3(kScanThreads), 0, ctl, qa, qb, (int64_t)0, g->prefix.p,
                                    tstate, g->tctr.p);
    cudaGraphNode_t t3 = add_kernel(T, {t2}, k_td_chunk_starts, g8, t256, 0, g->prefix.p, (int64_t)0, (int64_t)0,
                                    g->scratch64.p, ctl);
    add_kernel(T, {t3}, k_td_expand<false>, dim3(td_resident_grid<false>()), dim3(kTdThreads), 0, qa, g->prefix.p, g->scratch64.p, (int64_t)0,
               (int64_t)0, g->off.p, g->adj.p, g->visited.p, g->rec.p, pmap, qb, g->head.p, cnt, (int32_t)0, g->lo,
               g->hi, Remote{}, ctl, lrec);
    // bottom-up body
    cudaGraphNode_t u1 = add_kernel(U, {}, k_bu_prep, g8, t256, 0, ctl, g->front.p, g->next.p, words);
    cudaGraphNode_t u2 = add_kernel(U, {u1}, k_q2b_dev, g8, t256, 0, ctl, qa, qb, g->front.p, g->next.p);
    const int64_t nbatches = (words + 31) / 32;
    const int bu_grid = grid_for(nbatches * 32, kBuWarps * 32, kBuCtas);
    const int grab = (int)std::max<int64_t>(1, nbatches / ((int64_t)bu_grid * kBuWarps * 8));
    add_kernel(U, {u2}, k_bu_batch, dim3(bu_grid), dim3(kBuWarps * 32), 0, g->off.p, g->head.p, g->adj.p, g->visited.p,
               g->front.p, g->next.p, g->rec.p, pmap, g->reindexed ? g->hpar.p : nullptr, words, g->lo, (int32_t)0,
               cnt, grab, bu_long_setting(), bu_dense_setting(), ctl, lrec);
    BFS_CUDA(cudaGraphInstantiate(&g->loop_exec, G, 0));
    g->loop_graph = G;
}

void bfs_release_loop(bfs_graph_s* g) {
    if (g->loop_exec) cudaGraphExecDestroy(g->loop_exec);
    if (g->loop_graph) cudaGraphDestroy(g->loop_graph);
    if (g->h_ctl) cudaFreeHost(g->h_ctl);
    if (g->h_lrec) cudaFreeHost(g->h_lrec);
    g->loop_exec = nullptr;
    g->loop_graph = nullptr;
    g->h_ctl = g->h_lrec = nullptr;
}

// graphs up to this many arcs use the persistent kernel in auto mode (BFS_PERSIST_MAX_ARCS)
static int64_t persist_max_arcs() {
    const char* e = getenv("BFS_PERSIST_MAX_ARCS");
    return e ? atoll(e) : (int64_t)1 << 22;
}

static int pers_blocks_per_sm() {
    const char* e = getenv("BFS_PERSIST_BLOCKS");   // tuning only
    return e ? std::max(1, atoi(e)) : 1;
}

// co-resident CTAs of the persistent kernel (cooperative launch limit)
static int pers_grid() {
    static const int gsz = [] {
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bfs_persistent, kPersThreads, 0) != cudaSuccess ||
            per < 1) {
            cudaGetLastError();
            per = 1;
        }
        // fewer CTAs make every grid barrier cheaper; small graphs need no more
        return std::min(per, pers_blocks_per_sm()) * num_sms();
    }();
    return gsz;
}

// One search with the device-driven loop: the loop graph, or (persistent) the
// one-kernel search.  Returns false (nothing to report) if the search ran past
// kGraphMaxLevels levels; the caller reruns it host-driven.
static bool bfs_run_graph(bfs_graph_s* g, int64_t root, int32_t* od, int32_t* op, int32_t* parent_out,
                          int32_t* depth_out, bool persistent) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    if (persistent) {
        if (!g->ctl.p) build_loop_graph(g);   // the state buffers (the graph itself stays unused)
        if (!g->big.p) g->big.alloc((size_t)(g->arcs_local / kPersBig + 4), s);   // + 2 barrier words
    }
    // the graph bakes the tuning knobs into its kernel arguments: rebuild if they changed
    const std::vector<int> key{bu_long_setting(), bu_dense_setting()};
    if (!persistent && g->loop_exec && g->loop_key != key) {
        BFS_CUDA(cudaStreamSynchronize(s));
        cudaGraphExecDestroy(g->loop_exec);
        cudaGraphDestroy(g->loop_graph);
        g->loop_exec = nullptr;
        g->loop_graph = nullptr;
    }
    if (!persistent && !g->loop_exec) {
        build_loop_graph(g);
        g->loop_key = key;
    }
    Ctl* ctl = reinterpret_cast<Ctl*>(g->ctl.p);
    const Queue qa{g->q0.p, g->qd0.p};
    const int64_t pw = reset_words(g);
    const bool lt = g->policy.level_times != 0;
    BFS_CUDA(cudaEventRecord(g->ev[0], s));
    k_init_dev<<<grid_for(pw, 256), 256, 0, s>>>(g->visited.p, g->skip.p, pw, root, g->reindexed ? g->label.p : nullptr,
                                                 g->rec.p, qa, g->head.p, (unsigned long long*)g->cnt.p, ctl, g->policy,
                                                 g->n, g->arcs_global, kGraphMaxLevels);
    BFS_CHECK_LAUNCH();
    BFS_CUDA(cudaEventRecord(g->ev[2], s));
    if (persistent) {
        const int64_t words = loop_words(g);
        const Queue qb{g->q1.p, g->qd1.p};
        LevelRec* lrec = reinterpret_cast<LevelRec*>(g->lrec.p);
        const int32_t* pmap = g->reindexed ? g->ilabel.p : nullptr;
        const int32_t* hpar = g->reindexed ? g->hpar.p : nullptr;
        unsigned long long* cntp = (unsigned long long*)g->cnt.p;
        // barrier words live in the tail of the big-row list buffer; zeroed per search
        unsigned* bar = reinterpret_cast<unsigned*>(g->big.p + g->big.count - 2);
        BFS_CUDA(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s));
        k_bfs_persistent<<<pers_grid(), kPersThreads, 0, s>>>(g->off.p, g->head.p, g->adj.p, g->visited.p, g->front.p,
                                                              g->next.p, words, g->rec.p, pmap, hpar, qa, qb, cntp,
                                                              g->big.p, ctl, lrec, GridBar{bar, bar + 1});
        BFS_CHECK_LAUNCH();
    } else {
        BFS_CUDA(cudaGraphLaunch(g->loop_exec, s));
    }
    BFS_CUDA(cudaEventRecord(g->ev[3], s));
    int64_t launches = 1;
    if (od || op) {
        if (g->reindexed) {
            k_mark_unreached<<<grid_for(words_of(g->n_active), 256), 256, 0, s>>>(g->visited.p, g->skip.p, g->n_active,
                                                                                   g->rec.p);
            BFS_CHECK_LAUNCH();
            k_emit_perm<<<grid_for(g->n, 128, 16), 128, 0, s>>>(g->rec.p, g->label.p, g->n, g->n_active, 0, od, op, ctl);
            launches += 2;
        } else {
            k_emit<<<grid_for(nl, 256), 256, 0, s>>>(g->visited.p, g->skip.p, g->rec.p, nl, 0, od, op, ctl);
            launches += 1;
        }
        BFS_CHECK_LAUNCH();
    }
    BFS_CUDA(cudaEventRecord(g->ev[1], s));
    if (depth_out && od != depth_out) BFS_CUDA(cudaMemcpyAsync(depth_out, od, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
    if (parent_out && op != parent_out)
        BFS_CUDA(cudaMemcpyAsync(parent_out, op, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
    // the one read-back of the search: loop state plus the first kLrecHead step records
    BFS_CUDA(cudaMemcpyAsync(g->h_ctl, g->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaMemcpyAsync(g->h_lrec, g->lrec.p, kLrecHead * sizeof(LevelRec), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
    const Ctl c = *reinterpret_cast<const Ctl*>(g->h_ctl);
    if (c.overflow) return false;
    if (c.d > kLrecHead) {
        BFS_CUDA(cudaMemcpyAsync(g->h_lrec + kLrecHead * sizeof(LevelRec) / 8, g->lrec.p + kLrecHead * sizeof(LevelRec) / 8,
                                 (size_t)(c.d - kLrecHead) * sizeof(LevelRec), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
    }
    const LevelRec* R = reinterpret_cast<const LevelRec*>(g->h_lrec);
    double comp = 0;
    for (int d = 0; d < c.d; ++d) {
        bfs_level_stats L{};
        L.level = d;
        L.direction = R[d].dir;
        L.frontier = R[d].n_f;
        L.discovered = R[d].discovered;
        L.m_f = R[d].m_f;
        L.m_u = R[d].m_u;
        L.inspections = R[d].insp;
        L.scanned = R[d].scanned;
        if (lt) {
            L.ms = (float)((double)(R[d].te - R[d].ts) * 1e-6);
            L.kernel_ms = R[d].k1 > R[d].k0 ? (float)((double)(R[d].k1 - R[d].k0) * 1e-6) : 0.f;
            comp += L.kernel_ms;
        }
        g->levels.push_back(L);
        launches += persistent ? 0 : 2 + (R[d].dir == 0 ? 4 : 3);
    }
    float ms = 0, ms_init = 0, ms_loop = 0;
    BFS_CUDA(cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]));
    BFS_CUDA(cudaEventElapsedTime(&ms_init, g->ev[0], g->ev[2]));
    BFS_CUDA(cudaEventElapsedTime(&ms_loop, g->ev[2], g->ev[3]));
    g->run.ms_total = ms;
    g->run.ms_init = ms_init;
    g->run.ms_compute = lt ? comp : ms_loop;
    g->run.levels = c.d;
    g->run.reached = c.reached;
    g->run.kernel_launches = launches + (persistent ? 1 : 0);
    g->last_root_l = c.root_i;
    g->run.component_edge_tuples = -1;
    return true;
}

void bfs_run_impl(bfs_graph_s* g, int64_t root, int32_t* parent_out, int32_t* depth_out) {
    if (root < 0 || root >= g->n)
        fail(BFS_ERR_OUT_OF_RANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(g->n) + ")");
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    const bool mg = multi(g);
    const int p = mg ? g->comm->nranks : 1;
    const int me = mg ? g->comm->rank : 0;
    unsigned long long* cnt = (unsigned long long*)g->cnt.p;
    int64_t* h = g->h_cnt;

    // the steps record (depth, parent) per discovered vertex in `rec` (internal
    // order); k_emit writes the caller's arrays (device) or staging buffers (host)
    const bool dev_depth = depth_out && is_device_ptr(depth_out);
    const bool dev_parent = parent_out && is_device_ptr(parent_out);
    int2* rec = g->rec.p;
    const int32_t* pmap = g->reindexed ? g->ilabel.p : nullptr;
    int32_t* od = dev_depth ? depth_out : nullptr;
    int32_t* op = dev_parent ? parent_out : nullptr;
    if (depth_out && !dev_depth) {
        if (!g->tmp_depth.p) g->tmp_depth.alloc((size_t)std::max<int64_t>(nl, 1), s);
        od = g->tmp_depth.p;
    }
    if (parent_out && !dev_parent) {
        if (!g->tmp_parent.p) g->tmp_parent.alloc((size_t)std::max<int64_t>(nl, 1), s);
        op = g->tmp_parent.p;
    }

    g->levels.clear();
    g->run = bfs_run_stats{};
    g->run.root = root;
    static const bool env_host_loop = [] {
        const char* e = getenv("BFS_HOST_LOOP");   // A/B experiments only
        return e && e[0] == '1';
    }();
    // level loop: 0 auto (persistent kernel for small graphs, loop graph otherwise),
    // 1 host, 2 loop graph, 3 persistent kernel; p ranks always host-driven
    int loop = g->policy.loop;
    if (env_host_loop) loop = 1;
    if (loop == 0) loop = g->arcs_local <= persist_max_arcs() ? 3 : 2;
    if (!mg && g->nparts == 1 && loop != 1) {
        if (bfs_run_graph(g, root, od, op, parent_out, depth_out, loop == 3)) return;
        g->levels.clear();   // deeper than the graph's record capacity: host loop below
        g->run = bfs_run_stats{};
        g->run.root = root;
    }
    // ---------------- host-driven level loop (p ranks, or policy.host_loop)
    int64_t root_i = root;
    if (g->reindexed) {
        int32_t r;
        BFS_CUDA(cudaMemcpy(&r, g->label.p + root, sizeof(int32_t), cudaMemcpyDeviceToHost));
        root_i = r;
    }
    const bool own_root = root_i >= g->lo && root_i < g->hi;
    const int64_t root_l = own_root ? root_i - g->lo : -1;

    int64_t launches = 0;
    // per-step events: [4d] step start, [4d+1] main kernel start, [4d+2] main kernel end,
    // [4d+3] exchange end (p > 1)
    const bool lt = g->policy.level_times != 0;
    constexpr int kMaxTimed = 64;
    if (lt && g->lev_ev.empty()) {
        g->lev_ev.resize(4 * kMaxTimed + 1);
        for (auto& e : g->lev_ev) BFS_CUDA(cudaEventCreate(&e));
    }

    BFS_CUDA(cudaEventRecord(g->ev[0], s));
    const int64_t pw = reset_words(g);
    Queue qcur{g->q0.p, g->qd0.p};
    Queue qnxt{g->q1.p, g->qd1.p};
    k_init<<<grid_for(pw, 256), 256, 0, s>>>(g->visited.p, g->skip.p, pw, root_l, (int32_t)root_i, rec, (int32_t)root, qcur,
                                             g->head.p, cnt);
    BFS_CHECK_LAUNCH();
    ++launches;
    if (mg) BFS_CUDA(cudaMemsetAsync(g->seen.p, 0, g->seen.bytes(), s));
    sync_counters(g);
    BFS_CUDA(cudaEventRecord(g->ev[2], s));  // end of init

    uint32_t* front = g->front.p;
    uint32_t* next = g->next.p;
    bool have_queue = true;
    int dir = 0;  // 0 TD, 1 BU
    int64_t n_f = h[C_GLOBAL + C_NEXT], m_f = h[C_GLOBAL + C_MF];
    int64_t nf_loc = h[C_NEXT], mf_loc = h[C_MF];
    int64_t prev_nf = 0, seen = 0, reached = 0;
    int64_t m_fc = h[C_GLOBAL + C_COORD], bu_done = 0;  // policy 3: coordinator m_f, BU steps taken
    bool returned = false;
    const int64_t words = loop_words(g);
    const size_t slice_bytes = mg ? (size_t)(g->nb / 8) : 0;
    uint64_t nvl_total = 0;
    std::vector<size_t> sendb(p), recvb(p);
    std::vector<const void*> sendp(p);
    std::vector<void*> recvp(p);
    for (int d = 0; n_f > 0; ++d) {
        if (d >= (1 << 30)) fail(BFS_ERR_INTERNAL, "level loop did not terminate");
        reached += n_f;
        seen += m_f;
        const int64_t m_u = g->arcs_global - seen;
        // direction for the step that builds level d+1 (R2)
        switch (g->policy.mode) {
            case 1: dir = 0; break;
            case 2: dir = d >= g->policy.bu_from_level ? 1 : 0; break;
            case 3:  // the paper's rule (section 3.3; R23)
                if (dir == 0) {
                    if (!returned && m_fc * 10000 >= g->policy.alpha * g->arcs_global) dir = 1;
                } else if (bu_done >= g->policy.beta) {
                    dir = 0;
                    returned = true;
                }
                if (dir == 1) ++bu_done;
                break;
            default:
                if (dir == 0) {
                    if (m_f * g->policy.alpha > m_u) dir = 1;
                } else {
                    if (n_f * g->policy.beta < g->n && n_f < prev_nf) dir = 0;
                }
        }
        const bool timed = lt && d < kMaxTimed;
        if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d], s));
        BFS_CUDA(cudaMemsetAsync(g->cnt.p, 0, 8 * sizeof(int64_t), s));
        int64_t insp = -1, scanned = -1;
        uint64_t nvl = 0;
        if (dir == 0) {
            // ---------------- top-down (Alg. 1, push Alg. 2)
            if (!have_queue) {
                k_b2q<<<grid_for(words, 256), 256, 0, s>>>(front, words, g->lo, g->head.p, qcur, cnt);
                BFS_CHECK_LAUNCH();
                ++launches;
                have_queue = true;
            }
            const int64_t E = mf_loc;
            Remote rm{};
            if (mg) {
                rm.nb = g->nb;
                rm.cap = std::max<int64_t>(1, std::min<int64_t>(g->nb, E));
                ensure(g->out_list, (size_t)(p * rm.cap), s);
                rm.seen = g->seen.p;
                rm.out = g->out_list.p;
                rm.out_cnt = (unsigned long long*)g->out_cnt.p;
                BFS_CUDA(cudaMemsetAsync(g->out_cnt.p, 0, (size_t)p * sizeof(int64_t), s));
            }
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 1], s));
            if (E > 0) {
                l2_window(g, g->visited.p, g->visited.bytes());
                // single-pass scan of the queue degrees (the loop graph's kernel, host-sized)
                BFS_CUDA(cudaMemsetAsync(g->tstate.p, 0, (size_t)((nf_loc + kScanTile - 1) / kScanTile) * 8, s));
                BFS_CUDA(cudaMemsetAsync(g->tctr.p, 0, sizeof(uint32_t), s));
                k_scan_dev<<<grid_for((nf_loc + kScanTile - 1) / kScanTile * kScanThreads, kScanThreads), kScanThreads, 0,
                             s>>>(nullptr, qcur, qcur, nf_loc, g->prefix.p, (unsigned long long*)g->tstate.p,
                                  g->tctr.p);
                BFS_CHECK_LAUNCH();
                ++launches;
                const int64_t nchunks = (E + kTdChunk - 1) / kTdChunk;
                k_td_chunk_starts<<<grid_for(nchunks, 256), 256, 0, s>>>(g->prefix.p, nf_loc, nchunks, g->scratch64.p,
                                                                          nullptr);
                BFS_CHECK_LAUNCH();
                const int grid = (int)std::min<int64_t>(nchunks, mg ? td_resident_grid<true>() : td_resident_grid<false>());
                if (mg)
                    k_td_expand<true><<<grid, kTdThreads, 0, s>>>(qcur, g->prefix.p, g->scratch64.p, nf_loc, E, g->off.p,
                                                                  g->adj.p, g->visited.p, rec, pmap, qnxt, g->head.p, cnt, d + 1,
                                                                  g->lo, g->hi, rm, nullptr, nullptr);
                else
                    k_td_expand<false><<<grid, kTdThreads, 0, s>>>(qcur, g->prefix.p, g->scratch64.p, nf_loc, E,
                                                                   g->off.p, g->adj.p, g->visited.p, rec, pmap, qnxt, g->head.p, cnt,
                                                                   d + 1, g->lo, g->hi, rm, nullptr, nullptr);
                BFS_CHECK_LAUNCH();
                launches += 2;
            }
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 2], s));
            if (mg) {
                // push: counts matrix (allgather), then claims to their owners (alltoallv)
                BFS_CUDA(cudaMemcpyAsync(g->cnt_mat.p + (size_t)me * p, g->out_cnt.p, (size_t)p * 8,
                                         cudaMemcpyDeviceToDevice, s));
                g->comm->allgather_inplace(g->cnt_mat.p, (size_t)p * 8, s);
                BFS_CUDA(cudaMemcpyAsync(g->h_cnt_mat, g->cnt_mat.p, (size_t)p * p * 8, cudaMemcpyDeviceToHost, s));
                BFS_CUDA(cudaStreamSynchronize(s));
                int64_t R = 0;
                for (int q = 0; q < p; ++q) R += q == me ? 0 : g->h_cnt_mat[(size_t)q * p + me];
                ensure(g->in_list, (size_t)std::max<int64_t>(R, 1), s);
                int64_t roff = 0;
                for (int q = 0; q < p; ++q) {
                    const int64_t out_q = q == me ? 0 : g->h_cnt_mat[(size_t)me * p + q];
                    const int64_t in_q = q == me ? 0 : g->h_cnt_mat[(size_t)q * p + me];
                    sendp[q] = g->out_list.p + (size_t)q * rm.cap;
                    sendb[q] = (size_t)out_q * sizeof(int2);
                    recvp[q] = g->in_list.p + roff;
                    recvb[q] = (size_t)in_q * sizeof(int2);
                    roff += in_q;
                    nvl += sendb[q];
                }
                g->comm->alltoallv(sendp.data(), sendb.data(), recvp.data(), recvb.data(), s);
                if (R > 0) {
                    k_td_merge<<<grid_for(R, 256), 256, 0, s>>>(g->in_list.p, R, g->head.p, g->visited.p, rec, qnxt,
                                                                cnt, d + 1, g->lo);
                    BFS_CHECK_LAUNCH();
                    ++launches;
                }
            }
            std::swap(qcur, qnxt);
            insp = E;
            scanned = nf_loc;
        } else {
            // ---------------- bottom-up (Alg. 1, pull Alg. 3)
            // Pull (Alg. 3) adapts to the frontier's density: a sparse global
            // frontier (4 bytes per vertex below the bitmap slices' size) travels as
            // vertex lists -- each rank sends its owned frontier vertices to every peer and
            // rebuilds the whole bitmap locally -- a dense one as bitmap slices (allgather).
            // Every rank sees the same global n_f, so all take the same branch.
            const bool sparse_pull = mg && (uint64_t)n_f * 4 < (uint64_t)slice_bytes * (uint64_t)(p - 1);
            if (sparse_pull) {
                // this rank's frontier as a vertex list: the TD queue, or its bitmap slice
                const int32_t* mine = qcur.v;
                if (!have_queue) {
                    k_b2q<<<grid_for(words, 256), 256, 0, s>>>(front, words, g->lo, g->head.p, qnxt, cnt);
                    BFS_CHECK_LAUNCH();
                    ++launches;
                    mine = qnxt.v;
                }
                BFS_CUDA(cudaMemsetAsync(g->cnt_mat.p, 0, (size_t)p * 8, s));
                BFS_CUDA(cudaMemcpyAsync(g->cnt_mat.p + me, &g->h_cnt[C_NEXT], 8, cudaMemcpyHostToDevice, s));
                g->comm->allgather_inplace(g->cnt_mat.p, 8, s);
                BFS_CUDA(cudaMemcpyAsync(g->h_cnt_mat, g->cnt_mat.p, (size_t)p * 8, cudaMemcpyDeviceToHost, s));
                BFS_CUDA(cudaStreamSynchronize(s));
                int64_t R = 0;
                for (int q = 0; q < p; ++q) R += q == me ? 0 : g->h_cnt_mat[q];
                ensure(g->flist, (size_t)std::max<int64_t>(R, 1), s);
                int64_t roff = 0;
                for (int q = 0; q < p; ++q) {
                    const int64_t in_q = q == me ? 0 : g->h_cnt_mat[q];
                    sendp[q] = mine;
                    sendb[q] = q == me ? 0 : (size_t)nf_loc * 4;
                    recvp[q] = g->flist.p + roff;
                    recvb[q] = (size_t)in_q * 4;
                    roff += in_q;
                    nvl += sendb[q];
                }
                g->comm->alltoallv(sendp.data(), sendb.data(), recvp.data(), recvb.data(), s);
                BFS_CUDA(cudaMemsetAsync(front, 0, (size_t)p * slice_bytes, s));
                if (nf_loc) {
                    k_q2b<<<grid_for(nf_loc, 256), 256, 0, s>>>(mine, nf_loc, front);
                    BFS_CHECK_LAUNCH();
                    ++launches;
                }
                if (R) {
                    k_q2b<<<grid_for(R, 256), 256, 0, s>>>(g->flist.p, R, front);
                    BFS_CHECK_LAUNCH();
                    ++launches;
                }
                have_queue = false;
            } else {
                if (have_queue) {
                    BFS_CUDA(cudaMemsetAsync(front + (g->lo >> 5), 0, (size_t)words_of(nl) * 4, s));
                    if (nf_loc) {
                        k_q2b<<<grid_for(nf_loc, 256), 256, 0, s>>>(qcur.v, nf_loc, front);
                        BFS_CHECK_LAUNCH();
                        ++launches;
                    }
                    have_queue = false;
                }
                if (mg) {
                    g->comm->allgather_inplace(front, slice_bytes, s);
                    nvl = slice_bytes * (size_t)(p - 1);
                }
            }
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 1], s));
            l2_window(g, front, g->front.bytes());
            const int64_t nbatches = (words + 31) / 32;
            const int bu_grid = grid_for(nbatches * 32, kBuWarps * 32, kBuCtas);
            const int grab = (int)std::max<int64_t>(1, nbatches / ((int64_t)bu_grid * kBuWarps * 8));
            k_bu_batch<<<bu_grid, kBuWarps * 32, 0, s>>>(g->off.p, g->head.p, g->adj.p, g->visited.p, front, next, rec,
                                                         pmap, g->reindexed ? g->hpar.p : nullptr, words, g->lo,
                                                         d + 1, cnt, grab, bu_long_setting(), bu_dense_setting(), nullptr,
                                                         nullptr);
            BFS_CHECK_LAUNCH();
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 2], s));
            ++launches;
            std::swap(front, next);
        }
        if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 3], s));
        sync_counters(g);
        bfs_level_stats L{};
        L.level = d;
        L.direction = dir;
        L.frontier = n_f;
        L.discovered = h[C_GLOBAL + C_NEXT];
        L.m_f = m_f;
        L.m_u = m_u;
        L.inspections = dir == 0 ? m_f : h[C_GLOBAL + C_INSP];
        L.scanned = dir == 0 ? n_f : h[C_GLOBAL + C_SCAN];
        L.nvlink_bytes = nvl;
        (void)insp;
        (void)scanned;
        nvl_total += nvl;
        g->levels.push_back(L);
        prev_nf = n_f;
        n_f = h[C_GLOBAL + C_NEXT];
        m_f = h[C_GLOBAL + C_MF];
        m_fc = h[C_GLOBAL + C_COORD];
        nf_loc = h[C_NEXT];
        mf_loc = h[C_MF];
    }
    const int ntimed = lt ? (int)std::min<size_t>(g->levels.size(), kMaxTimed) : 0;
    if (lt) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * ntimed], s));
    if (od || op) {
        if (g->reindexed) {
            k_mark_unreached<<<grid_for(words_of(g->n_active), 256), 256, 0, s>>>(g->visited.p, g->skip.p, g->n_active,
                                                                                   rec);
            BFS_CHECK_LAUNCH();
            ++launches;
            k_emit_perm<<<grid_for(g->n, 128, 16), 128, 0, s>>>(rec, g->label.p, g->n,
                                                            g->n_active, root_l, od, op, nullptr);
        } else {
            k_emit<<<grid_for(nl, 256), 256, 0, s>>>(g->visited.p, g->skip.p, rec, nl, root_l, od, op, nullptr);
        }
        BFS_CHECK_LAUNCH();
        ++launches;
    }
    l2_window(g, nullptr, 0);
    BFS_CUDA(cudaEventRecord(g->ev[1], s));
    if (depth_out && !dev_depth) BFS_CUDA(cudaMemcpyAsync(depth_out, od, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
    if (parent_out && !dev_parent) BFS_CUDA(cudaMemcpyAsync(parent_out, op, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
    float ms = 0, ms_init = 0;
    BFS_CUDA(cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]));
    BFS_CUDA(cudaEventElapsedTime(&ms_init, g->ev[0], g->ev[2]));
    g->run.ms_total = ms;
    g->run.ms_init = ms_init;
    g->run.levels = (int)g->levels.size();
    g->run.reached = reached;
    g->run.kernel_launches = launches;
    g->run.nvlink_bytes = nvl_total;
    double push = 0, pull = 0, comp = 0;
    for (int d = 0; d < ntimed; ++d) {
        float x = 0, k = 0, xe = 0;
        BFS_CUDA(cudaEventElapsedTime(&x, g->lev_ev[4 * d], g->lev_ev[4 * d + 4]));
        BFS_CUDA(cudaEventElapsedTime(&k, g->lev_ev[4 * d + 1], g->lev_ev[4 * d + 2]));
        BFS_CUDA(cudaEventElapsedTime(&xe, g->lev_ev[4 * d + 2], g->lev_ev[4 * d + 3]));
        g->levels[d].ms = x;
        g->levels[d].kernel_ms = k;
        comp += k;
        if (mg) {
            if (g->levels[d].direction == 0) {
                push += xe;
            } else {
                float pre = 0;
                BFS_CUDA(cudaEventElapsedTime(&pre, g->lev_ev[4 * d], g->lev_ev[4 * d + 1]));
                pull += pre;
            }
        }
    }
    g->run.ms_compute = lt ? comp : ms - ms_init;
    g->run.ms_push = push;
    g->run.ms_pull = pull;
    g->last_root_l = root_l;
    g->run.component_edge_tuples = -1;  // computed lazily by bfs_stats
}

int64_t component_tuples_impl(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    BFS_CUDA(cudaMemsetAsync(g->cnt.p + C_TUPLES, 0, sizeof(int64_t), s));
    k_component_degree<<<grid_for(g->nl(), 256), 256, 0, s>>>(g->visited.p, g->skip.p, g->deg_raw.p, g->nl(),
                                                              g->last_root_l, (unsigned long long*)g->cnt.p + C_TUPLES);
    BFS_CHECK_LAUNCH();
    if (multi(g)) g->comm->allreduce_sum_i64(g->cnt.p + C_TUPLES, 1, s);
    int64_t v = 0;
    BFS_CUDA(cudaMemcpyAsync(&v, g->cnt.p + C_TUPLES, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
    return v / 2;
}

void sample_roots_impl(bfs_graph_s* g, uint32_t scale, uint64_t seed, int64_t count, int64_t* roots, int64_t* found) {
    cudaStream_t s = g->stream;
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    const int64_t max_cand = 64 * count + 4 * g->n;
    const int64_t B = 4096;
    std::vector<int32_t> cand;
    std::vector<int64_t> deg(B);
    DevBuf<int32_t> dcand, dint;
    DevBuf<int64_t> ddeg;
    dcand.alloc(B, s);
    dint.alloc(B, s);
    ddeg.alloc(B, s);
    int64_t got = 0;
    for (int64_t k0 = 0; k0 < max_cand && got < count; k0 += B) {
        cand.clear();
        for (int64_t k = k0; k < std::min(max_cand, k0 + B); ++k) {
            uint32_t ctr[4] = {(uint32_t)((uint64_t)k & 0xffffffffu), (uint32_t)((uint64_t)k >> 32), 0u, 2u}, w[4];
            philox4x32_10_host(ctr, key, w);
            const int64_t r = scale == 0 ? 0 : (int64_t)(w[0] >> (32 - scale));
            cand.push_back(r < g->n ? (int32_t)r : -1);
        }
        const int64_t K = (int64_t)cand.size();
        BFS_CUDA(cudaMemcpyAsync(dcand.p, cand.data(), (size_t)K * 4, cudaMemcpyHostToDevice, s));
        const int32_t* di = dcand.p;
        if (g->reindexed) {
            k_gather_labels<<<grid_for(K, 256), 256, 0, s>>>(g->label.p, dcand.p, K, dint.p);
            BFS_CHECK_LAUNCH();
            di = dint.p;
        }
        k_nonloop_degree<<<grid_for(K * 32, 256), 256, 0, s>>>(di, K, g->off.p, g->adj.p, g->lo, g->hi, ddeg.p);
        BFS_CHECK_LAUNCH();
        if (multi(g)) g->comm->allreduce_sum_i64(ddeg.p, (int)K, s);
        BFS_CUDA(cudaMemcpyAsync(deg.data(), ddeg.p, (size_t)K * 8, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        for (int64_t t = 0; t < K && got < count; ++t) {
            if (cand[t] < 0 || deg[t] == 0) continue;
            bool dup = false;
            for (int64_t x = 0; x < got; ++x)
                if (roots[x] == cand[t]) { dup = true; break; }
            if (!dup) roots[got++] = cand[t];
        }
    }
    *found = got;
}

}  // namespace bfsb
