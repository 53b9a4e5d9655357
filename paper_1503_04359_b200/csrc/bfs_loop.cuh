// Device-driven level loops: the loop-graph kernels (the step kernel,
// TD / BU prologues, single-pass look-back scan) and the persistent one-kernel search.
// Included once, inside namespace bfsb::{anonymous}, by bfs.cu (a single translation
// unit: the kernels, device helpers and the host launch code share one file scope).
#pragma once

// ============================================================ device-driven level loop
// (SURVEY f3).  On one GPU the whole level loop is one CUDA graph: a WHILE node
// whose body is k_step (roll the counters of the step that just ran and record it,
// then the alpha/beta decision on the device, or stop when the frontier is empty)
// -> IF(top-down) {k_td_prep -> k_scan_dev -> k_td_chunk_starts -> k_td_expand} and
// IF(bottom-up) {k_bu_prep -> k_q2b_dev -> k_bu_batch}.  The host launches it once
// per search and synchronises once, instead of once per level.

// init on the device: the root's internal label, visited <- skip | root, root
// record, the first queue, the loop state (policy included)
struct InitArgs {
    uint32_t* visited;
    const uint32_t* skip;
    int64_t pw, root;
    const int32_t* label;
    int2* out;
    Queue q;
    const int2* head;
    unsigned long long* cnt;
    Ctl* ctl;
    bfs_policy pol;
    int64_t n, arcs;
    int max_levels;
    int64_t claim_min, tile_min, td_small;
    unsigned long long* pcnt;   // persistent / cluster search: its three counter sets (zeroed)
    unsigned* bar;              // grid-barrier words (zeroed)
};

__device__ __forceinline__ void init_body(const InitArgs& a) {
    const int64_t ri = a.label ? (int64_t)__ldg(a.label + a.root) : a.root;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < a.pw; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = a.skip[w];
        if (w == (ri >> 5)) x |= 1u << (ri & 31);
        a.visited[w] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) a.cnt[i] = 0;
        a.out[ri] = make_int2(0, (int32_t)a.root);
        const int32_t dg = a.head[ri].y;
        queue_put(a.q, 0, (int32_t)ri, dg);
        Ctl c{};
        c.n_f = 1;
        c.m_f = c.m_fc = dg;
        c.root_i = ri;
        c.alpha = a.pol.alpha;
        c.beta = a.pol.beta;
        c.n = a.n;
        c.arcs = a.arcs;
        c.have_queue = 1;
        c.mode = a.pol.mode;
        c.bu_from = a.pol.bu_from_level;
        c.max_levels = a.max_levels;
        c.claim_min = a.claim_min;
        c.tile_min = a.tile_min;
        c.td_small = a.td_small;
        *a.ctl = c;
        if (a.pcnt)
            for (int i = 0; i < 48; ++i) a.pcnt[i] = 0;
        if (a.bar) a.bar[0] = a.bar[1] = 0u;
    }
}
__global__ void k_init_dev(InitArgs a) { init_body(a); }

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

// the step's record and the roll of the counters into the loop state (k_step and
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
        c.front_ok = 0;
        if (c.claim) {            // the next frontier is a bitmap only (k_td_finish)
            c.fsel ^= 1;
            c.have_queue = 0;
        }
    } else {
        c.fsel ^= 1;
        c.have_queue = 0;
        c.front_ok = 0;
    }
    c.claim = 0;
    c.tile = 0;
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

// One kernel per level of the loop graph: the roll of the step that just ran (its record,
// the counters into the loop state; nothing on the first call) and, if the search goes
// on, the alpha/beta decision and the IF handles of the next step; otherwise the WHILE
// handle drops to 0 and no IF body runs.  (Round 1 had a begin and an end kernel per
// level: one single-thread launch more per level.)
enum { kStepSmallTd = 0, kStepTd = 1, kStepBuConv = 2, kStepBu = 3, kStepNone = 4 };
__global__ void k_step(Ctl* ctl, LevelRec* lrec, unsigned long long* cnt, cudaGraphConditionalHandle h_loop,
                       cudaGraphConditionalHandle h_sw) {
    Ctl c = *ctl;
    if (c.started && !step_finish(c, lrec[c.d], cnt)) {
        *ctl = c;
        cudaGraphSetConditional(h_loop, 0u);
        return;   // the SWITCH handle keeps its default (no body)
    }
    c.started = 1;
    const long long t = gtimer();
    const long long m_u = step_decide(c);
    c.E = c.m_f;
    c.nchunks = (c.E + kTdChunk - 1) / kTdChunk;
    // k_td_small (neither claim-only nor tiled): few arcs, and no hub among the frontier
    // vertices on average (a long row is one warp's work there)
    const bool small = c.dir == 0 && c.E <= c.td_small && c.E <= 64 * c.n_f;
    c.tile = c.dir == 0 && !small && c.tile_min >= 0 && c.E >= c.tile_min;
    c.claim = c.dir == 0 && !small && (c.E >= c.claim_min || c.tile);
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
    cudaGraphSetConditional(h_sw, c.dir == 0 ? (small ? kStepSmallTd : kStepTd)
                                             : ((c.have_queue && !c.front_ok) ? kStepBuConv : kStepBu));
}

// A small top-down step (m_f <= td_small arcs and at most 64 per frontier vertex: the
// first levels from a low-degree root and the last levels of a search) as ONE kernel instead of the prologue / scan /
// chunk / expand / finish chain: warp per frontier vertex, lanes over its arcs,
// claims by atomicOr on the visited word, winners record (depth, parent) and append
// to the next queue (one atomic per warp instruction).  The frontier is the queue or,
// after a bottom-up step, the bitmap (its set bits are expanded in place: no b2q).
__global__ void k_td_small(const Ctl* ctl, Queue qa, Queue qb, const uint32_t* __restrict__ f0,
                           const uint32_t* __restrict__ f1, int64_t words, const int64_t* __restrict__ off,
                           const int32_t* __restrict__ adj, const int2* __restrict__ head, uint32_t* __restrict__ visited,
                           int2* __restrict__ rec, const int32_t* __restrict__ pmap, unsigned long long* __restrict__ cnt,
                           LevelRec* lrec) {
    const Ctl& c = *ctl;
    if (c.dir != 0 || c.E > c.td_small || c.E > 64 * c.n_f) return;
    stamp_begin(lrec, ctl);
    const int lane = threadIdx.x & 31;
    const int32_t level = c.d + 1;
    const Queue qn = c.qsel ? qa : qb;
    unsigned long long my_mf = 0;
    constexpr int kU = 4;   // 32-arc groups of a row in flight per warp
    auto expand = [&](int32_t u) {   // warp-uniform u
        const int64_t jb = __ldg(off + u), je = __ldg(off + u + 1);
        const int32_t par = pmap ? __ldg(pmap + u) : u;
        for (int64_t j0 = jb; j0 < je; j0 += 32 * kU) {
            int32_t v[kU];
            uint32_t w[kU];
#pragma unroll
            for (int q = 0; q < kU; ++q) {
                const int64_t j = j0 + q * 32 + lane;
                v[q] = j < je ? __ldg(adj + j) : -1;
            }
#pragma unroll
            for (int q = 0; q < kU; ++q) w[q] = v[q] >= 0 ? __ldcg(visited + (v[q] >> 5)) : kFull;
#pragma unroll
            for (int q = 0; q < kU; ++q) {
                const uint32_t bit = v[q] >= 0 ? 1u << (v[q] & 31) : 0u;
                const bool win = v[q] >= 0 && !(w[q] & bit) && !(atomicOr(visited + (v[q] >> 5), bit) & bit);
                const unsigned m = __ballot_sync(kFull, win);
                if (!m) continue;
                unsigned long long base = 0;
                if (lane == __ffs(m) - 1) base = atomicAdd(cnt + C_NEXT, (unsigned long long)__popc(m));
                base = __shfl_sync(kFull, base, __ffs(m) - 1);
                if (win) {
                    const int32_t dg = __ldg(head + v[q]).y;
                    rec[v[q]] = make_int2(level, par);
                    queue_put(qn, base + __popc(m & lanemask_lt()), v[q], dg);
                    my_mf += (unsigned long long)dg;
                }
            }
        }
    };
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (c.have_queue) {
        const int32_t* qv = c.qsel ? qb.v : qa.v;
        for (int64_t i = gw; i < c.n_f; i += nw) expand(__ldg(qv + i));
    } else {
        const uint32_t* fr = c.fsel ? f1 : f0;
        for (int64_t b0 = gw * 32; b0 < words; b0 += nw * 32) {
            const uint32_t x = b0 + lane < words ? __ldcg(fr + b0 + lane) : 0u;
            unsigned todo = __ballot_sync(kFull, x != 0u);
            while (todo) {
                const int q = __ffs(todo) - 1;
                todo &= todo - 1;
                uint32_t bits = __shfl_sync(kFull, x, q);
                while (bits) {
                    const int k = __ffs(bits) - 1;
                    bits &= bits - 1;
                    expand((int32_t)((b0 + q) * 32 + k));
                }
            }
        }
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
    if (lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}


// top-down prologue: frontier bitmap -> queue when the previous step was bottom-up,
// and a fresh tile state for the single-pass scan
__global__ void k_td_prep(const Ctl* ctl, uint32_t* __restrict__ f0, uint32_t* __restrict__ f1,
                          int64_t words, const int2* __restrict__ head, Queue qa, Queue qb,
                          unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ tstate,
                          unsigned int* __restrict__ tctr, const uint32_t* __restrict__ visited,
                          unsigned* __restrict__ hcount, unsigned* __restrict__ lcnt, int64_t nwl,
                          cudaGraphConditionalHandle h_tile, int has_tile) {
    const int64_t tiles = (ctl->n_f + 2047) / 2048;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tiles; i += (int64_t)gridDim.x * blockDim.x)
        tstate[i] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *tctr = 0u;
        if (hcount) *hcount = 0u;   // heavy list (tile mode)
        if (has_tile) cudaGraphSetConditional(h_tile, ctl->tile ? 1u : 0u);
    }
    if (ctl->tile && lcnt)   // light-row record buckets (tile mode)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nwl; i += (int64_t)gridDim.x * blockDim.x)
            lcnt[i] = 0u;

    if (ctl->claim) {   // claim-only step: snapshot visited into the spare bitmap (k_td_finish)
        uint32_t* snap = ctl->fsel ? f0 : f1;
        for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
            snap[w] = __ldcs(visited + w);
    }
    if (!ctl->have_queue) b2q_body(ctl->fsel ? f1 : f0, words, 0, head, ctl->qsel ? qb : qa, cnt);
}

__global__ void k_td_finish_dev(const Ctl* ctl, const uint32_t* __restrict__ visited, uint32_t* __restrict__ f0,
                                uint32_t* __restrict__ f1, int64_t words, const int2* __restrict__ head, Queue qa,
                                Queue qb, unsigned long long* __restrict__ cnt) {
    if (!ctl->claim) return;
    td_finish_body(visited, ctl->fsel ? f0 : f1, words, head, cnt);
}

// Single-pass exclusive scan of the current queue's degrees (decoupled look-back:
// tiles are taken in order from a counter, each publishes its aggregate, then its
// inclusive prefix once the look-back over its predecessors resolves).  n+1 outputs.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

// Tile mode (td_tile.cuh): queue entries with label < nh (heavy rows) count 0 arcs
// here -- the tiled kernel expands them (k_tile_list lists them).
__global__ void __launch_bounds__(kScanThreads) k_scan_dev(const Ctl* ctl, Queue qa, Queue qb, int64_t n_host,
                                                           int64_t* __restrict__ out, unsigned long long* tstate,
                                                           unsigned int* tctr, int64_t nh, int tile_host) {
    __shared__ long long s_tile, s_excl;
    __shared__ long long s_warp[kScanThreads / 32];
    // loop graph: size and queue from the loop state; host loop: qa holds the queue
    const long long n = ctl ? ctl->n_f : n_host;
    const int32_t* __restrict__ deg = (ctl && ctl->qsel) ? qb.deg : qa.deg;
    const int32_t* __restrict__ qv = (ctl && ctl->qsel) ? qb.v : qa.v;
    const bool tile = ctl ? ctl->tile != 0 : tile_host != 0;
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
            const bool in = base + k < n;
            const int32_t u = (tile && in) ? qv[base + k] : INT32_MAX;
            v[k] = (in && u >= nh) ? (long long)deg[base + k] : 0;   // heavy row (u < nh): k_td_tile expands it
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
    if (!ctl->have_queue || ctl->front_ok) return;
    uint32_t* f = ctl->fsel ? f1 : f0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
        f[w] = 0u;
}
__global__ void k_q2b_dev(const Ctl* ctl, Queue qa, Queue qb, uint32_t* __restrict__ f0, uint32_t* __restrict__ f1) {
    if (!ctl->have_queue || ctl->front_ok) return;
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
constexpr int kPersBig = 128;    // rows at least this long are split over the grid (a hub row of a
                                 // few thousand arcs was 60+ dependent warp steps: ~90 us at K16)

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

// Thread-block-cluster barrier (one cluster runs the whole search: the hardware
// barrier.cluster with release/acquire semantics at cluster scope replaces the
// atomic-and-spin grid barrier).
struct ClusterBar {
    __device__ __forceinline__ void sync() const {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
};

__device__ __forceinline__ bool pers_in_front(const uint32_t* front, int32_t u) {
    return (__ldcg(front + (u >> 5)) >> (u & 31)) & 1u;
}

// the output pass the persistent search runs after its last level (mode 0: none,
// 1: labels unchanged (emit_body), 2: degree-reindexed (mark_unreached + emit_perm))
struct PersOut {
    int mode;
    const uint32_t* skip;
    const int32_t* label;
    int64_t n, n_active;
    int32_t* depth;
    int32_t* parent;
};

// Bar = GridBar: one resident wave over every SM; Bar = ClusterBar: ONE thread-block
// cluster (up to 16 CTAs) whose levels are separated by barrier.cluster.
template <class Bar, int kThreads>
__global__ void __launch_bounds__(kThreads) k_bfs_persistent(
    const int64_t* __restrict__ off, const int2* __restrict__ head, const int32_t* __restrict__ adj,
    uint32_t* visited, uint32_t* f0, uint32_t* f1, int64_t words, int2* __restrict__ rec,
    const int32_t* __restrict__ pmap, const int32_t* __restrict__ hpar, Queue qa, Queue qb,
    unsigned long long* cnt3, int32_t* big, Ctl* ctl, LevelRec* lrec, Bar grid, PersOut po, InitArgs ia,
    int do_init) {
    // One grid barrier per level: the counters are triple-buffered (level d accumulates
    // into set d % 3, zeroed by thread 0 two levels ahead), and every thread rolls its own
    // copy of the loop state from them after the barrier (the same arithmetic on the
    // same numbers, so all copies agree); thread 0 keeps the step records and publishes
    // the final state.
    const int lane = threadIdx.x & 31;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t gwarp = gtid >> 5, nwarps = nthr >> 5;
    if (do_init) {   // the search's init in the same kernel (cluster search: one launch per search)
        init_body(ia);
        grid.sync();
    }
    Ctl c;
    {
        const long long* cw = reinterpret_cast<const long long*>(ctl);
        long long* cp = reinterpret_cast<long long*>(&c);
        for (int i = 0; i < (int)(sizeof(Ctl) / 8); ++i) cp[i] = __ldcg(cw + i);
    }
    for (;;) {
        unsigned long long* cnt = cnt3 + 16 * (c.d % 3);
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
            // big rows: up to 4 arcs per thread of a CTA -> one CTA each (round robin);
            // longer ones -> the whole grid, arc per thread
            for (int k = blockIdx.x; k < nbig; k += gridDim.x) {
                const int32_t u = __ldcg(big + k);
                const int64_t b = __ldg(off + u), e = __ldg(off + u + 1);
                if (e - b > 4 * (int64_t)blockDim.x) continue;
                const int32_t pu = pmap ? __ldg(pmap + u) : u;
                for (int64_t j0 = b + threadIdx.x - lane; j0 < e; j0 += blockDim.x) {
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
            for (int k = 0; k < nbig; ++k) {
                const int32_t u = __ldcg(big + k);
                const int64_t b = __ldg(off + u), e = __ldg(off + u + 1);
                if (e - b <= 4 * (int64_t)blockDim.x) continue;
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
        unsigned long long cv[8];
        for (int i = 0; i < 8; ++i) cv[i] = __ldcg(cnt + i);
        LevelRec r{};
        r.n_f = c.n_f;
        r.m_f = c.m_f;
        r.m_u = m_u;
        r.dir = c.dir;
        r.ts = ts;
        r.k0 = ts;
        const bool cont = step_finish(c, r, cv);
        r.k1 = r.te;
        if (gtid == 0) {
            lrec[c.d - 1] = r;
            unsigned long long* z = cnt3 + 16 * ((c.d + 1) % 3);   // the set of level d + 2
            for (int i = 0; i < 16; ++i) z[i] = 0;
            if (!cont) *ctl = c;
        }
        if (!cont) break;
    }
    // the output pass in the same kernel (saves two launches per search on small graphs)
    if (po.mode) {
        if (po.mode == 2) {   // degree-reindexed: reset unreached records, then the permuted pass
            mark_unreached_body(visited, po.skip, po.n_active, rec);
            grid.sync();
            emit_perm_body(rec, po.label, po.n, po.n_active, c.root_i, po.depth, po.parent);
        } else {
            emit_body(visited, po.skip, rec, po.n, c.root_i, po.depth, po.parent);
        }
    }
}

