// Tiled top-down step for hub frontiers (Alg. 1 TD branch P:87-97 on one GPU with the
// section 3.4 degree reindex).  Included once, inside namespace bfsb::{anonymous},
// by bfs.cu (single translation unit).
//
// Why: the top-down levels whose frontier holds hubs (m_f = 10^7..10^9 arcs from
// 10^3..10^5 vertices) are bound by random L2 probes and atomicOr claims on the
// visited bitmap -- one per arc, ~100 G/s -- and by the partial-sector writes of
// scattered records (a DRAM read-modify-write each), far below the 4-byte-per-arc
// streaming rate of HBM.
//
// How: the reindexed labels [0, n_active) are cut into T tiles of about equal arc mass
// (sum of degrees), each at most BFS_TILE_WORDS visited words.  For every HEAVY row
// (labels [0, nh): the degree reindex puts the highest degrees first) a build-time
// table bnd[u][t] holds the position in u's row of its first arc whose target lies in
// tile t (rows are sorted ascending, so the arcs into one tile are contiguous).  A
// top-down step with m_f >= BFS_TILE_MIN arcs runs in tile mode:
//   light frontier vertices (label >= nh): the edge-balanced claim-only expansion
//     (k_scan_dev masks the heavy rows' degrees and lists the heavy vertices); its
//     winners log (vertex, parent) into the bucket of their (tile, window);
//   heavy frontier vertices: k_td_tile, one CTA per tile (hub tiles split over several
//     CTAs): the tile's visited words go to shared memory, the CTA streams the heavy
//     frontier rows' segments into its tile, probes and claims in shared memory
//     (atomicOr: exact winners), logs its winners per window, stores the words back;
//   k_tile_rec: per (tile, window) the logged parents go to shared memory and the
//     window's records are stored in vertex order, a whole 32-byte sector at a time;
//   k_td_finish: winners = visited & ~snapshot in vertex order (degrees, queue, n_f,
//     m_f), as for every claim-only step.
// The set of winners is the set a plain top-down step discovers (every arc of F(d) is
// examined once, claims are exact), so depths and every per-step counter are
// unchanged; parents are frontier neighbours (Alg. 1 P:95 "parent = u").

constexpr int kTileThreads = 512;
constexpr int kTileItems = 8;               // consecutive arcs per thread per round
constexpr int kTileMaxWordsDefault = 16384; // 2^19 labels, 64 KB of shared memory

// tile of label v: largest t with ts[t] <= v (ts ascending, ts[0] = 0)
__device__ __forceinline__ int tile_of(const int32_t* ts, int T, int32_t v) {
    int a = 0, b = T - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (ts[m] <= v) a = m;
        else b = m - 1;
    }
    return a;
}

// bnd[u*(T+1) + t] = arcs of heavy row u with target < ts[t], t in [0, T]; warp per row.
// Every entry is written exactly once: the entries of the tiles from the previous
// arc's tile (exclusive) to this arc's tile (inclusive) get this arc's position.
__global__ void k_tile_bnd(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                           const int32_t* __restrict__ ts_g, int T, int64_t nh, int32_t* __restrict__ bnd) {
    extern __shared__ int32_t s_ts[];
    for (int i = threadIdx.x; i <= T; i += blockDim.x) s_ts[i] = ts_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = gw; u < nh; u += nw) {
        const int64_t rb = off[u], re = off[u + 1];
        int32_t* row = bnd + u * (int64_t)(T + 1);
        int prev = -1;   // tile of the previous arc (-1 before the first)
        for (int64_t j0 = rb; j0 < re; j0 += 32) {
            const int64_t j = j0 + lane;
            const int tt = j < re ? tile_of(s_ts, T, __ldg(adj + j)) : T;
            int tp = __shfl_up_sync(kFull, tt, 1);
            if (lane == 0) tp = prev;
            if (j < re)
                for (int t = tp + 1; t <= tt; ++t) row[t] = (int32_t)(j - rb);
            prev = __shfl_sync(kFull, tt, 31);
            if (j0 + 32 >= re) {   // the last arc's lane fills the tiles after it
                const int last = (int)((re - 1 - j0) & 31);
                const int tl = __shfl_sync(kFull, tt, last);
                if (lane == 0)
                    for (int t = tl + 1; t <= T; ++t) row[t] = (int32_t)(re - rb);
            }
        }
        if (re == rb && lane == 0)
            for (int t = 0; t <= T; ++t) row[t] = 0;
    }
}

__global__ void k_gather_stride(const int64_t* __restrict__ off, int64_t step, int64_t K, int64_t* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = off[k * step];
}

// Records of a tile-mode step.  A scattered 8-byte record store is a partial-sector
// write, which DRAM serves as a 32-byte read plus a 32-byte write; at 10^7..10^8
// winners per step that costs more than the claims.  So the tile kernel logs each
// winner's (vertex, parent) in its unit's log, one bucket per 2^kWinShift-label window
// of the tile (appends to a bucket are sequential, so its sectors fill completely),
// and k_tile_rec stores each window's records in vertex order a whole sector at a time.
constexpr int kWinShift = 14;
constexpr int kWin = 1 << kWinShift;
constexpr int kMaxWin = 128;   // windows per tile (tiles of at most kMaxWin * kWin labels)
struct TileLog {
    int2* pool;                // unit u's bucket k: pool[base[u] + k * kWin ...]
    const int64_t* base;       // [units]
    unsigned* cnt;             // [units * kMaxWin] entries per bucket
    // winners of the light-row expansion (k_td_expand): one bucket per (tile, window)
    int2* lpool;               // [nwl * kWin]
    unsigned* lcnt;            // [nwl]
    const int32_t* ts;         // [T + 1] tile starts
    const int32_t* wf;         // [T] first (tile, window) index of each tile
    int T;
};

// light-row winner's record into its (tile, window) bucket; every lane of the calling
// (possibly partial) warp must call it, `win` says whether it has a record
__device__ __forceinline__ int light_window(const TileLog& lg, int32_t v) {
    int t = 0, hi_ = lg.T - 1;   // tile of v (global starts: binary search)
    while (t < hi_) {
        const int m = (t + hi_ + 1) >> 1;
        if (__ldg(lg.ts + m) <= v) t = m;
        else hi_ = m - 1;
    }
    return __ldg(lg.wf + t) + ((v - __ldg(lg.ts + t)) >> kWinShift);
}
// All kN items of a thread at once: the windows first, then one warp-aggregated
// atomicAdd per (item, window group) with every item's atomic in flight before any
// result is used, then the stores -- one atomic round trip per call instead of kN.
template <int kN>
__device__ __forceinline__ void light_log_all(const TileLog& lg, const bool (&win)[kN], const int32_t (&v)[kN],
                                              const int32_t (&par)[kN]) {
    const unsigned act = __activemask();
    const int lane = threadIdx.x & 31;
    int w[kN];
#pragma unroll
    for (int j = 0; j < kN; ++j) w[j] = win[j] ? light_window(lg, v[j]) : 0;
    unsigned peers[kN], base[kN];
#pragma unroll
    for (int j = 0; j < kN; ++j) {
        const unsigned m = __ballot_sync(act, win[j]);
        peers[j] = 0u;
        base[j] = 0u;
        if (win[j]) {
            peers[j] = __match_any_sync(m, w[j]);
            if (lane == __ffs(peers[j]) - 1) base[j] = atomicAdd(lg.lcnt + w[j], (unsigned)__popc(peers[j]));
        }
    }
#pragma unroll
    for (int j = 0; j < kN; ++j) {
        if (win[j]) {
            const unsigned pos = __shfl_sync(peers[j], base[j], __ffs(peers[j]) - 1) + __popc(peers[j] & lanemask_lt());
            lg.lpool[((int64_t)w[j] << kWinShift) + pos] = make_int2(v[j], par[j]);
        }
    }
}

// The heavy frontier vertices (label < nh) of the current queue into hlist (count
// *hcount, zeroed by the prologue): warp-aggregated appends.  ctl == nullptr: host loop,
// qa is the queue and F its length.
__global__ void k_tile_list(const Ctl* ctl, Queue qa, Queue qb, int64_t F, int64_t nh, int32_t* __restrict__ hlist,
                            unsigned* __restrict__ hcount) {
    const int32_t* qv = qa.v;
    if (ctl) {
        if (!ctl->tile) return;
        qv = ctl->qsel ? qb.v : qa.v;
        F = ctl->n_f;
    }
    const int lane = threadIdx.x & 31;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < F;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b0 + lane;
        const int32_t u = i < F ? __ldg(qv + i) : INT32_MAX;
        const bool heavy = u < nh;
        const unsigned m = __ballot_sync(kFull, heavy);
        if (!m) continue;
        unsigned pos = 0;
        if (lane == __ffs(m) - 1) pos = atomicAdd(hcount, (unsigned)__popc(m));
        pos = __shfl_sync(kFull, pos, __ffs(m) - 1);
        if (heavy) hlist[pos + __popc(m & lanemask_lt())] = u;
    }
}

// One CTA per work unit (grid = number of units).  A unit is (tile t, part s of S):
// a tile whose arc mass exceeds the per-unit target (the hub labels) is split over S
// CTAs, part s taking heavy-list entries s, s + S, ...; each part claims in its own
// shared copy and merges its new bits into `visited` with atomicOr (a vertex two parts
// both claim is logged twice with two valid same-depth parents; k_td_finish counts it
// once).  Unit encoding: unit[i] = (t, s | S << 16).  Tile mode only (ctl->tile);
// ctl == nullptr: host loop.
__global__ void __launch_bounds__(kTileThreads, 2)
k_td_tile(const Ctl* ctl, const int32_t* __restrict__ ts, int T, const int2* __restrict__ unit,
          const int32_t* __restrict__ bnd, const int32_t* __restrict__ hlist, const unsigned* __restrict__ hcount,
          const int64_t* __restrict__ off, const int32_t* __restrict__ adj, uint32_t* __restrict__ visited,
          const int32_t* __restrict__ pmap, TileLog lg, LevelRec* lrec) {
    extern __shared__ uint32_t s_vis[];   // [nw] live words; split units: [nw, 2nw) the words as loaded
    __shared__ int64_t s_base[kTileThreads];
    __shared__ int32_t s_pre[kTileThreads + 1];
    __shared__ int32_t s_par[kTileThreads];
    __shared__ int32_t s_warp[kTileThreads / 32];
    __shared__ unsigned s_wc[kMaxWin];
    if (ctl) {
        if (!ctl->tile) return;
        stamp_begin(lrec, ctl);
    }
    const int2 un = unit[blockIdx.x];
    const int t = un.x, part = un.y & 0xffff, nparts = un.y >> 16;
    const int32_t a = ts[t], b = ts[t + 1];
    const int64_t wa = a >> 5;
    const int nw = (b - a) >> 5;
    const int nwin = (b - a + kWin - 1) >> kWinShift;
    for (int i = threadIdx.x; i < nw; i += kTileThreads) {
        const uint32_t x = __ldcg(visited + wa + i);
        s_vis[i] = x;
        if (nparts > 1) s_vis[nw + i] = x;
    }
    for (int i = threadIdx.x; i < nwin; i += kTileThreads) s_wc[i] = 0u;
    int2* const logb = lg.pool + lg.base[blockIdx.x];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t H = (int64_t)*hcount;
    const int64_t stride = T + 1;
    const int64_t step = (int64_t)kTileThreads * nparts;
    // segment of heavy-list entry i in this tile: (len, address of its first arc, parent label)
    auto seg = [&](int64_t i, int32_t& len, int64_t& base, int32_t& par) {
        len = 0;
        base = 0;
        par = 0;
        if (i < H) {
            const int32_t u = __ldg(hlist + i);
            const int32_t* row = bnd + (int64_t)u * stride + t;
            const int32_t s0 = __ldg(row), e0 = __ldg(row + 1);
            len = e0 - s0;
            if (len > 0) {
                base = __ldg(off + u) + s0;
                par = pmap ? __ldg(pmap + u) : u;
            }
        }
    };
    int32_t len, par;
    int64_t base;
    seg((int64_t)threadIdx.x * nparts + part, len, base, par);
    __syncthreads();
    for (int64_t b0 = 0; b0 < H; b0 += step) {
        // the next batch's segments are loaded while this one is expanded
        int32_t nlen, npar;
        int64_t nbase;
        seg(b0 + step + (int64_t)threadIdx.x * nparts + part, nlen, nbase, npar);
        // block exclusive scan of len
        int inc = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += y;
        }
        if (lane == 31) s_warp[wid] = inc;
        __syncthreads();
        if (threadIdx.x < 32) {
            const int x = threadIdx.x < kTileThreads / 32 ? s_warp[threadIdx.x] : 0;
            int xi = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(kFull, xi, d);
                if (lane >= d) xi += y;
            }
            if (threadIdx.x < kTileThreads / 32) s_warp[threadIdx.x] = xi - x;
            if (threadIdx.x == 31) s_pre[kTileThreads] = xi;
        }
        __syncthreads();
        const int32_t pre = s_warp[wid] + inc - len;
        s_pre[threadIdx.x] = pre;
        s_base[threadIdx.x] = base - pre;   // address of arc k of this segment: s_base + k
        s_par[threadIdx.x] = par;
        __syncthreads();
        const int32_t L = s_pre[kTileThreads];
        for (int32_t k0 = threadIdx.x * kTileItems; k0 < L; k0 += kTileThreads * kTileItems) {
            // segment of arc k0: largest j with s_pre[j] <= k0 (a non-empty segment)
            int lo_ = 0, hi_ = kTileThreads - 1;
            while (lo_ < hi_) {
                const int m = (lo_ + hi_ + 1) >> 1;
                if (s_pre[m] <= k0) lo_ = m;
                else hi_ = m - 1;
            }
            int j = lo_;
            int32_t nxt = s_pre[j + 1];
            int64_t sb = s_base[j];
            int32_t v[kTileItems], pj[kTileItems];
#pragma unroll
            for (int q = 0; q < kTileItems; ++q) {
                const int32_t k = k0 + q;
                v[q] = -1;
                pj[q] = j;
                if (k < L) {
                    while (k >= nxt) {
                        ++j;
                        nxt = s_pre[j + 1];
                        sb = s_base[j];
                    }
                    v[q] = __ldg(adj + sb + k);
                    pj[q] = j;
                }
            }
#pragma unroll
            for (int q = 0; q < kTileItems; ++q) {
                if (v[q] < 0) continue;
                const int32_t lv = v[q] - a;
                const uint32_t bit = 1u << (lv & 31);
                uint32_t* wp = s_vis + (lv >> 5);
                if (!(*wp & bit) && !(atomicOr(wp, bit) & bit)) {
                    const int wk = lv >> kWinShift;
                    const unsigned pos = atomicAdd(&s_wc[wk], 1u);
                    __stcg(logb + ((int64_t)wk << kWinShift) + pos, make_int2(v[q], s_par[pj[q]]));
                }
            }
        }
        len = nlen;
        base = nbase;
        par = npar;
        __syncthreads();   // s_pre / s_base / s_par are rewritten by the next batch
    }
    if (nparts == 1) {
        for (int i = threadIdx.x; i < nw; i += kTileThreads) visited[wa + i] = s_vis[i];
    } else {
        for (int i = threadIdx.x; i < nw; i += kTileThreads) {
            const uint32_t nb = s_vis[i] & ~s_vis[nw + i];
            if (nb) atomicOr(visited + wa + i, nb);
        }
    }
    for (int i = threadIdx.x; i < nwin; i += kTileThreads) lg.cnt[(int64_t)blockIdx.x * kMaxWin + i] = s_wc[i];
    if (ctl && lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}

// Records of a tile-mode step, one CTA per (tile, window) = wl[i]: the window's
// buckets (one per unit of the tile, plus the light-row bucket) put the winners'
// parents into shared memory, then the window's records are stored in vertex order a
// whole 32-byte sector (4 vertices) at a time.  A sector with a winner also rewrites
// its vertices visited before (their old record) and fills its unvisited ones with
// (-1, -1) (a later discovery or k_mark_unreached overwrites those).  Winners =
// visited & ~snapshot; every winner is in some bucket.  fu[t] = first unit of tile t.
constexpr int kWinThreads = 512;
__global__ void __launch_bounds__(kWinThreads)
k_tile_rec(const Ctl* ctl, int32_t level_in, const int2* __restrict__ wl, const int32_t* __restrict__ fu,
           const int2* __restrict__ unit, TileLog lg, const uint32_t* __restrict__ visited,
           const uint32_t* __restrict__ f0, const uint32_t* __restrict__ f1, int2* __restrict__ rec, LevelRec* lrec) {
    extern __shared__ int32_t s_p[];   // [kWin] parent of each winner of the window
    const uint32_t* snap = f0;
    int32_t level = level_in;
    if (ctl) {
        if (!ctl->tile) return;
        snap = ctl->fsel ? f0 : f1;
        level = ctl->d + 1;
    }
    const int2 tw = wl[blockIdx.x];
    const int t = tw.x, k = tw.y;
    const int32_t v0 = lg.ts[t] + (k << kWinShift);
    const int32_t v1 = min(lg.ts[t + 1], v0 + kWin);
    const int u0 = fu[t], parts = unit[u0].y >> 16;
    unsigned any = lg.lcnt[blockIdx.x];
    for (int u = u0; u < u0 + parts; ++u) any |= lg.cnt[(int64_t)u * kMaxWin + k];
    if (!any) return;   // no winner in this window
    for (int i = threadIdx.x; i < (v1 - v0); i += kWinThreads) s_p[i] = -1;
    __syncthreads();
    for (int u = u0; u <= u0 + parts; ++u) {
        const bool light = u == u0 + parts;
        const unsigned n = light ? lg.lcnt[blockIdx.x] : lg.cnt[(int64_t)u * kMaxWin + k];
        const int2* P = light ? lg.lpool + ((int64_t)blockIdx.x << kWinShift)
                              : lg.pool + lg.base[u] + ((int64_t)k << kWinShift);
        // a vertex two parts of a split tile both claimed has two (valid) entries: the
        // larger parent label wins, deterministically.  4 entries per thread in flight.
        for (unsigned i0 = threadIdx.x; i0 < n; i0 += 4 * kWinThreads) {
            int2 e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned i = i0 + q * kWinThreads;
                e[q] = i < n ? __ldcs(P + i) : make_int2(-1, 0);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (e[q].x >= 0) atomicMax(s_p + (e[q].x - v0), e[q].y);
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nwd = (v1 - v0) >> 5;
    // a warp takes 32 words at a time: one coalesced load of each bitmap, then word by word
    for (int wb = wid * 32; wb < nwd; wb += kWinThreads) {
        const int64_t gw = (v0 >> 5) + wb + lane;
        uint32_t sbl = 0, nbl = 0;
        if (wb + lane < nwd) {
            sbl = __ldcg(snap + gw);
            nbl = __ldcg(visited + gw) & ~sbl;
        }
        unsigned todo = __ballot_sync(kFull, nbl != 0u);
        while (todo) {
            const int q = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t nb = __shfl_sync(kFull, nbl, q), sb = __shfl_sync(kFull, sbl, q);
            if (!((nb >> (lane & ~3)) & 0xfu)) continue;
            const int i = (wb + q) * 32 + lane;
            const int64_t v = (int64_t)v0 + i;
            int2 r = make_int2(-1, -1);
            if ((nb >> lane) & 1u) r = make_int2(level, s_p[i]);
            else if ((sb >> lane) & 1u) r = __ldcg(rec + v);
            __stcs(rec + v, r);
        }
    }
    if (ctl && lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}
