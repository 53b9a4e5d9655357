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

#include "bfs_common.cuh"
#include "td_tile.cuh"
#include "bfs_steps.cuh"
#include "bfs_loop.cuh"

int grid_for(int64_t items, int threads, int per_sm = 8) {
    const int64_t b = (items + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    return (int)std::max<int64_t>(1, std::min(b, cap));
}

// Planes of bottom-up second-probe blocks used (arcs 1+4p..4+4p of every row,
// build.cu k_nb4): all that were built unless BFS_BU_NB4 asks for fewer (tuning only)
static int bu_nbp(const bfs_graph_s* g) {
    const char* e = getenv("BFS_BU_NB4");
    const int want = e ? std::max(0, atoi(e)) : g->nb4_planes;
    return g->nb4.p ? std::min(want, g->nb4_planes) : 0;
}
static const int4* bu_nb4(const bfs_graph_s* g) { return bu_nbp(g) ? g->nb4.p : nullptr; }

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

// p ranks: top-down steps whose global m_f reaches this push bitmaps instead of (vertex,
// parent) claim lists: 8 bytes per claim against (p - 1) slices of nb / 8 bytes; m_f
// bounds the claims, so n / 64 arcs (BFS_TD_BITMAP_MIN overrides: tests, tuning)
static int64_t td_bitmap_min(const bfs_graph_s* g) {
    const char* e = getenv("BFS_TD_BITMAP_MIN");
    return e ? atoll(e) : std::max<int64_t>(1, g->n / 64);
}

// top-down steps with at least this many arcs run claim-only + k_td_finish
// (single partition; BFS_TD_CLAIM_MIN overrides: tuning only)
static int64_t td_claim_min() {
    const char* e = getenv("BFS_TD_CLAIM_MIN");
    return e ? atoll(e) : (int64_t)1 << 26;
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

// tiled top-down (td_tile.cuh) knobs; the BFS_TILE* variables are for tuning and tests
static int64_t env_i64(const char* name, int64_t dflt) {
    const char* e = getenv(name);
    return e && *e ? atoll(e) : dflt;
}
// top-down steps with at least this many arcs run tiled when the graph has a tile index
static int64_t tile_min_setting() { return env_i64("BFS_TILE_MIN", (int64_t)1 << 24); }
// top-down steps with at most this many arcs run as one kernel on the device loop
// (k_td_small; BFS_TD_SMALL=-1 disables it)
// top-down steps of at most this many arcs (and <= 64 per frontier vertex) run as the one
// kernel k_td_small; 2^18 from the round-2 sweep (ER22 +2.2%, K26 +0.6%, K29 +0.1% vs 2^15;
// 2^22 loses: profiles/r02_td_small_sweep.txt)
static int64_t td_small_setting() { return env_i64("BFS_TD_SMALL", (int64_t)1 << 18); }

TileLog tile_log(const bfs_graph_s* g) {
    return TileLog{g->tile_pool.p, g->tile_ubase.p, g->tile_ucnt.p, g->tile_lpool.p, g->tile_lcnt.p,
                   g->tile_start.p, g->tile_wf.p, g->tile_T};
}

}  // namespace

// The tile index of td_tile.cuh for a degree-reindexed graph on one GPU: heavy rows
// [0, nh) are those of degree >= H (the reindex orders labels by decreasing degree, so
// they form a prefix); tiles of about equal arc mass, each at most `maxw` visited
// words; per heavy row and tile the first arc into the tile (k_tile_bnd).
void bfs_build_tiles(bfs_graph_s* g) {
    g->tile_T = 0;
    g->tile_nh = 0;
    if (!active_range(g) || env_i64("BFS_TILE", 1) == 0) return;
    cudaStream_t s = g->stream;
    const int64_t na = g->n_active;
    if (na < 64) return;
    auto degree = [&](int64_t v) {
        int64_t b[2];
        BFS_CUDA(cudaMemcpy(b, g->off.p + v, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
        return b[1] - b[0];
    };
    // offsets sampled at every word boundary (32 labels), plus the end
    const int64_t step = 32;
    const int64_t K = (na + step - 1) / step;
    std::vector<int64_t> so((size_t)K + 1);
    {
        DevBuf<int64_t> d;
        d.alloc((size_t)K, s);
        k_gather_stride<<<grid_for(K, 256), 256, 0, s>>>(g->off.p, step, K, d.p);
        BFS_CHECK_LAUNCH();
        BFS_CUDA(cudaMemcpyAsync(so.data(), d.p, (size_t)K * 8, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaMemcpyAsync(&so[K], g->off.p + na, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
    }
    const int64_t maxw = std::max<int64_t>(1, std::min<int64_t>(env_i64("BFS_TILE_WORDS", kTileMaxWordsDefault),
                                                                std::min(48 * 1024, kMaxWin * kWin / 32)));
    const int64_t vmax = maxw * 32;
    const int64_t target = std::max<int64_t>(1, env_i64("BFS_TILE_COUNT", 4 * (int64_t)num_sms()));
    const int64_t mass = std::max<int64_t>(1, (so[K] - so[0]) / target);
    std::vector<int32_t> ts{0};
    int64_t cur = 0;
    for (int64_t k = 1; k < K; ++k)
        if (so[k] - so[cur] >= mass || (k + 1 - cur) * step > vmax) {
            ts.push_back((int32_t)(k * step));
            cur = k;
        }
    ts.push_back((int32_t)(words_of(na) * 32));
    const int T = (int)ts.size() - 1;
    if (T > 16384) return;   // k_tile_bnd keeps the starts in shared memory
    // work units: a tile heavier than the mass target is split over up to 64 CTAs
    // (only tiles of at most maxw/2 words: a split part keeps a second copy of its words)
    std::vector<int2> units;
    int64_t wmax = 0;
    for (int t = 0; t < T; ++t) {
        const int64_t w = (ts[t + 1] - ts[t]) / 32;
        const int64_t m = so[std::min<int64_t>(K, ts[t + 1] / step)] - so[ts[t] / step];
        int parts = (int)std::min<int64_t>(64, std::max<int64_t>(1, (m + mass - 1) / mass));
        if (2 * w > maxw) parts = 1;
        for (int q = 0; q < parts; ++q) units.push_back(make_int2(t, q | (parts << 16)));
        wmax = std::max<int64_t>(wmax, parts > 1 ? 2 * w : w);
    }
    // heavy rows: degree >= H (binary search on the non-increasing degrees); H doubles
    // until the table fits the budget
    const int64_t budget = env_i64("BFS_TILE_BUDGET", (int64_t)8 << 30);
    int64_t H = std::max<int64_t>(1, env_i64("BFS_TILE_H", 4096)), nh = 0;
    for (;;) {
        int64_t lo = 0, hi = na;   // first label with degree < H
        while (lo < hi) {
            const int64_t m = (lo + hi) / 2;
            if (degree(m) >= H) lo = m + 1;
            else hi = m;
        }
        nh = lo;
        if (nh * (int64_t)(T + 1) * 4 <= budget) break;
        H *= 2;
    }
    if (nh == 0) return;
    cudaEvent_t e0, e1;
    BFS_CUDA(cudaEventCreate(&e0));
    BFS_CUDA(cudaEventCreate(&e1));
    BFS_CUDA(cudaEventRecord(e0, s));
    g->tile_start.alloc((size_t)T + 1, s);
    BFS_CUDA(cudaMemcpyAsync(g->tile_start.p, ts.data(), (size_t)(T + 1) * 4, cudaMemcpyHostToDevice, s));
    g->tile_unit.alloc(units.size(), s);
    BFS_CUDA(cudaMemcpyAsync(g->tile_unit.p, units.data(), units.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    g->tile_bnd.alloc((size_t)nh * (T + 1), s);
    g->tile_hlist.alloc((size_t)nh, s);
    g->tile_hcnt.alloc(1, s);
    // record log: unit u owns one kWin-entry bucket per window of its tile
    {
        std::vector<int64_t> ub(units.size());
        std::vector<int32_t> fu((size_t)T, -1), wf((size_t)T, 0);
        std::vector<int2> wl;
        int64_t tot = 0;
        for (size_t u = 0; u < units.size(); ++u) {
            const int t = units[u].x;
            const int64_t nwin = ((int64_t)ts[t + 1] - ts[t] + kWin - 1) / kWin;
            ub[u] = tot;
            tot += nwin * kWin;
            if (fu[t] < 0) {
                fu[t] = (int32_t)u;
                wf[t] = (int32_t)wl.size();
                for (int k = 0; k < nwin; ++k) wl.push_back(make_int2(t, k));
            }
        }
        g->tile_pool.alloc((size_t)tot, s);
        g->tile_ubase.alloc(ub.size(), s);
        g->tile_ucnt.alloc(units.size() * kMaxWin, s);
        g->tile_wl.alloc(wl.size(), s);
        g->tile_fu.alloc((size_t)T, s);
        g->tile_wf.alloc((size_t)T, s);
        g->tile_lpool.alloc(wl.size() * kWin, s);
        g->tile_lcnt.alloc(wl.size(), s);
        BFS_CUDA(cudaMemcpyAsync(g->tile_wf.p, wf.data(), wf.size() * 4, cudaMemcpyHostToDevice, s));
        BFS_CUDA(cudaMemcpyAsync(g->tile_ubase.p, ub.data(), ub.size() * 8, cudaMemcpyHostToDevice, s));
        BFS_CUDA(cudaMemcpyAsync(g->tile_wl.p, wl.data(), wl.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
        BFS_CUDA(cudaMemcpyAsync(g->tile_fu.p, fu.data(), fu.size() * 4, cudaMemcpyHostToDevice, s));
        BFS_CUDA(cudaStreamSynchronize(s));   // the host vectors go out of scope
        g->tile_nwl = (int)wl.size();
    }
    BFS_CUDA(cudaFuncSetAttribute(k_tile_rec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kWin * 4)));
    const size_t smem_bnd = (size_t)(T + 1) * 4;
    if (smem_bnd > 48 * 1024)
        BFS_CUDA(cudaFuncSetAttribute(k_tile_bnd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bnd));
    k_tile_bnd<<<grid_for(nh * 32, 256), 256, smem_bnd, s>>>(g->off.p, g->adj.p, g->tile_start.p, T, nh, g->tile_bnd.p);
    BFS_CHECK_LAUNCH();
    BFS_CUDA(cudaFuncSetAttribute(k_td_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wmax * 4)));
    BFS_CUDA(cudaEventRecord(e1, s));
    BFS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    BFS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    g->tile_build_ms = ms;
    g->tile_T = T;
    g->tile_units = (int)units.size();
    g->tile_nh = nh;
    g->tile_maxw = (int)wmax;
}

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
        const size_t want = std::max(count, b.count * 2);   // geometric growth: few reallocations
        b.reset();
        b.alloc(want, s);
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
        // loop state and step records in one buffer: one read-back per search
        g->ctl.alloc((sizeof(Ctl) + (size_t)kGraphMaxLevels * sizeof(LevelRec)) / 8, s);
        BFS_CUDA(cudaMallocHost(&g->h_ctl, sizeof(Ctl) + kLrecHead * sizeof(LevelRec)));
        BFS_CUDA(cudaMallocHost(&g->h_lrec, (size_t)kGraphMaxLevels * sizeof(LevelRec)));
    }
    Ctl* ctl = reinterpret_cast<Ctl*>(g->ctl.p);
    LevelRec* lrec = reinterpret_cast<LevelRec*>(g->ctl.p + sizeof(Ctl) / 8);
    unsigned long long* cnt = (unsigned long long*)g->cnt.p;
    unsigned long long* tstate = (unsigned long long*)g->tstate.p;
    const Queue qa{g->q0.p, g->qd0.p}, qb{g->q1.p, g->qd1.p};
    const int32_t* pmap = g->reindexed ? g->ilabel.p : nullptr;
    const int sms = num_sms();
    const dim3 g8(sms * 8), t256(256);

    cudaGraph_t G;
    BFS_CUDA(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle h_loop;
    BFS_CUDA(cudaGraphConditionalHandleCreate(&h_loop, G, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t n_while, n_sw;
    cudaGraph_t B = add_cond(G, {}, h_loop, cudaGraphCondTypeWhile, &n_while);
    // one SWITCH node per level: body 0 small top-down, 1 top-down, 2 bottom-up after a
    // queue -> bitmap conversion, 3 bottom-up (k_step selects; 4 = none, the last call)
    cudaGraphConditionalHandle h_sw;
    BFS_CUDA(cudaGraphConditionalHandleCreate(&h_sw, B, kStepNone, cudaGraphCondAssignDefault));
    cudaGraphNode_t n_begin = add_kernel(B, {}, k_step, dim3(1), dim3(1), 0, ctl, lrec, cnt, h_loop, h_sw);
    cudaGraph_t SW[4];
    {
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h_sw;
        cp.conditional.type = cudaGraphCondTypeSwitch;
        cp.conditional.size = 4;
        BFS_CUDA(cudaGraphAddNode(&n_sw, B, &n_begin, 1, &cp));
        for (int i = 0; i < 4; ++i) SW[i] = cp.conditional.phGraph_out[i];
    }
    cudaGraph_t S = SW[kStepSmallTd], T = SW[kStepTd], C = SW[kStepBuConv], U = SW[kStepBu];
    // small top-down step: one kernel
    add_kernel(S, {}, k_td_small, dim3(sms * 4), t256, 0, (const Ctl*)ctl, qa, qb, (const uint32_t*)g->front.p,
               (const uint32_t*)g->next.p, words, (const int64_t*)g->off.p, (const int32_t*)g->adj.p,
               (const int2*)g->head.p, g->visited.p, g->rec.p, pmap, cnt, lrec);
    // top-down body
    unsigned* hcnt = g->tile_T ? g->tile_hcnt.p : nullptr;
    const TileLog lg = tile_log(g);
    cudaGraphConditionalHandle h_tile{};
    if (g->tile_T) BFS_CUDA(cudaGraphConditionalHandleCreate(&h_tile, T, 0, cudaGraphCondAssignDefault));
    cudaGraphNode_t t1 = add_kernel(T, {}, k_td_prep, g8, t256, 0, ctl, g->front.p, g->next.p, words, g->head.p, qa, qb,
                                    cnt, tstate, g->tctr.p, (const uint32_t*)g->visited.p, hcnt, g->tile_lcnt.p,
                                    (int64_t)g->tile_nwl, h_tile, g->tile_T ? 1 : 0);
    cudaGraphNode_t t2 = add_kernel(T, {t1}, k_scan_dev, g8, dim3(kScanThreads), 0, ctl, qa, qb, (int64_t)0, g->prefix.p,
                                    tstate, g->tctr.p, g->tile_nh, 0);
    cudaGraphNode_t t3 = add_kernel(T, {t2}, k_td_chunk_starts, g8, t256, 0, g->prefix.p, (int64_t)0, (int64_t)0,
                                    g->scratch64.p, ctl);
    cudaGraphNode_t t4 = add_kernel(T, {t3}, k_td_expand<false>, dim3(td_resident_grid<false>()), dim3(kTdThreads), 0,
                                    qa, g->prefix.p, g->scratch64.p, (int64_t)0, (int64_t)0, g->off.p, g->adj.p,
                                    g->visited.p, g->rec.p, pmap, qb, g->head.p, cnt, (int32_t)0, g->lo, g->hi, Remote{},
                                    ctl, lrec, -1, lg);
    if (g->tile_T) {   // heavy frontier rows and the records of a tile-mode step (IF node set by k_td_prep)
        cudaGraphNode_t n_tile;
        cudaGraph_t TT = add_cond(T, {t4}, h_tile, cudaGraphCondTypeIf, &n_tile);
        cudaGraphNode_t tl = add_kernel(TT, {}, k_tile_list, g8, t256, 0, (const Ctl*)ctl, qa, qb, (int64_t)0,
                                        g->tile_nh, g->tile_hlist.p, hcnt);
        cudaGraphNode_t t5 = add_kernel(TT, {tl}, k_td_tile, dim3(g->tile_units), dim3(kTileThreads), (size_t)g->tile_maxw * 4,
                        (const Ctl*)ctl, (const int32_t*)g->tile_start.p, g->tile_T, (const int2*)g->tile_unit.p,
                        (const int32_t*)g->tile_bnd.p, (const int32_t*)g->tile_hlist.p, (const unsigned*)hcnt,
                        (const int64_t*)g->off.p, (const int32_t*)g->adj.p, g->visited.p, pmap, lg, lrec);
        add_kernel(TT, {t5}, k_tile_rec, dim3(g->tile_nwl), dim3(kWinThreads), (size_t)kWin * 4, (const Ctl*)ctl,
                        (int32_t)0, (const int2*)g->tile_wl.p, (const int32_t*)g->tile_fu.p,
                        (const int2*)g->tile_unit.p, lg, (const uint32_t*)g->visited.p, (const uint32_t*)g->front.p,
                        (const uint32_t*)g->next.p, g->rec.p, lrec);
        t4 = n_tile;
    }
    const int64_t nbatches = (words + 31) / 32;
    const int bu_grid = grid_for(nbatches * 32, kBuWarps * 32, kBuCtas);
    const int grab = (int)std::max<int64_t>(1, nbatches / ((int64_t)bu_grid * kBuWarps * 8));
    add_kernel(T, {t4}, k_td_finish_dev, g8, t256, 0, ctl, (const uint32_t*)g->visited.p, g->front.p, g->next.p, words,
               g->head.p, qa, qb, cnt);
    // bottom-up body
    // queue -> bitmap before a bottom-up step that follows a top-down one (IF node)
    cudaGraphNode_t u1 = add_kernel(C, {}, k_bu_prep, g8, t256, 0, ctl, g->front.p, g->next.p, words);
    cudaGraphNode_t u2 = add_kernel(C, {u1}, k_q2b_dev, g8, t256, 0, ctl, qa, qb, g->front.p, g->next.p);
    for (cudaGraph_t X : {C, U})
        add_kernel(X, X == C ? std::vector<cudaGraphNode_t>{u2} : std::vector<cudaGraphNode_t>{}, k_bu_batch,
                   dim3(bu_grid), dim3(kBuWarps * 32), 0, g->off.p, g->head.p, g->adj.p, g->visited.p, g->front.p,
                   g->next.p, g->rec.p, pmap, g->reindexed ? g->hpar.p : nullptr, bu_nb4(g), g->nb4_rows, bu_nbp(g),
                   words, g->lo, (int32_t)0, cnt, grab, bu_long_setting(), bu_dense_setting(), ctl, lrec);
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

// graphs up to this many arcs use the one-cluster search in auto mode (BFS_CLUSTER_MAX_ARCS):
// K16 (1.5 M arcs) 80 vs 95 us per search; at s20 (31 M arcs) the full-device wave wins
static int64_t cluster_max_arcs() {
    const char* e = getenv("BFS_CLUSTER_MAX_ARCS");
    return e ? atoll(e) : (int64_t)1 << 21;
}

static int pers_blocks_per_sm() {
    const char* e = getenv("BFS_PERSIST_BLOCKS");   // tuning only
    return e ? std::max(1, atoi(e)) : 1;
}

// co-resident CTAs of the persistent kernel (cooperative launch limit).
// BFS_PERSIST_GRID overrides it (tests: a grid too large to be co-resident must make
// the cooperative launch fail and the search run as the loop graph instead).
static int pers_grid() {
    if (const char* e = getenv("BFS_PERSIST_GRID")) return std::max(1, atoi(e));
    static const int gsz = [] {
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bfs_persistent<GridBar, kPersThreads>, kPersThreads,
                                                          0) != cudaSuccess ||
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
// CTAs of the one-cluster search (BFS_CLUSTER: tuning; 16 needs the non-portable
// cluster size, 8 is portable)
static int cluster_size() {
    const char* e = getenv("BFS_CLUSTER");
    return e ? std::max(1, std::min(16, atoi(e))) : 16;
}
constexpr int kClusterThreads = 1024;

static bool bfs_run_graph(bfs_graph_s* g, int64_t root, int32_t* od, int32_t* op, int32_t* parent_out,
                          int32_t* depth_out, int mode) {
    bool persistent = mode != 0;   // 1: one resident wave (grid barrier), 2: one thread-block cluster
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    if (persistent) {
        if (!g->ctl.p) {   // the state buffers (the graph itself is the fallback)
            build_loop_graph(g);
            g->loop_key = {bu_long_setting(), bu_dense_setting(), bu_nbp(g)};
        }
        if (!g->big.p) g->big.alloc((size_t)(g->arcs_local / kPersBig + 4), s);   // + 2 barrier words
        if (!g->pcnt.p) g->pcnt.alloc(48, s);
    }
    // the graph bakes the tuning knobs into its kernel arguments: rebuild if they changed
    const std::vector<int> key{bu_long_setting(), bu_dense_setting(), bu_nbp(g)};
    auto ensure_loop_graph = [&] {
        if (g->loop_exec && g->loop_key != key) {
            BFS_CUDA(cudaStreamSynchronize(s));
            cudaGraphExecDestroy(g->loop_exec);
            cudaGraphDestroy(g->loop_graph);
            g->loop_exec = nullptr;
            g->loop_graph = nullptr;
        }
        if (!g->loop_exec) build_loop_graph(g);
        g->loop_key = key;
    };
    if (!persistent) ensure_loop_graph();
    Ctl* ctl = reinterpret_cast<Ctl*>(g->ctl.p);
    const Queue qa{g->q0.p, g->qd0.p};
    const int64_t pw = reset_words(g);
    const bool lt = g->policy.level_times != 0;
    BFS_CUDA(cudaEventRecord(g->ev[0], s));
    const InitArgs ia{g->visited.p, g->skip.p, pw, root, g->reindexed ? g->label.p : nullptr, g->rec.p, qa, g->head.p,
                      (unsigned long long*)g->cnt.p, ctl, g->policy, g->n, g->arcs_global, kGraphMaxLevels,
                      td_claim_min(), (persistent || !g->tile_T) ? (int64_t)-1 : tile_min_setting(), td_small_setting(),
                      persistent ? (unsigned long long*)g->pcnt.p : nullptr,
                      persistent ? reinterpret_cast<unsigned*>(g->big.p + g->big.count - 2) : nullptr};
    // the one-cluster search runs the init itself (its barrier needs no memory words)
    const bool fused_init = mode == 2;
    if (!fused_init) {
        k_init_dev<<<grid_for(pw, 256), 256, 0, s>>>(ia);
        BFS_CHECK_LAUNCH();
    }
    BFS_CUDA(cudaEventRecord(g->ev[2], s));
    if (persistent) {
        const int64_t words = loop_words(g);
        const Queue qb{g->q1.p, g->qd1.p};
        LevelRec* lrec = reinterpret_cast<LevelRec*>(g->ctl.p + sizeof(Ctl) / 8);
        const int32_t* pmap = g->reindexed ? g->ilabel.p : nullptr;
        const int32_t* hpar = g->reindexed ? g->hpar.p : nullptr;
        // barrier words live in the tail of the big-row list buffer; the three counter sets
        // start at zero except what k_init_dev put in set 0
        // (zeroed by k_init_dev, which also put the root's counters in set 0)
        unsigned* bar = reinterpret_cast<unsigned*>(g->big.p + g->big.count - 2);
        // the grid barrier needs every CTA resident at once: a cooperative launch
        // guarantees it or fails (instead of hanging when other work holds SMs)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(pers_grid());
        cfg.blockDim = dim3(kPersThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const PersOut po{(od || op) ? (g->reindexed ? 2 : 1) : 0, g->skip.p, g->label.p, g->reindexed ? g->n : nl,
                         g->n_active, od, op};
        cudaError_t e;
        if (mode == 2) {
            // one cluster: hardware barrier.cluster between phases, guaranteed co-scheduled
            static const bool attr_ok = [] {
                const bool ok = cudaFuncSetAttribute(k_bfs_persistent<ClusterBar, kClusterThreads>,
                                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
                cudaGetLastError();
                return ok;
            }();
            cfg.gridDim = dim3(attr_ok ? cluster_size() : std::min(8, cluster_size()));
            cfg.blockDim = dim3(kClusterThreads);
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cfg.gridDim.x;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            e = cudaLaunchKernelEx(&cfg, k_bfs_persistent<ClusterBar, kClusterThreads>, (const int64_t*)g->off.p,
                                   (const int2*)g->head.p, (const int32_t*)g->adj.p, g->visited.p, g->front.p,
                                   g->next.p, words, g->rec.p, pmap, hpar, qa, qb, (unsigned long long*)g->pcnt.p,
                                   g->big.p, ctl, lrec, ClusterBar{}, po, ia, 1);
        } else {
            e = cudaLaunchKernelEx(&cfg, k_bfs_persistent<GridBar, kPersThreads>, (const int64_t*)g->off.p,
                                   (const int2*)g->head.p, (const int32_t*)g->adj.p, g->visited.p, g->front.p,
                                   g->next.p, words, g->rec.p, pmap, hpar, qa, qb, (unsigned long long*)g->pcnt.p,
                                   g->big.p, ctl, lrec, GridBar{bar, bar + 1}, po, ia, 0);
        }
        if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorLaunchOutOfResources ||
            e == cudaErrorInvalidClusterSize) {
            // the persistent grid cannot be co-resident now: the loop graph runs the
            // same steps from the state k_init_dev wrote
            cudaGetLastError();
            persistent = false;
            if (fused_init) {
                k_init_dev<<<grid_for(pw, 256), 256, 0, s>>>(ia);
                BFS_CHECK_LAUNCH();
            }
            ensure_loop_graph();
            BFS_CUDA(cudaGraphLaunch(g->loop_exec, s));
            ++g->coop_fallbacks;
        } else {
            BFS_CUDA(e);
        }
    } else {
        BFS_CUDA(cudaGraphLaunch(g->loop_exec, s));
    }
    BFS_CUDA(cudaEventRecord(g->ev[3], s));
    int64_t launches = (fused_init && persistent) ? 0 : 1;   // k_init_dev
    if ((od || op) && !persistent) {   // (the persistent search ran the output pass itself)
        const int64_t dw = words_of(g->reindexed ? g->n_active : nl);
        k_l2_demote<<<grid_for((dw + 31) / 32, 256), 256, 0, s>>>(g->front.p, g->next.p, dw);
        ++launches;
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
    BFS_CUDA(cudaMemcpyAsync(g->h_ctl, g->ctl.p, sizeof(Ctl) + kLrecHead * sizeof(LevelRec), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
    const Ctl c = *reinterpret_cast<const Ctl*>(g->h_ctl);
    if (c.overflow) return false;
    const LevelRec* R = reinterpret_cast<const LevelRec*>(g->h_ctl + sizeof(Ctl) / 8);
    if (c.d > kLrecHead) {   // a deep search: every record
        BFS_CUDA(cudaMemcpyAsync(g->h_lrec, g->ctl.p + sizeof(Ctl) / 8, (size_t)c.d * sizeof(LevelRec),
                                 cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        R = reinterpret_cast<const LevelRec*>(g->h_lrec);
    }
    // kernels the loop graph launched for step d (after its k_step)
    const int64_t tmin = g->tile_T ? tile_min_setting() : INT64_MAX, tsmall = td_small_setting(), cmin = td_claim_min();
    auto small = [&](int d) { return R[d].m_f <= tsmall && R[d].m_f <= 64 * R[d].n_f; };
    auto claimed = [&](int d) { return R[d].dir == 0 && !small(d) && (R[d].m_f >= cmin || R[d].m_f >= tmin); };
    auto step_kernels = [&](int d) -> int64_t {
        if (R[d].dir == 0) return small(d) ? 1 : 5 + (R[d].m_f >= tmin ? 3 : 0);
        const bool conv = d == 0 || (R[d - 1].dir == 0 && !claimed(d - 1));   // queue -> bitmap first
        return 1 + (conv ? 2 : 0);
    };
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
        launches += persistent ? 0 : 1 + step_kernels(d);
    }
    if (!persistent) ++launches;   // the last k_step, which ends the loop
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
    // level loop: 0 auto (one cluster for small graphs, the persistent kernel up to 2^22 arcs,
    // the loop graph above),
    // 1 host, 2 loop graph, 3 persistent kernel, 4 one-cluster search; p ranks always host-driven
    int loop = g->policy.loop;
    if (env_host_loop) loop = 1;
    if (loop == 0) loop = g->arcs_local <= cluster_max_arcs() ? 4 : g->arcs_local <= persist_max_arcs() ? 3 : 2;
    if (!mg && g->nparts == 1 && loop != 1) {
        if (bfs_run_graph(g, root, od, op, parent_out, depth_out, loop == 3 ? 1 : loop == 4 ? 2 : 0)) return;
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
    bool front_ok = false;   // `front` also holds the current frontier (after a claim-mode TD step)
    int dir = 0;  // 0 TD, 1 BU
    int64_t n_f = h[C_GLOBAL + C_NEXT], m_f = h[C_GLOBAL + C_MF];
    int64_t nf_loc = h[C_NEXT], mf_loc = h[C_MF];
    int64_t prev_nf = 0, seen = 0, reached = 0;
    int64_t m_fc = h[C_GLOBAL + C_COORD], bu_done = 0;  // policy 3: coordinator m_f, BU steps taken
    bool returned = false;
    const int64_t words = loop_words(g);
    const size_t slice_bytes = mg ? (size_t)(g->nb / 8) : 0;
    uint64_t nvl_total = 0;
    bool used_bitmap = false;   // some top-down step pushed bitmaps: parent logs to send at the end
    if (g->plog_cnt.p) BFS_CUDA(cudaMemsetAsync(g->plog_cnt.p, 0, (size_t)p * 8, s));
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
            bool claim_mode = false;
            front_ok = false;
            Remote rm{};
            // dense levels push bitmaps (every rank decides on the same global m_f)
            const bool bitmap_mode = mg && m_f >= td_bitmap_min(g);
            if (mg) {
                rm.nb = g->nb;
                rm.seen = g->seen.p;
                if (bitmap_mode) {
                    if (!g->plog.p) {
                        g->outbox.alloc((size_t)p * (g->nb / 32), s);
                        g->inbox.alloc((size_t)p * (g->nb / 32), s);
                        g->plog.alloc((size_t)p * g->nb, s);
                        g->plog_cnt.alloc((size_t)p, s);
                        BFS_CUDA(cudaMemsetAsync(g->plog_cnt.p, 0, (size_t)p * 8, s));   // this search's logs
                    }
                    BFS_CUDA(cudaMemsetAsync(g->outbox.p, 0, g->outbox.bytes(), s));
                    rm.outbox = g->outbox.p;
                    rm.plog = g->plog.p;
                    rm.plog_cnt = (unsigned long long*)g->plog_cnt.p;
                    used_bitmap = true;
                } else {
                    rm.cap = std::max<int64_t>(1, std::min<int64_t>(g->nb, E));
                    ensure(g->out_list, (size_t)(p * rm.cap), s);
                    rm.out = g->out_list.p;
                    rm.out_cnt = (unsigned long long*)g->out_cnt.p;
                    BFS_CUDA(cudaMemsetAsync(g->out_cnt.p, 0, (size_t)p * sizeof(int64_t), s));
                }
            }
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 1], s));
            // tile mode (td_tile.cuh): heavy frontier rows expanded per tile, the rest below
            const bool tile_mode = !mg && g->tile_T > 0 && E >= tile_min_setting();
            if (E > 0) {
                l2_window(g, g->visited.p, g->visited.bytes());
                // single-pass scan of the queue degrees (the loop graph's kernel, host-sized)
                BFS_CUDA(cudaMemsetAsync(g->tstate.p, 0, (size_t)((nf_loc + kScanTile - 1) / kScanTile) * 8, s));
                BFS_CUDA(cudaMemsetAsync(g->tctr.p, 0, sizeof(uint32_t), s));
                if (tile_mode) {
                    BFS_CUDA(cudaMemsetAsync(g->tile_hcnt.p, 0, sizeof(uint32_t), s));
                    BFS_CUDA(cudaMemsetAsync(g->tile_lcnt.p, 0, (size_t)g->tile_nwl * 4, s));
                }
                const TileLog lg = tile_mode ? tile_log(g) : TileLog{};
                k_scan_dev<<<grid_for((nf_loc + kScanTile - 1) / kScanTile * kScanThreads, kScanThreads), kScanThreads, 0,
                             s>>>(nullptr, qcur, qcur, nf_loc, g->prefix.p, (unsigned long long*)g->tstate.p,
                                  g->tctr.p, g->tile_nh, tile_mode ? 1 : 0);
                BFS_CHECK_LAUNCH();
                ++launches;
                int64_t El = E;   // arcs of the edge-balanced expansion (tile mode: light rows)
                if (tile_mode) {
                    BFS_CUDA(cudaMemcpyAsync(&El, g->prefix.p + nf_loc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                    BFS_CUDA(cudaStreamSynchronize(s));
                }
                const int64_t nchunks = (El + kTdChunk - 1) / kTdChunk;
                k_td_chunk_starts<<<grid_for(nchunks, 256), 256, 0, s>>>(g->prefix.p, nf_loc, nchunks, g->scratch64.p,
                                                                          nullptr);
                BFS_CHECK_LAUNCH();
                const int grid = (int)std::min<int64_t>(nchunks, mg ? td_resident_grid<true>() : td_resident_grid<false>());
                // large single-partition steps: claims + records only, the winners' degrees
                // and the next queue from k_td_finish in vertex order (visited snapshot in
                // `next`, which becomes the next frontier bitmap)
                claim_mode = !mg && (E >= td_claim_min() || tile_mode);
                if (claim_mode) {
                    BFS_CUDA(cudaMemcpyAsync(next, g->visited.p, (size_t)words * 4, cudaMemcpyDeviceToDevice, s));
                    if (El > 0) {
                        k_td_expand<false><<<std::max(1, grid), kTdThreads, 0, s>>>(
                            qcur, g->prefix.p, g->scratch64.p, nf_loc, El, g->off.p, g->adj.p, g->visited.p, rec, pmap, qnxt,
                            g->head.p, cnt, d + 1, g->lo, g->hi, rm, nullptr, nullptr, tile_mode ? 2 : 1, lg);
                        BFS_CHECK_LAUNCH();
                    }
                    if (tile_mode) {
                        k_tile_list<<<grid_for(nf_loc, 256), 256, 0, s>>>(nullptr, qcur, qcur, nf_loc, g->tile_nh,
                                                                          g->tile_hlist.p, g->tile_hcnt.p);
                        BFS_CHECK_LAUNCH();
                        k_td_tile<<<g->tile_units, kTileThreads, (size_t)g->tile_maxw * 4, s>>>(
                            nullptr, g->tile_start.p, g->tile_T, g->tile_unit.p, g->tile_bnd.p, g->tile_hlist.p,
                            g->tile_hcnt.p, g->off.p, g->adj.p, g->visited.p, pmap, lg, nullptr);
                        BFS_CHECK_LAUNCH();
                        k_tile_rec<<<g->tile_nwl, kWinThreads, (size_t)kWin * 4, s>>>(
                            nullptr, (int32_t)(d + 1), g->tile_wl.p, g->tile_fu.p, g->tile_unit.p, lg, g->visited.p,
                            next, nullptr, rec, nullptr);
                        BFS_CHECK_LAUNCH();
                        launches += 3;
                    }
                    k_td_finish<<<grid_for(words * 32, 256), 256, 0, s>>>(g->visited.p, next, words, g->head.p, cnt);
                    BFS_CHECK_LAUNCH();
                    launches += 2;
                } else if (mg)
                    k_td_expand<true><<<grid, kTdThreads, 0, s>>>(qcur, g->prefix.p, g->scratch64.p, nf_loc, E, g->off.p,
                                                                  g->adj.p, g->visited.p, rec, pmap, qnxt, g->head.p, cnt, d + 1,
                                                                  g->lo, g->hi, rm, nullptr, nullptr, 0, TileLog{});
                else
                    k_td_expand<false><<<grid, kTdThreads, 0, s>>>(qcur, g->prefix.p, g->scratch64.p, nf_loc, E,
                                                                   g->off.p, g->adj.p, g->visited.p, rec, pmap, qnxt, g->head.p, cnt,
                                                                   d + 1, g->lo, g->hi, rm, nullptr, nullptr, 0, TileLog{});
                BFS_CHECK_LAUNCH();
                launches += 2;
            }
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[4 * d + 2], s));
            if (bitmap_mode) {
                // push as bitmaps (Alg. 2 NextFrontier[P] with parents deferred): slice q
                // of the outbox to peer q, the received slices ORed into this rank's claims
                const int64_t nbw = g->nb / 32;
                for (int q = 0; q < p; ++q) {
                    sendp[q] = g->outbox.p + (size_t)q * nbw;
                    sendb[q] = q == me ? 0 : (size_t)nbw * 4;
                    recvp[q] = g->inbox.p + (size_t)q * nbw;
                    recvb[q] = q == me ? 0 : (size_t)nbw * 4;
                    nvl += sendb[q];
                }
                g->comm->alltoallv(sendp.data(), sendb.data(), recvp.data(), recvb.data(), s);
                k_td_inbox<<<grid_for(words, 256), 256, 0, s>>>(g->inbox.p, p, me, nbw, words, g->visited.p, g->head.p,
                                                                rec, qnxt, cnt, d + 1, g->lo);
                BFS_CHECK_LAUNCH();
                ++launches;
            } else if (mg) {
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
            if (claim_mode) {
                std::swap(front, next);   // the next frontier as a bitmap only: BU needs no q2b,
                have_queue = false;       // a top-down step builds its queue with b2q
            }
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
                if (have_queue && !front_ok) {
                    BFS_CUDA(cudaMemsetAsync(front + (g->lo >> 5), 0, (size_t)words_of(nl) * 4, s));
                    if (nf_loc) {
                        k_q2b<<<grid_for(nf_loc, 256), 256, 0, s>>>(qcur.v, nf_loc, front);
                        BFS_CHECK_LAUNCH();
                        ++launches;
                    }
                }
                have_queue = false;
                front_ok = false;
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
                                                         pmap, g->reindexed ? g->hpar.p : nullptr, bu_nb4(g), g->nb4_rows,
                                                         bu_nbp(g), words, g->lo, d + 1, cnt, grab, bu_long_setting(), bu_dense_setting(), nullptr,
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
    if (used_bitmap) {
        // final aggregation: the parent logs of the bitmap-mode levels to their owners
        BFS_CUDA(cudaEventRecord(g->ev[3], s));
        BFS_CUDA(cudaMemcpyAsync(g->cnt_mat.p + (size_t)me * p, g->plog_cnt.p, (size_t)p * 8, cudaMemcpyDeviceToDevice,
                                 s));
        g->comm->allgather_inplace(g->cnt_mat.p, (size_t)p * 8, s);
        BFS_CUDA(cudaMemcpyAsync(g->h_cnt_mat, g->cnt_mat.p, (size_t)p * p * 8, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        int64_t R = 0;
        for (int q = 0; q < p; ++q) R += q == me ? 0 : g->h_cnt_mat[(size_t)q * p + me];
        ensure(g->plog_in, (size_t)std::max<int64_t>(R, 1), s);
        int64_t roff = 0;
        uint64_t nvl_agg = 0;
        for (int q = 0; q < p; ++q) {
            const int64_t out_q = q == me ? 0 : g->h_cnt_mat[(size_t)me * p + q];
            const int64_t in_q = q == me ? 0 : g->h_cnt_mat[(size_t)q * p + me];
            sendp[q] = g->plog.p + (size_t)q * g->nb;
            sendb[q] = (size_t)out_q * sizeof(int4);
            recvp[q] = g->plog_in.p + roff;
            recvb[q] = (size_t)in_q * sizeof(int4);
            roff += in_q;
            nvl_agg += sendb[q];
        }
        g->comm->alltoallv(sendp.data(), sendb.data(), recvp.data(), recvb.data(), s);
        if (R) {
            k_plog_resolve<<<grid_for(R, 256), 256, 0, s>>>(g->plog_in.p, R, rec, g->lo);
            BFS_CHECK_LAUNCH();
            ++launches;
        }
        nvl_total += nvl_agg;
    }
    if ((od || op) && g->reindexed && mg) {
        // partition-local reindex: every owned output is produced on this rank
        k_emit_local<<<grid_for(nl, 256), 256, 0, s>>>(g->visited.p, g->skip.p, rec, g->label.p, g->lo, nl, root_l, od,
                                                       op);
        BFS_CHECK_LAUNCH();
        ++launches;
    } else if (od || op) {
        if (!mg) {
            const int64_t dw = words_of(g->reindexed ? g->n_active : nl);
            k_l2_demote<<<grid_for((dw + 31) / 32, 256), 256, 0, s>>>(g->front.p, g->next.p, dw);
            ++launches;
        }
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
    if (used_bitmap) {
        float ma = 0;
        BFS_CUDA(cudaEventElapsedTime(&ma, g->ev[3], g->ev[1]));
        g->run.ms_aggregate = ma;
    }
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
