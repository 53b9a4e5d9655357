// The hot path: level-synchronous direction-optimized BFS on one GPU
// (Alg. 1; Beamer via P:16; switch rule
// P:151-155 read as DESIGN.md R2/R3/R17/R19).
//
// Data layout in HBM (internal labels, owned range [lo, hi), nl = hi - lo):
//   off     int64[nl+1]   CSR offsets          adj   int32[arcs] global IDs
//   visited u32[nl/32]    1 = visited or degree 0 (initialised from the skip mask)
//   front / next u32[n/32] frontier bitmaps (bottom-up input / output)
//   q0 / q1 int32[nl]     frontier queues (top-down input / output)
//   depth / parent int32[nl]  outputs, each entry written exactly once
//
// Kernels:
//   k_init        visited <- skip | root, root outputs, counters
//   k_td_expand   top-down step, edge-balanced: a device scan of frontier degrees
//                 gives every CTA a contiguous 2048-arc chunk; arcs are mapped back
//                 to their frontier vertex by binary search in shared memory;
//                 unvisited targets are claimed with atomicOr on the visited word;
//                 winners write depth/parent and append to the next queue with one
//                 warp-aggregated atomicAdd; m_f of the next frontier is fused.
//   k_bu_step     bottom-up step, one warp per 32-vertex visited word: lanes scan
//                 their own row for up to kBuLaneSteps arcs (first frontier
//                 neighbour wins: `break for`), then rows still unresolved
//                 are scanned by the whole warp 32 arcs at a time with a ballot
//                 (lowest lane = first in row order).  n_f, m_f, inspections fused.
//   k_q2b / k_b2q frontier queue <-> bitmap on direction switches (ballot/popc +
//                 warp prefix sums, one atomicAdd per warp)
//   k_finalize    parent = depth = -1 for unreached vertices (write-once outputs)
#include <algorithm>
#include <cstring>

#include "internal.cuh"

namespace bfsb {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTdThreads = 256;
constexpr int kTdItems = 8;
constexpr int kTdChunk = kTdThreads * kTdItems;  // arcs per CTA iteration
constexpr int kBuThreads = 256;
constexpr int kBuLaneSteps = 4;

// counter slots
enum { C_NEXT = 0, C_MF = 1, C_INSP = 2, C_B2Q = 3, C_SCAN = 4, C_TUPLES = 8 };

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
    return x;
}

__global__ void k_init(uint32_t* visited, const uint32_t* skip, int64_t pw, int64_t root_l, int32_t root_g,
                       int32_t* depth, int32_t* parent, int32_t* q, const int64_t* off, unsigned long long* cnt) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < pw; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = skip[w];
        if (w == (root_l >> 5)) x |= 1u << (root_l & 31);
        visited[w] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        depth[root_l] = 0;
        parent[root_l] = root_g;
        q[0] = root_g;
        cnt[C_NEXT] = 1;
        cnt[C_MF] = (unsigned long long)(off[root_l + 1] - off[root_l]);
        cnt[C_INSP] = 0;
    }
}

// chunk c of the top-down arc range starts inside frontier entry starts[c]
__global__ void k_td_chunk_starts(const int64_t* prefix, int64_t F, int64_t nchunks, int64_t* starts) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = c * kTdChunk;
        // largest i in [0, F) with prefix[i] <= e (prefix non-decreasing, prefix[0] = 0)
        int64_t lo = 0, hi = F - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        starts[c] = lo;
    }
}

__global__ void __launch_bounds__(kTdThreads)
k_td_expand(const int32_t* __restrict__ q, const int64_t* __restrict__ prefix, const int64_t* __restrict__ starts,
            int64_t F, int64_t E, const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
            uint32_t* __restrict__ visited, int32_t* __restrict__ depth, int32_t* __restrict__ parent,
            int32_t* __restrict__ qnext, unsigned long long* __restrict__ cnt, int32_t next_level, int64_t lo) {
    __shared__ int64_t s_pre[kTdChunk + 2];
    __shared__ int64_t s_beg[kTdChunk + 1];
    __shared__ int32_t s_u[kTdChunk + 1];
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0;
    const int64_t nchunks = (E + kTdChunk - 1) / kTdChunk;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const int64_t e0 = c * kTdChunk;
        const int64_t e1 = min(E, e0 + kTdChunk);
        const int64_t i0 = starts[c];
        const int64_t i1 = (c + 1 < nchunks) ? starts[c + 1] : F - 1;
        const int64_t cntv = min(i1 - i0 + 1, F - i0);
        const bool fits = cntv <= kTdChunk;
        if (fits) {
            for (int k = threadIdx.x; k <= cntv; k += kTdThreads) {
                s_pre[k] = prefix[i0 + k];
                if (k < cntv) {
                    int32_t u = q[i0 + k];
                    s_u[k] = u;
                    s_beg[k] = off[u - lo];
                }
            }
        }
        __syncthreads();
#pragma unroll 2
        for (int j = 0; j < kTdItems; ++j) {
            const int64_t e = e0 + (int64_t)j * kTdThreads + threadIdx.x;
            bool win = false;
            int32_t v = 0, u = 0;
            if (e < e1) {
                int64_t beg, pre;
                if (fits) {
                    int a = 0, b = (int)cntv - 1;
                    while (a < b) {
                        int mid = (a + b + 1) >> 1;
                        if (s_pre[mid] <= e) a = mid;
                        else b = mid - 1;
                    }
                    u = s_u[a];
                    beg = s_beg[a];
                    pre = s_pre[a];
                } else {
                    int64_t a = i0, b = F - 1;
                    while (a < b) {
                        int64_t mid = (a + b + 1) >> 1;
                        if (prefix[mid] <= e) a = mid;
                        else b = mid - 1;
                    }
                    u = q[a];
                    beg = off[u - lo];
                    pre = prefix[a];
                }
                v = __ldg(adj + beg + (e - pre));
                const uint32_t bit = 1u << (v & 31);
                uint32_t* wp = visited + ((v - lo) >> 5);
                if (!(__ldcg(wp) & bit)) win = !(atomicOr(wp, bit) & bit);
            }
            const unsigned m = __ballot_sync(kFull, win);
            if (m) {
                const int leader = __ffs(m) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(cnt + C_NEXT, (unsigned long long)__popc(m));
                base = __shfl_sync(kFull, base, leader);
                if (win) {
                    const int64_t vl = v - lo;
                    qnext[base + __popc(m & lanemask_lt())] = v;
                    depth[vl] = next_level;
                    parent[vl] = u;
                    my_mf += (unsigned long long)(off[vl + 1] - off[vl]);
                }
            }
        }
        __syncthreads();
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
}

__device__ __forceinline__ bool in_front(const uint32_t* __restrict__ front, int32_t u) {
    return (__ldg(front + (u >> 5)) >> (u & 31)) & 1u;
}

__global__ void __launch_bounds__(kBuThreads)
k_bu_step(const int64_t* __restrict__ off, const int32_t* __restrict__ adj, uint32_t* __restrict__ visited,
          const uint32_t* __restrict__ front, uint32_t* __restrict__ next, int32_t* __restrict__ depth,
          int32_t* __restrict__ parent, int64_t words, int64_t lo, int32_t next_level,
          unsigned long long* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t wbase = lo >> 5;  // first global word of the owned range
    unsigned long long my_nf = 0, my_mf = 0, my_insp = 0, my_scan = 0;
    for (int64_t w = gw; w < words; w += nw) {
        const uint32_t vis = visited[w];
        if (vis == kFull) {
            if (lane == 0) next[wbase + w] = 0u;
            continue;
        }
        const int64_t vl = w * 32 + lane;
        const bool todo = !((vis >> lane) & 1u);
        if (lane == 0) my_scan += __popc(~vis);
        int64_t b = 0, e = 0;
        if (todo) {
            b = off[vl];
            e = off[vl + 1];
        }
        int64_t j = b;
        bool found = false;
        int32_t par = -1;
        // phase 1: each lane walks its own row (virtual warp of 1)
#pragma unroll
        for (int t = 0; t < kBuLaneSteps; ++t) {
            if (!found && j < e) {
                int32_t u = __ldg(adj + j);
                if (in_front(front, u)) {
                    found = true;
                    par = u;
                } else {
                    ++j;
                }
            }
        }
        // phase 2: unresolved rows, one at a time, scanned by the whole warp
        unsigned rem = __ballot_sync(kFull, !found && j < e);
        while (rem) {
            const int src = __ffs(rem) - 1;
            rem &= rem - 1;
            const int64_t jb = __shfl_sync(kFull, j, src);
            const int64_t je = __shfl_sync(kFull, e, src);
            int64_t hit_j = je;
            int32_t hit_u = -1;
            for (int64_t j0 = jb; j0 < je; j0 += 32) {
                const int64_t jj = j0 + lane;
                int32_t u = -1;
                bool h = false;
                if (jj < je) {
                    u = __ldg(adj + jj);
                    h = in_front(front, u);
                }
                const unsigned hm = __ballot_sync(kFull, h);
                if (hm) {
                    const int first = __ffs(hm) - 1;
                    hit_j = j0 + first;
                    hit_u = __shfl_sync(kFull, u, first);
                    break;
                }
            }
            if (lane == src) {
                j = hit_j;
                if (hit_u >= 0) {
                    found = true;
                    par = hit_u;
                }
            }
        }
        if (found) {
            depth[vl] = next_level;
            parent[vl] = par;
        }
        const unsigned nb = __ballot_sync(kFull, found);
        if (lane == 0) {
            next[wbase + w] = nb;
            visited[w] = vis | nb;
            my_nf += __popc(nb);
        }
        if (todo) {
            my_insp += (unsigned long long)(found ? (j - b + 1) : (e - b));
            if (found) my_mf += (unsigned long long)(e - b);
        }
    }
    my_nf = warp_sum_u64(my_nf);
    my_mf = warp_sum_u64(my_mf);
    my_insp = warp_sum_u64(my_insp);
    if (lane == 0 && my_scan) atomicAdd(cnt + C_SCAN, my_scan);
    if (lane == 0) {
        if (my_nf) atomicAdd(cnt + C_NEXT, my_nf);
        if (my_mf) atomicAdd(cnt + C_MF, my_mf);
        if (my_insp) atomicAdd(cnt + C_INSP, my_insp);
    }
}

// queue -> bitmap (front cleared beforehand)
__global__ void k_q2b(const int32_t* __restrict__ q, int64_t F, uint32_t* __restrict__ front) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = q[i];
        atomicOr(front + (v >> 5), 1u << (v & 31));
    }
}

// bitmap (owned words) -> queue of global IDs
__global__ void k_b2q(const uint32_t* __restrict__ bm, int64_t words, int64_t lo, int32_t* __restrict__ q,
                      unsigned long long* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t wbase = lo >> 5;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < words;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = b0 + lane;
        uint32_t bits = w < words ? bm[wbase + w] : 0u;
        int c = __popc(bits);
        int inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int y = __shfl_up_sync(kFull, inc, d);
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
            q[pos++] = (int32_t)(lo + w * 32 + k);
        }
    }
}

// unreached -> -1 (write-once outputs: discovered entries were written by the steps)
__global__ void k_finalize(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip, int64_t nl,
                           int64_t root_l, int32_t* __restrict__ depth, int32_t* __restrict__ parent) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = v >> 5;
        const uint32_t r = visited[w] & ~skip[w];
        if (!((r >> (v & 31)) & 1u) && v != root_l) {
            depth[v] = -1;
            parent[v] = -1;
        }
    }
}

// original-label outputs from internal-label ones (degree reindex)
__global__ void k_remap_out(const int32_t* __restrict__ label, const int32_t* __restrict__ ilabel,
                            const int32_t* __restrict__ dep_i, const int32_t* __restrict__ par_i, int64_t n,
                            int32_t* __restrict__ dep_o, int32_t* __restrict__ par_o) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t iv = label[v];
        if (dep_o) dep_o[v] = dep_i[iv];
        if (par_o) {
            const int32_t p = par_i[iv];
            par_o[v] = p < 0 ? -1 : ilabel[p];
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

// non-self-loop arc count of candidate roots (internal labels), one warp per candidate
__global__ void k_nonloop_degree(const int32_t* __restrict__ cand, int64_t k, const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ adj, int64_t lo, int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = gw; t < k; t += nw) {
        const int32_t r = cand[t];
        const int64_t b = off[r - lo], e = off[r - lo + 1];
        int64_t c = 0;
        for (int64_t j = b + lane; j < e; j += 32) c += adj[j] != r;
        for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
        if (lane == 0) out[t] = c;
    }
}

int grid_for(int64_t items, int threads, int per_sm = 8) {
    int64_t b = (items + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * per_sm;
    return (int)std::max<int64_t>(1, std::min(b, cap));
}

}  // namespace

void bfs_alloc_state(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    g->visited.alloc((size_t)padded_words(nl), s);
    g->front.alloc((size_t)padded_words(g->n), s);
    g->next.alloc((size_t)padded_words(g->n), s);
    BFS_CUDA(cudaMemsetAsync(g->front.p, 0, g->front.bytes(), s));
    BFS_CUDA(cudaMemsetAsync(g->next.p, 0, g->next.bytes(), s));
    g->q0.alloc((size_t)std::max<int64_t>(nl, 1), s);
    g->q1.alloc((size_t)std::max<int64_t>(nl, 1), s);
    g->prefix.alloc((size_t)nl + 1, s);
    g->cnt.alloc(16, s);
    g->scratch64.alloc((size_t)(g->arcs_local / kTdChunk + 2), s);  // TD chunk starts
    if (!g->h_cnt) BFS_CUDA(cudaMallocHost(&g->h_cnt, 16 * sizeof(int64_t)));
    for (auto& e : g->ev)
        if (!e) BFS_CUDA(cudaEventCreate(&e));
}

static void read_counters(bfs_graph_s* g) {
    BFS_CUDA(cudaMemcpyAsync(g->h_cnt, g->cnt.p, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, g->stream));
    BFS_CUDA(cudaStreamSynchronize(g->stream));
}

void bfs_run_impl(bfs_graph_s* g, int64_t root, int32_t* parent_out, int32_t* depth_out) {
    if (root < 0 || root >= g->n)
        fail(BFS_ERR_OUT_OF_RANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(g->n) + ")");
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    unsigned long long* cnt = (unsigned long long*)g->cnt.p;
    int64_t* h = g->h_cnt;

    int64_t root_i = root;
    if (g->reindexed) {
        int32_t r;
        BFS_CUDA(cudaMemcpy(&r, g->label.p + root, sizeof(int32_t), cudaMemcpyDeviceToHost));
        root_i = r;
    }
    const int64_t root_l = root_i - g->lo;

    // where the kernels write (internal order)
    const bool dev_depth = depth_out && is_device_ptr(depth_out);
    const bool dev_parent = parent_out && is_device_ptr(parent_out);
    int32_t* kd = (!g->reindexed && dev_depth) ? depth_out : nullptr;
    int32_t* kp = (!g->reindexed && dev_parent) ? parent_out : nullptr;
    if (!kd) {
        if (!g->tmp_depth.p) g->tmp_depth.alloc((size_t)std::max<int64_t>(nl, 1), s);
        kd = g->tmp_depth.p;
    }
    if (!kp) {
        if (!g->tmp_parent.p) g->tmp_parent.alloc((size_t)std::max<int64_t>(nl, 1), s);
        kp = g->tmp_parent.p;
    }

    g->levels.clear();
    g->run = bfs_run_stats{};
    g->run.root = root;
    int64_t launches = 0;
    // per-step events: [3d] step start, [3d+1] main kernel start, [3d+2] main kernel end
    const bool lt = g->policy.level_times != 0;
    constexpr int kMaxTimed = 64;
    if (lt && g->lev_ev.empty()) {
        g->lev_ev.resize(3 * kMaxTimed + 1);
        for (auto& e : g->lev_ev) BFS_CUDA(cudaEventCreate(&e));
    }

    BFS_CUDA(cudaEventRecord(g->ev[0], s));
    const int64_t pw = padded_words(nl);
    k_init<<<grid_for(pw, 256), 256, 0, s>>>(g->visited.p, g->skip.p, pw, root_l, (int32_t)root_i, kd, kp, g->q0.p,
                                             g->off.p, cnt);
    BFS_CHECK_LAUNCH();
    ++launches;
    read_counters(g);

    int32_t* qcur = g->q0.p;
    int32_t* qnxt = g->q1.p;
    uint32_t* front = g->front.p;
    uint32_t* next = g->next.p;
    bool have_queue = true;
    int dir = 0;  // 0 TD, 1 BU
    int64_t n_f = h[C_NEXT], m_f = h[C_MF], prev_nf = 0, seen = 0, reached = 0;
    const int64_t words = words_of(nl);
    for (int d = 0; n_f > 0; ++d) {
        if (d >= (1 << 30)) fail(BFS_ERR_INTERNAL, "level loop did not terminate");
        reached += n_f;
        seen += m_f;
        const int64_t m_u = g->arcs_global - seen;
        // direction for the step that builds level d+1 (R2)
        switch (g->policy.mode) {
            case 1: dir = 0; break;
            case 2: dir = d >= g->policy.bu_from_level ? 1 : 0; break;
            default:
                if (dir == 0) {
                    if (m_f * g->policy.alpha > m_u) dir = 1;
                } else {
                    if (n_f * g->policy.beta < g->n && n_f < prev_nf) dir = 0;
                }
        }
        const bool timed = lt && d < kMaxTimed;
        if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d], s));
        BFS_CUDA(cudaMemsetAsync(g->cnt.p, 0, 8 * sizeof(int64_t), s));
        int64_t insp, scanned;
        if (dir == 0) {
            if (!have_queue) {
                k_b2q<<<grid_for(words, 256), 256, 0, s>>>(front, words, g->lo, qcur, cnt);
                BFS_CHECK_LAUNCH();
                ++launches;
                have_queue = true;
            }
            const int64_t E = m_f;
            if (E > 0) {
                launches += scan_queue_degrees(qcur, n_f, g->off.p, g->lo, g->prefix.p, s);
                const int64_t nchunks = (E + kTdChunk - 1) / kTdChunk;
                k_td_chunk_starts<<<grid_for(nchunks, 256), 256, 0, s>>>(g->prefix.p, n_f, nchunks, g->scratch64.p);
                BFS_CHECK_LAUNCH();
                if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d + 1], s));
                k_td_expand<<<grid_for(nchunks * kTdThreads, kTdThreads, 8), kTdThreads, 0, s>>>(
                    qcur, g->prefix.p, g->scratch64.p, n_f, E, g->off.p, g->adj.p, g->visited.p, kd, kp, qnxt, cnt,
                    d + 1, g->lo);
                BFS_CHECK_LAUNCH();
                if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d + 2], s));
                launches += 2;
            } else if (timed) {
                BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d + 1], s));
                BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d + 2], s));
            }
            std::swap(qcur, qnxt);
            insp = E;
            scanned = n_f;
        } else {
            if (have_queue) {
                BFS_CUDA(cudaMemsetAsync(front, 0, g->front.bytes(), s));
                k_q2b<<<grid_for(n_f, 256), 256, 0, s>>>(qcur, n_f, front);
                BFS_CHECK_LAUNCH();
                ++launches;
                have_queue = false;
            }
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d + 1], s));
            k_bu_step<<<grid_for(words * 32, kBuThreads, 8), kBuThreads, 0, s>>>(
                g->off.p, g->adj.p, g->visited.p, front, next, kd, kp, words, g->lo, d + 1, cnt);
            BFS_CHECK_LAUNCH();
            if (timed) BFS_CUDA(cudaEventRecord(g->lev_ev[3 * d + 2], s));
            ++launches;
            std::swap(front, next);
            insp = -1;
            scanned = -1;
        }
        read_counters(g);
        bfs_level_stats L{};
        L.level = d;
        L.direction = dir;
        L.frontier = n_f;
        L.discovered = h[C_NEXT];
        L.m_f = m_f;
        L.m_u = m_u;
        L.inspections = insp >= 0 ? insp : h[C_INSP];
        L.scanned = scanned >= 0 ? scanned : h[C_SCAN];
        g->levels.push_back(L);
        prev_nf = n_f;
        n_f = h[C_NEXT];
        m_f = h[C_MF];
    }
    const int ntimed = lt ? (int)std::min<size_t>(g->levels.size(), kMaxTimed) : 0;
    if (lt) BFS_CUDA(cudaEventRecord(g->lev_ev[3 * ntimed], s));
    k_finalize<<<grid_for(nl, 256), 256, 0, s>>>(g->visited.p, g->skip.p, nl, root_l, kd, kp);
    BFS_CHECK_LAUNCH();
    ++launches;
    if (g->reindexed) {
        int32_t* od = dev_depth ? depth_out : nullptr;
        int32_t* op = dev_parent ? parent_out : nullptr;
        // host outputs: remap into staging buffers, then copy
        DevBuf<int32_t> hd, hp;
        if (depth_out && !dev_depth) { hd.alloc((size_t)nl, s); od = hd.p; }
        if (parent_out && !dev_parent) { hp.alloc((size_t)nl, s); op = hp.p; }
        k_remap_out<<<grid_for(g->n, 256), 256, 0, s>>>(g->label.p, g->ilabel.p, kd, kp, g->n, od, op);
        BFS_CHECK_LAUNCH();
        ++launches;
        BFS_CUDA(cudaEventRecord(g->ev[1], s));
        if (hd.p) BFS_CUDA(cudaMemcpyAsync(depth_out, hd.p, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
        if (hp.p) BFS_CUDA(cudaMemcpyAsync(parent_out, hp.p, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
    } else {
        BFS_CUDA(cudaEventRecord(g->ev[1], s));
        if (depth_out && !dev_depth) BFS_CUDA(cudaMemcpyAsync(depth_out, kd, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
        if (parent_out && !dev_parent) BFS_CUDA(cudaMemcpyAsync(parent_out, kp, (size_t)nl * 4, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
    }
    float ms = 0;
    BFS_CUDA(cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]));
    g->run.ms_total = ms;
    g->run.ms_compute = ms;
    g->run.levels = (int)g->levels.size();
    g->run.reached = reached;
    g->run.kernel_launches = launches;
    for (int d = 0; d < ntimed; ++d) {
        float x = 0, k = 0;
        BFS_CUDA(cudaEventElapsedTime(&x, g->lev_ev[3 * d], g->lev_ev[3 * d + 3]));
        BFS_CUDA(cudaEventElapsedTime(&k, g->lev_ev[3 * d + 1], g->lev_ev[3 * d + 2]));
        g->levels[d].ms = x;
        g->levels[d].kernel_ms = k;
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
    std::vector<int32_t> cand_i;
    std::vector<int64_t> deg(B);
    DevBuf<int32_t> dcand;
    DevBuf<int64_t> ddeg;
    dcand.alloc(B, s);
    ddeg.alloc(B, s);
    int64_t got = 0;
    for (int64_t k0 = 0; k0 < max_cand && got < count; k0 += B) {
        cand.clear();
        for (int64_t k = k0; k < std::min(max_cand, k0 + B); ++k) {
            uint32_t ctr[4] = {(uint32_t)((uint64_t)k & 0xffffffffu), (uint32_t)((uint64_t)k >> 32), 0u, 2u}, w[4];
            philox4x32_10_host(ctr, key, w);
            int64_t r = scale == 0 ? 0 : (int64_t)(w[0] >> (32 - scale));
            cand.push_back(r < g->n ? (int32_t)r : -1);
        }
        // map to internal labels, count non-self-loop arcs on the device
        std::vector<int32_t> valid;
        for (int32_t r : cand) valid.push_back(r < 0 ? 0 : r);
        BFS_CUDA(cudaMemcpyAsync(dcand.p, valid.data(), valid.size() * 4, cudaMemcpyHostToDevice, s));
        if (g->reindexed) {
            // gather label[cand] in place via a tiny copy (host loop is fine: B small)
            cand_i.resize(valid.size());
            for (size_t t = 0; t < valid.size(); ++t)
                BFS_CUDA(cudaMemcpyAsync(&cand_i[t], g->label.p + valid[t], 4, cudaMemcpyDeviceToHost, s));
            BFS_CUDA(cudaStreamSynchronize(s));
            BFS_CUDA(cudaMemcpyAsync(dcand.p, cand_i.data(), cand_i.size() * 4, cudaMemcpyHostToDevice, s));
        }
        k_nonloop_degree<<<grid_for((int64_t)valid.size() * 32, 256), 256, 0, s>>>(dcand.p, (int64_t)valid.size(),
                                                                                 g->off.p, g->adj.p, g->lo, ddeg.p);
        BFS_CHECK_LAUNCH();
        BFS_CUDA(cudaMemcpyAsync(deg.data(), ddeg.p, valid.size() * 8, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        for (size_t t = 0; t < cand.size() && got < count; ++t) {
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
