// Graph500 validation of one search's outputs on the device (P:168
// "experimental methodology defined by Graph500"): the benchmark's own check that a
// reported search is a BFS tree of the graph --
//   V1 parent[root] = root, depth[root] = 0, and depth 0 only at the root
//   V2 the tree edge {parent[v], v} of every reached v != root is an arc of the graph
//   V3 depth[parent[v]] = depth[v] - 1
//   V4 no arc joins a reached and an unreached vertex or spans more than one level
//   V5 unreached <=> parent = depth = -1; parent in [0, n)
// This is the product's self-check (bench.py runs it outside the timed region on
// every root); parity itself is proven against the independent CPU oracle in tests/.
// Single-partition graphs (the outputs and the CSR live on one device).
#include "internal.cuh"

namespace bfsb {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ void vfail(unsigned long long* fails, int rule) { atomicAdd(fails + rule, 1ull); }

// per vertex (internal label iv, original o): V1, V2, V3, V5; writes depth in internal
// order for the arc pass
__global__ void k_val_vertices(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                               const int32_t* __restrict__ ilabel, const int32_t* __restrict__ label, int64_t n,
                               int64_t root, const int32_t* __restrict__ depth, const int32_t* __restrict__ parent,
                               int32_t* __restrict__ dint, int sorted_rows, unsigned long long* __restrict__ fails) {
    for (int64_t iv = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; iv < n; iv += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = ilabel ? (int64_t)ilabel[iv] : iv;
        const int32_t d = depth[o], p = parent[o];
        dint[iv] = d;
        if (o == root && (p != root || d != 0)) vfail(fails, 0);
        if ((d >= 0) != (p >= 0) || d < -1 || p < -1 || p >= n) {
            vfail(fails, 4);
            continue;
        }
        if (d < 0) continue;
        if (d == 0 && o != root) vfail(fails, 0);
        if (o == root) continue;
        if (depth[p] != d - 1) vfail(fails, 2);
        const int32_t pi = label ? label[p] : p;
        int64_t b = off[iv], e = off[iv + 1];
        bool found = false;
        if (sorted_rows) {   // rows ascending by internal label: lower bound of pi
            while (b < e) {
                const int64_t mid = (b + e) >> 1;
                if (adj[mid] < pi) b = mid + 1;
                else e = mid;
            }
            found = b < off[iv + 1] && adj[b] == pi;
        } else {
            for (int64_t j = b; j < e && !found; ++j) found = adj[j] == pi;
        }
        if (!found) vfail(fails, 1);
    }
}

// V4 over every stored arc: a warp per row, lanes stride the row
__global__ void k_val_arcs(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                           const int32_t* __restrict__ dint, int64_t n, unsigned long long* __restrict__ fails) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long bad = 0;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
        const int64_t b = off[v], e = off[v + 1];
        if (b == e) continue;
        const int32_t dv = dint[v];
        for (int64_t j = b + lane; j < e; j += 32) {
            const int32_t du = dint[adj[j]];
            if ((dv >= 0) != (du >= 0) || (dv >= 0 && (dv - du > 1 || du - dv > 1))) ++bad;
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) bad += __shfl_xor_sync(kFullMask, bad, s);
    if (lane == 0 && bad) atomicAdd(fails + 3, bad);
}

}  // namespace

void validate_impl(bfs_graph_s* g, int64_t root, const int32_t* parent, const int32_t* depth, int64_t fails[5]) {
    if ((g->comm && g->comm->nranks > 1) || g->nparts > 1)
        fail(BFS_ERR_INVALID_ARG, "bfs_validate needs a single-partition graph");
    if (root < 0 || root >= g->n) fail(BFS_ERR_OUT_OF_RANGE, "root outside [0, n)");
    if (!parent || !depth) fail(BFS_ERR_INVALID_ARG, "parent and depth are required");
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    DevBuf<int32_t> dp, pp, dint;
    DevBuf<unsigned long long> f;
    const int32_t* dd = depth;
    const int32_t* pd = parent;
    if (!is_device_ptr(depth)) {
        dp.alloc((size_t)n, s);
        BFS_CUDA(cudaMemcpyAsync(dp.p, depth, (size_t)n * 4, cudaMemcpyHostToDevice, s));
        dd = dp.p;
    }
    if (!is_device_ptr(parent)) {
        pp.alloc((size_t)n, s);
        BFS_CUDA(cudaMemcpyAsync(pp.p, parent, (size_t)n * 4, cudaMemcpyHostToDevice, s));
        pd = pp.p;
    }
    dint.alloc((size_t)n, s);
    f.alloc(5, s);
    BFS_CUDA(cudaMemsetAsync(f.p, 0, 5 * sizeof(unsigned long long), s));
    // rows are ascending by internal label unless built unsorted or by neighbour degree
    const int sorted = g->opts.sort_rows == 1 || (g->opts.sort_rows != 0 && g->reindexed);
    const int grid = num_sms() * 8;
    k_val_vertices<<<grid, 256, 0, s>>>(g->off.p, g->adj.p, g->reindexed ? g->ilabel.p : nullptr,
                                        g->reindexed ? g->label.p : nullptr, n, root, dd, pd, dint.p, sorted, f.p);
    BFS_CHECK_LAUNCH();
    k_val_arcs<<<grid, 256, 0, s>>>(g->off.p, g->adj.p, dint.p, n, f.p);
    BFS_CHECK_LAUNCH();
    unsigned long long h[5];
    BFS_CUDA(cudaMemcpyAsync(h, f.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 5; ++i) fails[i] = (int64_t)h[i];
}

}  // namespace bfsb
