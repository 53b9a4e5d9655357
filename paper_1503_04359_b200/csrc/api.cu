// The C ABI (include/bfs.h): argument checking, error model, handles.
// Every entry point converts internal failures into bfs_status + a thread-local
// message; nothing here computes on the host -- all work is in the kernels.
#include <cstring>
#include <exception>
#include <new>
#include <numeric>

#include "internal.cuh"

namespace bfsb {

struct Failure {
    bfs_status code;
    std::string msg;
};

static thread_local std::string tl_error;

void set_error(const std::string& msg) { tl_error = msg; }

void fail(bfs_status code, const std::string& msg) { throw Failure{code, msg}; }

static void* (*g_alloc_fn)(size_t, void*, void*) = nullptr;
static void (*g_free_fn)(void*, void*) = nullptr;
static void* g_alloc_ctx = nullptr;

void* dev_alloc(size_t bytes, cudaStream_t s) {
    // every buffer gets a 16-byte tail: aligned 16-byte vector loads that straddle
    // the logical end (the bottom-up adjacency reads) stay inside the allocation
    bytes = (bytes + 31) & ~(size_t)15;
    if (g_alloc_fn) {
        void* p = g_alloc_fn(bytes, (void*)s, g_alloc_ctx);
        if (!p) fail(BFS_ERR_OUT_OF_MEMORY, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes");
        return p;
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        fail(e == cudaErrorMemoryAllocation ? BFS_ERR_OUT_OF_MEMORY : BFS_ERR_CUDA,
             "device allocation of " + std::to_string(bytes) + " bytes failed (" + cudaGetErrorString(e) +
                 "; free " + std::to_string(fr) + " of " + std::to_string(tot) + ")");
    }
    return p;
}

void dev_free(void* p, cudaStream_t s) {
    if (!p) return;
    if (g_free_fn) {
        g_free_fn(p, g_alloc_ctx);
        return;
    }
    cudaFreeAsync(p, s);  // errors here are not actionable (destructor path)
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        BFS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        cached[dev] = v > 0 ? v : 1;
    }
    return cached[dev];
}

static bfs_build_opts default_opts() { return bfs_build_opts{1, 1, 0, 1}; }

}  // namespace bfsb

using namespace bfsb;

#define API_BEGIN try {
#define API_END                                                   \
    }                                                             \
    catch (const Failure& f) {                                    \
        set_error(f.msg);                                         \
        return f.code;                                            \
    }                                                             \
    catch (const std::bad_alloc&) {                               \
        set_error("host allocation failed");                      \
        return BFS_ERR_OUT_OF_MEMORY;                             \
    }                                                             \
    catch (const std::exception& e) {                             \
        set_error(std::string("internal error: ") + e.what());    \
        return BFS_ERR_INTERNAL;                                  \
    }                                                             \
    catch (...) {                                                 \
        set_error("internal error");                              \
        return BFS_ERR_INTERNAL;                                  \
    }                                                             \
    return BFS_OK;

extern "C" {

int bfs_abi_version(void) { return BFS_ABI_VERSION; }

const char* bfs_last_error(void) { return tl_error.c_str(); }

bfs_status bfs_set_allocator(void* (*alloc_fn)(size_t, void*, void*), void (*free_fn)(void*, void*), void* ctx) {
    API_BEGIN
    if ((alloc_fn == nullptr) != (free_fn == nullptr)) fail(BFS_ERR_INVALID_ARG, "alloc_fn and free_fn must be both set or both NULL");
    g_alloc_fn = alloc_fn;
    g_free_fn = free_fn;
    g_alloc_ctx = ctx;
    API_END
}

bfs_status bfs_graph_create(const bfs_graph_desc* desc, bfs_comm_t comm, void* cuda_stream, bfs_graph_t* out) {
    bfs_graph_s* g = nullptr;
    API_BEGIN
    if (!desc || !out) fail(BFS_ERR_INVALID_ARG, "desc and out must be non-NULL");
    *out = nullptr;
    bfs_graph_desc d = *desc;
    int64_t n = d.n;
    switch (d.kind) {
        case BFS_SRC_KRONECKER:
            validate_kron_spec(&d.kron);
            n = (int64_t)1 << d.kron.scale;
            break;
        case BFS_SRC_EDGES:
            if (d.m < 0) fail(BFS_ERR_INVALID_ARG, "m must be >= 0");
            if (d.m > 0 && !d.uv) fail(BFS_ERR_INVALID_ARG, "uv is NULL");
            break;
        case BFS_SRC_CSR:
            if (!d.offsets) fail(BFS_ERR_INVALID_ARG, "offsets is NULL");
            break;
        default:
            fail(BFS_ERR_INVALID_ARG, "unknown source kind");
    }
    if (n < 1) fail(BFS_ERR_INVALID_ARG, "n must be >= 1");
    if (n > 0x7fffffffLL) fail(BFS_ERR_CAPACITY, "n = " + std::to_string(n) + " exceeds int32 vertex IDs");
    if (d.opts.reindex_by_degree && comm && comm->nranks > 1 && n % (32 * (int64_t)comm->nranks) != 0)
        fail(BFS_ERR_INVALID_ARG, "reindex_by_degree on p ranks permutes equal word-aligned blocks and needs n "
                                  "divisible by 32*p");
    if (d.opts.reindex_by_degree && d.kind == BFS_SRC_CSR)
        fail(BFS_ERR_INVALID_ARG, "reindex_by_degree needs an EDGES or KRONECKER source");
    g = new bfs_graph_s();
    if (comm) {
        BFS_CUDA(cudaSetDevice(comm->device));
        g->device = comm->device;
    } else {
        BFS_CUDA(cudaGetDevice(&g->device));
    }
    g->stream = (cudaStream_t)cuda_stream;
    {
        // keep freed blocks in the stream-ordered pool: construction and the TD scans
        // free and re-allocate GiB-sized temporaries, and returning them to the
        // driver at every synchronisation costs far more than the kernels
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    }
    g->n = n;
    g->comm = comm;
    if (comm && comm->nranks > 1) {
        g->nb = part_block(n, comm->nranks);
        g->lo = std::min<int64_t>(n, (int64_t)comm->rank * g->nb);
        g->hi = std::min<int64_t>(n, g->lo + g->nb);
    } else {
        g->nb = n;
        g->lo = 0;
        g->hi = n;
    }
    g->opts = d.opts;
    cudaEvent_t e0, e1;
    BFS_CUDA(cudaEventCreate(&e0));
    BFS_CUDA(cudaEventCreate(&e1));
    BFS_CUDA(cudaEventRecord(e0, g->stream));
    build_graph(g, &d);
    bfs_build_tiles(g);   // tiled top-down index (eligible graphs only)
    if (comm && comm->nranks > 1) {
        // global arc count for the switch rule (m_u)
        DevBuf<int64_t> a;
        a.alloc(1, g->stream);
        BFS_CUDA(cudaMemcpyAsync(a.p, &g->arcs_local, sizeof(int64_t), cudaMemcpyHostToDevice, g->stream));
        comm->allreduce_sum_i64(a.p, 1, g->stream);
        BFS_CUDA(cudaMemcpyAsync(&g->arcs_global, a.p, sizeof(int64_t), cudaMemcpyDeviceToHost, g->stream));
        BFS_CUDA(cudaStreamSynchronize(g->stream));
    }
    BFS_CUDA(cudaEventRecord(e1, g->stream));
    BFS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    BFS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    g->build_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    bfs_alloc_state(g);
    BFS_CUDA(cudaStreamSynchronize(g->stream));
    {
        // hand construction temporaries back to the driver (the caller's allocator
        // may need the memory); run-time temporaries stay pooled
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        cudaGetLastError();
    }
    *out = g;
    g = nullptr;
    }
    catch (const Failure& f) {
        delete g;
        set_error(f.msg);
        return f.code;
    }
    catch (...) {
        delete g;
        set_error("internal error during graph construction");
        return BFS_ERR_INTERNAL;
    }
    return BFS_OK;
}

bfs_status bfs_graph_create_kronecker(const bfs_kron_spec* spec, const bfs_build_opts* opts, bfs_comm_t comm,
                                      void* cuda_stream, bfs_graph_t* out) {
    if (!spec) {
        set_error("spec is NULL");
        return BFS_ERR_INVALID_ARG;
    }
    bfs_graph_desc d{};
    d.kind = BFS_SRC_KRONECKER;
    d.kron = *spec;
    d.opts = opts ? *opts : default_opts();
    return bfs_graph_create(&d, comm, cuda_stream, out);
}

bfs_status bfs_graph_create_edges(const int32_t* uv, int64_t m, int64_t n, const bfs_build_opts* opts,
                                  bfs_comm_t comm, void* cuda_stream, bfs_graph_t* out) {
    bfs_graph_desc d{};
    d.kind = BFS_SRC_EDGES;
    d.uv = uv;
    d.m = m;
    d.n = n;
    d.opts = opts ? *opts : default_opts();
    return bfs_graph_create(&d, comm, cuda_stream, out);
}

bfs_status bfs_graph_create_csr(const int64_t* offsets, const int32_t* adj, int64_t n, const bfs_build_opts* opts,
                                bfs_comm_t comm, void* cuda_stream, bfs_graph_t* out) {
    bfs_graph_desc d{};
    d.kind = BFS_SRC_CSR;
    d.offsets = offsets;
    d.adj = adj;
    d.n = n;
    d.opts = opts ? *opts : default_opts();
    return bfs_graph_create(&d, comm, cuda_stream, out);
}

bfs_status bfs_graph_info(bfs_graph_t g, int64_t* n, int64_t* arcs, int64_t* local_begin, int64_t* local_end) {
    API_BEGIN
    if (!g) fail(BFS_ERR_INVALID_ARG, "graph is NULL");
    if (n) *n = g->n;
    if (arcs) *arcs = g->arcs_global;
    if (local_begin) *local_begin = g->lo;
    if (local_end) *local_end = g->hi;
    API_END
}

bfs_status bfs_graph_active(bfs_graph_t g, int64_t* n_active) {
    API_BEGIN
    if (!g || !n_active) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    const bool active = g->reindexed && !(g->comm && g->comm->nranks > 1) && g->nparts == 1;
    *n_active = active ? g->n_active : g->nl();
    API_END
}

bfs_status bfs_graph_tiles(bfs_graph_t g, int64_t* heavy_rows, int64_t* tiles, double* build_ms) {
    API_BEGIN
    if (!g) fail(BFS_ERR_INVALID_ARG, "graph is NULL");
    if (heavy_rows) *heavy_rows = g->tile_T ? g->tile_nh : 0;
    if (tiles) *tiles = g->tile_T;
    if (build_ms) *build_ms = g->tile_build_ms;
    API_END
}

bfs_status bfs_graph_build_ms(bfs_graph_t g, double* ms) {
    API_BEGIN
    if (!g || !ms) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    *ms = g->build_ms;
    API_END
}

bfs_status bfs_set_policy(bfs_graph_t g, const bfs_policy* p) {
    API_BEGIN
    if (!g || !p) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    if (p->mode < 0 || p->mode > 3) fail(BFS_ERR_INVALID_ARG, "policy.mode must be 0, 1, 2 or 3");
    if (p->alpha < 1 || p->alpha > (1 << 24) || p->beta < 1 || p->beta > (1 << 24))
        fail(BFS_ERR_INVALID_ARG, "alpha and beta must be in [1, 2^24]");
    if (p->bu_from_level < 0) fail(BFS_ERR_INVALID_ARG, "bu_from_level must be >= 0");
    if (p->loop < 0 || p->loop > 4)
        fail(BFS_ERR_INVALID_ARG, "loop must be 0 (auto), 1 (host), 2 (graph), 3 (persistent) or 4 (cluster)");
    g->policy = *p;
    API_END
}

bfs_status bfs_run(bfs_graph_t g, int64_t root, int32_t* parent_out, int32_t* depth_out) {
    API_BEGIN
    if (!g) fail(BFS_ERR_INVALID_ARG, "graph is NULL");
    BFS_CUDA(cudaSetDevice(g->device));
    bfs_run_impl(g, root, parent_out, depth_out);
    g->has_run = true;
    API_END
}

bfs_status bfs_stats(bfs_graph_t g, bfs_run_stats* out, bfs_level_stats* levels, int max_levels) {
    API_BEGIN
    if (!g || !out) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    if (!g->has_run) fail(BFS_ERR_INVALID_ARG, "bfs_stats before any bfs_run");
    BFS_CUDA(cudaSetDevice(g->device));
    *out = g->run;
    if (levels)
        for (int i = 0; i < max_levels && i < (int)g->levels.size(); ++i) levels[i] = g->levels[i];
    API_END
}

bfs_status bfs_component_tuples(bfs_graph_t g, int64_t* tuples) {
    API_BEGIN
    if (!g || !tuples) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    if (!g->has_run) fail(BFS_ERR_INVALID_ARG, "bfs_component_tuples before any bfs_run");
    BFS_CUDA(cudaSetDevice(g->device));
    if (g->run.component_edge_tuples < 0) g->run.component_edge_tuples = component_tuples_impl(g);
    *tuples = g->run.component_edge_tuples;
    API_END
}

bfs_status bfs_validate(bfs_graph_t g, int64_t root, const int32_t* parent, const int32_t* depth, int64_t fails[5]) {
    API_BEGIN
    if (!g || !fails) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    BFS_CUDA(cudaSetDevice(g->device));
    validate_impl(g, root, parent, depth, fails);
    API_END
}

bfs_status bfs_graph_destroy(bfs_graph_t g) {
    API_BEGIN
    if (!g) return BFS_OK;
    cudaSetDevice(g->device);
    cudaStreamSynchronize(g->stream);
    for (auto& e : g->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : g->lev_ev) cudaEventDestroy(e);
    if (g->h_cnt) cudaFreeHost(g->h_cnt);
    if (g->h_cnt_mat) cudaFreeHost(g->h_cnt_mat);
    bfsb::bfs_release_loop(g);
    delete g;
    cudaDeviceSynchronize();
    API_END
}

bfs_status bfs_comm_unique_id(uint8_t id[128]) {
    API_BEGIN
    if (!id) fail(BFS_ERR_INVALID_ARG, "id is NULL");
    comm_unique_id(id);
    API_END
}

bfs_status bfs_comm_create(int nranks, int rank, const uint8_t id[128], int device, bfs_comm_t* out) {
    API_BEGIN
    if (!id || !out) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    *out = comm_create_nccl(nranks, rank, id, device);
    API_END
}

bfs_status bfs_comm_create_local(int nparts, int device, bfs_comm_t* out) {
    API_BEGIN
    if (!out) fail(BFS_ERR_INVALID_ARG, "out is NULL");
    comm_create_local(nparts, device, out);
    API_END
}

bfs_status bfs_comm_destroy(bfs_comm_t comm) {
    API_BEGIN
    delete comm;
    API_END
}

bfs_status bfs_partition_range(int64_t n, int nranks, int rank, int64_t* local_begin, int64_t* local_end) {
    API_BEGIN
    if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks || !local_begin || !local_end)
        fail(BFS_ERR_INVALID_ARG, "bad partition arguments");
    const int64_t nb = nranks > 1 ? part_block(n, nranks) : n;
    *local_begin = std::min<int64_t>(n, (int64_t)rank * nb);
    *local_end = std::min<int64_t>(n, *local_begin + nb);
    API_END
}

bfs_status bfs_kronecker_edges(const bfs_kron_spec* spec, int64_t first, int64_t count, int32_t* uv_out,
                               void* cuda_stream) {
    API_BEGIN
    if (!uv_out && count > 0) fail(BFS_ERR_INVALID_ARG, "uv_out is NULL");
    if (count > 0 && !is_device_ptr(uv_out)) fail(BFS_ERR_INVALID_ARG, "uv_out must be device memory");
    kron_edges_device(spec, first, count, uv_out, (cudaStream_t)cuda_stream);
    BFS_CUDA(cudaStreamSynchronize((cudaStream_t)cuda_stream));
    API_END
}

bfs_status bfs_graph_export_csr(bfs_graph_t g, int64_t* offsets_out, int32_t* adj_out) {
    API_BEGIN
    if (!g) fail(BFS_ERR_INVALID_ARG, "graph is NULL");
    BFS_CUDA(cudaSetDevice(g->device));
    if (offsets_out)
        BFS_CUDA(cudaMemcpyAsync(offsets_out, g->off.p, ((size_t)g->nl() + 1) * sizeof(int64_t), cudaMemcpyDefault,
                                 g->stream));
    if (adj_out && g->arcs_local)
        BFS_CUDA(cudaMemcpyAsync(adj_out, g->adj.p, (size_t)g->arcs_local * sizeof(int32_t), cudaMemcpyDefault,
                                 g->stream));
    BFS_CUDA(cudaStreamSynchronize(g->stream));
    API_END
}

bfs_status bfs_graph_export_row(bfs_graph_t g, int64_t v, int32_t* out, int64_t cap, int64_t* degree) {
    API_BEGIN
    if (!g || !degree) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    if (v < 0 || v >= g->nl()) fail(BFS_ERR_OUT_OF_RANGE, "row outside the local range");
    BFS_CUDA(cudaSetDevice(g->device));
    int64_t be[2];
    BFS_CUDA(cudaMemcpyAsync(be, g->off.p + v, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, g->stream));
    BFS_CUDA(cudaStreamSynchronize(g->stream));
    *degree = be[1] - be[0];
    const int64_t k = std::min<int64_t>(cap, be[1] - be[0]);
    if (out && k > 0)
        BFS_CUDA(cudaMemcpyAsync(out, g->adj.p + be[0], (size_t)k * sizeof(int32_t), cudaMemcpyDefault, g->stream));
    BFS_CUDA(cudaStreamSynchronize(g->stream));
    API_END
}

bfs_status bfs_graph_export_labels(bfs_graph_t g, int32_t* new_label_out) {
    API_BEGIN
    if (!g || !new_label_out) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    BFS_CUDA(cudaSetDevice(g->device));
    if (g->reindexed) {
        BFS_CUDA(cudaMemcpyAsync(new_label_out, g->label.p, (size_t)g->n * 4, cudaMemcpyDefault, g->stream));
    } else {
        std::vector<int32_t> id((size_t)g->n);
        std::iota(id.begin(), id.end(), 0);
        BFS_CUDA(cudaMemcpyAsync(new_label_out, id.data(), (size_t)g->n * 4, cudaMemcpyDefault, g->stream));
    }
    BFS_CUDA(cudaStreamSynchronize(g->stream));
    API_END
}

bfs_status bfs_sample_roots(bfs_graph_t g, uint32_t scale, uint64_t seed, int64_t count, int64_t* roots_out,
                            int64_t* found) {
    API_BEGIN
    if (!g || !roots_out || !found) fail(BFS_ERR_INVALID_ARG, "NULL argument");
    if (count < 0) fail(BFS_ERR_INVALID_ARG, "count must be >= 0");
    if (scale > 31) fail(BFS_ERR_INVALID_ARG, "scale must be <= 31");
    BFS_CUDA(cudaSetDevice(g->device));
    sample_roots_impl(g, scale, seed, count, roots_out, found);
    API_END
}

}  // extern "C"
