// Internal declarations shared by the library's translation units.
// Product code only: nothing here is shared with oracle/ (DESIGN.md section 3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/bfs.h"

namespace bfsb {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);

struct Error {
    bfs_status code;
    std::string msg;
};

// Throwing inside the library, converted to bfs_status at the C-ABI boundary.
[[noreturn]] void fail(bfs_status code, const std::string& msg);

#define BFS_CUDA(expr)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            ::bfsb::fail(_e == cudaErrorMemoryAllocation ? BFS_ERR_OUT_OF_MEMORY : BFS_ERR_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" __FILE__ ":" + \
                             std::to_string(__LINE__) + ")");                                   \
    } while (0)

#define BFS_CHECK_LAUNCH() BFS_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- memory
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, cudaStream_t s);

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p; count = o.count; s = o.s;
            o.p = nullptr; o.count = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void alloc(size_t n, cudaStream_t st) {
        reset();
        s = st;
        count = n;
        p = static_cast<T*>(dev_alloc((n ? n : 1) * sizeof(T), st));
    }
    void reset() {
        if (p) dev_free(p, s);
        p = nullptr;
        count = 0;
    }
    size_t bytes() const { return count * sizeof(T); }
};

bool is_device_ptr(const void* p);

// ---------------------------------------------------------------- geometry
inline int64_t words_of(int64_t nbits) { return (nbits + 31) / 32; }
// bitmap words padded to a multiple of 4 (16-byte vector access)
inline int64_t padded_words(int64_t nbits) { return (words_of(nbits) + 3) / 4 * 4; }

int num_sms();

// ---------------------------------------------------------------- scan (scan.cu)
// out[i] = sum_{k<i} f(k) for i in [0, n], i.e. n+1 outputs (out[n] = total).
// Input is int32 or int64 array; out may alias in only when both are int64.
int scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
int scan_exclusive_i32(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s);

}  // namespace bfsb

// ---------------------------------------------------------------- communication (comm.cu)
// The opaque bfs_comm_t of the C ABI: one rank's endpoint.  Backends: NCCL (one
// process per GPU) and local (p host threads of one process on one device).
struct bfs_comm_s {
    int nranks = 1, rank = 0, device = 0;
    virtual ~bfs_comm_s() = default;
    // buf holds nranks slices of bytes_per_rank; slice `rank` is the input, all slices the output
    virtual void allgather_inplace(void* buf, size_t bytes_per_rank, cudaStream_t s) = 0;
    virtual void allreduce_sum_i64(int64_t* buf, int count, cudaStream_t s) = 0;
    virtual void allreduce_max_i64(int64_t* buf, int count, cudaStream_t s) = 0;
    // variable-size all-to-all; entries for q == rank are ignored
    virtual void alltoallv(const void* const* sendp, const size_t* sendb, void* const* recvp, const size_t* recvb,
                           cudaStream_t s) = 0;
};

namespace bfsb {
using Comm = bfs_comm_s;
void comm_unique_id(uint8_t id[128]);
Comm* comm_create_nccl(int nranks, int rank, const uint8_t id[128], int device);
void comm_create_local(int nparts, int device, Comm** out);
// 1D block partition: every rank owns a word-aligned contiguous range
inline int64_t part_block(int64_t n, int p) { return ((n + p - 1) / p + 31) / 32 * 32; }
}  // namespace bfsb

// ---------------------------------------------------------------- the handle
struct bfs_graph_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t n = 0;          // global vertices
    int64_t lo = 0, hi = 0; // owned internal-label range (whole graph on one GPU)
    int64_t arcs_local = 0; // arcs stored on this rank
    int64_t arcs_global = 0;
    int64_t tuples = 0;     // raw input tuples
    double build_ms = 0;
    bfs_build_opts opts{};
    bfs_comm_t comm = nullptr;
    int nparts = 1;         // partitions held by this process (>1 only for a local comm)
    int part0 = 0;          // first partition index held here

    // CSR of owned rows (internal labels); adjacency holds global internal IDs
    bfsb::DevBuf<int64_t> off;      // [nl + 1]
    bfsb::DevBuf<int32_t> adj;      // [arcs_local]
    bfsb::DevBuf<int32_t> deg_raw;  // [nl] raw arcs per vertex (TEPS numerator)
    bfsb::DevBuf<uint32_t> skip;    // [padded words of nl] bit set = CSR degree 0
    bfsb::DevBuf<int2> head;        // [nl] (first neighbour or -1, degree): the bottom-up fast path,
                                    // and the degree of a vertex discovered top-down
    bfsb::DevBuf<int32_t> hpar;     // [nl] reindexed only: ORIGINAL label of the first neighbour
    bfsb::DevBuf<int4> nb4;         // [planes][nb4_rows] plane p: arcs 1+4p..4+4p of each row (-1 past
                                    // the degree): the bottom-up second probes read along the miss list
    int64_t nb4_rows = 0;
    int nb4_planes = 0;
    // reindex (identity when absent)
    bool reindexed = false;
    int64_t n_active = 0;            // reindexed: labels >= n_active are isolated
    bool visited_tail_ok = false;    // visited words past n_active hold their skip bits
    bfsb::DevBuf<int32_t> label;    // [n] original -> internal
    bfsb::DevBuf<int32_t> ilabel;   // [n] internal -> original

    // BFS state
    bfsb::DevBuf<uint32_t> visited;  // [padded words of nl]
    bfsb::DevBuf<uint32_t> front;    // [padded words of n] global frontier bitmap
    bfsb::DevBuf<uint32_t> next;     // [padded words of n] global next bitmap
    bfsb::DevBuf<int32_t> q0, q1;    // [nl] frontier queues (global internal IDs)
    bfsb::DevBuf<int32_t> qd0, qd1;  // [nl] degree of each queued vertex
    bfsb::DevBuf<int64_t> prefix;    // [nl + 1] TD degree prefix
    bfsb::DevBuf<int64_t> cnt;       // [8] device counters
    int64_t* h_cnt = nullptr;        // pinned mirror
    bfsb::DevBuf<int32_t> tmp_depth, tmp_parent;  // host-output staging
    bfsb::DevBuf<int2> rec;          // [nl] (depth, parent) recorded at discovery, internal order
    bfsb::DevBuf<int64_t> scratch64; // TD chunk starts
    // 1D partition (p > 1)
    int64_t nb = 0;                  // block size: rank r owns [r*nb, min(n, (r+1)*nb))
    bfsb::DevBuf<uint32_t> seen;     // [n/32] remote vertices already claimed this BFS
    bfsb::DevBuf<int2> out_list, in_list;  // (vertex, parent) claims
    bfsb::DevBuf<int32_t> flist;     // sparse pull: frontier vertices received from peers
    bfsb::DevBuf<int64_t> out_cnt;   // [p]
    // bitmap-mode top-down push (dense levels): outbox / inbox bitmaps (p slices of nb/32
    // words) and the per-owner parent logs (p * nb entries) sent after the last level
    bfsb::DevBuf<uint32_t> outbox, inbox;
    bfsb::DevBuf<int4> plog, plog_in;
    bfsb::DevBuf<int64_t> plog_cnt;  // [p]
    bfsb::DevBuf<int64_t> cnt_mat;   // [p*p] claim counts, row = sender
    int64_t* h_cnt_mat = nullptr;    // pinned mirror

    // device-driven level loop (one GPU): state, per-step records, scan tile states,
    // the instantiated loop graph and pinned mirrors for the one read-back per search
    bfsb::DevBuf<int64_t> ctl, tstate;   // ctl: loop state followed by the step records
    bfsb::DevBuf<uint32_t> tctr;
    cudaGraph_t loop_graph = nullptr;
    cudaGraphExec_t loop_exec = nullptr;
    std::vector<int> loop_key;       // tuning knobs the graph was built with
    int64_t* h_ctl = nullptr;
    int64_t* h_lrec = nullptr;

    // tiled top-down (td_tile.cuh; degree-reindexed graphs on one GPU): heavy rows
    // [0, tile_nh), tile_T tiles of internal labels, per heavy row the first arc of
    // each tile; tile_T == 0: no index (tile mode off)
    int64_t tile_nh = 0;
    int tile_T = 0, tile_maxw = 0;
    int tile_units = 0;
    bfsb::DevBuf<int32_t> tile_start;  // [T + 1] first label of each tile (multiples of 32), then the end
    bfsb::DevBuf<int2> tile_unit;      // [units] (tile, part | parts << 16): hub tiles split over several CTAs
    bfsb::DevBuf<int32_t> tile_bnd;    // [nh * (T + 1)]
    bfsb::DevBuf<int32_t> tile_hlist;  // [nh] heavy frontier vertices of the current step
    bfsb::DevBuf<uint32_t> tile_hcnt;  // [1] heavy-list length
    // tile-mode record log (td_tile.cuh): per unit one bucket per 2^kWinShift-label window
    int tile_nwl = 0;                  // (tile, window) pairs
    bfsb::DevBuf<int2> tile_pool;      // (vertex, parent) entries
    bfsb::DevBuf<int64_t> tile_ubase;  // [units] first entry of each unit's buckets
    bfsb::DevBuf<uint32_t> tile_ucnt;  // [units * kMaxWin] entries per bucket
    bfsb::DevBuf<int2> tile_wl;        // [nwl] (tile, window)
    bfsb::DevBuf<int32_t> tile_fu;     // [T] first unit of each tile
    bfsb::DevBuf<int32_t> tile_wf;     // [T] first (tile, window) index of each tile
    bfsb::DevBuf<int2> tile_lpool;     // [nwl * kWin] light-row winners per (tile, window)
    bfsb::DevBuf<uint32_t> tile_lcnt;  // [nwl]
    double tile_build_ms = 0;

    bfs_policy policy{0, 15, 18, 0, 0, 0};
    bfsb::DevBuf<int32_t> big;       // persistent kernel: big frontier rows of a top-down step
    bfsb::DevBuf<int64_t> pcnt;      // persistent kernel: three counter sets
    int64_t coop_fallbacks = 0;      // persistent searches that ran as the loop graph (grid not co-resident)
    std::vector<bfs_level_stats> levels;
    bfs_run_stats run{};
    int64_t last_root_l = 0;
    bool has_run = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> lev_ev;

    int64_t nl() const { return hi - lo; }
};

namespace bfsb {
// build.cu
void build_graph(bfs_graph_s* g, const bfs_graph_desc* d);
// sort.cu: stable ascending sort of (key, value) pairs in place
void radix_sort_pairs(uint32_t* keys, int32_t* vals, int64_t n, int key_bits, cudaStream_t s);
void kron_edges_device(const bfs_kron_spec* spec, int64_t first, int64_t count, int32_t* uv, cudaStream_t s);
void validate_kron_spec(const bfs_kron_spec* spec);
// bfs.cu
void bfs_alloc_state(bfs_graph_s* g);
void bfs_build_tiles(bfs_graph_s* g);
void bfs_run_impl(bfs_graph_s* g, int64_t root, int32_t* parent_out, int32_t* depth_out);
void bfs_release_loop(bfs_graph_s* g);
int64_t component_tuples_impl(bfs_graph_s* g);
// validate.cu
void validate_impl(bfs_graph_s* g, int64_t root, const int32_t* parent, const int32_t* depth, int64_t fails[5]);
void sample_roots_impl(bfs_graph_s* g, uint32_t scale, uint64_t seed, int64_t count, int64_t* roots, int64_t* found);
// host-side Philox (product's own; used for root candidates)
void philox4x32_10_host(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
}  // namespace bfsb
