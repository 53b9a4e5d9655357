/*
 * include/bfs.h -- C ABI of libbfsb200.so, the B200-native direction-optimized BFS.
 *
 * What the library computes (citation keys: P:n = PAPER.md line n, S:n = SPEC.md
 * line n of arxiv 1503.04359's reference text; DESIGN.md lists every reading):
 *   level-synchronous direction-optimized BFS (Beamer's top-down push and
 *   bottom-up pull steps alternating under the alpha/beta rule; P:16, P:45-47,
 *   Alg. 1) over a CSR that stores each undirected edge as two arcs
 *   (P:168), producing a BFS parent array and per-vertex depth from a root
 *   ("computing the BFS parent of each vertex").
 *
 * Conventions shared by every call:
 *   - Every call returns bfs_status; on failure bfs_last_error() returns a
 *     thread-local, NUL-terminated message valid until the next failing call
 *     on the same thread.
 *   - Vertex IDs are int32 (n <= 2^31 - 1, Kronecker scale <= 30); arc offsets
 *     are int64.
 *   - Input arrays are BORROWED for the duration of the call only and may be
 *     host or device pointers (detected with cudaPointerGetAttributes); the
 *     library copies what it keeps.
 *   - A graph handle OWNS its device memory (on the device current at creation)
 *     and all of its work is stream-ordered on the stream given at creation
 *     (NULL = the legacy default stream).  A handle is not thread-safe.
 *   - Nothing here ever falls back to the CPU: every step of graph construction
 *     and traversal runs in the library's CUDA kernels; if no device is usable
 *     the call fails with BFS_ERR_CUDA.
 */
#ifndef BFS_B200_H
#define BFS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFS_ABI_VERSION 1

typedef struct bfs_graph_s* bfs_graph_t;
typedef struct bfs_comm_s* bfs_comm_t;

typedef enum {
    BFS_OK = 0,
    BFS_ERR_INVALID_ARG = 1,     /* NULL handle/pointer, bad option value */
    BFS_ERR_OUT_OF_RANGE = 2,    /* root outside [0, n) */
    BFS_ERR_MALFORMED_INPUT = 3, /* edge endpoint >= n, non-monotone offsets, ... */
    BFS_ERR_CAPACITY = 4,        /* scale > 30 or n beyond int32 IDs, before any allocation */
    BFS_ERR_OUT_OF_MEMORY = 5,   /* device allocation failed */
    BFS_ERR_CUDA = 6,            /* CUDA runtime failure (message carries cudaGetErrorString) */
    BFS_ERR_NCCL = 7,            /* NCCL failure or NCCL library not loadable */
    BFS_ERR_INTERNAL = 8         /* consistency check failed (a library bug) */
} bfs_status;

/* Graph500 Kronecker generator spec ("Graph500 reference code generator and
 * parameters").  n = 2^scale vertices, M = edgefactor * 2^scale
 * edge tuples; (a, b, c) are initiator probabilities per 10000 and d = 10000-a-b-c.
 * Graph500: a=5700 b=1900 c=1900.  Uniform (Erdos-Renyi-like) graph: 2500 each.
 * Edge i is a pure function of (scale, seed, a, b, c, i): Philox4x32-10 keyed by
 * seed, then a bijective label scramble (R12, R18). */
typedef struct {
    uint32_t scale, edgefactor;
    uint64_t seed;
    uint32_t a, b, c;
} bfs_kron_spec;

/* CSR build options (R4, R13).  Defaults used by the benchmark: all 1
 * except reindex_by_degree.
 *   dedup             remove repeated neighbours within a row
 *   drop_self_loops   remove arcs v->v
 *   sort_rows         rows in canonical order: ascending neighbour ID, or, with
 *                     reindex_by_degree, ascending neighbour position (degree
 *                     descending, ID ascending; "decreasing order of vertex
 *                     connectivity").  0 = arbitrary fill order.
 *   reindex_by_degree relabel vertices by (degree desc, ID asc) (section 3.4;
 *                     S:177-185); bfs_run still takes and returns ORIGINAL labels. */
typedef struct {
    int dedup, drop_self_loops, reindex_by_degree, sort_rows;
} bfs_build_opts;

/* Direction policy (R2, R3, R17, R19).
 *   mode 0  auto: start top-down (TD); in TD go bottom-up (BU) for the step that
 *           builds level d+1 iff m_f(d)*alpha > m_u(d); in BU go TD iff
 *           n_f(d)*beta < n and n_f(d) < n_f(d-1).  Integer arithmetic only.
 *   mode 1  TD only (classic BFS, "top-down (classic)")
 *   mode 2  TD for steps d < bu_from_level, BU for every step d >= bu_from_level
 *   mode 3  the paper's own rule (section 3.3; R23):
 *           in TD go BU iff m_fc(d)*10000 >= alpha*arcs, m_fc = degree sum of the
 *           frontier vertices partition 0 (the coordinator) owns, alpha = the
 *           "static percent" in units of 1/10000 (500 = 0.05); after beta BU
 *           steps ("a fixed number of steps") return to TD for the rest of the search.
 * level_times != 0 records per-step device times into bfs_level_stats.ms / kernel_ms.
 * loop (who drives the levels): 0 = auto: on one GPU a device-driven loop,
 *   the one-cluster search for graphs up to 2^21 arcs, the persistent one-kernel
 *   search up to 2^22 arcs, the CUDA loop graph (conditional WHILE/IF nodes) above; on p ranks the host (the exchange sizes are
 *   host decisions).  1 = host-driven loop (one synchronisation per level).  2 = the
 *   loop graph, 3 = the persistent kernel (one GPU; else host), 4 = the persistent
 *   search as ONE thread-block cluster (up to 16 CTAs; levels separated by the
 *   hardware cluster barrier; one GPU).  All give identical outputs and statistics
 *   (one host synchronisation per search on the device loops).
 * Defaults: mode 0, alpha 15, beta 18, bu_from_level 0, level_times 0, loop 0. */
typedef struct {
    int mode;
    int64_t alpha, beta;
    int bu_from_level;
    int level_times;
    int loop;
} bfs_policy;

/* One record per BFS step d (the step that builds level d+1 from frontier d). */
typedef struct {
    int level;              /* d */
    int direction;          /* 0 TD, 1 BU */
    int64_t frontier;       /* n_f(d)  = |{depth == d}| (global) */
    int64_t discovered;     /* n_f(d+1) */
    int64_t m_f;            /* sum of CSR degrees over frontier d */
    int64_t m_u;            /* sum of CSR degrees over {depth > d or unreached} */
    int64_t inspections;    /* TD: m_f(d); BU: sum over scanned vertices of arcs read up to and including the hit */
    int64_t scanned;        /* TD: frontier vertices expanded; BU: unvisited non-isolated vertices scanned */
    float ms;               /* device time of the whole step (0 unless policy.level_times) */
    float kernel_ms;        /* device time of the step's main kernel: TD expand or BU scan (0 unless level_times) */
    uint64_t nvlink_bytes;  /* bytes this rank sent to peers in the step (0 on one GPU) */
} bfs_level_stats;

typedef struct {
    int64_t root;                   /* original label */
    int64_t reached;                /* vertices with depth >= 0 (global) */
    int64_t component_edge_tuples;  /* input tuples with both ends reached: the TEPS numerator (R5) */
    int levels;                     /* number of steps recorded */
    double ms_total;                /* device time of bfs_run from init to the last output write (R6) */
    double ms_init, ms_compute, ms_push, ms_pull, ms_aggregate; /* Fig. 3 breakdown; 0 when not collected */
    uint64_t nvlink_bytes;
    int64_t kernel_launches;        /* CUDA kernels this rank launched inside bfs_run */
} bfs_run_stats;

typedef enum { BFS_SRC_EDGES = 0, BFS_SRC_CSR = 1, BFS_SRC_KRONECKER = 2 } bfs_source_kind;

/* Graph description for bfs_graph_create.
 *   EDGES     : uv = m tuples as int32 [m][2] (host or device), n vertices.
 *   CSR       : offsets int64[n+1], adj int32[offsets[n]] (host or device); the rows
 *               are taken as given (then sorted / deduplicated per opts).  The CSR
 *               must be symmetric for BFS on an undirected graph; not checked.
 *   KRONECKER : kron; n is ignored (2^scale); generated on the device. */
typedef struct {
    bfs_source_kind kind;
    int64_t n;
    const int32_t* uv;
    int64_t m;
    const int64_t* offsets;
    const int32_t* adj;
    bfs_kron_spec kron;
    bfs_build_opts opts;
} bfs_graph_desc;

/* ---- graph construction ----
 * comm == NULL: one GPU holds the whole graph.  comm != NULL: 1D vertex partition;
 * this rank owns vertices [local_begin, local_end) (see bfs_graph_info) and keeps
 * the arcs whose source it owns; every rank must make the same call.
 * cuda_stream: a cudaStream_t (may be NULL).  *out receives the handle. */
bfs_status bfs_graph_create(const bfs_graph_desc* desc, bfs_comm_t comm, void* cuda_stream, bfs_graph_t* out);
bfs_status bfs_graph_create_kronecker(const bfs_kron_spec* spec, const bfs_build_opts* opts, bfs_comm_t comm,
                                      void* cuda_stream, bfs_graph_t* out);
bfs_status bfs_graph_create_edges(const int32_t* uv, int64_t m, int64_t n, const bfs_build_opts* opts,
                                  bfs_comm_t comm, void* cuda_stream, bfs_graph_t* out);
bfs_status bfs_graph_create_csr(const int64_t* offsets, const int32_t* adj, int64_t n, const bfs_build_opts* opts,
                                bfs_comm_t comm, void* cuda_stream, bfs_graph_t* out);

/* n = global vertex count; arcs = global arc count (after dedup/self-loop removal);
 * [local_begin, local_end) = vertices owned by this rank (internal labels when
 * reindexed; the outputs of bfs_run are in original labels either way). */
bfs_status bfs_graph_info(bfs_graph_t g, int64_t* n, int64_t* arcs, int64_t* local_begin, int64_t* local_end);

/* Vertices the per-search bitmaps and bottom-up scans cover on this rank: with the
 * degree reindex on one GPU the non-isolated prefix [0, n_active) of the internal
 * labels (isolated vertices sit at the tail and never change state), else the
 * owned range.  Lets measurements charge bitmap bytes per launch exactly. */
bfs_status bfs_graph_active(bfs_graph_t g, int64_t* n_active);

/* Tiled top-down index (degree-reindexed graphs on one GPU):
 * *heavy_rows = rows [0, heavy_rows) whose frontier arcs a tile-mode top-down step
 * expands per label tile in shared memory, *tiles = number of label tiles (0: no
 * index, every top-down step uses the edge-balanced expansion), *build_ms = device
 * time of the index build (included in bfs_graph_build_ms).  Any pointer may be NULL. */
bfs_status bfs_graph_tiles(bfs_graph_t g, int64_t* heavy_rows, int64_t* tiles, double* build_ms);

/* Construction time of the last bfs_graph_create on this handle (device ms). */
bfs_status bfs_graph_build_ms(bfs_graph_t g, double* ms);

bfs_status bfs_set_policy(bfs_graph_t g, const bfs_policy* policy);

/* ---- the hot path (Alg. 1-3) ----
 * BFS from `root` (original label).  parent_out/depth_out: caller-owned buffers of
 * (local_end - local_begin) int32 each -- all n on one GPU (in original label
 * order), the owned slice on p GPUs -- host or device memory.  Device buffers are
 * written by the kernels only (each entry exactly once); host buffers are filled
 * by a device-to-host copy at the end of the call.
 * Output convention: parent[root] = root, depth[root] = 0; unreached
 * vertices get parent = depth = -1.  Depth is the exact hop distance; parent is
 * some valid BFS tree (bottom-up steps pick the first frontier neighbour in row
 * order).  Either output pointer may be NULL to skip that copy for host buffers.
 * Returns after the work completed; bfs_stats is valid afterwards.
 * Errors: BFS_ERR_OUT_OF_RANGE for root outside [0, n).  An isolated
 * root is not an error: one reached vertex, one step. */
bfs_status bfs_run(bfs_graph_t g, int64_t root, int32_t* parent_out, int32_t* depth_out);

/* Stats of the last bfs_run (host copy only, no device work).  levels may be NULL;
 * at most max_levels records are copied (run_stats.levels says how many exist).
 * component_edge_tuples is -1 until bfs_component_tuples has been called for
 * this run. */
bfs_status bfs_stats(bfs_graph_t g, bfs_run_stats* out, bfs_level_stats* levels, int max_levels);
/* TEPS numerator of the last bfs_run: input tuples with both endpoints reached
 * (R5) = sum of raw degrees over reached vertices / 2, reduced on
 * the device (collective on p ranks).  Meant to be called outside timed regions. */
bfs_status bfs_component_tuples(bfs_graph_t g, int64_t* tuples);

/* Graph500 validation of a search's outputs on the device: the
 * benchmark's self-check, run outside timed regions.  parent/depth: the n-entry
 * outputs of bfs_run for `root` (original labels; host or device).  fails[0..5)
 * receive the number of violations of V1 (root: parent = root, depth 0; depth 0
 * only at the root), V2 (tree edge {parent[v], v} is a stored arc), V3
 * (depth[parent[v]] = depth[v] - 1), V4 (no stored arc joins reached and unreached
 * vertices or spans more than one level) and V5 (unreached <=> parent = depth = -1;
 * parent < n).  All zero = a valid BFS tree with exact depths (the theorem in
 * oracle/oracle.c).  Returns BFS_OK whether or not the outputs are valid; errors
 * only for bad arguments (BFS_ERR_INVALID_ARG on a multi-partition graph). */
bfs_status bfs_validate(bfs_graph_t g, int64_t root, const int32_t* parent, const int32_t* depth, int64_t fails[5]);

bfs_status bfs_graph_destroy(bfs_graph_t g);

/* ---- multi-GPU (SURVEY e; Alg. 2/3) ----
 * 1D vertex partition: rank r owns [r*nb, min(n, (r+1)*nb)) with
 * nb = ceil(ceil(n/p)/32)*32 (bfs_partition_range).  Per level, bottom-up steps
 * allgather the next-frontier bitmap slices (Alg. 3 PullFrontiers); sparse top-down
 * steps send (vertex, parent) claims for remote vertices to their owners with grouped
 * send/recv after an allgather of the p x p claim counts, dense ones (global m_f >=
 * n/64) send per-peer outbox bitmaps and the parents of those claims follow in one
 * final aggregation after the last level (Alg. 2 PushFrontiers);
 * the four switch counters are allreduced, so every rank takes the same direction.
 * DESIGN.md section 7.  With reindex_by_degree the
 * reindex is partition-local (the block partition of the original labels
 * first, then each rank permutes its own local IDs by degree), so every rank
 * produces the outputs of its own original labels (n must be divisible by 32*p).
 * One process per GPU: rank 0 calls bfs_comm_unique_id and ships the 128 bytes to
 * the other ranks (e.g. torch.distributed broadcast); every rank then calls
 * bfs_comm_create with its rank and CUDA device.  NCCL is loaded at run time
 * (dlopen "libnccl.so.2"); BFS_ERR_NCCL if it is unavailable.  Every rank must
 * issue the same sequence of graph / run / stats calls (collective semantics). */
bfs_status bfs_comm_unique_id(uint8_t id[128]);
bfs_status bfs_comm_create(int nranks, int rank, const uint8_t id[128], int device, bfs_comm_t* out);
/* Testing aid: out[0..nparts) receives nparts rank endpoints that live in ONE
 * process on ONE device and exchange through device copies instead of NCCL.  Each
 * endpoint is driven from its own host thread exactly like a separate process
 * (same calls, same kernels, same host logic); only the transport differs. */
bfs_status bfs_comm_create_local(int nparts, int device, bfs_comm_t* out);
bfs_status bfs_comm_destroy(bfs_comm_t comm);
/* Host arithmetic only (no device needed): the vertex range rank `rank` of
 * `nranks` owns for an n-vertex graph. */
bfs_status bfs_partition_range(int64_t n, int nranks, int rank, int64_t* local_begin, int64_t* local_end);

const char* bfs_last_error(void);

/* ---- test / introspection exports (parity hooks; never on the timed path) ---- */
/* Edge tuples [first, first+count) of the Kronecker graph into uv_out, a DEVICE
 * buffer of int32 [count][2], generated by the library's GPU generator. */
bfs_status bfs_kronecker_edges(const bfs_kron_spec* spec, int64_t first, int64_t count, int32_t* uv_out,
                               void* cuda_stream);
/* Local CSR (internal labels) into caller buffers (host or device):
 * offsets_out int64[local_n + 1] (starting at 0), adj_out int32[local arcs]. */
bfs_status bfs_graph_export_csr(bfs_graph_t g, int64_t* offsets_out, int32_t* adj_out);
/* One local row (internal labels) into a caller buffer (host or device): writes
 * min(degree, cap) neighbours in stored order and *degree.  v is a local index
 * in [0, local_end - local_begin).  Lets tests sample rows of graphs too large to
 * export whole. */
bfs_status bfs_graph_export_row(bfs_graph_t g, int64_t v, int32_t* out, int64_t cap, int64_t* degree);
/* Internal label of every original vertex (identity unless reindexed), host or device int32[n]. */
bfs_status bfs_graph_export_labels(bfs_graph_t g, int32_t* new_label_out);
/* Root sampling (R8): candidates k = 0, 1, ... are Philox4x32-10
 * (ctr = (k lo, k hi, 0, 2), key = seed) word 0 >> (32 - scale); a candidate is
 * rejected if it has no non-self-loop arc or repeats.  roots_out: host int64[count];
 * *found = number written (< count only if candidates ran out: max 64*count + 4n). */
bfs_status bfs_sample_roots(bfs_graph_t g, uint32_t scale, uint64_t seed, int64_t count, int64_t* roots_out,
                            int64_t* found);
/* Optional allocator hook (e.g. torch's caching allocator); NULL restores cudaMalloc. */
bfs_status bfs_set_allocator(void* (*alloc_fn)(size_t bytes, void* stream, void* ctx),
                             void (*free_fn)(void* ptr, void* ctx), void* ctx);
int bfs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BFS_B200_H */
