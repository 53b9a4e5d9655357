// Graph construction on the device:
//   Kronecker generator fused into a degree-count
//   pass and a fill pass (the 2M-arc edge list is never materialised),
//   exclusive scan to int64 offsets, canonical per-row sort, optional
//   dedup / self-loop removal with compaction (R4, R13), the
//   degree-0 skip bitmap, and the optional section 3.4 degree reindex.
//
// Everything is integer work.  The generator is ALU-bound (10-round Philox per
// 4 levels); count/fill are bound by random 4/8-byte atomics into the degree /
// cursor arrays; the row sort is binned by row length:
//   len 2..32      one warp per row, bitonic network over lanes (shuffles)
//   len 33..32768  one CTA per row, bitonic sort in shared memory (pow2 classes)
//   len > 32768    one CTA per row: 32768-element chunks sorted in shared memory,
//                  then merge-path passes ping-ponging with a scratch buffer.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace bfsb {

// BFS_VERBOSE=1 prints wall-clock construction phases (synchronising at each mark)
struct PhaseLog {
    bool on = getenv("BFS_VERBOSE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what, cudaStream_t s) {
        if (!on) return;
        cudaStreamSynchronize(s);
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[bfs build] %-24s %9.2f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// ============================================================== Philox4x32-10
// (Salmon et al. SC'11).  Product-side implementation; the oracle has its own.
__host__ __device__ __forceinline__ void philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                  uint32_t k1, uint32_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void philox4x32_10_host(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    philox10(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1], out);
}

namespace {

struct KronParams {
    uint32_t scale, key0, key1;
    uint32_t a, ab, abc;  // cumulative quadrant thresholds per 10000
    uint32_t sk[4];       // scramble keys
    uint32_t mask;
    uint64_t m;           // number of tuples
};

KronParams make_params(const bfs_kron_spec* s) {
    KronParams P{};
    P.scale = s->scale;
    P.key0 = (uint32_t)(s->seed & 0xffffffffu);
    P.key1 = (uint32_t)(s->seed >> 32);
    P.a = s->a;
    P.ab = s->a + s->b;
    P.abc = s->a + s->b + s->c;
    uint32_t ctr[4] = {0, 0, 0, 1}, key[2] = {P.key0, P.key1};
    philox4x32_10_host(ctr, key, P.sk);
    P.mask = (uint32_t)((1ull << s->scale) - 1ull);
    P.m = (uint64_t)s->edgefactor << s->scale;
    return P;
}

__device__ __forceinline__ uint32_t scramble(const KronParams& P, uint32_t x) {
    x = ((x + P.sk[0]) * (P.sk[1] | 1u)) & P.mask;
    x = __brev(x) >> (32 - P.scale);
    x = ((x + P.sk[2]) * (P.sk[3] | 1u)) & P.mask;
    x = __brev(x) >> (32 - P.scale);
    return x;
}

// Edge i: per level a Philox word picks one initiator quadrant (row bit of u, column bit of v).
__device__ __forceinline__ void kron_edge(const KronParams& P, uint64_t i, uint32_t& u, uint32_t& v) {
    uint32_t uu = 0, vv = 0;
    for (uint32_t l = 0; l < P.scale; l += 4) {
        uint32_t w[4];
        philox10((uint32_t)i, (uint32_t)(i >> 32), l >> 2, 0u, P.key0, P.key1, w);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (l + t < P.scale) {
                uint32_t q = __umulhi(w[t], 10000u);
                uint32_t row = q >= P.ab;
                uint32_t col = (q >= P.a && q < P.ab) || q >= P.abc;
                uu |= row << (l + t);
                vv |= col << (l + t);
            }
        }
    }
    u = scramble(P, uu);
    v = scramble(P, vv);
}

__global__ void k_kron_edges(KronParams P, uint64_t first, uint64_t count, int2* uv) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count; e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u, v;
        kron_edge(P, first + e, u, v);
        uv[e] = make_int2((int)u, (int)v);
    }
}

// ---- edge sources: generated (Kronecker) or an explicit tuple array; with a
// label array both endpoints are relabeled (second pass of the degree reindex)
struct KronSource {
    KronParams P;
    const int32_t* label;
    __device__ void get(uint64_t i, uint32_t& u, uint32_t& v) const {
        kron_edge(P, i, u, v);
        if (label) {
            u = (uint32_t)label[u];
            v = (uint32_t)label[v];
        }
    }
};
struct ArraySource {
    const int2* uv;
    const int32_t* label;
    __device__ void get(uint64_t i, uint32_t& u, uint32_t& v) const {
        int2 t = uv[i];
        u = (uint32_t)t.x;
        v = (uint32_t)t.y;
        if (label) {
            u = (uint32_t)label[u];
            v = (uint32_t)label[v];
        }
    }
};

// head[v] = (first neighbour in row order or -1, degree): with rows in canonical
// order most bottom-up searches end at the first neighbour, so a dense
// coalesced 8-byte record per vertex replaces the offsets pair + a random
// adjacency sector on that path.
__global__ void k_head(const int64_t* off, const int32_t* adj, int64_t nl, int2* head) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = off[v], e = off[v + 1];
        head[v] = make_int2(e > b ? adj[b] : -1, (int)(e - b));
    }
}

// hpar[v] = original label of v's first neighbour (reindexed graphs): the parent a
// first-probe bottom-up hit writes, read coalesced beside head[v]
__global__ void k_head_parent(const int2* head, const int32_t* ilabel, int64_t nl, int32_t* hpar) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = head[v].x;
        hpar[v] = f >= 0 ? ilabel[f] : -1;
    }
}

// nb4[v] = arcs 1..4 of row v (-1 past the degree): the bottom-up step probes them
// for the rows that miss on the first arc, reading 16 dense bytes per row along its
// miss list instead of the row's offsets and a row-aligned adjacency sector
__global__ void k_nb4(const int64_t* off, const int32_t* adj, int64_t rows, int planes, int4* nb4) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < rows; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = off[v], d = off[v + 1] - b;
        for (int p = 0; p < planes; ++p) {
            const int64_t k = 1 + 4 * p;
            nb4[p * rows + v] = make_int4(d > k ? adj[b + k] : -1, d > k + 1 ? adj[b + k + 1] : -1,
                                          d > k + 2 ? adj[b + k + 2] : -1, d > k + 3 ? adj[b + k + 3] : -1);
        }
    }
}

// planes of second-probe blocks built (BFS_NB_PLANES, default 2: arcs 1..8; 16 bytes
// per plane and row).  K29 same-box A/B, 64 roots: 0 planes 1583 GTEPS, 1: 1693,
// 2: 1707, 3: 1706 (profiles/r02_nb4_ab.txt)
static int nb_planes_setting() {
    const char* e = getenv("BFS_NB_PLANES");
    return e ? std::max(0, std::min(8, atoi(e))) : 2;
}

// Degree reindex on p ranks ("after partitioning ... permutation of local IDs";
// the oracle's orc_degree_reindex_local): the 1D block partition of the ORIGINAL labels
// comes first, then every block numbers its own vertices by (degree desc, ID asc).  A
// stable sort of the global (degree desc, ID asc) order by block gives, at index i,
// the vertex with internal label i (all blocks but the last hold exactly nb labels).
// Ownership is unchanged, so the outputs of a rank's vertices stay on the rank.
__global__ void k_block_keys(const int32_t* order, int64_t n, int64_t nb, uint32_t* keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        keys[k] = (uint32_t)(order[k] / nb);
}
__global__ void k_labels_of(const int32_t* sorted, int64_t n, int32_t* label, int32_t* ilabel) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        label[sorted[i]] = (int32_t)i;
        ilabel[i] = sorted[i];
    }
}
// out[i] = a[b[i]]
__global__ void k_compose(const int32_t* a, const int32_t* b, int64_t n, int32_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[b[i]];
}

// degree-order helpers: key = maxdeg - deg (ascending key = descending degree)
__global__ void k_local_degree(const int64_t* off, int64_t nl, int32_t* deg) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x)
        deg[v] = (int32_t)(off[v + 1] - off[v]);
}

__global__ void k_degree_max(const int32_t* deg, int64_t n, unsigned int* mx) {
    unsigned int m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned int)deg[v]);
    for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

__global__ void k_degree_keys(const int32_t* deg, int64_t n, unsigned int mx, uint32_t* keys, int32_t* vals) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        keys[v] = mx - (unsigned int)deg[v];
        vals[v] = (int32_t)v;
    }
}

__global__ void k_count_active(const int64_t* off, int64_t nl, unsigned long long* cnt) {
    unsigned long long c = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x)
        c += off[v + 1] > off[v];
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// order[k] = vertex at position k  ->  rank[vertex] = k
__global__ void k_rank_of(const int32_t* order, int64_t n, int32_t* rank) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        rank[order[k]] = (int32_t)k;
}

// adj[j] <- map[adj[j]]
__global__ void k_map_ids(int32_t* adj, int64_t arcs, const int32_t* map) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < arcs; j += (int64_t)gridDim.x * blockDim.x)
        adj[j] = map[adj[j]];
}

// N1: raw arc count of owned endpoints (a self-loop counts 2)
template <class Src>
__global__ void k_count(Src src, uint64_t m, uint32_t lo, uint32_t hi, unsigned int* deg) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u, v;
        src.get(e, u, v);
        if (u >= lo && u < hi) atomicAdd(deg + (u - lo), 1u);
        if (v >= lo && v < hi) atomicAdd(deg + (v - lo), 1u);
    }
}

// N3: fill arcs u->v and v->u at atomically claimed row positions
template <class Src>
__global__ void k_fill(Src src, uint64_t m, uint32_t lo, uint32_t hi, unsigned long long* cursor, int32_t* adj) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u, v;
        src.get(e, u, v);
        if (u >= lo && u < hi) adj[atomicAdd(cursor + (u - lo), 1ull)] = (int32_t)v;
        if (v >= lo && v < hi) adj[atomicAdd(cursor + (v - lo), 1ull)] = (int32_t)u;
    }
}

// first tuple with an endpoint outside [0, n)
__global__ void k_check_edges(const int2* uv, uint64_t m, int64_t n, unsigned long long* first_bad) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        int2 t = uv[e];
        if (t.x < 0 || t.x >= n || t.y < 0 || t.y >= n) atomicMin(first_bad, (unsigned long long)e);
    }
}

// CSR input checks: offsets[0]==0, non-decreasing; adj entries in range
__global__ void k_check_csr(const int64_t* off, int64_t n, const int32_t* adj, int64_t arcs, unsigned long long* bad) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        if (off[i + 1] < off[i]) atomicMin(bad, (unsigned long long)i);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < arcs; j += stride)
        if (adj[j] < 0 || adj[j] >= n) atomicMin(bad, (unsigned long long)(n + 1 + j));
}

// CSR input: raw degree of owned rows, and copy rows
__global__ void k_csr_degree(const int64_t* off, int64_t lo, int64_t nl, unsigned int* deg) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x)
        deg[v] = (unsigned int)(off[lo + v + 1] - off[lo + v]);
}

// ============================================================== segmented sort
constexpr int32_t kPad = 0x7fffffff;
constexpr int kCtaSortMax = 32768;  // largest row sorted entirely in shared memory

// Bin rows by length class: 0 = len<=1 (nothing), 1 = 2..32 (warp), c>=2: CTA class
// with pow2 capacity 2^(c+4) (64 .. 32768), kBigClass = longer.
constexpr int kNumClasses = 13;  // 0,1, 2..11 (64..32768), 12 big
constexpr int kBigClass = 12;

__device__ __forceinline__ int len_class(int64_t len) {
    if (len <= 1) return 0;
    if (len <= 32) return 1;
    if (len > kCtaSortMax) return kBigClass;
    int c = 64 - __clzll((unsigned long long)(len - 1));  // ceil(log2 len)
    return c - 4;                                         // 64 -> 2, 32768 -> 11
}

__global__ void k_class_count(const int64_t* off, int64_t nl, unsigned long long* class_count) {
    __shared__ unsigned long long sc[kNumClasses];
    for (int c = threadIdx.x; c < kNumClasses; c += blockDim.x) sc[c] = 0;
    __syncthreads();
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        int c = len_class(off[v + 1] - off[v]);
        if (c) atomicAdd(sc + c, 1ull);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kNumClasses; c += blockDim.x)
        if (sc[c]) atomicAdd(class_count + c, sc[c]);
}

// append row v to the list of its class: lists[base[c] + cursor[c]++]
__global__ void k_bin_rows(const int64_t* off, int64_t nl, const unsigned long long* base, unsigned long long* cursor,
                           int32_t* lists) {
    const int lane = threadIdx.x & 31;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < nl;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = b0 + lane;
        int c = v < nl ? len_class(off[v + 1] - off[v]) : 0;
        unsigned peers = __match_any_sync(0xffffffffu, c);
        int leader = __ffs(peers) - 1;
        unsigned long long pos = 0;
        if (lane == leader && c != 0) pos = atomicAdd(cursor + c, (unsigned long long)__popc(peers));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (c != 0) lists[base[c] + pos + __popc(peers & ((1u << lane) - 1u))] = (int32_t)v;
    }
}

// class 1: one warp per row (len 2..32), bitonic over lanes
__global__ void k_sort_warp_rows(const int32_t* rows, unsigned long long count, const int64_t* off, int32_t* adj) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = wid; t < (int64_t)count; t += nw) {
        int64_t v = rows[t];
        int64_t b = off[v];
        int len = (int)(off[v + 1] - b);
        int32_t x = lane < len ? adj[b + lane] : kPad;
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                int32_t y = __shfl_xor_sync(0xffffffffu, x, j);
                bool up = ((lane & k) == 0);
                bool lower = ((lane & j) == 0);
                // lower lane keeps min when ascending
                int32_t mn = min(x, y), mx = max(x, y);
                x = (lower == up) ? mn : mx;
            }
        }
        if (lane < len) adj[b + lane] = x;
    }
}

// bitonic sort of s[0..cap) in shared memory by the whole CTA (cap pow2)
__device__ void cta_bitonic(int32_t* s, int cap) {
    for (int k = 2; k <= cap; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < cap / 2; i += blockDim.x) {
                // i-th compare pair: index with bit j cleared
                int lo_i = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                int hi_i = lo_i | j;
                bool up = (lo_i & k) == 0;
                int32_t a = s[lo_i], c = s[hi_i];
                if ((a > c) == up) { s[lo_i] = c; s[hi_i] = a; }
            }
            __syncthreads();
        }
    }
}

// classes 2..11: one CTA per row, row fits in shared memory (capacity cap)
__global__ void k_sort_cta_rows(const int32_t* rows, unsigned long long count, const int64_t* off, int32_t* adj, int cap) {
    extern __shared__ int32_t s[];
    for (int64_t t = blockIdx.x; t < (int64_t)count; t += gridDim.x) {
        int64_t v = rows[t];
        int64_t b = off[v];
        int len = (int)(off[v + 1] - b);
        for (int i = threadIdx.x; i < cap; i += blockDim.x) s[i] = i < len ? adj[b + i] : kPad;
        __syncthreads();
        cta_bitonic(s, cap);
        for (int i = threadIdx.x; i < len; i += blockDim.x) adj[b + i] = s[i];
        __syncthreads();
    }
}

// merge path: number of elements taken from A for output diagonal d
__device__ __forceinline__ int64_t merge_path(const int32_t* A, int64_t na, const int32_t* B, int64_t nb, int64_t d) {
    int64_t lo = d > nb ? d - nb : 0;
    int64_t hi = d < na ? d : na;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        // take mid from A, d-mid from B: valid if A[mid] > B[d-mid-1] ... standard: A[mid] <= B[d-1-mid] -> go right
        if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// class 12: rows longer than kCtaSortMax. One CTA per row: chunk sort, then merge passes.
__global__ void k_sort_big_rows(const int32_t* rows, unsigned long long count, const int64_t* off, int32_t* adj,
                                int32_t* scratch) {
    extern __shared__ int32_t s[];
    constexpr int kItems = 8;
    for (int64_t t = blockIdx.x; t < (int64_t)count; t += gridDim.x) {
        int64_t v = rows[t];
        int64_t b = off[v];
        int64_t len = off[v + 1] - b;
        int32_t* src = adj + b;
        int32_t* dst = scratch + b;
        // 1) sort chunks of kCtaSortMax in shared memory
        for (int64_t c0 = 0; c0 < len; c0 += kCtaSortMax) {
            int clen = (int)min((int64_t)kCtaSortMax, len - c0);
            for (int i = threadIdx.x; i < kCtaSortMax; i += blockDim.x) s[i] = i < clen ? src[c0 + i] : kPad;
            __syncthreads();
            cta_bitonic(s, kCtaSortMax);
            for (int i = threadIdx.x; i < clen; i += blockDim.x) src[c0 + i] = s[i];
            __syncthreads();
        }
        // 2) merge runs of length L pairwise until one run remains
        for (int64_t L = kCtaSortMax; L < len; L <<= 1) {
            for (int64_t p0 = 0; p0 < len; p0 += 2 * L) {
                int64_t na = min(L, len - p0);
                int64_t nb = min(L, len - p0 - na);
                const int32_t* A = src + p0;
                const int32_t* B = A + na;
                int64_t tot = na + nb;
                for (int64_t d0 = (int64_t)threadIdx.x * kItems; d0 < tot; d0 += (int64_t)blockDim.x * kItems) {
                    int64_t ia = merge_path(A, na, B, nb, d0);
                    int64_t ib = d0 - ia;
                    int64_t dend = min(tot, d0 + kItems);
                    for (int64_t d = d0; d < dend; ++d) {
                        bool takeA = ib >= nb || (ia < na && A[ia] <= B[ib]);
                        dst[p0 + d] = takeA ? A[ia++] : B[ib++];
                    }
                }
            }
            __syncthreads();
            int32_t* tmp = src; src = dst; dst = tmp;
        }
        // sorted data is in src; copy back to adj if it ended in scratch
        if (src != adj + b)
            for (int64_t i = threadIdx.x; i < len; i += blockDim.x) adj[b + i] = src[i];
        __syncthreads();
    }
}

// ---- dedup / self-loop removal on sorted rows: kept count per row, then compaction
__device__ __forceinline__ bool keep_arc(const int32_t* row, int64_t j, int64_t v, int dedup, int drop_loops) {
    int32_t x = row[j];
    if (drop_loops && x == v) return false;
    if (dedup && j > 0 && row[j - 1] == x) return false;
    return true;
}

__global__ void k_kept_count(const int64_t* off, const int32_t* adj, int64_t nl, int64_t lo, int dedup, int drop_loops,
                             int64_t* newdeg) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = wid; v < nl; v += nw) {
        int64_t b = off[v], len = off[v + 1] - b;
        int64_t kept = 0;
        for (int64_t j0 = 0; j0 < len; j0 += 32) {
            int64_t j = j0 + lane;
            bool k = j < len && keep_arc(adj + b, j, v + lo, dedup, drop_loops);
            kept += __popc(__ballot_sync(0xffffffffu, k));
        }
        if (lane == 0) newdeg[v] = kept;
    }
}

__global__ void k_compact(const int64_t* off, const int32_t* adj, const int64_t* noff, int32_t* nadj, int64_t nl,
                          int64_t lo, int dedup, int drop_loops) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = wid; v < nl; v += nw) {
        int64_t b = off[v], len = off[v + 1] - b;
        int64_t w = noff[v];
        for (int64_t j0 = 0; j0 < len; j0 += 32) {
            int64_t j = j0 + lane;
            bool k = j < len && keep_arc(adj + b, j, v + lo, dedup, drop_loops);
            unsigned m = __ballot_sync(0xffffffffu, k);
            if (k) nadj[w + __popc(m & ((1u << lane) - 1u))] = adj[b + j];
            w += __popc(m);
        }
    }
}

// skip bitmap: bit set = degree 0 (also set for padding bits past nl)
__global__ void k_skip_bits(const int64_t* off, int64_t nl, int64_t pwords, uint32_t* skip) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < pwords; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t bits = 0;
        for (int k = 0; k < 32; ++k) {
            int64_t v = w * 32 + k;
            if (v >= nl || off[v + 1] == off[v]) bits |= 1u << k;
        }
        skip[w] = bits;
    }
}

int grid_for(int64_t items, int threads, int per_sm = 8) {
    int64_t b = (items + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * per_sm;
    return (int)std::max<int64_t>(1, std::min(b, cap));
}

}  // namespace

void validate_kron_spec(const bfs_kron_spec* s) {
    if (!s) fail(BFS_ERR_INVALID_ARG, "kron spec is NULL");
    if (s->scale < 1) fail(BFS_ERR_INVALID_ARG, "scale must be >= 1");
    if (s->scale > 30) fail(BFS_ERR_CAPACITY, "scale " + std::to_string(s->scale) + " > 30 exceeds int32 vertex IDs");
    if (s->edgefactor < 1) fail(BFS_ERR_INVALID_ARG, "edgefactor must be >= 1");
    if ((uint64_t)s->a + s->b + s->c > 10000) fail(BFS_ERR_INVALID_ARG, "a + b + c must be <= 10000");
}

void kron_edges_device(const bfs_kron_spec* spec, int64_t first, int64_t count, int32_t* uv, cudaStream_t s) {
    validate_kron_spec(spec);
    KronParams P = make_params(spec);
    if (first < 0 || count < 0 || (uint64_t)(first + count) > P.m) fail(BFS_ERR_OUT_OF_RANGE, "edge range outside [0, M)");
    if (count == 0) return;
    k_kron_edges<<<grid_for(count, 256, 16), 256, 0, s>>>(P, (uint64_t)first, (uint64_t)count, (int2*)uv);
    BFS_CHECK_LAUNCH();
}

// Sort rows (canonical order) then optionally drop self-loops / duplicates and
// compact.  off/adj are replaced in g.
static void sort_and_compact(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    const bool filter = g->opts.dedup || g->opts.drop_self_loops;
    DevBuf<int32_t> scratch;
    if (g->opts.sort_rows || filter) {
        // ---- bin rows by length class (exact-size lists)
        DevBuf<unsigned long long> ccount;
        ccount.alloc(2 * kNumClasses, s);
        BFS_CUDA(cudaMemsetAsync(ccount.p, 0, ccount.bytes(), s));
        k_class_count<<<grid_for(nl, 256), 256, 0, s>>>(g->off.p, nl, ccount.p);
        BFS_CHECK_LAUNCH();
        unsigned long long hc[kNumClasses], hb[kNumClasses];
        BFS_CUDA(cudaMemcpyAsync(hc, ccount.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        unsigned long long total = 0;
        for (int c = 0; c < kNumClasses; ++c) { hb[c] = total; total += (c ? hc[c] : 0); }
        DevBuf<int32_t> lists;
        lists.alloc((size_t)std::max<unsigned long long>(total, 1), s);
        BFS_CUDA(cudaMemcpyAsync(ccount.p + kNumClasses, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
        BFS_CUDA(cudaMemsetAsync(ccount.p, 0, kNumClasses * sizeof(unsigned long long), s));
        k_bin_rows<<<grid_for(nl, 256), 256, 0, s>>>(g->off.p, nl, ccount.p + kNumClasses, ccount.p, lists.p);
        BFS_CHECK_LAUNCH();
        if (hc[1]) {
            k_sort_warp_rows<<<grid_for((int64_t)hc[1] * 32, 256), 256, 0, s>>>(lists.p + hb[1], hc[1], g->off.p, g->adj.p);
            BFS_CHECK_LAUNCH();
        }
        for (int c = 2; c <= 11; ++c) {
            if (!hc[c]) continue;
            int cap = 1 << (c + 4);
            int threads = std::min(1024, std::max(32, cap / 2));
            size_t smem = (size_t)cap * sizeof(int32_t);
            if (smem > 48 * 1024)
                BFS_CUDA(cudaFuncSetAttribute(k_sort_cta_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int blocks = (int)std::min<unsigned long long>(hc[c], (unsigned long long)num_sms() * 8);
            k_sort_cta_rows<<<blocks, threads, smem, s>>>(lists.p + hb[c], hc[c], g->off.p, g->adj.p, cap);
            BFS_CHECK_LAUNCH();
        }
        if (hc[kBigClass]) {
            scratch.alloc((size_t)g->arcs_local, s);
            size_t smem = (size_t)kCtaSortMax * sizeof(int32_t);
            BFS_CUDA(cudaFuncSetAttribute(k_sort_big_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int blocks = (int)std::min<unsigned long long>(hc[kBigClass], (unsigned long long)num_sms());
            k_sort_big_rows<<<blocks, 1024, smem, s>>>(lists.p + hb[kBigClass], hc[kBigClass], g->off.p,
                                                      g->adj.p, scratch.p);
            BFS_CHECK_LAUNCH();
        }
    }
    if (filter) {
        DevBuf<int64_t> newdeg, noff;
        newdeg.alloc(nl + 1, s);
        k_kept_count<<<grid_for(nl * 32, 256), 256, 0, s>>>(g->off.p, g->adj.p, nl, g->lo, g->opts.dedup,
                                                            g->opts.drop_self_loops, newdeg.p);
        BFS_CHECK_LAUNCH();
        noff.alloc(nl + 1, s);
        scan_exclusive_i64(newdeg.p, noff.p, nl, s);
        int64_t narcs = 0;
        BFS_CUDA(cudaMemcpyAsync(&narcs, noff.p + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        newdeg.reset();
        DevBuf<int32_t> nadj;
        if (scratch.p && (int64_t)scratch.count >= narcs) {
            nadj = std::move(scratch);
        } else {
            scratch.reset();
            nadj.alloc((size_t)std::max<int64_t>(narcs, 1), s);
        }
        k_compact<<<grid_for(nl * 32, 256), 256, 0, s>>>(g->off.p, g->adj.p, noff.p, nadj.p, nl, g->lo,
                                                         g->opts.dedup, g->opts.drop_self_loops);
        BFS_CHECK_LAUNCH();
        g->adj = std::move(nadj);
        g->off = std::move(noff);
        g->arcs_local = narcs;
    }
}

static void build_pass(bfs_graph_s* g, const bfs_graph_desc* d, const int32_t* label) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    PhaseLog log;
    log.mark("start", s);
    DevBuf<unsigned int> deg;
    deg.alloc((size_t)std::max<int64_t>(nl, 1), s);
    BFS_CUDA(cudaMemsetAsync(deg.p, 0, deg.bytes(), s));
    DevBuf<int2> uv_dev;  // device copy of an EDGES input
    KronParams P{};
    uint64_t m = 0;
    const uint32_t lo = (uint32_t)g->lo, hi = (uint32_t)g->hi;

    if (d->kind == BFS_SRC_KRONECKER) {
        P = make_params(&d->kron);
        m = P.m;
        g->tuples = (int64_t)m;
        k_count<<<grid_for((int64_t)m, 256, 16), 256, 0, s>>>(KronSource{P, label}, m, lo, hi, deg.p);
        BFS_CHECK_LAUNCH();
    } else if (d->kind == BFS_SRC_EDGES) {
        m = (uint64_t)d->m;
        g->tuples = d->m;
        uv_dev.alloc((size_t)std::max<int64_t>(d->m, 1), s);
        if (m) BFS_CUDA(cudaMemcpyAsync(uv_dev.p, d->uv, m * sizeof(int2), cudaMemcpyDefault, s));
        DevBuf<unsigned long long> bad;
        bad.alloc(1, s);
        BFS_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
        if (m) {
            k_check_edges<<<grid_for((int64_t)m, 256), 256, 0, s>>>(uv_dev.p, m, g->n, bad.p);
            BFS_CHECK_LAUNCH();
        }
        unsigned long long hb = 0;
        BFS_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        if (hb != ~0ull) {
            int2 t;
            BFS_CUDA(cudaMemcpy(&t, uv_dev.p + hb, sizeof(t), cudaMemcpyDeviceToHost));
            fail(BFS_ERR_MALFORMED_INPUT, "tuple " + std::to_string(hb) + " = (" + std::to_string(t.x) + ", " +
                                              std::to_string(t.y) + ") has an endpoint outside [0, " +
                                              std::to_string(g->n) + ")");
        }
        if (m) {
            k_count<<<grid_for((int64_t)m, 256, 16), 256, 0, s>>>(ArraySource{uv_dev.p, label}, m, lo, hi, deg.p);
            BFS_CHECK_LAUNCH();
        }
    }

    if (d->kind == BFS_SRC_CSR) {
        // copy the owned rows as given
        std::vector<int64_t> hoff(2);
        DevBuf<int64_t> off_in;
        off_in.alloc((size_t)g->n + 1, s);
        BFS_CUDA(cudaMemcpyAsync(off_in.p, d->offsets, ((size_t)g->n + 1) * sizeof(int64_t), cudaMemcpyDefault, s));
        int64_t total = 0, first = 0;
        BFS_CUDA(cudaMemcpyAsync(&first, off_in.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaMemcpyAsync(&total, off_in.p + g->n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        if (first != 0 || total < 0) fail(BFS_ERR_MALFORMED_INPUT, "offsets[0] must be 0 and offsets[n] >= 0");
        DevBuf<int32_t> adj_in;
        adj_in.alloc((size_t)std::max<int64_t>(total, 1), s);
        if (total) BFS_CUDA(cudaMemcpyAsync(adj_in.p, d->adj, (size_t)total * sizeof(int32_t), cudaMemcpyDefault, s));
        DevBuf<unsigned long long> bad;
        bad.alloc(1, s);
        BFS_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
        k_check_csr<<<grid_for(std::max<int64_t>(g->n, total), 256), 256, 0, s>>>(off_in.p, g->n, adj_in.p, total, bad.p);
        BFS_CHECK_LAUNCH();
        unsigned long long hb = 0;
        BFS_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        if (hb != ~0ull) {
            if ((int64_t)hb < g->n) fail(BFS_ERR_MALFORMED_INPUT, "offsets decrease at row " + std::to_string(hb));
            fail(BFS_ERR_MALFORMED_INPUT, "adj[" + std::to_string(hb - g->n - 1) + "] outside [0, n)");
        }
        int64_t b = 0, e = 0;
        BFS_CUDA(cudaMemcpy(&b, off_in.p + g->lo, sizeof(int64_t), cudaMemcpyDeviceToHost));
        BFS_CUDA(cudaMemcpy(&e, off_in.p + g->hi, sizeof(int64_t), cudaMemcpyDeviceToHost));
        g->off.alloc((size_t)nl + 1, s);
        // local offsets = off_in[lo..hi] - b
        k_csr_degree<<<grid_for(nl, 256), 256, 0, s>>>(off_in.p, g->lo, nl, deg.p);
        BFS_CHECK_LAUNCH();
        scan_exclusive_i32((const int32_t*)deg.p, g->off.p, nl, s);
        g->arcs_local = e - b;
        g->adj.alloc((size_t)std::max<int64_t>(g->arcs_local, 1), s);
        if (g->arcs_local)
            BFS_CUDA(cudaMemcpyAsync(g->adj.p, adj_in.p + b, (size_t)g->arcs_local * sizeof(int32_t),
                                     cudaMemcpyDeviceToDevice, s));
        g->tuples = total / 2;
    } else {
        // offsets from raw degrees, then the fill pass
        g->off.alloc((size_t)nl + 1, s);
        scan_exclusive_i32((const int32_t*)deg.p, g->off.p, nl, s);
        BFS_CUDA(cudaMemcpyAsync(&g->arcs_local, g->off.p + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        g->adj.alloc((size_t)std::max<int64_t>(g->arcs_local, 1), s);
        DevBuf<unsigned long long> cursor;
        cursor.alloc((size_t)nl + 1, s);
        BFS_CUDA(cudaMemcpyAsync(cursor.p, g->off.p, ((size_t)nl + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        if (d->kind == BFS_SRC_KRONECKER)
            k_fill<<<grid_for((int64_t)m, 256, 16), 256, 0, s>>>(KronSource{P, label}, m, lo, hi, cursor.p, g->adj.p);
        else if (m)
            k_fill<<<grid_for((int64_t)m, 256, 16), 256, 0, s>>>(ArraySource{uv_dev.p, label}, m, lo, hi, cursor.p, g->adj.p);
        BFS_CHECK_LAUNCH();
        cursor.reset();
        uv_dev.reset();
    }
    log.mark("count+scan+fill", s);
    // raw degree (TEPS numerator) is what the count pass produced
    g->deg_raw.alloc((size_t)std::max<int64_t>(nl, 1), s);
    BFS_CUDA(cudaMemcpyAsync(g->deg_raw.p, deg.p, (size_t)nl * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    deg.reset();

    sort_and_compact(g);
    log.mark("sort+compact", s);

    BFS_CUDA(cudaStreamSynchronize(s));
    g->arcs_global = g->arcs_local;
}

// Section 3.4 degree reindex ("reorder vertices in memory to improve local
// partition access locality" and adjacency lists "in decreasing order of vertex
// connectivity").  Pass 1 builds the CSR in original labels to get the
// final (deduplicated) degrees; a stable radix sort orders vertices by (degree
// desc, ID asc); the position becomes the internal label; pass 2 regenerates the
// graph with relabeled endpoints, so ascending internal IDs in a row are exactly
// "decreasing connectivity, ties by original ID".  Isolated vertices end up
// contiguous at the top of the label range, hubs at the bottom.
// Position of every vertex in the (degree desc, ID asc) order of the CURRENT
// graph: rank[v] = position, order[position] = v.  On p ranks the owned degree
// slices are allgathered first, so every rank computes the same order.
static void degree_order(bfs_graph_s* g, DevBuf<int32_t>& rank, DevBuf<int32_t>& order) {
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    const bool mg = g->comm && g->comm->nranks > 1;
    const int64_t slots = mg ? (int64_t)g->comm->nranks * g->nb : n;
    DevBuf<int32_t> deg;
    deg.alloc((size_t)slots, s);
    BFS_CUDA(cudaMemsetAsync(deg.p, 0, deg.bytes(), s));
    k_local_degree<<<grid_for(g->nl(), 256), 256, 0, s>>>(g->off.p, g->nl(), deg.p + g->lo);
    BFS_CHECK_LAUNCH();
    if (mg) g->comm->allgather_inplace(deg.p, (size_t)g->nb * sizeof(int32_t), s);
    DevBuf<unsigned int> mx;
    mx.alloc(1, s);
    BFS_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned int), s));
    k_degree_max<<<grid_for(n, 256), 256, 0, s>>>(deg.p, n, mx.p);
    BFS_CHECK_LAUNCH();
    unsigned int hmx = 0;
    BFS_CUDA(cudaMemcpyAsync(&hmx, mx.p, sizeof(hmx), cudaMemcpyDeviceToHost, s));
    BFS_CUDA(cudaStreamSynchronize(s));
    DevBuf<uint32_t> keys;
    keys.alloc((size_t)n, s);
    order.alloc((size_t)n, s);
    k_degree_keys<<<grid_for(n, 256), 256, 0, s>>>(deg.p, n, hmx, keys.p, order.p);
    BFS_CHECK_LAUNCH();
    deg.reset();
    const int bits = hmx ? 32 - __builtin_clz(hmx) : 0;
    radix_sort_pairs(keys.p, order.p, n, bits, s);
    keys.reset();
    rank.alloc((size_t)n, s);
    k_rank_of<<<grid_for(n, 256), 256, 0, s>>>(order.p, n, rank.p);
    BFS_CHECK_LAUNCH();
}

static void finish_graph(bfs_graph_s* g) {
    cudaStream_t s = g->stream;
    const int64_t nl = g->nl();
    const int64_t pw = padded_words(nl);
    g->skip.alloc((size_t)pw, s);
    k_skip_bits<<<grid_for(pw, 256), 256, 0, s>>>(g->off.p, nl, pw, g->skip.p);
    BFS_CHECK_LAUNCH();
    g->head.alloc((size_t)std::max<int64_t>(nl, 1), s);
    k_head<<<grid_for(nl, 256), 256, 0, s>>>(g->off.p, g->adj.p, nl, g->head.p);
    BFS_CHECK_LAUNCH();
    if (g->reindexed) {
        g->hpar.alloc((size_t)std::max<int64_t>(nl, 1), s);
        k_head_parent<<<grid_for(nl, 256), 256, 0, s>>>(g->head.p, g->ilabel.p, nl, g->hpar.p);
        BFS_CHECK_LAUNCH();
    }
    // one GPU, reindexed: rows >= n_active are empty and never listed
    const bool mg = g->comm && g->comm->nranks > 1;
    const int64_t rows = (g->reindexed && !mg) ? g->n_active : nl;
    g->nb4_planes = nb_planes_setting();
    g->nb4_rows = rows;
    g->nb4.reset();
    if (g->nb4_planes > 0) {
        g->nb4.alloc((size_t)std::max<int64_t>(rows * g->nb4_planes, 1), s);
        k_nb4<<<grid_for(rows, 256), 256, 0, s>>>(g->off.p, g->adj.p, rows, g->nb4_planes, g->nb4.p);
        BFS_CHECK_LAUNCH();
    }
    BFS_CUDA(cudaStreamSynchronize(s));
}

void build_graph(bfs_graph_s* g, const bfs_graph_desc* d) {
    cudaStream_t s = g->stream;
    build_pass(g, d, nullptr);
    if (d->opts.reindex_by_degree) {
        DevBuf<int32_t> rank, order;
        degree_order(g, rank, order);
        // pass-1 graph is no longer needed
        g->adj.reset();
        g->off.reset();
        g->deg_raw.reset();
        const bool mg = g->comm && g->comm->nranks > 1;
        const int p = mg ? g->comm->nranks : 1;
        DevBuf<int32_t> pos_of_id, id_of_pos;   // p ranks: internal label <-> global degree position
        if (mg) {
            // partition-local labels (nb = n / p, checked by the ABI): stable sort of the
            // global degree order by block
            DevBuf<uint32_t> keys;
            DevBuf<int32_t> sorted, lab, ilab;
            keys.alloc((size_t)g->n, s);
            sorted.alloc((size_t)g->n, s);
            BFS_CUDA(cudaMemcpyAsync(sorted.p, order.p, (size_t)g->n * 4, cudaMemcpyDeviceToDevice, s));
            k_block_keys<<<grid_for(g->n, 256), 256, 0, s>>>(order.p, g->n, g->nb, keys.p);
            BFS_CHECK_LAUNCH();
            radix_sort_pairs(keys.p, sorted.p, g->n, 32 - __builtin_clz((unsigned)p), s);
            keys.reset();
            lab.alloc((size_t)g->n, s);
            ilab.alloc((size_t)g->n, s);
            k_labels_of<<<grid_for(g->n, 256), 256, 0, s>>>(sorted.p, g->n, lab.p, ilab.p);
            BFS_CHECK_LAUNCH();
            sorted.reset();
            pos_of_id.alloc((size_t)g->n, s);
            id_of_pos.alloc((size_t)g->n, s);
            k_compose<<<grid_for(g->n, 256), 256, 0, s>>>(rank.p, ilab.p, g->n, pos_of_id.p);
            k_compose<<<grid_for(g->n, 256), 256, 0, s>>>(lab.p, order.p, g->n, id_of_pos.p);
            BFS_CHECK_LAUNCH();
            rank.reset();
            order.reset();
            g->label = std::move(lab);
            g->ilabel = std::move(ilab);
        } else {
            g->label = std::move(rank);
            g->ilabel = std::move(order);
        }
        build_pass(g, d, g->label.p);
        if (mg) {
            // rows in global degree order, not in the order of the local labels
            k_map_ids<<<grid_for(g->arcs_local, 256), 256, 0, s>>>(g->adj.p, g->arcs_local, pos_of_id.p);
            BFS_CHECK_LAUNCH();
            const bfs_build_opts keep = g->opts;
            g->opts = bfs_build_opts{0, 0, 0, 1};
            sort_and_compact(g);
            g->opts = keep;
            k_map_ids<<<grid_for(g->arcs_local, 256), 256, 0, s>>>(g->adj.p, g->arcs_local, id_of_pos.p);
            BFS_CHECK_LAUNCH();
        }
        g->reindexed = true;
        // isolated vertices are last in (degree desc, ID asc) order
        DevBuf<unsigned long long> cntz;
        cntz.alloc(1, s);
        BFS_CUDA(cudaMemsetAsync(cntz.p, 0, sizeof(unsigned long long), s));
        k_count_active<<<grid_for(g->nl(), 256), 256, 0, s>>>(g->off.p, g->nl(), cntz.p);
        BFS_CHECK_LAUNCH();
        unsigned long long act = 0;
        BFS_CUDA(cudaMemcpyAsync(&act, cntz.p, sizeof(act), cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        g->n_active = (int64_t)act;
    } else if (d->opts.sort_rows == 2) {
        // rows in decreasing neighbour degree, ties by ID, labels
        // unchanged: sort each row by the neighbour's degree rank, then map back
        DevBuf<int32_t> rank, order;
        degree_order(g, rank, order);
        PhaseLog log;
        k_map_ids<<<grid_for(g->arcs_local, 256), 256, 0, s>>>(g->adj.p, g->arcs_local, rank.p);
        BFS_CHECK_LAUNCH();
        const bfs_build_opts keep = g->opts;
        g->opts = bfs_build_opts{0, 0, 0, 1};
        sort_and_compact(g);
        g->opts = keep;
        k_map_ids<<<grid_for(g->arcs_local, 256), 256, 0, s>>>(g->adj.p, g->arcs_local, order.p);
        BFS_CHECK_LAUNCH();
        log.mark("degree row order", s);
    }
    finish_graph(g);
}

}  // namespace bfsb
