/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain, slow, obviously-correct serial CPU implementation of what the
 * direction-optimized BFS hot path computes.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` leg may load this library.
 * The product path (paper_1503_04359_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with the
 * CUDA sources.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n
 * (the reference is not present on the GPU box; citations are for readers).
 *
 * Everything here is integer arithmetic: BFS has no floating point.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11; the Random123 reference).
 * SPEC S:127 asks for "a seedable counter-based generator so edge i is
 * computable independently"; reading R12 fixes Philox4x32-10.
 * Pinned by the Random123 known-answer vectors in tests/test_oracle_generator.py. */
static void philox_round(uint32_t ctr[4], const uint32_t key[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * ctr[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * ctr[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ ctr[1] ^ key[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ ctr[3] ^ key[1];
    uint32_t n3 = lo0;
    ctr[0] = n0; ctr[1] = n1; ctr[2] = n2; ctr[3] = n3;
}

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t ctr[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t key[2] = {key_in[0], key_in[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { key[0] += 0x9E3779B9u; key[1] += 0xBB67AE85u; }
        philox_round(ctr, key);
    }
    out[0] = ctr[0]; out[1] = ctr[1]; out[2] = ctr[2]; out[3] = ctr[3];
}

static void seed_key(uint64_t seed, uint32_t key[2]) {
    key[0] = (uint32_t)(seed & 0xffffffffu);
    key[1] = (uint32_t)(seed >> 32);
}

/* ------------------------------------------------------------------------- */
/* Graph500-style Kronecker generator ("built with the Graph500 reference
 * code generator and parameters"; R12, R18).
 * Edge i is a pure function of (scale, seed, a, b, c, i):
 *   for level l in 0..scale-1:
 *     r = Philox(ctr = (i lo, i hi, l/4, 0), key = seed)[l % 4]
 *     q = (r * 10000) >> 32                      -- uniform in [0, 10000)
 *     quadrant: q < a -> (0,0); q < a+b -> (0,1); q < a+b+c -> (1,0); else (1,1)
 *     u |= row << l;  v |= col << l
 *   then both endpoints go through the scramble bijection below. */

/* reverse the low `scale` bits of v */
static uint32_t bitrev_s(uint32_t v, int scale) {
    uint32_t r = 0;
    for (int b = 0; b < scale; ++b)
        r |= ((v >> b) & 1u) << (scale - 1 - b);   /* bit b of v -> bit scale-1-b */
    return r;
}

/* scramble keys: Philox(ctr = (0,0,0,1), key = seed) */
void orc_kron_scramble_keys(uint64_t seed, uint32_t k_out[4]) {
    uint32_t ctr[4] = {0, 0, 0, 1}, key[2];
    seed_key(seed, key);
    orc_philox4x32_10(ctr, key, k_out);
}

/* v -> ((v + k0) * (k1|1)) mod 2^s -> bitrev_s -> ((. + k2) * (k3|1)) mod 2^s -> bitrev_s.
 * Each stage is a bijection of [0, 2^s) (add, multiply by an odd number, bit
 * reversal), so the composition is a vertex relabeling ("vertex labels are
 * randomly permuted after generation"). */
uint32_t orc_kron_scramble(int scale, const uint32_t k[4], uint32_t v) {
    uint64_t mask = (scale >= 32) ? 0xffffffffull : ((1ull << scale) - 1ull);
    uint64_t x = v;
    x = ((x + k[0]) * (uint64_t)(k[1] | 1u)) & mask;
    x = bitrev_s((uint32_t)x, scale);
    x = ((x + k[2]) * (uint64_t)(k[3] | 1u)) & mask;
    x = bitrev_s((uint32_t)x, scale);
    return (uint32_t)x;
}

/* Edges [first, first+count) as int32 pairs uv[2k], uv[2k+1].
 * scramble = 0 returns the pre-permutation labels (used by the statistical pins). */
void orc_kron_edges(int scale, uint64_t seed, uint32_t a, uint32_t b, uint32_t c,
                    int64_t first, int64_t count, int scramble, int32_t* uv) {
    uint32_t key[2], k[4];
    seed_key(seed, key);
    orc_kron_scramble_keys(seed, k);
    for (int64_t e = 0; e < count; ++e) {
        uint64_t i = (uint64_t)(first + e);
        uint32_t u = 0, v = 0;
        uint32_t words[4] = {0, 0, 0, 0};
        for (int l = 0; l < scale; ++l) {
            if (l % 4 == 0) {
                uint32_t ctr[4] = {(uint32_t)(i & 0xffffffffu), (uint32_t)(i >> 32), (uint32_t)(l / 4), 0};
                orc_philox4x32_10(ctr, key, words);
            }
            uint32_t r = words[l % 4];
            uint32_t q = (uint32_t)(((uint64_t)r * 10000u) >> 32);
            /* the quadrant table above as comparisons (the same values, no data-
             * dependent branch: a K29 pass regenerates 8.6 G tuples, section 8(c4)):
             *   row = 1 iff q >= a+b             -- quadrants C, D
             *   col = 1 iff a <= q < a+b  or  q >= a+b+c   -- quadrants B, D */
            uint32_t row = (uint32_t)(q >= a + b);
            uint32_t col = ((uint32_t)(q >= a) & (uint32_t)(q < a + b)) | (uint32_t)(q >= a + b + c);
            u |= row << l;
            v |= col << l;
        }
        if (scramble) {
            u = orc_kron_scramble(scale, k, u);
            v = orc_kron_scramble(scale, k, v);
        }
        uv[2 * e] = (int32_t)u;
        uv[2 * e + 1] = (int32_t)v;
    }
}

/* ------------------------------------------------------------------------- */
/* CSR build ("represents each undirected edge as two directed edges";
 * S:44-52).  Each tuple {u,v} contributes arc u->v and arc v->u (a self-loop
 * gives two identical arcs u->u); rows are filled in input encounter order.
 * Options (R4, R13):
 *   sort_rows       : sort each row ascending by neighbour ID (canonical order)
 *   drop_self_loops : remove arcs v->v
 *   dedup           : keep only the first occurrence of each neighbour in a row
 * Returns 0, or -(k+1) when tuple k has an endpoint outside [0,n).
 * offsets: int64[n+1]; adj: capacity 2*m; *arcs_out = offsets[n]. */
static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

int64_t orc_build_csr(int64_t n, int64_t m, const int32_t* uv, int dedup, int drop_self_loops,
                      int sort_rows, int64_t* offsets, int32_t* adj, int64_t* arcs_out) {
    for (int64_t k = 0; k < m; ++k) {
        int32_t u = uv[2 * k], v = uv[2 * k + 1];
        if (u < 0 || u >= n || v < 0 || v >= n) return -(k + 1);
    }
    int64_t* deg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t k = 0; k < m; ++k) {
        deg[uv[2 * k]] += 1;
        deg[uv[2 * k + 1]] += 1;
    }
    offsets[0] = 0;
    for (int64_t v = 0; v < n; ++v) offsets[v + 1] = offsets[v] + deg[v];
    int64_t* cur = deg; /* reuse as fill cursor */
    for (int64_t v = 0; v < n; ++v) cur[v] = offsets[v];
    for (int64_t k = 0; k < m; ++k) {
        int32_t u = uv[2 * k], v = uv[2 * k + 1];
        adj[cur[u]++] = v;
        adj[cur[v]++] = u;
    }
    free(deg);
    if (sort_rows)
        for (int64_t v = 0; v < n; ++v)
            qsort(adj + offsets[v], (size_t)(offsets[v + 1] - offsets[v]), sizeof(int32_t), cmp_i32);
    if (dedup || drop_self_loops) {
        /* compact in place, row by row; rows only shrink so writes never overtake reads */
        int64_t w = 0;
        int64_t row_begin = offsets[0];
        for (int64_t v = 0; v < n; ++v) {
            int64_t row_end = offsets[v + 1];
            int64_t out_begin = w;
            for (int64_t j = row_begin; j < row_end; ++j) {
                int32_t x = adj[j];
                if (drop_self_loops && x == v) continue;
                if (dedup) {
                    int seen = 0;
                    if (sort_rows) {
                        /* sorted row: an earlier copy of x is the last kept entry */
                        seen = (w > out_begin && adj[w - 1] == x);
                    } else {
                        for (int64_t t = out_begin; t < w; ++t)
                            if (adj[t] == x) { seen = 1; break; }
                    }
                    if (seen) continue;
                }
                adj[w++] = x;
            }
            row_begin = row_end;
            offsets[v + 1] = w;
        }
    }
    *arcs_out = offsets[n];
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Optional degree reindex (section 3.4).
 * position k of vertex v = its place when all vertices are ordered by
 * (degree descending, ID ascending).  With p partitions, position k is dealt
 * round-robin: partition k % p, local index k / p, new label
 * (k % p) * (n / p) + k / p  (p must divide n).  p = 1 gives new label = k.
 * Outputs new_label[v] and position[v]. */
static const int64_t* g_sort_deg;
static int cmp_deg_desc_id_asc(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    if (g_sort_deg[a] != g_sort_deg[b]) return g_sort_deg[a] > g_sort_deg[b] ? -1 : 1;
    return (a > b) - (a < b);
}

int orc_degree_reindex(int64_t n, const int64_t* offsets, int64_t p, int64_t* new_label, int64_t* position) {
    if (p <= 0 || n % p != 0) return -1;
    int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* deg = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) { order[v] = v; deg[v] = offsets[v + 1] - offsets[v]; }
    g_sort_deg = deg;
    qsort(order, (size_t)n, sizeof(int64_t), cmp_deg_desc_id_asc);
    int64_t per = n / p;
    for (int64_t k = 0; k < n; ++k) {
        int64_t v = order[k];
        position[v] = k;
        new_label[v] = (k % p) * per + k / p;
    }
    free(order);
    free(deg);
    return 0;
}

/* Partition-local degree reindex ("after partitioning, a vertex is identified
 * by ... a global ID ... and a local ID ... permutation of local IDs ... reorder
 * vertices in memory to improve local partition access locality").  The 1D block
 * partition comes first: partition b holds the original labels [b*per, (b+1)*per),
 * per = n / p.  Each partition then numbers its own vertices by (degree descending,
 * ID ascending): new label = b*per + (index of v among partition b's vertices in that
 * order).  position[v] = v's place in the GLOBAL (degree desc, ID asc) order, which
 * orders the rows (decreasing connectivity).  p = 1 gives orc_degree_reindex.
 * Walking the global order once, each partition hands out its next local index. */
int orc_degree_reindex_local(int64_t n, const int64_t* offsets, int64_t p, int64_t* new_label, int64_t* position) {
    if (p <= 0 || n % p != 0) return -1;
    int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* deg = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* next = (int64_t*)calloc((size_t)p, sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) { order[v] = v; deg[v] = offsets[v + 1] - offsets[v]; }
    g_sort_deg = deg;
    qsort(order, (size_t)n, sizeof(int64_t), cmp_deg_desc_id_asc);
    int64_t per = n / p;
    for (int64_t k = 0; k < n; ++k) {
        int64_t v = order[k];
        int64_t b = v / per;
        position[v] = k;
        new_label[v] = b * per + next[b]++;
    }
    free(next);
    free(order);
    free(deg);
    return 0;
}

/* Relabel a CSR through new_label and order every row by the neighbour's
 * position (degree descending, ties by original ID: S:189).  Row of new vertex
 * new_label[v] = { new_label[x] : x in adj(v) }. */
static const int64_t* g_sort_pos;
static int cmp_by_pos(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    int64_t pa = g_sort_pos[a], pb = g_sort_pos[b];
    return (pa > pb) - (pa < pb);
}

void orc_relabel_csr(int64_t n, const int64_t* offsets, const int32_t* adj, const int64_t* new_label,
                     const int64_t* position, int64_t* offsets_out, int32_t* adj_out) {
    int64_t* inv = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) inv[new_label[v]] = v;
    offsets_out[0] = 0;
    for (int64_t nv = 0; nv < n; ++nv) {
        int64_t v = inv[nv];
        offsets_out[nv + 1] = offsets_out[nv] + (offsets[v + 1] - offsets[v]);
    }
    int64_t maxdeg = 0;
    for (int64_t v = 0; v < n; ++v)
        if (offsets[v + 1] - offsets[v] > maxdeg) maxdeg = offsets[v + 1] - offsets[v];
    int64_t* tmp = (int64_t*)malloc((size_t)(maxdeg > 0 ? maxdeg : 1) * sizeof(int64_t));
    g_sort_pos = position;
    for (int64_t nv = 0; nv < n; ++nv) {
        int64_t v = inv[nv];
        int64_t d = offsets[v + 1] - offsets[v];
        for (int64_t j = 0; j < d; ++j) tmp[j] = adj[offsets[v] + j];
        qsort(tmp, (size_t)d, sizeof(int64_t), cmp_by_pos);
        for (int64_t j = 0; j < d; ++j) adj_out[offsets_out[nv] + j] = (int32_t)new_label[tmp[j]];
    }
    free(tmp);
    free(inv);
}

/* Rows in "decreasing order of vertex connectivity, so that the highest degree
 * vertex in the adjacency list comes first", ties by ascending ID,
 * labels unchanged: every row of (offsets, adj) is re-sorted in place. */
static const int64_t* g_row_off;
static int cmp_nbr_deg_desc(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    int64_t da = g_row_off[a + 1] - g_row_off[a], db = g_row_off[b + 1] - g_row_off[b];
    if (da != db) return da > db ? -1 : 1;
    return (a > b) - (a < b);
}

void orc_sort_rows_by_degree(int64_t n, const int64_t* offsets, int32_t* adj) {
    g_row_off = offsets;
    for (int64_t v = 0; v < n; ++v)
        qsort(adj + offsets[v], (size_t)(offsets[v + 1] - offsets[v]), sizeof(int32_t), cmp_nbr_deg_desc);
}

/* ------------------------------------------------------------------------- */
/* Serial FIFO BFS -- the plain definition of BFS depth (section 2.2;
 * S:353-361).  depth[root]=0, parent[root]=root; pop u; for v in adj(u) in
 * stored order: if depth[v] < 0 then depth[v]=depth[u]+1, parent[v]=u, push v.
 * Unreached vertices keep -1.  No bitmaps, no direction logic.
 * Returns the number of reached vertices, or -1 if root is out of range. */
int64_t orc_bfs(int64_t n, const int64_t* offsets, const int32_t* adj, int64_t root,
                int32_t* depth, int32_t* parent) {
    if (root < 0 || root >= n) return -1;
    for (int64_t v = 0; v < n; ++v) { depth[v] = -1; parent[v] = -1; }
    int32_t* queue = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    int64_t head = 0, tail = 0;
    depth[root] = 0;
    parent[root] = (int32_t)root;
    queue[tail++] = (int32_t)root;
    while (head < tail) {
        int32_t u = queue[head++];
        for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
            int32_t v = adj[j];
            if (depth[v] < 0) {
                depth[v] = depth[u] + 1;
                parent[v] = u;
                queue[tail++] = v;
            }
        }
    }
    free(queue);
    return tail;
}

/* ------------------------------------------------------------------------- */
/* Graph500 validator ("experimental methodology defined by Graph500";
 * S:362-370).  Checks, counting failures per rule:
 *   V1 parent[root]=root, depth[root]=0, and depth 0 only at the root
 *   V2 every reached v != root has {parent[v], v} as a graph edge
 *   V3 depth[parent[v]] = depth[v] - 1 for every reached v != root
 *   V4 every arc {a,b}: both reached with |depth a - depth b| <= 1, or both unreached
 *   V5 unreached <=> parent = depth = -1 (and reached <=> both >= 0)
 *   V6 depth == ref_depth element-wise (skipped when ref_depth is NULL)
 * fails[6] receives the counts, first_bad[6] the first offending vertex (or -1).
 * Returns the total number of failures (0 = passed). */
int64_t orc_validate(int64_t n, const int64_t* offsets, const int32_t* adj, int64_t root,
                     const int32_t* depth, const int32_t* parent, const int32_t* ref_depth,
                     int64_t fails[6], int64_t first_bad[6]) {
    for (int r = 0; r < 6; ++r) { fails[r] = 0; first_bad[r] = -1; }
#define FAIL(r, v) do { if (fails[r]++ == 0) first_bad[r] = (v); } while (0)
    if (root < 0 || root >= n) { FAIL(0, root); return 1; }
    if (parent[root] != root || depth[root] != 0) FAIL(0, root);
    for (int64_t v = 0; v < n; ++v) {
        int reached_d = depth[v] >= 0, reached_p = parent[v] >= 0;
        if (reached_d != reached_p || depth[v] < -1 || parent[v] < -1 || parent[v] >= n) { FAIL(4, v); continue; }
        if (!reached_d) continue;
        if (depth[v] == 0 && v != root) FAIL(0, v);
        if (v == root) continue;
        int32_t p = parent[v];
        int found = 0;
        for (int64_t j = offsets[v]; j < offsets[v + 1]; ++j)
            if (adj[j] == p) { found = 1; break; }
        if (!found) FAIL(1, v);
        if (depth[p] != depth[v] - 1) FAIL(2, v);
    }
    for (int64_t a = 0; a < n; ++a) {
        for (int64_t j = offsets[a]; j < offsets[a + 1]; ++j) {
            int32_t b = adj[j];
            int ra = depth[a] >= 0, rb = depth[b] >= 0;
            if (ra != rb) { FAIL(3, a); break; }
            if (ra && (depth[a] - depth[b] > 1 || depth[b] - depth[a] > 1)) { FAIL(3, a); break; }
        }
    }
    if (ref_depth)
        for (int64_t v = 0; v < n; ++v)
            if (depth[v] != ref_depth[v]) FAIL(5, v);
#undef FAIL
    int64_t total = 0;
    for (int r = 0; r < 6; ++r) total += fails[r];
    return total;
}

/* ------------------------------------------------------------------------- */
/* Streaming Graph500 validator (P:168
 * "experimental methodology defined by Graph500").  The rules of orc_validate,
 * checked against the input TUPLES themselves (regenerated by orc_kron_edges)
 * instead of a CSR, for R searches of one graph at once, so it runs at scales
 * where the serial oracle's CSR does not fit in host memory.
 *
 * Why it pins depths exactly (SURVEY c4 theorem): if V1-V5 hold then
 *   - V2+V3+V1: following parents from a reached v walks real edges, one level
 *     down per step, and can only stop at the root, so dist(v) <= depth(v);
 *   - V4 along a shortest path r = x0, x1, ..., xk = v: depth(x_i) <= depth(x_{i-1}) + 1
 *     and every x_i is reached, so depth(v) <= k = dist(v);
 *   - V4 carries reachability across every edge, and V5 makes the unreached
 *     exactly the vertices with depth -1: the reached set is the root's component.
 * Hence depth == the hop distance == the serial oracle's depth, vertex by vertex.
 *
 * Layout (vertex-major so one tuple touches one cache line per endpoint per array):
 *   depth8[v * R + r]   int8  depth of v in search r, -1 unreached (callers check depth < 127)
 *   parent[v * R + r]   int32 parent of v in search r, -1 unreached
 *   witness[v * R + r]  uint8 set to 1 by the edge pass when a tuple {parent[v], v} exists
 *
 * Edge pass over tuples uv[0..count) (tuple indices index0...): for every tuple
 * {a, b} and search r
 *   V4: both reached with |depth a - depth b| <= 1, or both unreached;
 *   V2 witness: parent[b] == a  =>  witness[b] = 1;  parent[a] == b  =>  witness[a] = 1.
 * fails_v4[r] counts failing tuples, first_v4[r] = index of the first one (or -1).
 * Passes over disjoint tuple ranges may run concurrently: witness bytes only ever
 * go 0 -> 1 (atomic store). */
void orc_stream_validate_edges(int64_t n, int R, const int32_t* uv, int64_t count, int64_t index0,
                               const int8_t* depth8, const int32_t* parent, uint8_t* witness,
                               int64_t* fails_v4, int64_t* first_v4) {
    for (int64_t k = 0; k < count; ++k) {
        int64_t a = uv[2 * k], b = uv[2 * k + 1];
        if (a < 0 || a >= n || b < 0 || b >= n) continue;   /* not a tuple of this graph */
        for (int r = 0; r < R; ++r) {
            int da = depth8[a * R + r], db = depth8[b * R + r];
            int ra = da >= 0, rb = db >= 0;
            if (ra != rb || (ra && (da - db > 1 || db - da > 1))) {
                if (fails_v4[r]++ == 0) first_v4[r] = index0 + k;
            }
            if (parent[b * R + r] == (int32_t)a) __atomic_store_n(&witness[b * R + r], (uint8_t)1, __ATOMIC_RELAXED);
            if (parent[a * R + r] == (int32_t)b) __atomic_store_n(&witness[a * R + r], (uint8_t)1, __ATOMIC_RELAXED);
        }
    }
}

/* Vertex pass over v in [v0, v1), after every tuple went through the edge pass;
 * the per-vertex rules in orc_validate's order:
 *   V1 root: parent = root and depth 0; depth 0 only at the root
 *   V5 reached (depth >= 0) <=> parent >= 0; depth, parent >= -1; parent < n
 *   V2 every reached v != root has its witness (the tuple {parent[v], v} exists)
 *   V3 depth[parent[v]] = depth[v] - 1 for every reached v != root
 * fails[r * 5 + i] counts failures of rule V(i+1) (slot 3 = V4 belongs to the
 * edge pass and stays 0), first[r * 5 + i] the first offending vertex (or -1). */
void orc_stream_validate_vertices(int64_t n, int R, const int64_t* roots, const int8_t* depth8,
                                  const int32_t* parent, const uint8_t* witness, int64_t v0, int64_t v1,
                                  int64_t* fails, int64_t* first) {
#define SFAIL(r, i, v) do { if (fails[(r) * 5 + (i)]++ == 0) first[(r) * 5 + (i)] = (v); } while (0)
    for (int64_t v = v0; v < v1; ++v) {
        for (int r = 0; r < R; ++r) {
            int d = depth8[v * R + r];
            int32_t p = parent[v * R + r];
            int64_t root = roots[r];
            if (v == root && (p != (int32_t)root || d != 0)) SFAIL(r, 0, v);
            if ((d >= 0) != (p >= 0) || d < -1 || p < -1 || p >= n) { SFAIL(r, 4, v); continue; }
            if (d < 0) continue;
            if (d == 0 && v != root) SFAIL(r, 0, v);
            if (v == root) continue;
            if (!witness[v * R + r]) SFAIL(r, 1, v);
            if (depth8[(int64_t)p * R + r] != d - 1) SFAIL(r, 2, v);
        }
    }
#undef SFAIL
}

/* ------------------------------------------------------------------------- */
/* Direction-optimized BFS emulator (P:16, P:47 Beamer's
 * method; section 3.3).  From the oracle depth and the CSR
 * it derives, for every step d = 0, 1, ... (the step that builds level d+1 from
 * the frontier {depth == d}):
 *   n_f(d) = |{depth = d}|,   m_f(d) = sum of deg over {depth = d},
 *   m_u(d) = sum of deg over {depth > d or unreached}
 * and the direction the integer rule picks (start TD):
 *   mode TD: go BU for step d iff m_f(d) * alpha > m_u(d)
 *   mode BU: go TD for step d iff n_f(d) * beta < n  and  n_f(d) < n_f(d-1)
 * Policy: 0 = auto (rule above), 1 = TD only, 2 = BU for every step d >= bu_from,
 *   3 = the paper's own rule (section 3.3; R23):
 *       TD -> BU for step d iff m_fc(d) * 10000 >= alpha * arcs, where m_fc(d) is the
 *       degree sum of the frontier vertices the coordinator partition owns (labels
 *       [0, coord_hi); "the coordinator for switching can be the partition
 *       responsible for the high degree vertices") and alpha is the "static
 *       percent" in units of 1/10000; BU -> TD after beta BU steps ("a fixed number
 *       of steps"), never BU again.
 * Inspections of step d: TD -> m_f(d) (every arc of every frontier vertex).
 *   BU -> sum over v with depth > d or unreached, deg(v) > 0, of
 *         (index of v's first neighbour with depth d) + 1, or deg(v) if none
 *   (Alg. 1 P:98-111 with `break for` P:107, the membership test read as
 *    "Nbr in Frontier", R1).
 * bu_parent[v] (if non-NULL) = that first neighbour for every v discovered by a
 * BU step (-1 elsewhere): the parent a bottom-up step must choose.
 * Per step outputs (arrays of max_steps): dir (0 TD, 1 BU), n_f, m_f, m_u,
 * discovered (= n_f(d+1)), insp.  Returns the number of steps, -1 if max_steps
 * is too small.  The last step is the one whose discovered count is 0. */
int64_t orc_do_emulate(int64_t n, const int64_t* offsets, const int32_t* adj, const int32_t* depth,
                       int64_t alpha, int64_t beta, int policy, int64_t bu_from, int64_t max_steps,
                       int32_t* dir, int64_t* n_f, int64_t* m_f, int64_t* m_u, int64_t* discovered,
                       int64_t* insp, int32_t* bu_parent, int64_t coord_hi) {
    int32_t maxd = -1;
    int64_t arcs = offsets[n];
    for (int64_t v = 0; v < n; ++v) if (depth[v] > maxd) maxd = depth[v];
    int64_t steps = (int64_t)maxd + 1; /* steps d = 0..maxd; step maxd discovers nothing */
    if (steps > max_steps) return -1;
    if (bu_parent) for (int64_t v = 0; v < n; ++v) bu_parent[v] = -1;
    int64_t* cnt = (int64_t*)calloc((size_t)steps + 1, sizeof(int64_t));
    int64_t* dsum = (int64_t*)calloc((size_t)steps + 1, sizeof(int64_t));
    int64_t* csum = (int64_t*)calloc((size_t)steps + 1, sizeof(int64_t)); /* coordinator's share */
    for (int64_t v = 0; v < n; ++v)
        if (depth[v] >= 0) {
            cnt[depth[v]] += 1;
            dsum[depth[v]] += offsets[v + 1] - offsets[v];
            if (v < coord_hi) csum[depth[v]] += offsets[v + 1] - offsets[v];
        }
    int mode = 0; /* 0 TD, 1 BU */
    int64_t bu_done = 0, returned = 0; /* policy 3: BU steps taken; back in TD for good */
    int64_t seen_deg = 0;
    for (int64_t d = 0; d < steps; ++d) {
        seen_deg += dsum[d];
        n_f[d] = cnt[d];
        m_f[d] = dsum[d];
        m_u[d] = arcs - seen_deg;
        discovered[d] = cnt[d + 1];
        if (policy == 1) mode = 0;
        else if (policy == 2) mode = (d >= bu_from) ? 1 : 0;
        else if (policy == 3) {
            if (mode == 0) { if (!returned && csum[d] * 10000 >= alpha * arcs) mode = 1; }
            else if (bu_done >= beta) { mode = 0; returned = 1; }
            if (mode == 1) bu_done += 1;
        } else {
            if (mode == 0) { if (m_f[d] * alpha > m_u[d]) mode = 1; }
            else { if (n_f[d] * beta < n && n_f[d] < n_f[d - 1]) mode = 0; }
        }
        dir[d] = mode;
        if (mode == 0) {
            insp[d] = m_f[d];
        } else {
            int64_t s = 0;
            for (int64_t v = 0; v < n; ++v) {
                if (!(depth[v] > d || depth[v] < 0)) continue;
                int64_t b = offsets[v], e = offsets[v + 1];
                if (e == b) continue;
                int64_t j;
                for (j = b; j < e; ++j)
                    if (depth[adj[j]] == d) break;
                if (j < e) {
                    s += (j - b) + 1;
                    if (bu_parent) bu_parent[v] = adj[j];
                } else {
                    s += e - b;
                }
            }
            insp[d] = s;
        }
    }
    free(cnt);
    free(dsum);
    free(csum);
    return steps;
}

/* ------------------------------------------------------------------------- */
/* TEPS numerator ("undirected traversed edges per second"; S:408-416;
 * DESIGN.md R5): the number of input tuples {u,v} whose endpoints are both
 * reached (duplicates and self-loops included, each tuple counted once). */
int64_t orc_component_tuples(int64_t m, const int32_t* uv, const int32_t* depth) {
    int64_t c = 0;
    for (int64_t k = 0; k < m; ++k)
        if (depth[uv[2 * k]] >= 0 && depth[uv[2 * k + 1]] >= 0) c += 1;
    return c;
}

/* ------------------------------------------------------------------------- */
/* Root sampling (R8): candidate k = Philox(ctr = (k lo, k hi, 0, 2),
 * key = seed)[0] >> (32 - scale); candidates k = 0, 1, 2, ... are taken in order,
 * rejecting a vertex whose number of non-self-loop arcs is 0 or that was already
 * taken.  Stops after `count` roots or `max_candidates` candidates.
 * Returns the number of roots written. */
int64_t orc_sample_roots(int scale, uint64_t seed, int64_t n, const int64_t* offsets, const int32_t* adj,
                         int64_t count, int64_t max_candidates, int64_t* roots) {
    uint32_t key[2];
    seed_key(seed, key);
    int64_t got = 0;
    for (int64_t k = 0; k < max_candidates && got < count; ++k) {
        uint32_t ctr[4] = {(uint32_t)((uint64_t)k & 0xffffffffu), (uint32_t)((uint64_t)k >> 32), 0, 2}, w[4];
        orc_philox4x32_10(ctr, key, w);
        int64_t r = (int64_t)(scale == 0 ? 0 : (w[0] >> (32 - scale)));
        if (r >= n) continue;
        int64_t nonloop = 0;
        for (int64_t j = offsets[r]; j < offsets[r + 1]; ++j)
            if (adj[j] != r) nonloop += 1;
        if (nonloop == 0) continue;
        int dup = 0;
        for (int64_t t = 0; t < got; ++t)
            if (roots[t] == r) { dup = 1; break; }
        if (dup) continue;
        roots[got++] = r;
    }
    return got;
}
