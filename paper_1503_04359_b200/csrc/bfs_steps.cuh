// The BFS step kernels (Alg. 1): init, top-down
// expansion and the owner-side merge, bottom-up batches, queue <-> bitmap conversions,
// the output passes, TEPS numerator and root-sampling helpers.
// Included once, inside namespace bfsb::{anonymous}, by bfs.cu (a single translation
// unit: the kernels, device helpers and the host launch code share one file scope).
#pragma once

// root_l < 0 on ranks that do not own the root
__global__ void k_init(uint32_t* visited, const uint32_t* skip, int64_t pw, int64_t root_l, int32_t root_g,
                       int2* out, int32_t root_o, Queue q, const int2* head, unsigned long long* cnt) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < pw; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = skip[w];
        if (root_l >= 0 && w == (root_l >> 5)) x |= 1u << (root_l & 31);
        visited[w] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) cnt[i] = 0;
        if (root_l >= 0) {
            out[root_l] = make_int2(0, root_o);
            const int32_t dg = head[root_l].y;
            queue_put(q, 0, root_g, dg);
            cnt[C_NEXT] = 1;
            cnt[C_MF] = (unsigned long long)dg;
        }
    }
}

// chunk c of the top-down arc range starts inside frontier entry starts[c]
__global__ void k_td_chunk_starts(const int64_t* prefix, int64_t F, int64_t nchunks, int64_t* starts,
                                  const Ctl* ctl) {
    if (ctl) {   // E = prefix[F]: the arcs this expansion covers (tile mode: light rows only)
        F = ctl->n_f;
        nchunks = (prefix[F] + kTdChunk - 1) / kTdChunk;
    }
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = c * kTdChunk;
        // largest i in [0, F) with prefix[i] <= e (prefix non-decreasing, prefix[0] = 0)
        int64_t a = 0, b = F - 1;
        while (a < b) {
            const int64_t mid = (a + b + 1) >> 1;
            if (prefix[mid] <= e) a = mid;
            else b = mid - 1;
        }
        starts[c] = a;
    }
}

struct Remote {          // p > 1 only
    uint32_t* seen;      // global bitmap: remote vertices this rank already claimed in this BFS
    int2* out;           // list mode: claims (v, parent) for peer q at out[q * cap ...]
    unsigned long long* out_cnt;  // [p]
    int64_t cap;
    int64_t nb;          // partition block size
    // bitmap mode (dense levels): claims are bits of the global outbox
    // bitmap (peer q's slice goes to q); (v, parent, level) go to the parent log of the
    // owner, sent once after the last level
    uint32_t* outbox;    // null: list mode
    int4* plog;          // owner q's log at plog[q * nb ...]
    unsigned long long* plog_cnt;   // [p], kept across the levels of a search
};

// Top-down step (Alg. 1 TD branch).  Each CTA iteration handles one chunk of
// kTdChunk consecutive arcs in three phases so that the dependent loads of the
// kTdItems arcs of a thread overlap:
//   A  locate (binary search in shared memory) and load all targets v
//   B  probe the visited words, then atomicOr-claim the unvisited ones
//   C  winners write depth/parent and stage v in shared memory; one atomicAdd per
//      CTA chunk on the global queue tail, then a coalesced copy of the stage.
template <bool kMulti>
__global__ void __launch_bounds__(kTdThreads, 4)
k_td_expand(const Queue q_in, const int64_t* __restrict__ prefix, const int64_t* __restrict__ starts,
            int64_t F, int64_t E, const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
            uint32_t* __restrict__ visited, int2* __restrict__ out, const int32_t* __restrict__ pmap,
            const Queue qnext_in, const int2* __restrict__ head, unsigned long long* __restrict__ cnt,
            int32_t next_level, int64_t lo, int64_t hi, Remote rm, const Ctl* ctl, LevelRec* lrec, int claim_only_in,
            TileLog lg) {
    __shared__ int64_t s_pre[kTdStage + 2];
    __shared__ int64_t s_beg[kTdStage + 1];
    __shared__ int32_t s_u[kTdStage + 1];
    __shared__ int32_t s_q[kTdChunk];
    __shared__ int32_t s_qd[kTdChunk];
    __shared__ int s_qn;
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0;
    Queue qc = q_in, qnext = qnext_in;
    if (ctl) {   // device-driven loop: sizes and queue selector from the loop state
        F = ctl->n_f;
        E = prefix[F];   // = m_f, or the light rows' arcs in tile mode
        next_level = ctl->d + 1;
        if (ctl->qsel) { qc = qnext_in; qnext = q_in; }
        stamp_begin(lrec, ctl);
    }
    const Queue q = qc;
    const bool claim_only = claim_only_in > 0 || (claim_only_in < 0 && ctl && ctl->claim);   // < 0: the loop state decides
    // tile mode: the winners' records go to the (tile, window) buckets (k_tile_rec stores them)
    const bool use_log = lg.lpool && (claim_only_in == 2 || (claim_only_in < 0 && ctl && ctl->tile));
    const int64_t nchunks = (E + kTdChunk - 1) / kTdChunk;
    if (threadIdx.x == 0) s_qn = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const int64_t e0 = c * kTdChunk;
        const int64_t e1 = min(E, e0 + kTdChunk);
        const int64_t i0 = starts[c];
        const int64_t i1 = (c + 1 < nchunks) ? starts[c + 1] : F - 1;
        const int64_t cntv = min(i1 - i0 + 1, F - i0);
        const bool fits = cntv <= kTdStage;
        if (fits) {
            for (int k = threadIdx.x; k <= cntv; k += kTdThreads) {
                s_pre[k] = prefix[i0 + k];
                if (k < cntv) {
                    const int32_t uu = q.v[i0 + k];
                    s_u[k] = uu;
                    s_beg[k] = off[uu - lo];
                }
            }
        }
        __syncthreads();
        int32_t v[kTdItems], u[kTdItems];
        // A: targets.  Thread t takes kTdItems CONSECUTIVE arcs: one binary search for
        // the first, then a linear advance; the arcs of a row are sorted, so a thread's
        // targets are close together and its visited probes mostly share a sector (L1).
        {
            const int64_t et = e0 + (int64_t)threadIdx.x * kTdItems;
            int64_t a = 0;
            if (et < e1) {
                if (fits) {
                    int lo_ = 0, hi_ = (int)cntv - 1;
                    while (lo_ < hi_) {
                        const int mid = (lo_ + hi_ + 1) >> 1;
                        if (s_pre[mid] <= et) lo_ = mid;
                        else hi_ = mid - 1;
                    }
                    a = lo_;
                } else {
                    int64_t lo_ = i0, hi_ = F - 1;
                    while (lo_ < hi_) {
                        const int64_t mid = (lo_ + hi_ + 1) >> 1;
                        if (prefix[mid] <= et) lo_ = mid;
                        else hi_ = mid - 1;
                    }
                    a = lo_;
                }
            }
            int64_t pre = 0, nxt = 0, beg = 0;
            int32_t uu = 0;
            if (et < e1) {
                if (fits) {
                    pre = s_pre[a]; nxt = s_pre[a + 1]; beg = s_beg[a]; uu = s_u[a];
                } else {
                    pre = prefix[a]; nxt = prefix[a + 1]; uu = q.v[a]; beg = off[uu - lo];
                }
            }
#pragma unroll
            for (int j = 0; j < kTdItems; ++j) {
                const int64_t e = et + j;
                v[j] = -1;
                u[j] = 0;
                if (e < e1) {
                    while (e >= nxt) {   // the next frontier vertex (degree >= 1: one step each)
                        ++a;
                        if (fits) {
                            pre = s_pre[a]; nxt = s_pre[a + 1]; beg = s_beg[a]; uu = s_u[a];
                        } else {
                            pre = prefix[a]; nxt = prefix[a + 1]; uu = q.v[a]; beg = off[uu - lo];
                        }
                    }
                    u[j] = uu;
                    v[j] = __ldg(adj + beg + (e - pre));
                }
            }
        }
        // B: probe, then claim.  Owned targets in `visited`, remote ones in `seen`.
        bool own[kTdItems];
        uint32_t* wp[kTdItems];
        uint32_t wv[kTdItems];
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            own[j] = !kMulti || (v[j] >= lo && v[j] < hi);
            wp[j] = nullptr;
            if (v[j] >= 0) wp[j] = own[j] ? visited + ((v[j] - lo) >> 5) : rm.seen + (v[j] >> 5);
            // L1-cached probe: visited/seen bits only ever go 0 -> 1 during a step, so a
            // stale word can only send a claim to the atomicOr, which decides correctly
            wv[j] = wp[j] ? ld_ca(wp[j]) : kFull;
        }
        bool win[kTdItems];
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            const uint32_t bit = 1u << (v[j] & 31);
            win[j] = false;
            if (wp[j] && !(wv[j] & bit)) win[j] = !(atomicOr(wp[j], bit) & bit);
        }
        // claim-only mode (large steps, see k_td_finish): winners record (depth, parent)
        // -- only the claiming thread knows the parent -- but their degrees and the next
        // queue are produced in vertex order by k_td_finish
        if (claim_only) {
            if (use_log) {
                int32_t pj[kTdItems];
#pragma unroll
                for (int j = 0; j < kTdItems; ++j) pj[j] = win[j] ? (pmap ? __ldg(pmap + u[j]) : u[j]) : 0;
                light_log_all<kTdItems>(lg, win, v, pj);
            } else {
#pragma unroll
                for (int j = 0; j < kTdItems; ++j)
                    if (win[j]) __stcs(out + (v[j] - lo), make_int2(next_level, pmap ? __ldg(pmap + u[j]) : u[j]));
            }
            __syncthreads();
            continue;
        }
        // C: outputs + staged queue append; remote claims go to the owner's list
        // winners' degrees (8-byte head records) and parent labels: all loads issued
        // before any is consumed, so their latencies overlap instead of adding up
        int32_t dgs[kTdItems], par[kTdItems];
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            // one-shot random accesses stream through L2 with evict-first so the
            // visited words the probes and claims hit stay resident
            dgs[j] = (win[j] && own[j]) ? __ldcs(head + (v[j] - lo)).y : 0;
            par[j] = (win[j] && pmap) ? __ldg(pmap + u[j]) : u[j];   // original label (remote claims too)
        }
#pragma unroll
        for (int j = 0; j < kTdItems; ++j) {
            const bool lw = win[j] && own[j];
            const unsigned m = __ballot_sync(kFull, lw);
            if (m) {
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&s_qn, __popc(m));
                base = __shfl_sync(kFull, base, leader);
                if (lw) {
                    const int64_t vl = v[j] - lo;
                    const int slot = base + __popc(m & lanemask_lt());
                    s_q[slot] = v[j];
                    s_qd[slot] = dgs[j];
                    __stcs(out + vl, make_int2(next_level, par[j]));
                    my_mf += (unsigned long long)dgs[j];
                }
            }
            if (kMulti) {
                const bool rw = win[j] && !own[j];
                if (__ballot_sync(kFull, rw)) {
                    const int owner = rw ? (int)(v[j] / rm.nb) : -1;
                    const unsigned peers = __match_any_sync(kFull, owner);
                    const int leader = __ffs(peers) - 1;
                    unsigned long long pos = 0;
                    unsigned long long* ctr = rm.outbox ? rm.plog_cnt : rm.out_cnt;
                    if (rw && lane == leader) pos = atomicAdd(ctr + owner, (unsigned long long)__popc(peers));
                    pos = __shfl_sync(kFull, pos, leader) + __popc(peers & lanemask_lt());
                    if (rw) {
                        if (rm.outbox) {
                            atomicOr(rm.outbox + (v[j] >> 5), 1u << (v[j] & 31));
                            rm.plog[(int64_t)owner * rm.nb + (int64_t)pos] = make_int4(v[j], par[j], next_level, 0);
                        } else {
                            rm.out[(int64_t)owner * rm.cap + (int64_t)pos] = make_int2(v[j], par[j]);
                        }
                    }
                }
            }
        }
        __syncthreads();
        const int qn = s_qn;
        if (threadIdx.x == 0 && qn) s_base = atomicAdd(cnt + C_NEXT, (unsigned long long)qn);
        __syncthreads();
        for (int k = threadIdx.x; k < qn; k += kTdThreads) queue_put(qnext, s_base + k, s_q[k], s_qd[k]);
        __syncthreads();
        if (threadIdx.x == 0) s_qn = 0;
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
    if (ctl && lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}

// Second half of a large top-down step run in claim-only mode (single partition): the
// winners are the bits the claims set (visited now, not in the snapshot taken before the
// step), read back in vertex order: their count (n_f) and their head records' degrees
// (m_f of the next frontier) are coalesced reads.  The snapshot buffer becomes the next
// frontier bitmap, the ONLY form of that frontier: the bottom-up step that usually follows
// needs no conversion, and a top-down one builds its queue from the bitmap (b2q).
__device__ __forceinline__ void td_finish_body(const uint32_t* __restrict__ visited, uint32_t* __restrict__ snap,
                                               int64_t words, const int2* __restrict__ head,
                                               unsigned long long* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0, my_n = 0;
    for (int64_t b0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; b0 < words;
         b0 += (((int64_t)gridDim.x * blockDim.x) >> 5) * 32) {
        const int64_t w = b0 + lane;
        uint32_t nb = 0;
        if (w < words) {
            nb = __ldcg(visited + w) & ~__ldcg(snap + w);
            snap[w] = nb;
        }
        my_n += (unsigned long long)__popc(nb);
        unsigned todo = __ballot_sync(kFull, nb != 0u);
        while (todo) {   // word by word: the 32 lanes read 32 consecutive head records,
                         // 4 words' loads in flight before any is summed
            constexpr int kW = 4;
            int32_t dg[kW];
#pragma unroll
            for (int q = 0; q < kW; ++q) {
                dg[q] = 0;
                if (todo) {
                    const int k = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const uint32_t nk = __shfl_sync(kFull, nb, k);
                    if ((nk >> lane) & 1u) dg[q] = __ldg(head + (b0 + k) * 32 + lane).y;
                }
            }
#pragma unroll
            for (int q = 0; q < kW; ++q) my_mf += (unsigned long long)dg[q];
        }
    }
    my_mf = warp_sum_u64(my_mf);
    my_n = warp_sum_u64(my_n);
    if (lane == 0) {
        if (my_mf) atomicAdd(cnt + C_MF, my_mf);
        if (my_n) atomicAdd(cnt + C_NEXT, my_n);
    }
}
__global__ void k_td_finish(const uint32_t* __restrict__ visited, uint32_t* __restrict__ snap, int64_t words,
                            const int2* __restrict__ head, unsigned long long* __restrict__ cnt) {
    td_finish_body(visited, snap, words, head, cnt);
}

// Owner side of the top-down push: claims (v, parent) received from peers are
// claimed exactly like local top-down targets (Alg. 2 "(local) ==> (remote)").
__global__ void k_td_merge(const int2* __restrict__ in, int64_t R, const int2* __restrict__ head,
                           uint32_t* __restrict__ visited, int2* __restrict__ out,
                           const Queue qnext, unsigned long long* __restrict__ cnt, int32_t next_level,
                           int64_t lo) {
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < R;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b0 + lane;
        bool win = false;
        int2 c = make_int2(0, 0);
        if (i < R) {
            c = in[i];
            const uint32_t bit = 1u << (c.x & 31);
            uint32_t* wp = visited + ((c.x - lo) >> 5);
            if (!(__ldcg(wp) & bit)) win = !(atomicOr(wp, bit) & bit);
        }
        const unsigned m = __ballot_sync(kFull, win);
        if (m) {
            const int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(cnt + C_NEXT, (unsigned long long)__popc(m));
            base = __shfl_sync(kFull, base, leader);
            if (win) {
                const int64_t vl = c.x - lo;
                const int32_t dg = __ldg(head + vl).y;
                queue_put(qnext, base + __popc(m & lanemask_lt()), c.x, dg);
                out[vl] = make_int2(next_level, c.y);
                my_mf += (unsigned long long)dg;
            }
        }
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
}

// Owner side of a bitmap-mode top-down push: the p - 1 received outbox slices are ORed,
// the bits not yet visited are this rank's new vertices (claimed like local targets);
// their parents are not known yet: (depth, -1) until the parent logs arrive after the
// last level (k_plog_resolve).  inbox holds p slices of nbw words (own slice unused).
__global__ void k_td_inbox(const uint32_t* __restrict__ inbox, int p, int me, int64_t nbw, int64_t words,
                           uint32_t* __restrict__ visited, const int2* __restrict__ head, int2* __restrict__ out,
                           const Queue qnext, unsigned long long* __restrict__ cnt, int32_t next_level, int64_t lo) {
    const int lane = threadIdx.x & 31;
    unsigned long long my_mf = 0;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < words;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = b0 + lane;
        uint32_t nb = 0;
        if (w < words) {
            uint32_t x = 0;
            for (int q = 0; q < p; ++q)
                if (q != me) x |= __ldg(inbox + q * nbw + w);
            const uint32_t vis = visited[w];
            nb = x & ~vis;
            if (nb) visited[w] = vis | nb;
        }
        const int c = __popc(nb);
        int inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += y;
        }
        const int tot = __shfl_sync(kFull, inc, 31);
        if (!tot) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(cnt + C_NEXT, (unsigned long long)tot);
        base = __shfl_sync(kFull, base, 31);
        unsigned long long pos = base + (unsigned long long)(inc - c);
        while (nb) {
            const int k = __ffs(nb) - 1;
            nb &= nb - 1;
            const int64_t vl = w * 32 + k;
            const int32_t dg = __ldg(head + vl).y;
            out[vl] = make_int2(next_level, -1);
            queue_put(qnext, pos++, (int32_t)(lo + vl), dg);
            my_mf += (unsigned long long)dg;
        }
    }
    my_mf = warp_sum_u64(my_mf);
    if (lane == 0 && my_mf) atomicAdd(cnt + C_MF, my_mf);
}

// After the last level ("final aggregation"): the parent logs of every claimer,
// grouped by owner; an entry (v, parent, level) is a valid parent of v iff v was
// discovered at that level (a claimer may also have claimed v after its owner had
// discovered it), and only vertices still without a parent take one.
__global__ void k_plog_resolve(const int4* __restrict__ in, int64_t R, int2* __restrict__ out, int64_t lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = in[i];
        int2* r = out + (e.x - lo);
        if (r->x == e.z) atomicCAS(reinterpret_cast<int*>(r) + 1, -1, e.y);
    }
}

__device__ __forceinline__ bool in_front(const uint32_t* __restrict__ front, int32_t u) {
    return (__ldg(front + (u >> 5)) >> (u & 31)) & 1u;
}
__device__ __forceinline__ bool in_front_p(const uint32_t* __restrict__ front, uint64_t pol, int32_t u) {
    return (ldh(front + (u >> 5), pol) >> (u & 31)) & 1u;
}

constexpr int kBuLongDefault = 64;   // B200 sweep: 8 -> 64 is +1%; the warp path stays for hub rows
// lane-serial probes before a row is handed to the whole warp (BFS_BU_LONG: tuning only)
static int bu_long_setting() {
    const char* e = getenv("BFS_BU_LONG");
    return e ? std::max(1, atoi(e)) : kBuLongDefault;
}

// unvisited vertices of a 1024-vertex batch from which it is probed densely
// (BFS_BU_DENSE: tuning only)
static int bu_dense_setting() {
    const char* e = getenv("BFS_BU_DENSE");
    return e ? atoi(e) : 384;
}

// Bottom-up step (Alg. 1 BU branch, `break for` P:107, R1).
// A warp takes a batch of 32 visited words (1024 owned vertices) at a time from a
// global work counter:
//   1. one coalesced 128-byte load of the 32 visited words; an all-visited batch
//      costs only that load and a coalesced store of 32 zero next-words;
//   2. the unvisited vertices of the batch are compacted into a per-warp list in
//      shared memory (popc + warp prefix sum);
//   3. every lane keeps kBuSlots rows in flight and advances all of them each
//      round (independent adj[j] loads, then independent frontier-bit probes),
//      refilling a slot from the list as soon as its row resolves -- this hides
//      the off -> adj -> frontier dependent-load chain behind kBuSlots-way MLP
//      (the paper's "virtual warp" of one lane per vertex);
//   4. a row still unresolved after kBuLong lane-serial probes moves to a per-warp
//      list and is finished by the whole warp, 32 arcs per ballot (the lowest
//      hitting lane is the first frontier neighbour in row order);
//   5. the 32 next words are assembled in shared memory and stored coalesced.
constexpr int kBuWarps = 8;
constexpr int kBuCtas = 4;     // resident CTAs per SM (launch bound and grid; 5 spills: -10%)
constexpr int kBuSlots = 3;
constexpr int kBuIlp = 8;
constexpr int kBuVec = 4;      // arcs a slot reads (aligned vector loads: 2, 4 or 8) and probes per round
constexpr int kNbIlp = 4;     // listed rows per lane in flight in the second-probe phase
constexpr int kLongCap = 16;   // small: shared memory left to L1 matters more (B200-measured)

__global__ void __launch_bounds__(kBuWarps * 32, kBuCtas)
k_bu_batch(const int64_t* __restrict__ off, const int2* __restrict__ head, const int32_t* __restrict__ adj,
           uint32_t* __restrict__ visited,
           const uint32_t* __restrict__ front_in, uint32_t* __restrict__ next_in, int2* __restrict__ out,
           const int32_t* __restrict__ pmap, const int32_t* __restrict__ hpar, const int4* __restrict__ nb4,
           int64_t nb4_rows, int nbp, int64_t words, int64_t lo, int32_t next_level,
           unsigned long long* __restrict__ cnt, int grab, int blong, int dense_u, const Ctl* ctl,
           LevelRec* lrec) {
    __shared__ uint16_t s_list[kBuWarps][1024];
    __shared__ uint32_t s_nb[kBuWarps][32];
    __shared__ int64_t s_lj[kBuWarps][kLongCap];
    __shared__ int64_t s_le[kBuWarps][kLongCap];
    __shared__ int32_t s_lv[kBuWarps][kLongCap];
    __shared__ int32_t s_ld[kBuWarps][kLongCap];
    __shared__ int s_lcount[kBuWarps];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t* front = front_in;
    uint32_t* next = next_in;
    if (ctl) {   // device-driven loop: the bitmap pair flips every bottom-up step
        next_level = ctl->d + 1;
        if (ctl->fsel) {
            front = next_in;
            next = const_cast<uint32_t*>(front_in);
        }
        stamp_begin(lrec, ctl);
    }
    uint16_t* list = s_list[wid];
    uint32_t* nbw = s_nb[wid];
    const int64_t wbase = lo >> 5;
    // frontier probes with an L2 evict_last policy, so the bitmap outlives the once-read
    // head records, planes and rows streaming through L2 (K29 same-box A/B: loop 3.40 ->
    // 3.29 ms per search; profiles/r02_l2hint_ab.txt)
    const uint64_t pk = l2_evict_last();
    const int64_t nbatches = (words + 31) / 32;
    unsigned long long my_nf = 0, my_mf = 0, my_insp = 0, my_scan = 0;
    // batches are claimed `grab` at a time from the global counter (one atomic per
    // grab: a sparse level is otherwise bound by that single address)
    long long bt = 0, bt_end = 0;
    for (;; ++bt) {
        if (bt >= bt_end) {
            long long g0 = 0;
            if (lane == 0) g0 = (long long)atomicAdd(cnt + C_WORK, (unsigned long long)grab);
            g0 = __shfl_sync(kFull, g0, 0);
            if (g0 >= nbatches) break;
            bt = g0;
            bt_end = min(g0 + (long long)grab, (long long)nbatches);
        }
        const int64_t w = bt * 32 + lane;
        const uint32_t vis = w < words ? visited[w] : kFull;
        const uint32_t un = ~vis;
        if (!__ballot_sync(kFull, un != 0u)) {
            if (w < words) next[wbase + w] = 0u;
            continue;
        }
        const int c = __popc(un);
        const int U = __reduce_add_sync(kFull, c);
        nbw[lane] = 0u;
        if (lane == 0) s_lcount[wid] = 0;
        my_scan += (unsigned long long)c;
        const int64_t vbase = bt * 1024;
        int M = 0;  // warp-uniform count of rows that missed their first probe
        if (U >= dense_u) {
            // 3a'. dense batch (most vertices unvisited, the first bottom-up levels):
            //     lane j takes vertex j of every word, so head records load coalesced
            //     and the next word of the batch is one ballot -- no list to build and
            //     no shared-memory atomics.  Misses go to the list for 3b.
            uint32_t mynext = 0u;
            for (int k0 = 0; k0 < 32; k0 += kBuIlp) {
                int32_t sv[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) {
                    const uint32_t vk = __shfl_sync(kFull, vis, k0 + j);
                    sv[j] = ((vk >> lane) & 1u) ? -1 : (k0 + j) * 32 + lane;
                }
                int2 hd[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) hd[j] = sv[j] >= 0 ? __ldg(head + vbase + sv[j]) : make_int2(-1, 0);
                int32_t po[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) po[j] = (hpar && sv[j] >= 0) ? __ldg(hpar + vbase + sv[j]) : hd[j].x;
                bool hit[kBuIlp];
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) hit[j] = hd[j].y > 0 && in_front_p(front, pk, hd[j].x);
#pragma unroll
                for (int j = 0; j < kBuIlp; ++j) {
                    if (hd[j].y > 0) my_insp += 1;
                    if (hit[j]) {
                        __stcs(out + vbase + sv[j], make_int2(next_level, po[j]));
                        my_mf += (unsigned long long)hd[j].y;
                    }
                    const unsigned hm = __ballot_sync(kFull, hit[j]);
                    if (lane == k0 + j) mynext = hm;
                    const bool miss = !hit[j] && hd[j].y > 1;
                    const unsigned mm = __ballot_sync(kFull, miss);
                    if (miss) list[M + __popc(mm & lanemask_lt())] = (uint16_t)sv[j];
                    M += __popc(mm);
                }
            }
            nbw[lane] = mynext;
        } else {
            // 2. compact unvisited local indices (0..1023) into the per-warp list
            int inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(kFull, inc, d);
                if (lane >= d) inc += y;
            }
            {
                uint32_t bits = un;
                int p = inc - c;
                while (bits) {
                    const int k = __ffs(bits) - 1;
                    bits &= bits - 1;
                    list[p++] = (uint16_t)(lane * 32 + k);
                }
            }
            __syncwarp();
            // 3a. first probes: every unvisited vertex tries the first neighbour of its
            //     row from the dense head record (8 bytes, coalesced along the list);
            //     kBuIlp records per lane are loaded before any is probed.  With rows in
            //     canonical order this resolves most vertices.  Vertices that miss
            //     and have more neighbours are compacted in place at the front of the list.
            for (int t0 = 0; t0 < U; t0 += 32 * kBuIlp) {
                int32_t sv[kBuIlp];
                int2 hd[kBuIlp];
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) {
                    const int idx = t0 + k * 32 + lane;
                    sv[k] = idx < U ? (int32_t)list[idx] : -1;
                }
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) hd[k] = sv[k] >= 0 ? __ldg(head + vbase + sv[k]) : make_int2(-1, 0);
                // reindexed graphs: the first neighbour's ORIGINAL label comes from a dense
                // per-vertex array read beside the head record (coalesced), not from a
                // random ilabel[] lookup after the probe
                int32_t po[kBuIlp];
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) po[k] = (hpar && sv[k] >= 0) ? __ldg(hpar + vbase + sv[k]) : hd[k].x;
                bool hit[kBuIlp];
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) hit[k] = hd[k].y > 0 && in_front_p(front, pk, hd[k].x);
                __syncwarp();  // all lanes hold their entries of this block before misses overwrite it
#pragma unroll
                for (int k = 0; k < kBuIlp; ++k) {
                    if (hd[k].y > 0) my_insp += 1;
                    if (hit[k]) {
                        __stcs(out + vbase + sv[k], make_int2(next_level, po[k]));
                        atomicOr(nbw + (sv[k] >> 5), 1u << (sv[k] & 31));
                        my_mf += (unsigned long long)hd[k].y;
                    }
                    const bool miss = !hit[k] && hd[k].y > 1;
                    const unsigned mm = __ballot_sync(kFull, miss);
                    if (miss) list[M + __popc(mm & lanemask_lt())] = (uint16_t)sv[k];
                    M += __popc(mm);
                }
            }
        }
        __syncwarp();
        int skip0 = 1;   // arcs already probed per listed row
        for (int pl = 0; nb4 && pl < nbp && M > 0; ++pl) {
            // 3a''. second probes: arcs 1+4pl .. 4+4pl of every row still listed, from the
            //      dense 16-byte block of plane pl (nb4[pl * nb4_rows + v]) read along the
            //      list (consecutive misses share sectors) instead of an offsets load plus
            //      a row-aligned adjacency sector per row -- at a hub-frontier level most
            //      rows miss and most are short.  Rows with arcs past the plane and no hit
            //      stay listed for the next plane or for 3b.
            const int4* pb = nb4 + (int64_t)pl * nb4_rows;
            const int first = 1 + 4 * pl;
            int M2 = 0;
            for (int t0 = 0; t0 < M; t0 += 32 * kNbIlp) {
                // the block's -1 padding marks the row's end, so only the block is loaded
                // (the degree is read for the hits alone, for m_f)
                int32_t sv[kNbIlp];
                int4 x[kNbIlp];
#pragma unroll
                for (int k = 0; k < kNbIlp; ++k) {
                    const int idx = t0 + k * 32 + lane;
                    sv[k] = idx < M ? (int32_t)list[idx] : -1;
                }
#pragma unroll
                for (int k = 0; k < kNbIlp; ++k)
                    x[k] = sv[k] >= 0 ? __ldg(pb + vbase + sv[k]) : make_int4(-1, -1, -1, -1);
                __syncwarp();  // the block is in registers before survivors overwrite it
#pragma unroll
                for (int k = 0; k < kNbIlp; ++k) {
                    const bool h0 = x[k].x >= 0 && in_front_p(front, pk, x[k].x);
                    const bool h1 = x[k].y >= 0 && in_front_p(front, pk, x[k].y);
                    const bool h2 = x[k].z >= 0 && in_front_p(front, pk, x[k].z);
                    const bool h3 = x[k].w >= 0 && in_front_p(front, pk, x[k].w);
                    const int kh = h0 ? 0 : h1 ? 1 : h2 ? 2 : h3 ? 3 : -1;
                    if (sv[k] >= 0) {
                        if (kh >= 0) {
                            const int32_t hu = kh == 0 ? x[k].x : kh == 1 ? x[k].y : kh == 2 ? x[k].z : x[k].w;
                            my_insp += (unsigned long long)(kh + 1);
                            __stcs(out + vbase + sv[k], make_int2(next_level, pmap ? pmap[hu] : hu));
                            atomicOr(nbw + (sv[k] >> 5), 1u << (sv[k] & 31));
                            my_mf += (unsigned long long)__ldg(head + vbase + sv[k]).y;
                        } else {
                            my_insp += (unsigned long long)((x[k].x >= 0) + (x[k].y >= 0) + (x[k].z >= 0) +
                                                            (x[k].w >= 0));
                        }
                    }
                    // a full block without a hit: the row may go on (a row of exactly
                    // first + 4 arcs ends with an empty block or at once in 3b)
                    const bool miss = sv[k] >= 0 && kh < 0 && x[k].w >= 0;
                    const unsigned mm = __ballot_sync(kFull, miss);
                    if (miss) list[M2 + __popc(mm & lanemask_lt())] = (uint16_t)sv[k];
                    M2 += __popc(mm);
                }
            }
            M = M2;
            skip0 = first + 4;
            __syncwarp();
        }
        // 3b. rows that missed: each lane keeps kBuSlots rows in flight from position 1
        //     (1 + 4 nbp after 3a'')
        //     on and advances all of them each round (independent adj[j] loads, then
        //     independent frontier probes), refilling a slot as soon as its row
        //     resolves (the paper's "virtual warp" of one lane per vertex).
        {
            int t = lane;
            int32_t sv[kBuSlots], sd[kBuSlots];
            int64_t sj[kBuSlots], se[kBuSlots];
            bool sa[kBuSlots];
#pragma unroll
            for (int s = 0; s < kBuSlots; ++s) {
                sa[s] = false;
                sv[s] = sd[s] = 0;
                sj[s] = se[s] = 0;
                if (t < M) {
                    sv[s] = list[t];
                    t += 32;
                    sd[s] = __ldcs(head + vbase + sv[s]).y;
                    const int64_t o = __ldcs(off + vbase + sv[s]);
                    sj[s] = o + skip0;
                    se[s] = o + sd[s];
                    sa[s] = true;
                }
            }
            for (;;) {
                bool any = false;
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) any |= sa[s];
                if (!__any_sync(kFull, any)) break;
                // each slot reads the aligned kBuVec-arc group holding its next arc with
                // one vector load and probes every arc of it that lies in the row at once
                int32_t a[kBuSlots][kBuVec];
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) {
                    const int64_t b = sj[s] & ~(int64_t)(kBuVec - 1);
                    if (kBuVec == 8) {   // one whole 32-byte sector
                        const int4 x = sa[s] ? __ldg(reinterpret_cast<const int4*>(adj + b)) : make_int4(0, 0, 0, 0);
                        const int4 y = sa[s] ? __ldg(reinterpret_cast<const int4*>(adj + b) + 1) : make_int4(0, 0, 0, 0);
                        a[s][0] = x.x; a[s][1] = x.y; a[s][2 % kBuVec] = x.z; a[s][3 % kBuVec] = x.w;
                        a[s][4 % kBuVec] = y.x; a[s][5 % kBuVec] = y.y; a[s][6 % kBuVec] = y.z; a[s][7 % kBuVec] = y.w;
                    } else if (kBuVec == 4) {
                        const int4 x = sa[s] ? __ldg(reinterpret_cast<const int4*>(adj + b)) : make_int4(0, 0, 0, 0);
                        a[s][0] = x.x; a[s][1] = x.y; a[s][2 % kBuVec] = x.z; a[s][3 % kBuVec] = x.w;
                    } else if (kBuVec == 2) {
                        const int2 x = sa[s] ? __ldg(reinterpret_cast<const int2*>(adj + b)) : make_int2(0, 0);
                        a[s][0] = x.x; a[s][1 % kBuVec] = x.y;
                    } else {
                        a[s][0] = sa[s] ? __ldg(adj + b) : 0;
                    }
                }
                bool h[kBuSlots][kBuVec];
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) {
                    const int64_t b = sj[s] & ~(int64_t)(kBuVec - 1);
#pragma unroll
                    for (int k = 0; k < kBuVec; ++k)
                        h[s][k] = sa[s] && b + k >= sj[s] && b + k < se[s] && in_front_p(front, pk, a[s][k]);
                }
#pragma unroll
                for (int s = 0; s < kBuSlots; ++s) {
                    if (sa[s]) {
                        const int64_t b = sj[s] & ~(int64_t)(kBuVec - 1);
                        int kh = -1;
                        int32_t hu = 0;
#pragma unroll
                        for (int k = kBuVec - 1; k >= 0; --k)
                            if (h[s][k]) { kh = k; hu = a[s][k]; }
                        const int64_t nj = min(se[s], b + kBuVec);
                        if (kh >= 0) {
                            my_insp += (unsigned long long)(b + kh - sj[s] + 1);
                            __stcs(out + vbase + sv[s], make_int2(next_level, pmap ? pmap[hu] : hu));
                            atomicOr(nbw + (sv[s] >> 5), 1u << (sv[s] & 31));
                            my_mf += (unsigned long long)sd[s];
                            sa[s] = false;
                        } else if (my_insp += (unsigned long long)(nj - sj[s]), (sj[s] = nj) == se[s]) {
                            sa[s] = false;  // exhausted: no frontier neighbour this level
                        } else if (sd[s] - (se[s] - sj[s]) >= blong) {
                            const int idx = atomicAdd(s_lcount + wid, 1);
                            if (idx < kLongCap) {  // hand the rest of the row to the warp
                                s_lv[wid][idx] = sv[s];
                                s_lj[wid][idx] = sj[s];
                                s_le[wid][idx] = se[s];
                                s_ld[wid][idx] = sd[s];
                                sa[s] = false;
                            }
                        }
                    }
                    if (!sa[s] && t < M) {
                        sv[s] = list[t];
                        t += 32;
                        sd[s] = __ldcs(head + vbase + sv[s]).y;
                        const int64_t o = __ldcs(off + vbase + sv[s]);
                        sj[s] = o + skip0;
                        se[s] = o + sd[s];
                        sa[s] = true;
                    }
                }
            }
        }
        __syncwarp();
        // 4. long rows: whole warp, 32 arcs per ballot
        const int L = min(s_lcount[wid], kLongCap);
        for (int x = 0; x < L; ++x) {
            const int32_t lv = s_lv[wid][x];
            const int64_t jb = s_lj[wid][x], je = s_le[wid][x];
            int64_t hit = -1;
            int32_t hu = 0;
            for (int64_t j0 = jb; j0 < je; j0 += 32) {
                const int64_t jj = j0 + lane;
                int32_t uu = 0;
                bool hh = false;
                if (jj < je) {
                    uu = __ldg(adj + jj);
                    hh = in_front_p(front, pk, uu);
                }
                const unsigned hm = __ballot_sync(kFull, hh);
                if (hm) {
                    const int first = __ffs(hm) - 1;
                    hit = j0 + first;
                    hu = __shfl_sync(kFull, uu, first);
                    break;
                }
            }
            if (lane == 0) {
                if (hit >= 0) {
                    out[vbase + lv] = make_int2(next_level, pmap ? pmap[hu] : hu);
                    nbw[lv >> 5] |= 1u << (lv & 31);
                    my_mf += (unsigned long long)s_ld[wid][x];
                    my_insp += (unsigned long long)(hit - jb + 1);
                } else {
                    my_insp += (unsigned long long)(je - jb);
                }
            }
        }
        __syncwarp();
        // 5. coalesced next / visited words
        if (w < words) {
            const uint32_t nb = nbw[lane];
            next[wbase + w] = nb;
            if (nb) visited[w] = vis | nb;
            my_nf += (unsigned long long)__popc(nb);
        }
        __syncwarp();
    }
    my_nf = warp_sum_u64(my_nf);
    my_mf = warp_sum_u64(my_mf);
    my_insp = warp_sum_u64(my_insp);
    my_scan = warp_sum_u64(my_scan);
    if (lane == 0) {
        if (my_nf) atomicAdd(cnt + C_NEXT, my_nf);
        if (my_mf) atomicAdd(cnt + C_MF, my_mf);
        if (my_insp) atomicAdd(cnt + C_INSP, my_insp);
        if (my_scan) atomicAdd(cnt + C_SCAN, my_scan);
    }
    if (ctl && lrec) {
        __syncthreads();
        stamp_end(lrec, ctl);
    }
}

// queue -> bitmap (the owned slice of front is cleared beforehand)
__device__ __forceinline__ void q2b_body(const int32_t* __restrict__ q, int64_t F, uint32_t* __restrict__ front) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = q[i];
        atomicOr(front + (v >> 5), 1u << (v & 31));
    }
}
__global__ void k_q2b(const int32_t* __restrict__ q, int64_t F, uint32_t* __restrict__ front) { q2b_body(q, F, front); }

// owned slice of a bitmap -> queue of global IDs (with degree)
__device__ __forceinline__ void b2q_body(const uint32_t* __restrict__ bm, int64_t words, int64_t lo,
                                         const int2* __restrict__ head, const Queue q,
                                         unsigned long long* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t wbase = lo >> 5;
    for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; b0 < words;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = b0 + lane;
        uint32_t bits = w < words ? bm[wbase + w] : 0u;
        const int c = __popc(bits);
        int inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, d);
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
            const int64_t vl = w * 32 + k;
            queue_put(q, pos++, (int32_t)(lo + vl), __ldg(head + vl).y);
        }
    }
}

__global__ void k_b2q(const uint32_t* __restrict__ bm, int64_t words, int64_t lo, const int2* __restrict__ head,
                      const Queue q, unsigned long long* __restrict__ cnt) {
    b2q_body(bm, words, lo, head, q, cnt);
}

// Output pass (the only writer of the caller's arrays): every entry of depth and
// parent is written exactly once, in order, with full coalesced lines.  During
// the traversal the steps record (depth, parent) of each discovered vertex as one
// 8-byte `out` record in internal order; here reached vertices copy their record
// and unreached ones get -1.
//   one GPU / p ranks, labels unchanged: v = internal = original (owned slice)
//   degree reindex: v runs over ORIGINAL labels, iv = label[v] gathers the record;
//   isolated vertices sit at the tail of the internal order, so they skip the gather.
// n_active: internal labels >= n_active are isolated (degree reindex puts them last)
// and need neither the visited lookup nor the record gather.  Everything except the
// visited bitmap is touched once, so it streams with evict-first hints and the
// bitmap stays in L2 for the random lookups.
__device__ __forceinline__ void emit_body(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                                          const int2* __restrict__ rec, int64_t nl, int64_t root_l,
                                          int32_t* __restrict__ depth, int32_t* __restrict__ parent) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = v >> 5;
        const uint32_t r = visited[w] & ~skip[w];
        int2 o = make_int2(-1, -1);
        if (((r >> (v & 31)) & 1u) || v == root_l) o = rec[v];
        if (depth) depth[v] = o.x;
        if (parent) parent[v] = o.y;
    }
}
__global__ void k_emit(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                       const int2* __restrict__ rec, int64_t nl, int64_t root_l, int32_t* __restrict__ depth,
                       int32_t* __restrict__ parent, const Ctl* ctl) {
    emit_body(visited, skip, rec, nl, ctl ? ctl->root_i : root_l, depth, parent);
}

// Degree-reindexed variant: v runs over ORIGINAL labels and gathers the record of
// iv = label[v].  Internal labels >= n_active are isolated (the reindex puts them
// last) and need no gather unless one is the root.  Labels and outputs are touched
// once and stream with evict-first hints.
__device__ __forceinline__ void emit_perm_body(const int2* __restrict__ rec, const int32_t* __restrict__ label,
                                               int64_t n, int64_t n_active, int64_t root_l,
                                               int32_t* __restrict__ depth, int32_t* __restrict__ parent) {
    // kEmitV original vertices per thread: 16-byte label loads, then one record
    // gather per non-isolated vertex (k_mark_unreached has reset the records of the
    // unreached ones).  Same-degree vertices keep their original order in the
    // reindex (degree desc, ID asc), so the gathers form one ascending stream per
    // degree value.
    constexpr int kEmitV = 8;
    // a warp owns a tile of 32 * kEmitV consecutive vertices; part h of the tile is
    // 128 vertices, lane i holding vertices 4i..4i+3 of it, so every 16-byte label
    // load and output store of a warp instruction covers 512 contiguous bytes
    const bool vec = ((reinterpret_cast<uintptr_t>(depth) | reinterpret_cast<uintptr_t>(parent)) & 15) == 0 &&
                     depth && parent;
    const int lane = threadIdx.x & 31;
    const int64_t tiles = (n + 32 * kEmitV - 1) / (32 * kEmitV);
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // 32-byte aligned outputs: lane i takes the 8 consecutive vertices 8i..8i+7 of the
    // tile, one 256-bit label load and two 256-bit stores (half the memory instructions
    // of the 16-byte path below)
    const bool vec8 = ((reinterpret_cast<uintptr_t>(depth) | reinterpret_cast<uintptr_t>(parent) |
                        reinterpret_cast<uintptr_t>(label)) & 31) == 0 && depth && parent && kEmitV == 8;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < tiles; t += nwarps) {
        const int64_t t0 = t * 32 * kEmitV;
        const bool full = t0 + 32 * kEmitV <= n;
        if (vec8 && full) {
            const int64_t v0 = t0 + lane * 8;
            int32_t iv[8];
            asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(iv[0]), "=r"(iv[1]), "=r"(iv[2]), "=r"(iv[3]), "=r"(iv[4]), "=r"(iv[5]), "=r"(iv[6]),
                           "=r"(iv[7])
                         : "l"(label + v0));
            int2 o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const bool act = iv[k] >= 0 && (iv[k] < n_active || iv[k] == root_l);
                o[k] = act ? __ldg(rec + iv[k]) : make_int2(-1, -1);
            }
            asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(depth + v0), "r"(o[0].x),
                         "r"(o[1].x), "r"(o[2].x), "r"(o[3].x), "r"(o[4].x), "r"(o[5].x), "r"(o[6].x), "r"(o[7].x)
                         : "memory");
            asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(parent + v0), "r"(o[0].y),
                         "r"(o[1].y), "r"(o[2].y), "r"(o[3].y), "r"(o[4].y), "r"(o[5].y), "r"(o[6].y), "r"(o[7].y)
                         : "memory");
            continue;
        }
        int32_t iv[kEmitV];
#pragma unroll
        for (int h = 0; h < kEmitV / 4; ++h) {
            const int64_t v0 = t0 + h * 128 + lane * 4;
            if (full) {
                const int4 l4 = __ldcs(reinterpret_cast<const int4*>(label + v0));
                iv[4 * h] = l4.x; iv[4 * h + 1] = l4.y; iv[4 * h + 2] = l4.z; iv[4 * h + 3] = l4.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) iv[4 * h + j] = v0 + j < n ? label[v0 + j] : -1;
            }
        }
        // records of unreached active vertices were reset by k_mark_unreached, so the
        // record alone decides: no visited lookup
        int2 o[kEmitV];
#pragma unroll
        for (int k = 0; k < kEmitV; ++k) {
            const bool act = iv[k] >= 0 && (iv[k] < n_active || iv[k] == root_l);
            o[k] = act ? __ldg(rec + iv[k]) : make_int2(-1, -1);
        }
#pragma unroll
        for (int h = 0; h < kEmitV / 4; ++h) {
            const int64_t v0 = t0 + h * 128 + lane * 4;
            if (vec && full) {
                __stcs(reinterpret_cast<int4*>(depth + v0),
                       make_int4(o[4 * h].x, o[4 * h + 1].x, o[4 * h + 2].x, o[4 * h + 3].x));
                __stcs(reinterpret_cast<int4*>(parent + v0),
                       make_int4(o[4 * h].y, o[4 * h + 1].y, o[4 * h + 2].y, o[4 * h + 3].y));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (v0 + j >= n) break;
                    if (depth) depth[v0 + j] = o[4 * h + j].x;
                    if (parent) parent[v0 + j] = o[4 * h + j].y;
                }
            }
        }
    }
}

__global__ void k_emit_perm(const int2* __restrict__ rec, const int32_t* __restrict__ label, int64_t n,
                            int64_t n_active, int64_t root_l, int32_t* __restrict__ depth,
                            int32_t* __restrict__ parent, const Ctl* ctl) {
    emit_perm_body(rec, label, n, n_active, ctl ? ctl->root_i : root_l, depth, parent);
}

// The bottom-up probes left the frontier bitmaps at L2 evict_last priority: back to
// normal before the output pass streams its 9 GB (one thread per 128-byte line)
__global__ void k_l2_demote(const uint32_t* a, const uint32_t* b, int64_t words) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; (l + 1) * 32 <= words;   // whole lines
         l += (int64_t)gridDim.x * blockDim.x) {
        l2_demote_line(a + l * 32);
        l2_demote_line(b + l * 32);
    }
}

// rec <- (-1, -1) for every vertex of [0, nbits) with degree > 0 that this search did
// not reach (a few per search in a Kronecker graph: one coalesced pass over the
// bitmaps, scattered writes for the unreached only), so that the reindexed output
// pass can take every active vertex's record as is
__device__ __forceinline__ void mark_unreached_body(const uint32_t* __restrict__ visited,
                                                    const uint32_t* __restrict__ skip, int64_t nbits,
                                                    int2* __restrict__ rec) {
    const int64_t words = (nbits + 31) / 32;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = ~__ldcs(visited + w) & ~__ldcs(skip + w);
        if (w == words - 1 && (nbits & 31)) x &= (1u << (nbits & 31)) - 1u;
        while (x) {
            const int k = __ffs(x) - 1;
            x &= x - 1;
            rec[w * 32 + k] = make_int2(-1, -1);
        }
    }
}
__global__ void k_mark_unreached(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                                 int64_t nbits, int2* __restrict__ rec) {
    mark_unreached_body(visited, skip, nbits, rec);
}

// Output pass of a degree-reindexed search on p ranks: the reindex is partition-local
// (P:158), so the internal label of every owned original label is owned too and the
// outputs need no exchange.  v runs over the owned ORIGINAL labels, iv = label[v] - lo
// over the owned internal ones; unreached vertices get -1.
__global__ void k_emit_local(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ skip,
                             const int2* __restrict__ rec, const int32_t* __restrict__ label, int64_t lo, int64_t nl,
                             int64_t root_l, int32_t* __restrict__ depth, int32_t* __restrict__ parent) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nl; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t iv = (int64_t)__ldcs(label + lo + v) - lo;
        const uint32_t r = __ldg(visited + (iv >> 5)) & ~__ldg(skip + (iv >> 5));
        int2 o = make_int2(-1, -1);
        if (((r >> (iv & 31)) & 1u) || iv == root_l) o = rec[iv];
        if (depth) __stcs(depth + v, o.x);
        if (parent) __stcs(parent + v, o.y);
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

// non-self-loop arc count of owned candidate roots (internal labels), one warp per
// candidate; candidates outside [lo, hi) or negative contribute 0
__global__ void k_nonloop_degree(const int32_t* __restrict__ cand, int64_t k, const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ adj, int64_t lo, int64_t hi, int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = gw; t < k; t += nw) {
        const int32_t r = cand[t];
        int64_t c = 0;
        if (r >= lo && r < hi) {
            const int64_t b = off[r - lo], e = off[r - lo + 1];
            for (int64_t j = b + lane; j < e; j += 32) c += adj[j] != r;
        }
        for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
        if (lane == 0) out[t] = c;
    }
}

__global__ void k_gather_labels(const int32_t* __restrict__ label, const int32_t* __restrict__ in, int64_t k,
                                int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] < 0 ? -1 : label[in[i]];
}

