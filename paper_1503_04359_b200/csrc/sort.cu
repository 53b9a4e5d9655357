// Stable LSD radix sort of (uint32 key, int32 value) pairs on the device, used by
// the section 3.4 degree reindex: vertices ordered by
// (degree descending, ID ascending) = keys (maxdeg - deg) ascending over values
// (IDs) that start in ascending order, so stability gives the ID tie-break.
//
// One pass per 8-bit digit:
//   k_rs_hist     per-tile digit histogram, stored digit-major: hist[d * tiles + t]
//   scan          exclusive scan of hist -> base offset of (digit, tile)
//   k_rs_scatter  stable scatter: the tile is walked in 16 rounds of 256 consecutive
//                 elements; within a round a warp ranks equal digits with
//                 __match_any_sync, warps are ordered by a per-digit prefix over
//                 the 8 warps, and rounds accumulate a running per-digit base.
#include "internal.cuh"

namespace bfsb {
namespace {

constexpr int kRsThreads = 256;
constexpr int kRsRounds = 16;
constexpr int kRsTile = kRsThreads * kRsRounds;
constexpr int kRsWarps = kRsThreads / 32;

__global__ void __launch_bounds__(kRsThreads)
k_rs_hist(const uint32_t* __restrict__ keys, int64_t n, int shift, int32_t* __restrict__ hist, int64_t tiles) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsTile;
    for (int r = 0; r < kRsRounds; ++r) {
        const int64_t i = base + (int64_t)r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRsThreads)
k_rs_scatter(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin, int64_t n, int shift,
             const int64_t* __restrict__ base_off, int64_t tiles, uint32_t* __restrict__ kout,
             int32_t* __restrict__ vout) {
    __shared__ int s_wc[kRsWarps][256];   // per-warp digit counts of the current round
    __shared__ int s_run[256];            // running per-digit count over earlier rounds
    __shared__ int64_t s_base[256];       // global base of (digit, this tile)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    s_run[threadIdx.x] = 0;
    s_base[threadIdx.x] = base_off[(int64_t)threadIdx.x * tiles + blockIdx.x];
    const int64_t tile0 = (int64_t)blockIdx.x * kRsTile;
    for (int r = 0; r < kRsRounds; ++r) {
        for (int w = 0; w < kRsWarps; ++w) s_wc[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = tile0 + (int64_t)r * kRsThreads + threadIdx.x;
        const bool valid = i < n;
        uint32_t k = 0;
        int32_t v = 0;
        int dg = 256 + lane;  // distinct dummy digits for invalid lanes
        if (valid) {
            k = kin[i];
            v = vin[i];
            dg = (int)((k >> shift) & 255u);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) s_wc[wid][dg] = __popc(peers);
        __syncthreads();
        // per digit: exclusive prefix over warps (in warp order), then advance the run
        {
            const int d = threadIdx.x;
            int run = s_run[d];
            for (int w = 0; w < kRsWarps; ++w) {
                const int c = s_wc[w][d];
                s_wc[w][d] = run;
                run += c;
            }
            s_run[d] = run;
        }
        __syncthreads();
        if (valid) {
            const int64_t pos = s_base[dg] + s_wc[wid][dg] + rank;
            kout[pos] = k;
            vout[pos] = v;
        }
        __syncthreads();
    }
}

int grid_tiles(int64_t n) { return (int)((n + kRsTile - 1) / kRsTile); }

}  // namespace

// Sorts keys/vals in place (ascending keys, stable); key_bits = significant bits of the keys.
void radix_sort_pairs(uint32_t* keys, int32_t* vals, int64_t n, int key_bits, cudaStream_t s) {
    if (n <= 1 || key_bits <= 0) return;
    const int64_t tiles = grid_tiles(n);
    DevBuf<uint32_t> k2;
    DevBuf<int32_t> v2;
    k2.alloc((size_t)n, s);
    v2.alloc((size_t)n, s);
    DevBuf<int32_t> hist;
    DevBuf<int64_t> off;
    hist.alloc((size_t)(256 * tiles), s);
    off.alloc((size_t)(256 * tiles) + 1, s);
    uint32_t* ka = keys;
    int32_t* va = vals;
    uint32_t* kb = k2.p;
    int32_t* vb = v2.p;
    int passes = 0;
    for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
        k_rs_hist<<<(unsigned)tiles, kRsThreads, 0, s>>>(ka, n, shift, hist.p, tiles);
        BFS_CHECK_LAUNCH();
        scan_exclusive_i32(hist.p, off.p, 256 * tiles, s);
        k_rs_scatter<<<(unsigned)tiles, kRsThreads, 0, s>>>(ka, va, n, shift, off.p, tiles, kb, vb);
        BFS_CHECK_LAUNCH();
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) {
        BFS_CUDA(cudaMemcpyAsync(keys, ka, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
        BFS_CUDA(cudaMemcpyAsync(vals, va, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    }
    BFS_CUDA(cudaStreamSynchronize(s));
}

}  // namespace bfsb
