// Device-wide exclusive prefix sums: CSR offsets from degrees and
// the top-down frontier degree prefix used for edge-balanced expansion.
//
// Reduce-then-scan over tiles of 2048 elements (256 threads x 8 items): one
// pass reads the input to produce tile sums, the tile sums are scanned
// (recursively, at most 3 levels for n <= 2^31), and a second pass re-reads the
// input and writes the scanned output.  Traffic 2 reads + 1 write of the array;
// the input is at most a few GiB so both passes are HBM-streaming.
#include "internal.cuh"

namespace bfsb {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

struct LoadI64 {
    const int64_t* p;
    __device__ int64_t operator()(int64_t i) const { return p[i]; }
};
struct LoadI32 {
    const int32_t* p;
    __device__ int64_t operator()(int64_t i) const { return p[i]; }
};

__device__ __forceinline__ int64_t warp_incl_scan(int64_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    return x;
}

// exclusive block scan of one value per thread; returns the block total via *total
__device__ __forceinline__ int64_t block_excl_scan(int64_t x, int64_t* total) {
    __shared__ int64_t warp_sums[kThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t inc = warp_incl_scan(x);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < kThreads / 32 ? warp_sums[lane] : 0;
        int64_t wi = warp_incl_scan(w);
        if (lane < kThreads / 32) warp_sums[lane] = wi - w;
    }
    __syncthreads();
    int64_t res = inc - x + warp_sums[wid];
    if (total) {
        __shared__ int64_t tot;
        if (threadIdx.x == kThreads - 1) tot = res + x;
        __syncthreads();
        *total = tot;
    }
    __syncthreads();
    return res;
}

template <class F>
__global__ void __launch_bounds__(kThreads) k_tile_reduce(F f, int64_t n, int64_t* tile_sums) {
    int64_t base = (int64_t)blockIdx.x * kTile;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
        if (i < n) s += f(i);
    }
    // block reduce
    for (int d = 16; d > 0; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
    __shared__ int64_t ws[kThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += ws[w];
        tile_sums[blockIdx.x] = t;
    }
}

// each thread owns kItems consecutive elements; out has n+1 entries
template <class F>
__global__ void __launch_bounds__(kThreads) k_tile_scan(F f, int64_t n, const int64_t* tile_offsets, int64_t* out,
                                                        int write_total) {
    int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    int64_t v[kItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int64_t i = base + k;
        v[k] = i < n ? f(i) : 0;
        s += v[k];
    }
    int64_t tot;
    int64_t pre = block_excl_scan(s, &tot) + (tile_offsets ? tile_offsets[blockIdx.x] : 0);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int64_t i = base + k;
        if (i < n) out[i] = pre;
        pre += v[k];
    }
    if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
        out[n] = (tile_offsets ? tile_offsets[blockIdx.x] : 0) + tot;
}

template <class F>
int scan_impl(F f, int64_t n, int64_t* out, cudaStream_t s) {
    if (n <= 0) {
        BFS_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return 0;
    }
    int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles == 1) {
        k_tile_scan<<<1, kThreads, 0, s>>>(f, n, nullptr, out, 1);
        BFS_CHECK_LAUNCH();
        return 1;
    }
    // tile sums -> exclusive scan of tile sums (tiles+1 entries) -> final pass
    DevBuf<int64_t> sums, offs;
    sums.alloc(tiles, s);
    offs.alloc(tiles + 1, s);
    k_tile_reduce<<<(unsigned)tiles, kThreads, 0, s>>>(f, n, sums.p);
    BFS_CHECK_LAUNCH();
    int launches = 2 + scan_impl(LoadI64{sums.p}, tiles, offs.p, s);
    k_tile_scan<<<(unsigned)tiles, kThreads, 0, s>>>(f, n, offs.p, out, 1);
    BFS_CHECK_LAUNCH();
    return launches;
}

}  // namespace

int scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    // in == out is allowed: every thread reads its own items before the block
    // scan's barrier and writes only those items afterwards.
    return scan_impl(LoadI64{in}, n, out, s);
}

int scan_exclusive_i32(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    return scan_impl(LoadI32{in}, n, out, s);
}


}  // namespace bfsb
