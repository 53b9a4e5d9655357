// Micro-benchmark: random 4-byte probes into a bitmap of S MB, optionally with a
// concurrent evict-first stream over a large buffer (the TD/BU access mix).  Reports
// time; run under ncu for dram__bytes_read.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash32(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void probe(const unsigned* __restrict__ bm, size_t words, const int* __restrict__ stream, size_t slen,
                      int iters, unsigned long long* out, int mode) {
    unsigned long long acc = 0;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    for (int it = 0; it < iters; ++it) {
        const unsigned h = hash32((unsigned)(tid * 7919u + it * 104729u));
        const size_t w = h % words;
        unsigned x = mode & 1 ? __ldcg(bm + w) : __ldg(bm + w);
        acc += x;
        if (mode & 2) acc += __ldcs(stream + ((tid + (size_t)it * nt) % slen));
    }
    if (acc == 0x12345) out[0] = acc;
}
int main(int argc, char** argv) {
    const double mb = atof(argv[1]);
    const int mode = atoi(argv[2]);
    const size_t words = (size_t)(mb * 1e6 / 4);
    unsigned* bm; int* st; unsigned long long* out;
    const size_t slen = (size_t)4 << 30;  // 16 GB stream
    cudaMalloc(&bm, words * 4); cudaMalloc(&st, slen * 4); cudaMalloc(&out, 8);
    cudaMemset(bm, 0, words * 4); cudaMemset(st, 0, slen * 4);
    const int iters = 256;
    probe<<<148 * 8, 256>>>(bm, words, st, slen, iters, out, mode);  // warm
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<<<148 * 8, 256>>>(bm, words, st, slen, iters, out, mode);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double probes = 148.0 * 8 * 256 * iters;
    printf("bitmap %.1f MB mode %d: %.3f ms, %.1f G probes/s\n", mb, mode, ms, probes / ms / 1e6);
    return 0;
}
