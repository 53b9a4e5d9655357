// D2H bandwidth probe for the e2e leg: copy engine (cudaMemcpyAsync, 1 and 2 streams) vs an SM
// kernel storing straight into mapped pinned host memory (zero-copy).  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void k_store(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(dst + i, __ldcs(src + i));
}
int main() {
    const size_t bytes = (size_t)2 << 30;
    void *d, *h;
    CK(cudaMalloc(&d, bytes));
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaMemset(d, 1, bytes));
    cudaStream_t s[2]; cudaStreamCreateWithFlags(&s[0], cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s[1], cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, s[0]);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s[0]);
        cudaEventRecord(b, s[0]); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy 1 stream : %.1f GB/s\n", bytes / ms / 1e6);
        cudaEventRecord(a, s[0]); cudaStreamWaitEvent(s[1], a, 0);
        cudaMemcpyAsync(h, d, bytes / 2, cudaMemcpyDeviceToHost, s[0]);
        cudaMemcpyAsync((char*)h + bytes / 2, (char*)d + bytes / 2, bytes / 2, cudaMemcpyDeviceToHost, s[1]);
        cudaEvent_t c; cudaEventCreate(&c); cudaEventRecord(c, s[1]); cudaStreamWaitEvent(s[0], c, 0);
        cudaEventRecord(b, s[0]); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy 2 streams: %.1f GB/s\n", bytes / ms / 1e6);
        for (int g : {148, 296, 592, 1184, 2368}) for (int t : {256, 512}) {
            cudaEventRecord(a, s[0]);
            k_store<<<g, t, 0, s[0]>>>((const int4*)d, (int4*)h, bytes / 16);
            cudaEventRecord(b, s[0]); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("zero-copy kernel grid %d x %d: %.1f GB/s\n", g, t, bytes / ms / 1e6);
        }
    }
    // the bfs_run shape: two 2 GiB outputs, pooled device staging, separate host buffers
    void *d2, *h2;
    CK(cudaMallocAsync(&d2, bytes, s[0]));
    CK(cudaHostAlloc(&h2, bytes, cudaHostAllocDefault));
    CK(cudaMemsetAsync(d2, 2, bytes, s[0]));
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, s[0]);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s[0]);
        cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s[0]);
        cudaEventRecord(b, s[0]); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy 2 x 2 GiB sequential: %.1f GB/s\n", 2 * bytes / ms / 1e6);
        const size_t ch = (size_t)256 << 20;
        cudaEventRecord(a, s[0]);
        for (size_t o = 0; o < bytes; o += ch) {
            cudaMemcpyAsync((char*)h + o, (char*)d + o, ch, cudaMemcpyDeviceToHost, s[0]);
            cudaMemcpyAsync((char*)h2 + o, (char*)d2 + o, ch, cudaMemcpyDeviceToHost, s[0]);
        }
        cudaEventRecord(b, s[0]); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy 2 x 2 GiB in 256 MiB chunks: %.1f GB/s\n", 2 * bytes / ms / 1e6);
    }
    return 0;
}
