// Probe of NVLink SHARP (NVLS) multicast on this box: device attributes, a multicast
// object over the visible device(s), bound physical memory mapped at a unicast and a
// multicast address, multimem.st / multimem.ld_reduce.or through the multicast address,
// read back through the unicast one.  With one GPU the group has one member (the NVSwitch
// replication degenerates to a plain store), but every API and PTX step is exercised.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        CUresult r = (x);                                                                  \
        if (r != CUDA_SUCCESS) {                                                           \
            const char* m = nullptr;                                                       \
            cuGetErrorString(r, &m);                                                       \
            printf("FAIL %s: %d %s\n", #x, (int)r, m ? m : "?");                          \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

__global__ void k_mc_store(uint32_t* mc, const uint32_t* src, int64_t words) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = src[i];
        asm volatile("multimem.st.relaxed.sys.global.u32 [%0], %1;" ::"l"(mc + i), "r"(v) : "memory");
    }
}
__global__ void k_mc_or(const uint32_t* mc, uint32_t* dst, int64_t words) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b32 %0, [%1];" : "=r"(v) : "l"(mc + i) : "memory");
        dst[i] = v;
    }
}

int main() {
    CK(cuInit(0));
    int ndev = 0;
    CK(cuDeviceGetCount(&ndev));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc = 0, fab = 0, vmm = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    CK(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
    CK(cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev));
    printf("devices %d multicast_supported %d fabric_handles %d vmm %d\n", ndev, mc, fab, vmm);
    if (!mc) return 0;
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    const size_t want = 64 << 20;
    CUmulticastObjectProp mp{};
    mp.numDevices = 1;
    mp.size = want;
    size_t gran = 0, size = 0;
    CUmemGenericAllocationHandle mch{};
    bool ok = false;
    // handle types to try: none (single process), POSIX fd, fabric (cross-process over NVSwitch)
    const unsigned long long types[3] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
    for (unsigned nd : {1u, 2u})
    for (unsigned long long ht : types) {
        if (ok) break;
        mp.numDevices = nd;
        mp.handleTypes = ht;
        mp.size = want;
        if (cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) {
            printf("granularity(handleTypes %llu) failed\n", ht);
            continue;
        }
        size = (want + gran - 1) / gran * gran;
        mp.size = size;
        const CUresult r = cuMulticastCreate(&mch, &mp);
        const char* m = nullptr;
        cuGetErrorString(r, &m);
        printf("cuMulticastCreate(numDevices %u, handleTypes %llu, min granularity %zu, size %zu): %d %s\n", nd, ht,
               gran, size, (int)r, m ? m : "?");
        if (r == CUDA_SUCCESS) ok = nd == 1;
    }
    if (!ok) return 1;
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem, 0, size, 0));
    CUdeviceptr uva, mva;
    CK(cuMemAddressReserve(&uva, size, gran, 0, 0));
    CK(cuMemMap(uva, size, 0, mem, 0));
    CK(cuMemAddressReserve(&mva, size, gran, 0, 0));
    CK(cuMemMap(mva, size, 0, mch, 0));
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = dev;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva, size, &ad, 1));
    CK(cuMemSetAccess(mva, size, &ad, 1));
    const int64_t words = size / 4;
    std::vector<uint32_t> h(words);
    for (int64_t i = 0; i < words; ++i) h[i] = (uint32_t)(i * 2654435761u);
    uint32_t *src, *dst;
    cudaMalloc(&src, size);
    cudaMalloc(&dst, size);
    cudaMemcpy(src, h.data(), size, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_mc_store<<<148 * 4, 256>>>(reinterpret_cast<uint32_t*>(mva), src, words);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k_mc_store<<<148 * 4, 256>>>(reinterpret_cast<uint32_t*>(mva), src, words);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<uint32_t> back(words);
    cudaMemcpy(back.data(), reinterpret_cast<void*>(uva), size, cudaMemcpyDeviceToHost);
    int64_t bad = 0;
    for (int64_t i = 0; i < words; ++i) bad += back[i] != h[i];
    printf("multimem.st %zu MB: %lld mismatches through the unicast mapping; %.1f GB/s\n", size >> 20, (long long)bad,
           10.0 * size / (ms * 1e-3) / 1e9);
    k_mc_or<<<148 * 4, 256>>>(reinterpret_cast<const uint32_t*>(mva), dst, words);
    cudaMemcpy(back.data(), dst, size, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int64_t i = 0; i < words; ++i) bad += back[i] != h[i];
    printf("multimem.ld_reduce.or: %lld mismatches (one member: OR = the value); cuda error: %s\n", (long long)bad,
           cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
