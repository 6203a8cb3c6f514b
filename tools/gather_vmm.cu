// gather_vmm.cu — does mapping physical memory in large chunks (cuMemCreate /
// cuMemMap) extend the GPU's TLB reach for random sector gathers?  Not product code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gather_vmm tools/gather_vmm.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("CU %s at %d\n", s, __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__global__ void chase(const uint32_t* __restrict__ a, uint64_t nsec, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t h = mix(t * 0x9E3779B97F4A7C15ull);
    uint32_t acc = 0;
    for (int j = 0; j < iters; ++j) {
        uint32_t v0, v5, v3, d;
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v0), "=r"(d), "=r"(d), "=r"(v3), "=r"(d), "=r"(v5), "=r"(d), "=r"(d) : "l"(a + 8 * (h % nsec)));
        h = mix(h ^ v0 ^ v5); acc ^= v3;
    }
    if (acc == 0x12345678) sink[0] = acc;
}
__global__ void fill(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] = (uint32_t)mix(i);
}
int main(int argc, char** argv) {
    CU(cuInit(0));
    CUdevice dev; CU(cuDeviceGet(&dev, 0));
    CK(cudaSetDevice(0)); CK(cudaFree(0));
    double gb = argc > 1 ? atof(argv[1]) : 128;
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gmin, grec;
    CU(cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    CU(cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("granularity min %zu rec %zu\n", gmin, grec);
    uint32_t* sink; CK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (size_t chunk : {(size_t)2 << 20, (size_t)64 << 20, (size_t)1 << 30, (size_t)4 << 30}) {
        size_t total = ((size_t)(gb * 1e9) / chunk) * chunk;
        CUdeviceptr va;
        CU(cuMemAddressReserve(&va, total, (size_t)4 << 30, 0, 0));
        std::vector<CUmemGenericAllocationHandle> hs;
        for (size_t off = 0; off < total; off += chunk) {
            CUmemGenericAllocationHandle h;
            CU(cuMemCreate(&h, chunk, &prop, 0));
            CU(cuMemMap(va + off, chunk, 0, h, 0));
            hs.push_back(h);
        }
        CUmemAccessDesc acc = {};
        acc.location = prop.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CU(cuMemSetAccess(va, total, &acc, 1));
        uint32_t* a = (uint32_t*)va;
        fill<<<148 * 16, 256>>>(a, total / 4);
        CK(cudaDeviceSynchronize());
        for (double fp : {32.0, 64.0, 96.0, 128.0}) {
            if (fp * 1e9 > total) break;
            uint64_t nsec = (uint64_t)(fp * 1e9) / 32;
            int blocks = 148 * 8, it = 64;
            chase<<<blocks, 256>>>(a, nsec, it, sink); CK(cudaDeviceSynchronize());
            cudaEventRecord(e0); chase<<<blocks, 256>>>(a, nsec, it, sink); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("chunk %6zu MB  footprint %5.0f GB  %6.2f G sectors/s\n", chunk >> 20, fp, (double)blocks * 256 * it / ms / 1e6);
        }
        CU(cuMemUnmap(va, total));
        for (auto h : hs) CU(cuMemRelease(h));
        CU(cuMemAddressFree(va, total));
    }
    return 0;
}
