// l2_lookup.cu — independent random 8-B lookups into a table of S bytes on B200: the
// ceiling of the SkipGram pair kernel's rank lookups (node-guide entries).
// Not product code.  Each thread issues UNROLL independent loads per loop step (addresses
// from a hash of (thread, step), no dependence on loaded data), all SMs, full occupancy.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2l tools/l2_lookup.cu && /tmp/l2l
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t fmix(uint32_t h) {
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16; return h;
}
template <int UNROLL>
__global__ void __launch_bounds__(256) lookup(const uint2* __restrict__ t, uint32_t mask, int iters, uint32_t* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int j = 0; j < iters; ++j) {
        uint2 v[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) v[k] = __ldg(t + (fmix(tid * 0x9E3779B9u + (uint32_t)(j * UNROLL + k)) & mask));
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) acc += v[k].x ^ v[k].y;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void fill(uint2* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = make_uint2((uint32_t)i, (uint32_t)(i * 7));
}
int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint2* a; uint32_t* sink;
    const uint64_t maxb = 4ull << 30;
    CK(cudaMalloc(&a, maxb)); CK(cudaMalloc(&sink, 4));
    fill<<<sms * 8, 256>>>(a, maxb / 8);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    printf("table_MB  lookups_G_per_s(unroll1)  (unroll4)  (unroll8)\n");
    for (uint64_t mb : {4ull, 16ull, 32ull, 64ull, 96ull, 128ull, 256ull, 1024ull, 4096ull}) {
        const uint32_t mask = (uint32_t)((mb << 20) / 8 - 1);
        double r[3]; int ri = 0;
        for (int u : {1, 4, 8}) {
            const int blocks = sms * 8, it = 256 / u * 4;
            auto fn = [&] {
                if (u == 1) lookup<1><<<blocks, 256>>>(a, mask, it, sink);
                else if (u == 4) lookup<4><<<blocks, 256>>>(a, mask, it, sink);
                else lookup<8><<<blocks, 256>>>(a, mask, it, sink);
            };
            fn(); CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            for (int rep = 0; rep < 5; ++rep) fn();
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            r[ri++] = 5.0 * blocks * 256.0 * it * u / ms / 1e6;
        }
        printf("%8llu  %8.1f  %8.1f  %8.1f\n", (unsigned long long)mb, r[0], r[1], r[2]);
    }
    return 0;
}
