// gather_variants.cu — which load flavour moves how many sectors for one random
// 4-B read on B200 (run under ncu with dram__sectors_read.sum etc.).  Not product code.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
template <int K> __device__ __forceinline__ uint32_t ld(const uint32_t* p) {
    uint32_t r;
    if (K == 0) r = __ldg(p);
    if (K == 1) asm volatile("ld.global.u32 %0, [%1];" : "=r"(r) : "l"(p));
    if (K == 2) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
    if (K == 3) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(r) : "l"(p));
    if (K == 4) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    if (K == 5) asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(r) : "l"(p));
    if (K == 6) asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
    if (K == 7) asm volatile("ld.global.lu.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
template <int K> __global__ void rand4(const uint32_t* __restrict__ a, uint64_t n, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int j = 0; j < iters; j += 8) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ld<K>(a + (mix(t * 1315423911ull + j + k) & (n - 1)));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678) sink[0] = acc;
}
__global__ void fill(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] = (uint32_t)mix(i);
}
int main(int argc, char** argv) {
    int lg = argc > 1 ? atoi(argv[1]) : 30;
    uint64_t n = (1ull << lg) / 4;
    uint32_t *a, *sink;
    CK(cudaMalloc(&a, n * 4)); CK(cudaMalloc(&sink, 4));
    fill<<<148 * 16, 256>>>(a, n);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"ldg(.nc)", "ld(.ca)", "ld.cg", "ld.cs", "nc.L1::no_allocate", "ld.cv", "nc.L2::64B", "ld.lu"};
    int blocks = 148 * 16, it = 256;
    double loads = (double)blocks * 256 * it;
    auto run = [&](int k, auto fn) {
        fn(); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); fn(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-22s %7.3f ms  %6.2f G loads/s\n", names[k], ms, loads / ms / 1e6);
    };
    run(0, [&] { rand4<0><<<blocks, 256>>>(a, n, it, sink); });
    run(1, [&] { rand4<1><<<blocks, 256>>>(a, n, it, sink); });
    run(2, [&] { rand4<2><<<blocks, 256>>>(a, n, it, sink); });
    run(3, [&] { rand4<3><<<blocks, 256>>>(a, n, it, sink); });
    run(4, [&] { rand4<4><<<blocks, 256>>>(a, n, it, sink); });
    run(5, [&] { rand4<5><<<blocks, 256>>>(a, n, it, sink); });
    run(6, [&] { rand4<6><<<blocks, 256>>>(a, n, it, sink); });
    run(7, [&] { rand4<7><<<blocks, 256>>>(a, n, it, sink); });
    return 0;
}
