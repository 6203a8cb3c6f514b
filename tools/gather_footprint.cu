// gather_footprint.cu — random 32-B sector gather rate vs footprint on B200
// (TLB reach / DRAM page effects).  Not product code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gf tools/gather_footprint.cu && /tmp/gf 140
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
#ifndef LDQ
#define LDQ ""
#endif
__device__ __forceinline__ void ld8(const uint32_t* p, uint32_t (&v)[8]) {
    asm volatile("ld.global.nc" LDQ ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "l"(p));
}
// MLP independent chains per thread; each step's address depends on the previous load (like a walk)
template <int MLP>
__global__ void chase(const uint32_t* __restrict__ a, uint64_t nsec, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t h[MLP];
#pragma unroll
    for (int k = 0; k < MLP; ++k) h[k] = mix(t * 0x9E3779B97F4A7C15ull + k);
    uint32_t acc = 0;
    for (int j = 0; j < iters; ++j) {
        uint32_t v[MLP][8];
#pragma unroll
        for (int k = 0; k < MLP; ++k) ld8(a + 8 * (h[k] % nsec), v[k]);
#pragma unroll
        for (int k = 0; k < MLP; ++k) { h[k] = mix(h[k] ^ v[k][0] ^ v[k][5]); acc ^= v[k][3]; }
    }
    if (acc == 0x12345678) sink[0] = acc;
}
__global__ void fill(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] = (uint32_t)mix(i);
}
int main(int argc, char** argv) {
    double maxgb = argc > 1 ? atof(argv[1]) : 64;
    uint64_t bytes = (uint64_t)(maxgb * 1e9) & ~4095ull;
    uint32_t *a, *sink;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&sink, 4));
    fill<<<148 * 16, 256>>>(a, bytes / 4);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    if (argc > 2) {   // occupancy sweep at one footprint: resident threads per SM
        double fp = atof(argv[2]);
        uint64_t nsec = (uint64_t)(fp * 1e9) / 32;
        printf("footprint %.1f GB: threads/SM  mlp1_Gsec/s  mlp2_Gsec/s\n", fp);
        for (int bps : {1, 2, 3, 4, 6, 8}) {
            double r[2];
            int mi = 0;
            for (int mlp : {1, 2}) {
                int blocks = 148 * bps, it = 64;
                auto fn = [&] { if (mlp == 1) chase<1><<<blocks, 256>>>(a, nsec, it, sink); else chase<2><<<blocks, 256>>>(a, nsec, it, sink); };
                fn(); CK(cudaDeviceSynchronize());
                cudaEventRecord(e0); fn(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                r[mi++] = (double)blocks * 256 * it * mlp / ms / 1e6;
            }
            printf("%10d %12.2f %12.2f\n", bps * 256, r[0], r[1]);
        }
        return 0;
    }
    double fps[] = {0.5, 1, 2, 4, 8, 16, 32, 48, 56, 60, 64, 66, 68, 70, 72, 76, 80, 96, 128};
    printf("footprint_GB  mlp1_Gsec/s  mlp4_Gsec/s\n");
    for (double fp : fps) {
        if (fp * 1e9 > bytes) break;
        uint64_t nsec = (uint64_t)(fp * 1e9) / 32;
        double r[2];
        int mi = 0;
        for (int mlp : {1, 4}) {
            int blocks = 148 * 8, it = mlp == 1 ? 64 : 16;
            auto fn = [&] { if (mlp == 1) chase<1><<<blocks, 256>>>(a, nsec, it, sink); else chase<4><<<blocks, 256>>>(a, nsec, it, sink); };
            fn(); CK(cudaDeviceSynchronize());
            cudaEventRecord(e0); fn(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            r[mi++] = (double)blocks * 256 * it * mlp / ms / 1e6;
        }
        printf("%8.1f %12.2f %12.2f\n", fp, r[0], r[1]);
    }
    return 0;
}
