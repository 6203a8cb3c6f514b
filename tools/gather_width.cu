// gather_width.cu — dependent random reads of 32 / 64 / 128 / 256 B on B200: reads per
// second and (under ncu, dram__bytes_read.sum) DRAM bytes moved per read, at a table
// footprint like the walker's.  The verdict's question: does a 64-B or 128-B record cost a
// 32-B read's rate, i.e. could coarser reads carry more of the next step for free?
// Not product code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gw tools/gather_width.cu
//   /tmp/gw sweep                 # every width x footprint, CUDA events
//   /tmp/gw one <GB> <S> <MLP>    # one launch (for ncu --metrics dram__bytes_read.sum)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__device__ __forceinline__ void ld8(const uint32_t* p, uint32_t (&v)[8]) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "l"(p));
}
// MLP independent chains per thread; one read = S consecutive 32-B sectors of an aligned
// S*32-B block (S loads issued together); the next block depends on every sector read
template <int S, int MLP>
__global__ void chase(const uint32_t* __restrict__ a, uint64_t nblk, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t h[MLP];
#pragma unroll
    for (int k = 0; k < MLP; ++k) h[k] = mix(t * 0x9E3779B97F4A7C15ull + k);
    uint32_t acc = 0;
    for (int j = 0; j < iters; ++j) {
        uint32_t v[MLP][S][8];
#pragma unroll
        for (int k = 0; k < MLP; ++k)
#pragma unroll
            for (int q = 0; q < S; ++q) ld8(a + 8 * ((h[k] % nblk) * S + q), v[k][q]);
#pragma unroll
        for (int k = 0; k < MLP; ++k) {
            uint32_t f = 0;
#pragma unroll
            for (int q = 0; q < S; ++q) f ^= v[k][q][0] ^ v[k][q][5];
            h[k] = mix(h[k] ^ f);
            acc ^= v[k][0][3];
        }
    }
    if (acc == 0x12345678) sink[0] = acc;
}
__global__ void fill(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] = (uint32_t)mix(i);
}
template <int S, int MLP>
static float launch(const uint32_t* a, uint64_t fp_bytes, int blocks, int it, uint32_t* sink, bool timed) {
    const uint64_t nblk = fp_bytes / (32ull * S);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    if (timed) { chase<S, MLP><<<blocks, 256>>>(a, nblk, it, sink); CK(cudaDeviceSynchronize()); }
    cudaEventRecord(e0);
    chase<S, MLP><<<blocks, 256>>>(a, nblk, it, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}
template <int MLP>
static float run(int S, const uint32_t* a, uint64_t fp, int blocks, int it, uint32_t* sink, bool timed) {
    switch (S) {
    case 1: return launch<1, MLP>(a, fp, blocks, it, sink, timed);
    case 2: return launch<2, MLP>(a, fp, blocks, it, sink, timed);
    case 4: return launch<4, MLP>(a, fp, blocks, it, sink, timed);
    default: return launch<8, MLP>(a, fp, blocks, it, sink, timed);
    }
}
int main(int argc, char** argv) {
    const bool one = argc > 1 && !strcmp(argv[1], "one");
    const double maxgb = one ? atof(argv[2]) : 64.5;
    const uint64_t bytes = (uint64_t)(maxgb * 1e9) & ~4095ull;
    uint32_t *a, *sink;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&sink, 4));
    fill<<<148 * 16, 256>>>(a, bytes / 4);
    CK(cudaDeviceSynchronize());
    const int blocks = 148 * 8, it = 32;   // 2048 threads per SM (the walker's 1024 saturate too)
    if (one) {
        const int S = atoi(argv[3]), mlp = atoi(argv[4]);
        const float ms = mlp == 1 ? run<1>(S, a, bytes, blocks, it, sink, false) : run<4>(S, a, bytes, blocks, it, sink, false);
        const double reads = (double)blocks * 256 * it * mlp;
        printf("one: footprint %.1f GB, %d B reads, MLP %d: %.0f reads, %.3f ms, %.2f G reads/s\n",
               maxgb, 32 * S, mlp, reads, ms, reads / ms / 1e6);
        return 0;
    }
    printf("footprint_GB read_B  mlp1_Greads/s  mlp4_Greads/s  mlp4_GB/s(requested)\n");
    for (double fp : {2.0, 22.0, 64.0}) {
        for (int S : {1, 2, 4, 8}) {
            const uint64_t fb = (uint64_t)(fp * 1e9) & ~4095ull;
            const float m1 = run<1>(S, a, fb, blocks, it, sink, true);
            const float m4 = run<4>(S, a, fb, blocks, it / 4, sink, true);
            const double r1 = (double)blocks * 256 * it / m1 / 1e6, r4 = (double)blocks * 256 * it / m4 / 1e6;
            printf("%8.1f %6d %14.2f %14.2f %14.0f\n", fp, 32 * S, r1, r4, r4 * 32 * S);
        }
    }
    return 0;
}
