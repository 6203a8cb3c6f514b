// gather_roofline.cu — the random-access ceiling of B200 HBM for the walk kernels.
//
// Measures, over an array much larger than L2 (default 16 GiB):
//   (1) independent random 4-B loads, MLP 8 per thread  -> random-sector ceiling
//   (2) independent random 32-B (full-sector) loads      -> same sectors, all bytes used
//   (3) dependent random chains (pointer chasing), 1 per thread -> TLP-only ceiling
//   (4) dependent chains, 4 interleaved per thread
//   (5) streaming copy (read+write) for reference
// Reports sectors/s and "sector GB/s" (sectors x 32 B).  Not part of the product.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather tools/gather_roofline.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}

__global__ void fill(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)mix(i);
}

__global__ void rand4(const uint32_t* __restrict__ a, uint64_t n, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int j = 0; j < iters; j += 8) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(a + (mix(t * 1315423911ull + j + k) & (n - 1)));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678) sink[0] = acc;
}

__global__ void rand32(const uint4* __restrict__ a, uint64_t nsec, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int j = 0; j < iters; j += 8) {
        uint4 v[8], w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint64_t s = mix(t * 1315423911ull + j + k) & (nsec - 1);
            v[k] = __ldg(a + 2 * s);
            w[k] = __ldg(a + 2 * s + 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].w ^ w[k].y ^ w[k].z;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

__global__ void rand64(const uint4* __restrict__ a, uint64_t nline, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int j = 0; j < iters; j += 4) {
        uint4 v[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint64_t s = mix(t * 1315423911ull + j + k) & (nline - 1);
#pragma unroll
            for (int q = 0; q < 4; ++q) v[k][q] = __ldg(a + 4 * s + q);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc ^= v[k][0].x ^ v[k][1].y ^ v[k][2].z ^ v[k][3].w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

template <int CH>
__global__ void chase(const uint32_t* __restrict__ a, uint64_t n, int iters, uint32_t* sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t p[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) p[c] = mix(t * 7 + c) & (n - 1);
    for (int j = 0; j < iters; ++j) {
#pragma unroll
        for (int c = 0; c < CH; ++c) p[c] = (p[c] * 0x9E3779B97F4A7C15ull + __ldg(a + p[c])) >> 16 & (n - 1);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc ^= (uint32_t)p[c];
    if (acc == 0x12345678) sink[0] = acc;
}

__global__ void copyk(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main(int argc, char** argv) {
    int lg = argc > 1 ? atoi(argv[1]) : 34;   // array bytes = 2^lg (power of two: masks, not %)
    uint64_t n = (1ull << lg) / 4;
    if (argc > 2) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[2])));
    size_t gran = 0;
    CK(cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity));
    printf("array 2^%d bytes, L2 fetch granularity limit %zu B\n", lg, gran);
    uint32_t *a, *sink;
    CK(cudaMalloc(&a, n * 4));
    CK(cudaMalloc(&sink, 4));
    fill<<<148 * 16, 256>>>(a, n);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148 * 8, threads = 256;
    uint64_t nthr = (uint64_t)blocks * threads;
    auto run = [&](const char* name, auto launch, double sectors, double useful_bytes) {
        launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s %8.3f ms  %7.2f Gsectors/s  sector-GB/s %8.1f  useful-GB/s %8.1f\n", name, ms,
               sectors / ms / 1e6, sectors * 32 / ms / 1e6, useful_bytes / ms / 1e6);
    };
    int it = 256;
    run("random 4B loads (MLP 8)", [&] { rand4<<<blocks, threads>>>(a, n, it, sink); }, (double)nthr * it, (double)nthr * it * 4);
    run("random 32B sector loads (MLP 8)", [&] { rand32<<<blocks, threads>>>((const uint4*)a, n / 8, it, sink); }, (double)nthr * it, (double)nthr * it * 32);
    run("random 64B (2-sector) loads (MLP 4)", [&] { rand64<<<blocks, threads>>>((const uint4*)a, n / 16, it, sink); }, (double)nthr * it * 2, (double)nthr * it * 64);
    int blocks2 = 148 * 16;  // 2048 thr/SM
    uint64_t nthr2 = (uint64_t)blocks2 * threads;
    run("random 4B loads (MLP 8, 2048 thr/SM)", [&] { rand4<<<blocks2, threads>>>(a, n, it, sink); }, (double)nthr2 * it, (double)nthr2 * it * 4);
    int cit = 64;
    run("dependent chain x1 (2048 thr/SM)", [&] { chase<1><<<blocks2, threads>>>(a, n, cit, sink); }, (double)nthr2 * cit, (double)nthr2 * cit * 4);
    run("dependent chain x2 (2048 thr/SM)", [&] { chase<2><<<blocks2, threads>>>(a, n, cit, sink); }, (double)nthr2 * cit * 2, (double)nthr2 * cit * 8);
    run("dependent chain x4 (1024 thr/SM)", [&] { chase<4><<<blocks, threads>>>(a, n, cit, sink); }, (double)nthr * cit * 4, (double)nthr * cit * 16);
    uint64_t half = n / 8;  // uint4 count of half the array
    run("stream copy (read+write)", [&] { copyk<<<148 * 16, 256>>>((const uint4*)a, (uint4*)a + half, half); }, (double)half * 16 * 2 / 32, (double)half * 16 * 2);
    return 0;
}
