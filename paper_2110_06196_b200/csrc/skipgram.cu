// skipgram.cu — the SkipGram consumer of the walks on the device (SURVEY §8(f)
// row f3; include/grape_walk.h grape_skipgram_pairs): the
// (center, context) pairs of the sliding window and, per pair, K
// negatives from the out-degree ("scale-free") distribution, drawn as the node
// whose row holds a uniform arc index — the rank the paper implements on its
// Elias-Fano arrays.
//
// Rank on the device: a node guide over arc-index buckets of 2^sh arcs,
// gidx[b] = rank(b << sh), built once per graph (lazily, on the first call);
// rank(e) starts at gidx[e >> sh] and steps over rows that end at or before e
// (one node per bucket on average, so ~1-2 reads of off[] per negative).
//
// One thread per output word: slots p (center + context) in the first loop,
// (slot, k) pairs in the second, so every store of a warp is contiguous; the
// walk rows are re-read from L2.
#include <mutex>

#include "internal.h"
#include "philox.cuh"

namespace grape {
namespace {

constexpr uint32_t kPadSg = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t rank_search(const uint64_t* __restrict__ off, uint32_t n, uint64_t e)
{
    uint32_t lo = 0, hi = n - 1;   // off[lo] <= e < off[hi + 1]
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo + 1) / 2;
        if (off[mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void build_node_guide(const uint64_t* __restrict__ off, uint32_t n, uint32_t sh, uint64_t nb,
                                 uint32_t* __restrict__ gidx)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride)
        gidx[b] = rank_search(off, n, b << sh);
}

struct SgParams {
    const uint64_t* off;
    const uint32_t* gidx;
    uint32_t sh;
    uint64_t m;
    const uint32_t* walks;
    uint64_t num_walks;
    uint64_t base;
    uint32_t L, w, K;
    RoundKeys rk;
    uint32_t* centers;
    uint32_t* contexts;
    uint32_t* negs;
};

// slot p (local) -> row r, position i, offset j; valid iff both ends are live
__device__ __forceinline__ bool slot_of(const SgParams& P, uint64_t p, uint64_t& r, uint32_t& i, uint32_t& o,
                                        uint32_t& a, uint32_t& b)
{
    const uint64_t per_row = (uint64_t)P.L * 2 * P.w;
    r = p / per_row;
    const uint32_t rem = (uint32_t)(p - r * per_row);
    i = rem / (2 * P.w);
    o = rem - i * 2 * P.w;
    const int64_t j = o < P.w ? (int64_t)o - P.w : (int64_t)o - P.w + 1;
    const int64_t c = (int64_t)i + j;
    const uint32_t* row = P.walks + r * P.L;
    if (c < 0 || c >= (int64_t)P.L) return false;
    a = __ldg(row + i);
    b = __ldg(row + c);
    return a != kPadSg && b != kPadSg;
}

__global__ void __launch_bounds__(256) skipgram_kernel(const __grid_constant__ SgParams P)
{
    const uint64_t S = P.num_walks * P.L * 2 * P.w;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (uint64_t p = t0; p < S; p += stride) {
        uint64_t r;
        uint32_t i, o, a = 0, b = 0;
        const bool ok = slot_of(P, p, r, i, o, a, b);
        P.centers[p] = ok ? a : kPadSg;
        P.contexts[p] = ok ? b : kPadSg;
    }
    const uint64_t SK = S * P.K;
    for (uint64_t q = t0; q < SK; q += stride) {
        const uint64_t p = q / P.K;
        const uint32_t k = (uint32_t)(q - p * P.K);
        uint64_t r;
        uint32_t i, o, a = 0, b = 0;
        uint32_t v = kPadSg;
        if (slot_of(P, p, r, i, o, a, b) && P.m != 0) {
            const uint64_t slot = ((P.base + r) * P.L + i) * (uint64_t)(2 * P.w) + o;   // global slot id
            const Draw d = philox_draw_rk(P.rk, slot, 0xFFFFFFFFu, k);
            const uint64_t e = __umul64hi(d.x64, P.m);                                   // BOUNDED(x64, m)
            v = __ldg(P.gidx + (e >> P.sh));
            while (__ldg(P.off + v + 1) <= e) ++v;                                       // rows ending before e
        }
        P.negs[q] = v;
    }
}

}  // namespace

cudaError_t ensure_node_guide(grape_graph* g, cudaStream_t stream)
{
    std::lock_guard<std::mutex> lk(g->node_guide_mu);
    if (g->node_guide != nullptr || g->m == 0) return cudaSuccess;
    uint32_t sh = 0;
    while ((g->m >> sh) + 1 > (uint64_t)g->n) ++sh;   // about one bucket per node
    const uint64_t nb = (g->m >> sh) + 1;
    uint32_t* gidx = nullptr;
    cudaError_t e = cudaMalloc(&gidx, nb * 4);
    if (e != cudaSuccess) return e;
    const unsigned blocks = (unsigned)((nb + 255) / 256 < 4096 ? (nb + 255) / 256 : 4096);
    build_node_guide<<<blocks, 256, 0, stream>>>(g->off, g->n, sh, nb, gidx);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);   // later calls may use other streams
    if (e != cudaSuccess) {
        cudaFree(gidx);
        return e;
    }
    g->node_guide = gidx;
    g->node_guide_shift = sh;
    return cudaSuccess;
}

cudaError_t launch_skipgram(const grape_graph* g, const uint32_t* walks, uint64_t num_walks, uint64_t base,
                            uint32_t L, uint32_t window, uint32_t K, uint64_t seed, uint32_t* centers,
                            uint32_t* contexts, uint32_t* negs, cudaStream_t stream)
{
    SgParams P{};
    P.off = g->off;
    P.gidx = g->node_guide;
    P.sh = g->node_guide_shift;
    P.m = g->m;
    P.walks = walks;
    P.num_walks = num_walks;
    P.base = base;
    P.L = L;
    P.w = window;
    P.K = K;
    P.rk = philox_round_keys(seed);
    P.centers = centers;
    P.contexts = contexts;
    P.negs = negs;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const uint64_t work = num_walks * L * 2 * window * (K > 0 ? K : 1);
    uint64_t blocks = (work + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;   // 8 resident blocks of 256 per SM, grid-stride
    if (blocks > cap) blocks = cap;
    skipgram_kernel<<<(unsigned)blocks, 256, 0, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace grape
