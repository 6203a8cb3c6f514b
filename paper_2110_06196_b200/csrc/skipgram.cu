// skipgram.cu — the SkipGram consumer of the walks on the device (SURVEY §8(f)
// row f3; include/grape_walk.h grape_skipgram_pairs): the
// (center, context) pairs of the sliding window and, per pair, K
// negatives from the out-degree ("scale-free") distribution, drawn as the node
// whose row holds a uniform arc index — the rank the paper implements on its
// Elias-Fano arrays.
//
// Rank on the device: a node guide over arc-index buckets of 2^sh arcs (about 4
// or 1 per node, ensure_node_guide), 16-B entry b = {v0 = rank(b << sh), and where
// rows v0, v0 + 1, v0 + 2 end relative to the bucket}, built once per graph
// (lazily, on the first call).  A query reads its bucket's entry and is done unless
// three rows end at or before it inside the bucket; then it steps over off[].
//
// One block per walk row (staged in shared memory with its slots' validity bits);
// its threads write the row's slots, then its negatives, in order: every store of
// a warp is contiguous.
#include <cstdlib>
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

// entry b = {v0 = rank(b << sh), E1, E2, E3}: E_k = off[v0 + k] - (b << sh), the end of
// row v0 + k - 1 relative to the bucket (2^32 - 1 when past 2^32 - 1 or past row n - 1):
// a query at offset o into the bucket is row v0 + [o >= E1] + [o >= E2] + [o >= E3]
// unless o >= E3
__global__ void build_node_guide(const uint64_t* __restrict__ off, uint32_t n, uint32_t sh, uint64_t nb,
                                 uint4* __restrict__ gidx)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
        const uint64_t b0 = b << sh;
        const uint32_t v = rank_search(off, n, b0);
        uint32_t E[3];
        for (uint32_t k = 0; k < 3; ++k) {
            const uint64_t rel = v + 1 + k <= n ? off[v + 1 + k] - b0 : ~0ull;
            E[k] = rel < 0xFFFFFFFFull ? (uint32_t)rel : 0xFFFFFFFFu;
        }
        gidx[b] = make_uint4(v, E[0], E[1], E[2]);
    }
}

// n / d for 32-bit n and a divisor fixed per launch (Granlund-Montgomery, round-up
// multiplier): two multiplies instead of a division sequence
struct FastDiv {
    uint32_t d, m, s1;
    static FastDiv of(uint32_t d_)
    {
        FastDiv f{d_, 0, 0};
        if (d_ > 1) {
            uint32_t l = 0;
            while ((1ull << l) < d_) ++l;
            f.m = (uint32_t)((((1ull << 32) * ((1ull << l) - d_)) / d_) + 1);
            f.s1 = l - 1;
        }
        return f;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const
    {
        if (d == 1) return n;
        const uint32_t t = __umulhi(m, n);
        return (t + ((n - t) >> 1)) >> s1;
    }
};

struct SgParams {
    const uint64_t* off;
    uint32_t n;
    const uint4* gidx;
    uint32_t sh;
    uint64_t m;
    const uint32_t* walks;
    uint64_t num_walks;
    uint64_t base;
    uint32_t L, w, K;
    FastDiv tw_div, k_div;   // by 2w and by ceil(K / 2)
    RoundKeys rk;
    uint32_t* centers;
    uint32_t* contexts;
    uint32_t* negs;
};

constexpr uint32_t kRowSmemWords = 12288;
#ifndef GRAPE_SG_MIN_BLOCKS
#define GRAPE_SG_MIN_BLOCKS 8   // resident blocks of 256 per SM the pair kernel is compiled for
#endif   // a row and its slots' validity bits up to 48 KB are staged

// One block per walk row at a time (grid-stride over rows): the row is staged in
// shared memory, then the block's threads cover the row's L*2w slots (each slot's
// validity also kept as one bit in shared memory) and its L*2w*K negative words in
// order, so every store of a warp is contiguous and no 64-bit division is needed
// (32-bit index arithmetic within a row).
__global__ void __launch_bounds__(256, GRAPE_SG_MIN_BLOCKS) skipgram_kernel(const __grid_constant__ SgParams P)
{
    extern __shared__ uint32_t srow[];
    const uint32_t L = P.L, tw = 2 * P.w, K = P.K;
    const uint32_t per_row = L * tw;
    const uint32_t bit_words = (per_row + 31) / 32;
    const bool staged = L + bit_words <= kRowSmemWords;
    uint32_t* sbits = srow + L;   // staged: bit idx of word idx/32 = slot idx is valid
    for (uint64_t r = blockIdx.x; r < P.num_walks; r += gridDim.x) {
        const uint32_t* grow = P.walks + r * L;
        __syncthreads();   // the previous row's readers are done
        if (staged)
            for (uint32_t q = threadIdx.x; q < L; q += blockDim.x) srow[q] = __ldg(grow + q);
        __syncthreads();
        const uint32_t* row = staged ? srow : grow;
        auto ends = [&](uint32_t idx, uint32_t& a, uint32_t& b) {   // slot idx of this row: valid?
            const uint32_t i = P.tw_div.div(idx), o = idx - i * tw;
            const int32_t c = (int32_t)i + (o < P.w ? (int32_t)o - (int32_t)P.w : (int32_t)o - (int32_t)P.w + 1);
            if (c < 0 || c >= (int32_t)L) return false;
            a = row[i];
            b = row[c];
            return a != kPadSg && b != kPadSg;
        };
        const uint64_t o0 = r * per_row;                        // local slot offset of the row
        const uint64_t g0 = (P.base + r) * per_row;             // global slot id of its first slot
        // slots: whole warps step together over consecutive slots (the loop bound is
        // rounded up to a warp), so each warp's ballot is one word of validity bits
        const uint32_t per_row_w = (per_row + 31) & ~31u;
        for (uint32_t idx = threadIdx.x; idx < per_row_w; idx += blockDim.x) {
            uint32_t a = 0, b = 0;
            const bool in = idx < per_row;
            const bool ok = in && ends(idx, a, b);
            if (in) {
                P.centers[o0 + idx] = ok ? a : kPadSg;
                P.contexts[o0 + idx] = ok ? b : kPadSg;
            }
            const unsigned bits = __ballot_sync(0xffffffffu, ok);
            if (staged && (threadIdx.x & 31) == 0) sbits[idx >> 5] = bits;
        }
        if (staged) __syncthreads();   // the validity bits are complete
        // negatives 2kk and 2kk+1 of a slot come from one Philox block (words o1:o0 and
        // o3:o2): one thread per block, its two words stored side by side
        const uint32_t Kh = (K + 1) / 2;
        const uint32_t nk = per_row * Kh;
        auto rank = [&](uint64_t x64) {
            const uint64_t e = __umul64hi(x64, P.m);                 // BOUNDED(x64, m)
            const uint4 ge = __ldg(P.gidx + (e >> P.sh));
            const uint32_t o = (uint32_t)(e & ((1ull << P.sh) - 1));   // offset into the bucket
            uint32_t v = ge.x + (o >= ge.y) + (o >= ge.z) + (o >= ge.w);
            if (o >= ge.w)                                            // three rows end before e
                while (__ldg(P.off + v + 1) <= e) ++v;
            GRAPE_DCHECK(e < P.m && v < P.n && __ldg(P.off + v) <= e && e < __ldg(P.off + v + 1),
                         "negative = the row holding arc e");
            return v;
        };
        for (uint32_t idx = threadIdx.x; idx < nk; idx += blockDim.x) {
            const uint32_t sl = P.k_div.div(idx), kk = idx - sl * Kh;
            const uint32_t k0 = 2 * kk;
            uint32_t a = 0, b = 0, v0 = kPadSg, v1 = kPadSg;
            const bool ok = staged ? ((sbits[sl >> 5] >> (sl & 31)) & 1u) != 0 : ends(sl, a, b);
            if (ok && P.m != 0) {
                const uint4 o = philox_block_rk(P.rk, g0 + sl, 0xFFFFFFFFu, kk);
                v0 = rank((uint64_t)o.y << 32 | o.x);
                if (k0 + 1 < K) v1 = rank((uint64_t)o.w << 32 | o.z);
            }
            uint32_t* dst = P.negs + (o0 + sl) * K + k0;
            dst[0] = v0;
            if (k0 + 1 < K) dst[1] = v1;
        }
    }
}

}  // namespace

cudaError_t ensure_node_guide(grape_graph* g, cudaStream_t stream)
{
    std::lock_guard<std::mutex> lk(g->node_guide_mu);
    if (g->node_guide != nullptr || g->m == 0) return cudaSuccess;
    // buckets per node: 4 (64 B per node) while that guide stays L2-sized (<= 128 MB),
    // else 1 (16 B per node).  Each 16-B entry resolves a query up to three row ends
    // into its bucket (the 8-B entries of round 1 resolved one, at 8 and 2 per node:
    // configs[1] pair kernel 47.9 ms with those).  GRAPE_SG_GUIDE_PER_NODE overrides (A/B).
    uint32_t per_node = (uint64_t)g->n * 64 <= (128ull << 20) ? 4 : 1;
    if (const char* s = getenv("GRAPE_SG_GUIDE_PER_NODE")) per_node = (uint32_t)atoi(s) > 0 ? (uint32_t)atoi(s) : per_node;
    uint32_t sh = 0;
    while ((g->m >> sh) + 1 > (uint64_t)per_node * g->n) ++sh;
    const uint64_t nb = (g->m >> sh) + 1;
    uint4* gidx = nullptr;
    cudaError_t e = cudaMalloc(&gidx, nb * sizeof(uint4));
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
    P.n = g->n;
    P.gidx = g->node_guide;
    P.sh = g->node_guide_shift;
    P.m = g->m;
    P.walks = walks;
    P.num_walks = num_walks;
    P.base = base;
    P.L = L;
    P.w = window;
    P.K = K;
    P.tw_div = FastDiv::of(2 * window);
    P.k_div = FastDiv::of(K > 1 ? (K + 1) / 2 : 1);   // by ceil(K / 2): Philox blocks per slot
    P.rk = philox_round_keys(seed);
    P.centers = centers;
    P.contexts = contexts;
    P.negs = negs;
    int sms = 0;   // of the graph's device
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    if (sms < 1) sms = 1;
    uint64_t blocks = num_walks;
    const uint64_t cap = (uint64_t)sms * GRAPE_SG_MIN_BLOCKS;   // one wave of resident blocks, grid-stride over rows
    if (blocks > cap) blocks = cap;
    const uint64_t words = (uint64_t)L + ((uint64_t)L * 2 * window + 31) / 32;   // row + validity bits
    const size_t smem = words <= kRowSmemWords ? (size_t)words * 4 : 0;
    skipgram_kernel<<<(unsigned)blocks, 256, smem, stream>>>(P);
    return cudaGetLastError();
}


// ---- walks streamed into the SkipGram consumer (grape_walks_skipgram; §8(f) f3) ----
//
// The walk matrix is an intermediate of the pair stream: the walker fills one
// chunk of rows at a time into a device buffer and the pair kernel consumes the
// chunk while the walker fills the other buffer (two internal streams, events
// between them), so the walker's work overlaps the pair kernel's and the W*L*4-byte
// walk matrix is never materialised (two chunk buffers instead).  A persisting-L2
// access-policy window over the buffers was measured and dropped: the set-aside it
// needs stays reserved after the call and slowed the other kernels (the pair kernel
// of the two-call path 52 -> 70 ms on configs[1], 2e6 walks).  Results are the
// two-call results bit for bit: the same walk ids and slot ids.
cudaError_t launch_walks_skipgram(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                                  uint32_t window, uint32_t K, uint64_t pair_seed, uint32_t* centers,
                                  uint32_t* contexts, uint32_t* negs, uint64_t chunk_walks, cudaStream_t stream)
{
    const uint64_t L = a.L;
    uint64_t B = chunk_walks ? chunk_walks : a.num_walks;
    if (B > a.num_walks) B = a.num_walks;
    if (B == 0) return cudaSuccess;
    const uint64_t buf_bytes = ((B * L * 4 + 255) / 256) * 256;
    cudaStream_t sw = nullptr, sp = nullptr;
    cudaEvent_t start = nullptr, walked[2] = {}, paired[2] = {};
    char* buf = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&sw, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&walked[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&paired[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventRecord(start, stream);   // the caller's prior work (starts, outputs)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sw, start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sp, start, 0);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&buf, 2 * buf_bytes, sw);
    if (e == cudaSuccess) e = cudaEventRecord(walked[0], sw);   // the buffer exists before sp uses it
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sp, walked[0], 0);
    const uint64_t per_row = L * 2 * window;
    uint64_t k = 0;
    for (uint64_t lo = 0; lo < a.num_walks && e == cudaSuccess; lo += B, ++k) {
        const int b = (int)(k & 1);
        const uint64_t cnt = a.num_walks - lo < B ? a.num_walks - lo : B;
        uint32_t* rows = (uint32_t*)(buf + b * buf_bytes);
        if (k >= 2) e = cudaStreamWaitEvent(sw, paired[b], 0);   // the pair kernel has read this buffer
        WalkArgs c = a;
        c.starts = a.starts + lo;
        c.num_walks = cnt;
        c.walk_id_base = a.walk_id_base + lo;
        c.out = rows;
        if (e == cudaSuccess) e = launch_walks(g, c, node2vec, T, sw);
        if (e == cudaSuccess) e = cudaEventRecord(walked[b], sw);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sp, walked[b], 0);
        if (e == cudaSuccess)
            e = launch_skipgram(g, rows, cnt, a.walk_id_base + lo, a.L, window, K, pair_seed, centers + lo * per_row,
                                contexts + lo * per_row, negs ? negs + lo * per_row * K : nullptr, sp);
        if (e == cudaSuccess) e = cudaEventRecord(paired[b], sp);
    }
    // the caller's stream continues after the last pair kernel; the buffer is released
    // on the pair stream after its last reader
    // (the pair stream waited for every walker launch, so its end orders everything)
    cudaEvent_t done = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    if (buf) cudaFreeAsync(buf, sp);
    if (e == cudaSuccess) e = cudaEventRecord(done, sp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, done, 0);
    // destroying streams / events with work pending is allowed: resources are released
    // once the work completes
    if (sw) cudaStreamDestroy(sw);
    if (sp) cudaStreamDestroy(sp);
    if (start) cudaEventDestroy(start);
    for (int b = 0; b < 2; ++b) {
        if (walked[b]) cudaEventDestroy(walked[b]);
        if (paired[b]) cudaEventDestroy(paired[b]);
    }
    if (done) cudaEventDestroy(done);
    return e;
}

}  // namespace grape
