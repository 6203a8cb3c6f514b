// walk_cdf.cu — the paper's own node2vec sampler on the GPU (SURVEY §8(f) row
// f2; §4.3.2): per step, "1) the un-normalized transition
// probabilities to each neighbour of v according to the in-out and return
// biases; 2) their cumulative sum; 3) a uniform value between 0 and the total;
// 4) the corresponding index".  Rules (include/grape_walk.h,
// grape_walks_node2vec_cdf; oracle: oracle_walks_cdf): pi_x = w_vx * T_class(x)
// with the integer thresholds of §8(c) c9, exact 128-bit running sums, one draw
// per step (DRAW(seed, wid, s, 0), x64), r = floor(x64 * total / 2^64), the
// first index whose running sum exceeds r.  The first step is first-order.
//
// One warp per walk (walks from a shared counter), lanes over v's row in
// chunks of 32 arcs: the arc records give x, its weight (difference of
// consecutive prefix values, the predecessor's by shuffle) and the
// no-common-neighbour flag of (t, v); "x in N(t)" is an edge-hash probe.  Pass 1
// reduces the row's total and keeps each chunk's sum in a per-warp scratch; pass
// 2 finds the chunk holding r from those sums and rescans only that chunk —
// O(deg v) reads per step, the
// cost the paper's sampler has by construction.  It is the paper-faithful mode,
// not the fast one.
#include "walk_common.cuh"

namespace grape {
namespace {
using namespace walk;

constexpr uint32_t kEmpty = 0xFFFFFFFFu;

struct CdfParams {
    const NodeRec* nodes;
    const void* rec;
    const uint32_t* ehash;
    uint32_t n;
    const uint32_t* starts;
    uint64_t num_walks;
    uint64_t base;
    uint32_t L;
    RoundKeys rk;
    uint32_t* out;
    unsigned long long* steps_out;
    unsigned long long* next;      // walk counter
    uint64_t T[3];                 // T_p, T_1, T_q
    uint32_t h_mul, h_shift;       // floor(v / H)
    uint32_t xmask;                // compact records: x without flag bits
    bool notri;
    uint4* chunk_scratch;          // per resident warp: chunks_max x {sum lo, sum mid, sum hi, carry}
    uint64_t chunks_max;           // ceil(max degree / 32)
    uint64_t m_chk;                // arcs (checked build)
};

__device__ __forceinline__ uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

struct U128 {
    uint64_t lo, hi;
};

__device__ __forceinline__ U128 add128(U128 a, U128 b)
{
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
    return r;
}
__device__ __forceinline__ bool gt128(U128 a, U128 b) { return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo); }
__device__ __forceinline__ U128 shfl_up128(U128 a, int d)
{
    U128 r;
    r.lo = __shfl_up_sync(0xffffffffu, a.lo, d);
    r.hi = __shfl_up_sync(0xffffffffu, a.hi, d);
    return r;
}
__device__ __forceinline__ U128 shfl128(U128 a, int src)
{
    U128 r;
    r.lo = __shfl_sync(0xffffffffu, a.lo, src);
    r.hi = __shfl_sync(0xffffffffu, a.hi, src);
    return r;
}

// floor(x64 * S / 2^64) for S = (hi, lo): x64*hi + floor(x64*lo / 2^64) (< 2^128 since S < 2^92)
__device__ __forceinline__ U128 bounded128(uint64_t x64, U128 S)
{
    const uint64_t c = __umul64hi(x64, S.lo);
    U128 r;
    r.lo = x64 * S.hi;
    r.hi = __umul64hi(x64, S.hi);
    const uint64_t lo = r.lo + c;
    r.hi += lo < r.lo ? 1 : 0;
    r.lo = lo;
    return r;
}

__device__ __forceinline__ bool hash_has(const uint32_t* ehash, uint32_t base, uint32_t nb, uint32_t x)
{
    uint32_t b = (uint32_t)(((uint64_t)fmix32(x) * nb) >> 32);
    for (uint32_t tries = 0; tries < nb; ++tries) {
        const uint4* p = reinterpret_cast<const uint4*>(ehash + 8ull * (base + b));
        const uint4 a = __ldg(p), c = __ldg(p + 1);
        const bool f = a.x == x || a.y == x || a.z == x || a.w == x || c.x == x || c.y == x || c.z == x || c.w == x;
        if (f) return true;
        const bool e = a.x == kEmpty || a.y == kEmpty || a.z == kEmpty || a.w == kEmpty || c.x == kEmpty ||
                       c.y == kEmpty || c.z == kEmpty || c.w == kEmpty;
        if (e) return false;
        b = b + 1 == nb ? 0 : b + 1;
    }
    return false;
}

// Record fields of arc e: x, the prefix value hi (weighted) and the no-common-
// neighbour flag of the arc (bit "self").
template <bool WEIGHTED, bool COMPACT>
__device__ __forceinline__ void read_rec(const CdfParams& P, uint64_t e, uint32_t& x, uint32_t& hi, bool& nt)
{
    GRAPE_DCHECK(e < P.m_chk, "CDF sampler: arc record within the table");
    if constexpr (WEIGHTED && !COMPACT) {
        const uint4* r = reinterpret_cast<const uint4*>(P.rec) + 2 * e;
        const uint4 a = __ldg(r), b = __ldg(r + 1);
        x = a.x;
        hi = a.y;
        nt = ((b.y >> 29) & 1u) != 0;
    } else if constexpr (WEIGHTED) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(P.rec) + e);
        x = a.x & P.xmask;
        hi = a.y;
        nt = P.notri && (a.x >> 31) != 0;
    } else if constexpr (!COMPACT) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(P.rec) + e);
        x = a.x;
        hi = 0;
        nt = ((a.w >> 29) & 1u) != 0;
    } else {
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(P.rec) + e);
        x = a.x & P.xmask;
        hi = 0;
        nt = P.notri && (a.x >> 31) != 0;
    }
}

template <bool WEIGHTED, bool COMPACT>
__global__ void __launch_bounds__(256) walk_cdf_kernel(const __grid_constant__ CdfParams P)
{
    const int lane = threadIdx.x & 31;
    // per-warp chunk sums of the current row: {sum lo, sum hi, carry} x nchunks_max in global scratch
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint4* cs = P.chunk_scratch + gwarp * P.chunks_max;
    const uint32_t L = P.L;
    unsigned long long steps = 0;
    for (;;) {
        unsigned long long iw = 0;
        if (lane == 0) iw = atomicAdd(P.next, 1ull);
        iw = __shfl_sync(0xffffffffu, iw, 0);
        if (iw >= P.num_walks) break;
        const uint64_t wid = P.base + iw;
        uint32_t* row = P.out + iw * L;
        const uint32_t start = P.starts[iw];
        uint32_t s = 0;
        uint32_t buf = kPad;   // row entries s with s % 32 == lane, flushed every 32
        auto put = [&](uint32_t s_, uint32_t val) {
            if ((s_ & 31) == (uint32_t)lane) buf = val;
            if ((s_ & 31) == 31 || s_ + 1 == L) {   // flush entries [s_ & ~31, s_]
                const uint32_t b0 = s_ & ~31u;
                if ((uint32_t)lane <= (s_ & 31)) row[b0 + lane] = buf;
                buf = kPad;
            }
        };
        if (start < P.n) {
            put(0, start);
            s = 1;
            uint32_t t = kNone, tstart = 0, tdeg = 0, v = start;
            bool nt = false;   // no common neighbour of (t, v)
            for (; s < L; ++s) {
                const uint4 nr = __ldg(reinterpret_cast<const uint4*>(P.nodes) + v);
                const uint32_t vstart = nr.x, vdeg = nr.z;
                if (vdeg == 0) break;
                const Draw dr = philox_draw_rk(P.rk, wid, s, 0);
                const bool first = t == kNone;
                const uint32_t tb = first ? 0 : __umulhi(tstart, P.h_mul) >> P.h_shift;
                const uint32_t tnb = first ? 0 : (__umulhi(tdeg, P.h_mul) >> P.h_shift) + 1;
                // pi of arc e = vstart + k (all lanes; k < vdeg)
                auto pi_of = [&](uint32_t k, uint32_t& x, uint32_t& hi_carry, bool& xnt) -> uint64_t {
                    uint32_t hi = 0;
                    read_rec<WEIGHTED, COMPACT>(P, (uint64_t)vstart + k, x, hi, xnt);
                    uint64_t w = 1;
                    if constexpr (WEIGHTED) {
                        uint32_t prev = __shfl_up_sync(0xffffffffu, hi, 1);
                        if (lane == 0) prev = hi_carry;
                        if (k == 0) prev = 0;
                        w = hi - prev;
                        hi_carry = __shfl_sync(0xffffffffu, hi, 31);
                    }
                    uint64_t Tc = 1;
                    if (!first) {
                        if (x == t) Tc = P.T[0];
                        else if (nt) Tc = P.T[2];
                        else Tc = hash_has(P.ehash, tb + t, tnb, x) ? P.T[1] : P.T[2];
                    }
                    return w * Tc;
                };
                // pass 1: the total, and each 32-arc chunk's sum (and prefix carry) kept
                // in the warp's scratch
                U128 tot{0, 0};
                uint32_t carry = 0;
                for (uint32_t c0 = 0; c0 < vdeg; c0 += 32) {
                    const uint32_t k = c0 + lane;
                    uint32_t x = 0;
                    bool xnt = false;
                    uint64_t pi = 0;
                    const uint32_t carry_in = carry;
                    if (WEIGHTED || k < vdeg) {
                        // weighted: every lane takes part in the shuffles (out-of-row lanes read a
                        // valid record of the padded array and are masked below)
                        const uint32_t kk = k < vdeg ? k : vdeg - 1;
                        pi = pi_of(kk, x, carry, xnt);
                        if (k >= vdeg) pi = 0;
                    }
                    U128 a{pi, 0};
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        U128 b;
                        b.lo = __shfl_xor_sync(0xffffffffu, a.lo, o);
                        b.hi = __shfl_xor_sync(0xffffffffu, a.hi, o);
                        a = add128(a, b);
                    }
                    if (lane == 0)   // a chunk's sum < 2^69
                        cs[c0 >> 5] = make_uint4((uint32_t)a.lo, (uint32_t)(a.lo >> 32), (uint32_t)a.hi, carry_in);
                    tot = add128(tot, a);
                }
                const U128 r = bounded128(dr.x64, tot);
                __syncwarp();
                // pass 2: the first chunk whose running sum exceeds r (from the kept chunk
                // sums), then the running sum inside it
                U128 run{0, 0};
                uint32_t cfirst = 0;
                {
                    const uint32_t nch = (vdeg + 31) >> 5;
                    for (uint32_t b0 = 0; b0 < nch; b0 += 32) {
                        const uint32_t c = b0 + lane;
                        const uint4 e = c < nch ? cs[c] : make_uint4(0, 0, 0, 0);
                        U128 a{(uint64_t)e.y << 32 | e.x, (uint64_t)e.z};
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const U128 b = shfl_up128(a, o);
                            if (lane >= o) a = add128(a, b);
                        }
                        const U128 cum = add128(run, a);
                        const unsigned hit = __ballot_sync(0xffffffffu, c < nch && gt128(cum, r));
                        if (hit) {
                            const int src = __ffs(hit) - 1;
                            cfirst = b0 + src;
                            const U128 before = shfl128(a, src);   // inclusive sum up to chunk cfirst
                            const U128 mine{(uint64_t)e.y << 32 | e.x, (uint64_t)e.z};
                            const U128 own = shfl128(mine, src);
                            // run = (run + before) - own: the sum of the chunks before cfirst
                            U128 t2 = add128(run, before);
                            U128 negown;
                            negown.lo = ~own.lo + 1;
                            negown.hi = ~own.hi + (own.lo == 0 ? 1 : 0);
                            run = add128(t2, negown);
                            break;
                        }
                        run = add128(run, shfl128(a, 31));
                    }
                    carry = cs[cfirst].w;
                }
                __syncwarp();
                uint32_t xsel = 0;
                bool ntsel = false;
                for (uint32_t c0 = cfirst * 32; c0 < vdeg; c0 += 32) {
                    const uint32_t k = c0 + lane;
                    uint32_t x = 0;
                    bool xnt = false;
                    uint64_t pi = 0;
                    if (WEIGHTED || k < vdeg) {
                        const uint32_t kk = k < vdeg ? k : vdeg - 1;
                        pi = pi_of(kk, x, carry, xnt);
                        if (k >= vdeg) pi = 0;
                    }
                    U128 a{pi, 0};   // inclusive scan within the chunk
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const U128 b = shfl_up128(a, o);
                        if (lane >= o) a = add128(a, b);
                    }
                    const U128 cum = add128(run, a);
                    const unsigned hit = __ballot_sync(0xffffffffu, k < vdeg && gt128(cum, r));
                    if (hit) {
                        const int src = __ffs(hit) - 1;
                        xsel = __shfl_sync(0xffffffffu, x, src);
                        ntsel = __shfl_sync(0xffffffffu, xnt ? 1 : 0, src) != 0;
                        break;
                    }
                    run = add128(run, shfl128(a, 31));
                }
                put(s, xsel);
                ++steps;
                t = v;
                tstart = vstart;
                tdeg = vdeg;
                nt = ntsel;
                v = xsel;
            }
        }
        for (uint32_t q = s; q < L; ++q) put(q, kPad);
    }
    if (lane == 0 && steps && P.steps_out) atomicAdd(P.steps_out, steps);
}

template <bool WEIGHTED, bool COMPACT>
cudaError_t launch(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    CdfParams P{};
    P.nodes = g->nodes;
    P.rec = g->rec;
    P.m_chk = g->m;
    P.ehash = g->ehash;
    P.n = g->n;
    P.starts = a.starts;
    P.num_walks = a.num_walks;
    P.base = a.walk_id_base;
    P.L = a.L;
    P.rk = philox_round_keys(a.seed);
    P.out = a.out;
    P.steps_out = a.steps_out;
    P.T[0] = T.Tp;
    P.T[1] = T.T1;
    P.T[2] = T.Tq;
    if (g->hash_h == 6) { P.h_mul = 0xAAAAAAABu; P.h_shift = 2; }
    else { P.h_mul = 0x40000000u; P.h_shift = 0; }
    P.notri = g->notri;
    P.xmask = (g->notri && g->compact) ? 0x3FFFFFFFu : 0xFFFFFFFFu;
    const int resident = resident_blocks((const void*)walk_cdf_kernel<WEIGHTED, COMPACT>, 256, 0, g->device);
    uint64_t blocks = (a.num_walks * 32 + 255) / 256;
    if (blocks > (uint64_t)resident) blocks = resident;
    P.chunks_max = ((uint64_t)g->max_degree + 31) / 32 + 1;
    cudaError_t e = cudaMallocAsync((void**)&P.next, 8, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(P.next, 0, 8, stream);
    if (e == cudaSuccess)
        e = cudaMallocAsync((void**)&P.chunk_scratch, blocks * 8 * P.chunks_max * sizeof(uint4), stream);
    if (e == cudaSuccess) {
        walk_cdf_kernel<WEIGHTED, COMPACT><<<(unsigned)blocks, 256, 0, stream>>>(P);
        e = cudaGetLastError();
    }
    if (P.chunk_scratch) cudaFreeAsync(P.chunk_scratch, stream);
    cudaFreeAsync(P.next, stream);
    return e;
}

}  // namespace

cudaError_t launch_walks_cdf(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    const bool w = g->cw_bytes != 0;
    if (w && g->compact) return launch<true, true>(g, a, T, stream);
    if (w) return launch<true, false>(g, a, T, stream);
    if (g->compact) return launch<false, true>(g, a, T, stream);
    return launch<false, false>(g, a, T, stream);
}

}  // namespace grape
