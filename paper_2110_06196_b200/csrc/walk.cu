// walk.cu — first-order and node2vec walk kernels for sm_100a (no tensor cores:
// the path is a chain of dependent gathers, not a contraction).
//
// One thread owns one walk (wid = walk_id_base + i) and runs it to the end:
//   step s from v:  off[v], off[v+1]  -> deg, row start
//                   W_v = cw[end-1]   (weighted)
//   attempt a:      Philox(wid, s, a) -> x64, u                    (§8(c) c7)
//                   r = x64*W_v >> 64; i = upper_bound(cw row, r)
//                   x = col[off[v] + i]
//                   node2vec: class of x = p (x == t), 1 (x in N(t)), q (else)
//                    and accept iff u < T_class (§8(c) c9)
// Decision-identical shortcuts (§8(c) c12): x == t decided by a register
// compare; u < min(T_1,T_q) accepts and u >= max(T_1,T_q) rejects without the
// membership search; T_1 == T_q compiles the search out; on GRAPE_SYMMETRIC
// graphs "x in N(t)" is evaluated as "t in N(x)" when x's row is shorter.
// The node2vec path with p = q = 1 is dispatched to the first-order kernel
// (bit-identical by §8(c) c2).
#include <cstdint>
#include <type_traits>
#include "internal.h"
#include "philox.cuh"

namespace grape {
namespace {

constexpr uint32_t kPad = 0xFFFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kBlock = 256;

struct Unweighted {};

template <typename CW>
struct Csr {
    const uint64_t* __restrict__ off;
    const uint32_t* __restrict__ col;
    const CW* __restrict__ cw;
    uint32_t n;
};

// Smallest i in [0, d) with row[i] > r (row non-decreasing, row[d-1] > r).
template <typename CW>
__device__ __forceinline__ uint64_t upper_bound_row(const CW* __restrict__ row, uint64_t d, uint64_t r)
{
    uint64_t first = 0, len = d;
    while (len > 0) {
        const uint64_t half = len >> 1;
        if ((uint64_t)__ldg(row + first + half) <= r) {
            first += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return first;
}

// Is key in the sorted row col[lo, lo+d)?
__device__ __forceinline__ bool in_row(const uint32_t* __restrict__ col, uint64_t lo, uint64_t d, uint32_t key)
{
    uint64_t first = lo, len = d;
    while (len > 0) {
        const uint64_t half = len >> 1;
        if (__ldg(col + first + half) < key) {
            first += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return first < lo + d && __ldg(col + first) == key;
}

template <typename CW>
__device__ __forceinline__ uint32_t propose(const Csr<CW>& g, uint64_t lo, uint64_t d, uint64_t Wv, uint64_t x64)
{
    uint64_t i;
    if constexpr (std::is_same<CW, Unweighted>::value) {
        i = bounded64(x64, d);
    } else {
        const uint64_t r = bounded64(x64, Wv);
        i = upper_bound_row<CW>(g.cw + lo, d, r);
    }
    return __ldg(g.col + lo + i);
}

template <typename CW>
__device__ __forceinline__ uint64_t row_weight(const Csr<CW>& g, uint64_t lo, uint64_t d)
{
    if constexpr (std::is_same<CW, Unweighted>::value) return d;
    else return d ? (uint64_t)__ldg(g.cw + lo + d - 1) : 0;
}

__device__ __forceinline__ void add_steps(unsigned long long* steps_out, unsigned long long mine)
{
    if (steps_out == nullptr) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(steps_out, mine);
}

template <typename CW, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
__global__ void __launch_bounds__(kBlock)
walk_kernel(Csr<CW> g, const uint32_t* __restrict__ starts, uint64_t num_walks, uint64_t base,
            uint32_t L, uint32_t k0, uint32_t k1, uint32_t* __restrict__ out,
            unsigned long long* __restrict__ steps_out, uint64_t Tp, uint64_t T1, uint64_t Tq)
{
    const uint64_t Tlo = T1 < Tq ? T1 : Tq;
    const uint64_t Thi = T1 < Tq ? Tq : T1;
    const bool member_accepts = T1 > Tq;   // in [Tlo, Thi): accepted iff class has the larger T
    unsigned long long steps = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < num_walks; i += stride) {
        const uint64_t wid = base + i;
        uint32_t* __restrict__ row = out + i * (uint64_t)L;
        const uint32_t start = __ldg(starts + i);
        uint32_t s = 0;
        if (start < g.n) {
            row[0] = start;
            s = 1;
            uint32_t v = start, t = kNone;
            uint64_t ov = __ldg(g.off + v);
            uint64_t dv = __ldg(g.off + v + 1) - ov;
            uint64_t Wv = row_weight(g, ov, dv);
            uint64_t ot = 0, dt = 0;
            for (; s < L; ++s) {
                if (dv == 0) break;
                uint32_t x;
                if (!NODE2VEC || t == kNone) {
                    const Draw dr = philox_draw(k0, k1, wid, s, 0);
                    x = propose(g, ov, dv, Wv, dr.x64);
                } else {
                    for (uint32_t a = 0;; ++a) {
                        const Draw dr = philox_draw(k0, k1, wid, s, a);
                        x = propose(g, ov, dv, Wv, dr.x64);
                        const uint64_t u = dr.u;
                        if (x == t) {
                            if (u < Tp) break;
                            continue;
                        }
                        if constexpr (!NEED_MEMBER) {
                            if (u < T1) break;
                            continue;
                        } else {
                            if (u < Tlo) break;
                            if (u >= Thi) continue;
                            bool mem;
                            if constexpr (SYM) {
                                const uint64_t ox = __ldg(g.off + x);
                                const uint64_t dx = __ldg(g.off + x + 1) - ox;
                                mem = dx < dt ? in_row(g.col, ox, dx, t) : in_row(g.col, ot, dt, x);
                            } else {
                                mem = in_row(g.col, ot, dt, x);
                            }
                            if (mem == member_accepts) break;
                        }
                    }
                }
                row[s] = x;
                ++steps;
                t = v; ot = ov; dt = dv;
                v = x;
                ov = __ldg(g.off + v);
                dv = __ldg(g.off + v + 1) - ov;
                Wv = row_weight(g, ov, dv);
            }
        }
        for (; s < L; ++s) row[s] = kPad;
    }
    add_steps(steps_out, steps);
}

template <typename CW, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
cudaError_t launch_t(const grape_graph* gg, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    Csr<CW> g;
    g.off = gg->off;
    g.col = gg->col;
    g.cw = (const CW*)gg->cw;
    g.n = gg->n;
    uint64_t blocks = (a.num_walks + kBlock - 1) / kBlock;
    const uint64_t cap = 148ull * 8 * 64;   // grid-stride beyond this
    if (blocks > cap) blocks = cap;
    walk_kernel<CW, NODE2VEC, NEED_MEMBER, SYM><<<(unsigned)blocks, kBlock, 0, stream>>>(
        g, a.starts, a.num_walks, a.walk_id_base, a.L, (uint32_t)a.seed, (uint32_t)(a.seed >> 32),
        a.out, a.steps_out, T.Tp, T.T1, T.Tq);
    return cudaGetLastError();
}

template <typename CW>
cudaError_t dispatch_cw(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                        cudaStream_t stream)
{
    // Specialisation table ("eight specialized implementations"):
    //   weighted? x {p = q = 1 -> first order; T_1 == T_q -> no membership test;
    //   general} x {symmetric-membership trick}.  None changes a result.
    const bool all_equal = T.Tp == T.T1 && T.T1 == T.Tq;
    if (!node2vec || all_equal) return launch_t<CW, false, false, false>(g, a, T, stream);
    const bool need_member = T.T1 != T.Tq;
    if (!need_member) return launch_t<CW, true, false, false>(g, a, T, stream);
    if (g->flags & GRAPE_SYMMETRIC) return launch_t<CW, true, true, true>(g, a, T, stream);
    return launch_t<CW, true, true, false>(g, a, T, stream);
}

}  // namespace

cudaError_t launch_walks(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                         cudaStream_t stream)
{
    switch (g->cw_bytes) {
    case 0: return dispatch_cw<Unweighted>(g, a, node2vec, T, stream);
    case 4: return dispatch_cw<uint32_t>(g, a, node2vec, T, stream);
    default: return dispatch_cw<uint64_t>(g, a, node2vec, T, stream);
    }
}

}  // namespace grape
