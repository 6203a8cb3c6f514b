// walk.cu — first-order and node2vec walk kernels for sm_100a (no tensor cores:
// the path is a chain of dependent gathers, not a contraction).
//
// One thread owns one walk (wid = walk_id_base + i) and runs it to the end:
//   step s from v:  node record {start, deg, W_v}  (one 16-B load)
//   attempt a:      Philox(wid, s, a) -> x64, u                      (§8(c) c7)
//                   r = x64*W_v >> 64; i = first i with cw[i] > r
//                   x = col[start + i]
//                   node2vec: class of x = p (x == t), 1 (x in N(t)), q (else)
//                   (P:453-495); accept iff u < T_class               (§8(c) c9)
// Searches ("first i in a sorted row with A[i] >= key") use the fence levels
// built with the graph: a short binary search on the top fence level, then one
// aligned 32-B sector per level down to the answer.  They return
// exactly the index a plain binary search returns (§8(c) c11).
// Decision-identical shortcuts (§8(c) c12): x == t by a register compare;
// u < min(T_1,T_q) accepts and u >= max(T_1,T_q) rejects without the membership
// search; T_1 == T_q compiles the search out; on GRAPE_SYMMETRIC graphs
// "x in N(t)" is evaluated as "t in N(x)" when x's row is shorter.  The node2vec
// path with p = q = 1 is dispatched to the first-order kernel (bit-identical by
// §8(c) c2).
// Output: each thread stages its row in shared memory and writes every full,
// aligned 32-B sector of the walk matrix with two 16-B streaming stores.
// Index width: arc indices are u32 when m < 2^32 (IDX template), halving the
// registers of the search state.
#include "walk_common.cuh"

namespace grape {
namespace {
using namespace walk;

// First index i in [lo, hi) (lo < hi) with A[i] >= key, A sorted on [lo, hi); hi if
// none.  eq: whether A[i] == key.  Level l+1 candidates are the blocks
// [s_l / B, (e_l - 1) / B) of level l (the last block is the default answer).
// Reads: a binary search over the top level's slice (only when the row spans
// more than B^NL entries), then one aligned sector per level.
template <typename T, typename IDX>
__device__ __forceinline__ IDX lower_bound_fenced(const Levels<T>& lv, IDX lo, IDX hi, T key, bool& eq)
{
    constexpr IDX B = 32 / sizeof(T);
    IDX s[NL + 1], e[NL + 1];
    s[0] = lo;
    e[0] = hi;
    int top = 0;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        if (top == l && s[l] / B != (e[l] - 1) / B) {
            s[l + 1] = s[l] / B;
            e[l + 1] = (e[l] - 1) / B;
            top = l + 1;
        }
    }
    IDX k = 0;
    eq = false;
    if (top == NL) {   // plain binary search over the top level's slice
        IDX first = s[NL], len = e[NL] - s[NL];
        const T* __restrict__ f = lv.a[NL];
        while (len > 0) {
            const IDX half = len >> 1;
            if (ld_elem<T, kHot>(f + first + half) < key) {
                first += half + 1;
                len -= half + 1;
            } else {
                len = half;
            }
        }
        k = first;
    }
#pragma unroll
    for (int l = NL - 1; l >= 0; --l) {
        if (l <= top) {
            // l < top: the answer lies in block k of level l; l == top: in block s_l / B.
            const IDX blk = l < top ? k : s[l] / B;
            const IDX a = s[l] > blk * B ? s[l] : blk * B;
            const IDX b = e[l] < blk * B + B ? e[l] : blk * B + B;
            bool q;
            if (l == 0) {
                k = a + block_count_lt<T, IDX, kLeaf>(lv.a[l], blk, a, b, key, q);
                eq = q;
            } else {
                k = a + block_count_lt<T, IDX, kHot>(lv.a[l], blk, a, b, key, q);
            }
        }
    }
    return k;
}

template <typename CW, typename IDX>
__device__ __forceinline__ uint64_t row_weight(const Params<CW>& P, IDX start, uint32_t deg, uint32_t w32)
{
    if constexpr (std::is_same<CW, uint64_t>::value)
        return deg ? ld_u64<kLeaf>(P.cw.a[0] + start + deg - 1) : 0;
    else
        return w32;
}

template <typename CW, typename IDX>
__device__ __forceinline__ uint32_t propose(const Params<CW>& P, IDX lo, uint32_t d, uint64_t Wv, uint64_t x64)
{
    IDX i;
    if constexpr (std::is_same<CW, Unweighted>::value) {
        i = lo + (IDX)bounded64(x64, d);
    } else {
        const uint64_t r = bounded64(x64, Wv);   // r < W_v, so r + 1 fits CW
        bool eq;
        i = lower_bound_fenced<CW, IDX>(P.cw, lo, (IDX)(lo + d), (CW)(r + 1), eq);
    }
    return ld_u32<kLeaf>(P.col.a[0] + i);
}

template <typename IDX>
__device__ __forceinline__ bool in_row(const Levels<uint32_t>& col, IDX lo, uint32_t d, uint32_t key)
{
    bool eq;
    lower_bound_fenced<uint32_t, IDX>(col, lo, (IDX)(lo + d), key, eq);
    return eq;
}

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
__global__ void __launch_bounds__(kBlock, kMinBlocks) walk_kernel(const __grid_constant__ Params<CW> P)
{
    __shared__ uint32_t stage[8 * kBlock];
    unsigned long long steps = 0;
    RowWriter w;
    w.slot = stage + threadIdx.x;
    const uint32_t L = P.L;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.num_walks; i += stride) {
        const uint64_t wid = P.base + i;
        w.begin(P.out + i * L);
        const uint32_t start = __ldg(P.starts + i);
        uint32_t s = 0;
        if (start < P.n) {
            w.put(0, start);
            s = 1;
            uint32_t v = start, t = kNone;
            Node<IDX> rv = load_node<IDX>(P.nodes, v);
            uint64_t Wv = row_weight<CW, IDX>(P, rv.start, rv.deg, rv.w32);
            IDX ot = 0;
            uint32_t dt = 0;
            for (; s < L; ++s) {
                if (rv.deg == 0) break;
                uint32_t x;
                if (!NODE2VEC || t == kNone) {
                    const Draw dr = philox_draw(P.k0, P.k1, wid, s, 0);
                    x = propose<CW, IDX>(P, rv.start, rv.deg, Wv, dr.x64);
                } else {
                    for (uint32_t a = 0;; ++a) {
                        const Draw dr = philox_draw(P.k0, P.k1, wid, s, a);
                        x = propose<CW, IDX>(P, rv.start, rv.deg, Wv, dr.x64);
                        const uint32_t u = dr.u;
                        if (x == t) {
                            if (u <= P.tp_m1) break;
                            continue;
                        }
                        if constexpr (!NEED_MEMBER) {
                            if (u <= P.t1_m1) break;
                            continue;
                        } else {
                            if (u <= P.lo_m1) break;
                            if (u > P.hi_m1) continue;
                            bool mem;
                            if constexpr (SYM) {
                                const Node<IDX> rx = load_node<IDX>(P.nodes, x);
                                mem = rx.deg < dt ? in_row<IDX>(P.col, rx.start, rx.deg, t)
                                                  : in_row<IDX>(P.col, ot, dt, x);
                            } else {
                                mem = in_row<IDX>(P.col, ot, dt, x);
                            }
                            if (mem == P.member_accepts) break;
                        }
                    }
                }
                w.put(s, x);
                ++steps;
                t = v; ot = rv.start; dt = rv.deg;
                v = x;
                rv = load_node<IDX>(P.nodes, v);
                Wv = row_weight<CW, IDX>(P, rv.start, rv.deg, rv.w32);
            }
        }
        for (; s < L; ++s) w.put(s, kPad);
        w.finish(L);
    }
    add_steps(P.steps_out, steps);
}

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
cudaError_t launch_t(const grape_graph* gg, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    const Params<CW> P = make_params<CW>(gg, a, T);
    uint64_t blocks = (a.num_walks + kBlock - 1) / kBlock;
    const uint64_t cap = 148ull * 8 * 64;   // grid-stride beyond this
    if (blocks > cap) blocks = cap;
    walk_kernel<CW, IDX, NODE2VEC, NEED_MEMBER, SYM><<<(unsigned)blocks, kBlock, 0, stream>>>(P);
    return cudaGetLastError();
}

template <typename CW, typename IDX>
cudaError_t dispatch(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                     cudaStream_t stream)
{
    // Specialisation table ("eight specialized implementations"):
    //   weighted? x {p = q = 1 -> first order; T_1 == T_q -> no membership test;
    //   general} x {symmetric-membership trick}.  None changes a result.
    const bool all_equal = T.Tp == T.T1 && T.T1 == T.Tq;
    if (!node2vec || all_equal) return launch_t<CW, IDX, false, false, false>(g, a, T, stream);
    const bool need_member = T.T1 != T.Tq;
    if (!need_member) return launch_t<CW, IDX, true, false, false>(g, a, T, stream);
    if (g->flags & GRAPE_SYMMETRIC) return launch_t<CW, IDX, true, true, true>(g, a, T, stream);
    return launch_t<CW, IDX, true, true, false>(g, a, T, stream);
}

template <typename CW>
cudaError_t dispatch_idx(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                         cudaStream_t stream)
{
    if (g->m < (1ull << 32) - 64) return dispatch<CW, uint32_t>(g, a, node2vec, T, stream);
    return dispatch<CW, uint64_t>(g, a, node2vec, T, stream);
}

}  // namespace

cudaError_t launch_walks_structured(const grape_graph* g, const WalkArgs& a, bool node2vec,
                                    const Thresholds& T, cudaStream_t stream)
{
    switch (g->cw_bytes) {
    case 0: return dispatch_idx<Unweighted>(g, a, node2vec, T, stream);
    case 4: return dispatch_idx<uint32_t>(g, a, node2vec, T, stream);
    default: return dispatch_idx<uint64_t>(g, a, node2vec, T, stream);
    }
}

#ifndef GRAPE_WALKER
#define GRAPE_WALKER 3
#endif

// The walker used by the C-ABI: the v4 table walker (walk_tab.cu) when the
// graph has its sampling tables; otherwise 3 = convergent state machine over
// fenced searches (walk_sm.cu), 2 = structured thread-per-walk kernel (this
// file).  All produce identical walks.
cudaError_t launch_walks(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                         cudaStream_t stream)
{
    if (a.sampler == 1) return launch_walks_cdf(g, a, T, stream);
    if (g->tables) return launch_walks_tab(g, a, node2vec, T, stream);
    if (GRAPE_WALKER == 2) return launch_walks_structured(g, a, node2vec, T, stream);
    return launch_walks_sm(g, a, node2vec, T, stream);
}

}  // namespace grape
