// walk_sm.cu — convergent state-machine walkers ("v3").
//
// Same rules, same results as the structured kernels (include/grape_walk.h),
// organised for SIMT: every lane owns one walk, and every iteration of the
// kernel's single loop issues exactly ONE aligned 32-byte sector load per lane
// from one instruction (LDG.E.ENL2.256), whatever phase the lane is in:
//   ST_START  starts[i]                 -> begin walk i
//   ST_NODE   node record of v          -> {start, deg, W_v}
//   ST_WV     cw[end-1] of v (u64 rows) -> W_v
//   ST_SEARCH one probe of a fenced search (top-level bisection or a level scan)
//   ST_COL    col[i]                    -> proposal x
//   ST_XNODE  node record of x          -> shorter row for "x in N(t)" (§8(c) c12)
// followed by ALU-only bookkeeping (Philox, bounded draws, the accept test of
// P:453-495 with the integer thresholds of §8(c) c9, the staged row writer).
// A thread-per-walk kernel whose lanes sit in different phases executes their
// dependent load chains one after another; here the 32 lanes' loads are always
// in flight together, so a warp keeps up to 32 independent sectors outstanding.
#include "walk_common.cuh"

namespace grape {
namespace {
using namespace walk;

enum : uint32_t { ST_START = 0, ST_NODE, ST_WV, ST_SEARCH, ST_COL, ST_XNODE, ST_DONE };

__device__ __forceinline__ uint32_t pick8(const uint32_t (&w)[8], uint32_t j)
{
    const uint32_t a0 = (j & 1) ? w[1] : w[0], a1 = (j & 1) ? w[3] : w[2];
    const uint32_t a2 = (j & 1) ? w[5] : w[4], a3 = (j & 1) ? w[7] : w[6];
    const uint32_t b0 = (j & 2) ? a1 : a0, b1 = (j & 2) ? a3 : a2;
    return (j & 4) ? b1 : b0;
}

__device__ __forceinline__ const uint32_t* sector_of(const void* p)
{
    return reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(31));
}
__device__ __forceinline__ uint32_t word_of(const void* p)
{
    return (uint32_t)((reinterpret_cast<uintptr_t>(p) >> 2) & 7);
}

__device__ __forceinline__ void ld8(const uint32_t* p, uint32_t (&v)[8])
{
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}

// Lane-private count of the in-range entries of a u32 sector below key, and
// whether one equals key (branch-free; ja < jb <= 8).
__device__ __forceinline__ uint32_t sector_count_lt(const uint32_t (&w)[8], int ja, int jb, uint32_t key)
{
    uint32_t lt = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) lt |= (w[q] < key ? 1u : 0u) << q;
    const uint32_t in = (0xFFu >> (8 - jb)) & (0xFFu << ja);
    return __popc(lt & in);
}

__device__ __forceinline__ uint32_t sector_count_lt64(const uint32_t (&w)[8], int ja, int jb, uint64_t key, bool& eq)
{
    uint32_t lt = 0, ge = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint64_t val = ((uint64_t)w[2 * q + 1] << 32) | w[2 * q];
        lt |= (val < key ? 1u : 0u) << q;
        ge |= (val == key ? 1u : 0u) << q;
    }
    const uint32_t in = (0xFu >> (4 - jb)) & (0xFu << ja);
    eq = (ge & in) != 0;
    return __popc(lt & in);
}

// STATS: count every event of the walk (grape_walks_stats; diagnostics build of
// the same kernel — the timed path is compiled with STATS = false).
enum : int { C_LOADS = 0, C_NODE, C_XNODE, C_CWPROBE, C_COLPROBE, C_COL, C_ATTEMPT, C_MEMB, C_START, C_STEPS };

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM, bool STATS>
__global__ void __launch_bounds__(kBlock, kMinBlocks) walk_sm_kernel(const __grid_constant__ Params<CW> P)
{
    uint32_t cnt[kStatsWords];
    if (STATS) {
#pragma unroll
        for (int q = 0; q < kStatsWords; ++q) cnt[q] = 0;
    }
    constexpr bool WEIGHTED = !std::is_same<CW, Unweighted>::value;
    constexpr bool CW64 = WEIGHTED && sizeof(CwStore<CW>) == 8;
    using KeyT = CwStore<CW>;
    __shared__ uint32_t stage[8 * kBlock];
    RowWriter w;
    w.slot = stage + threadIdx.x;
    const uint32_t L = P.L;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t st = i < P.num_walks ? ST_START : ST_DONE;
    const void* nxt = P.starts + (i < P.num_walks ? i : 0);   // the address the next iteration loads
    unsigned long long steps = 0;

    uint32_t s = 0, a = 0, v = 0, t = kNone, x = 0, u = 0;
    IDX vstart = 0, tstart = 0;
    uint32_t vdeg = 0, tdeg = 0;
    uint64_t vW = 0;
    KeyT key = 0;          // search key (cw: r + 1; col: x or t)
    uint32_t sarr = 0;     // search array: 0 = cw, 1 = col
    IDX slo = 0, shi = 0, sfirst = 0, slast = 0;
    uint32_t slvl = 0;

    for (;;) {
        const bool active = st != ST_DONE;
        if (!__any_sync(0xffffffffu, active)) break;
        __syncwarp();
        uint32_t sec[8];
        if (active) ld8(sector_of(nxt), sec);
        const uint32_t j = word_of(nxt);
        if (STATS && active) {
            ++cnt[C_LOADS];
            cnt[C_NODE] += st == ST_NODE || st == ST_WV;
            cnt[C_XNODE] += st == ST_XNODE;
            cnt[C_CWPROBE] += st == ST_SEARCH && sarr == 0;
            cnt[C_COLPROBE] += st == ST_SEARCH && sarr == 1;
            cnt[C_COL] += st == ST_COL;
            cnt[C_START] += st == ST_START;
        }

        // ---- per-state extraction; sets at most one action
        bool emit = false, draw = false, fin = false, sinit = false;
        IDX ilo = 0, ihi = 0;
        if (st == ST_SEARCH) {
            const uint32_t lb = (CW64 && sarr == 0) ? 2 : 3;
            const IDX B = IDX(1) << lb;
            const IDX mid = sfirst + ((slast - sfirst) >> 1);
            const IDX sb = mid & ~(B - 1);
            const IDX lo_ = sfirst > sb ? sfirst : sb;
            const IDX hi_ = slast < sb + B ? slast : sb + B;
            bool eq = false;
            uint32_t c;
            if (CW64 && sarr == 0) {
                c = sector_count_lt64(sec, (int)(lo_ - sb), (int)(hi_ - sb), (uint64_t)key, eq);
            } else {
                c = sector_count_lt(sec, (int)(lo_ - sb), (int)(hi_ - sb), (uint32_t)key);
                // membership answer: the first entry >= key, if inside this sector, equals key?
                if (sarr && c < (uint32_t)(hi_ - lo_)) eq = pick8(sec, (uint32_t)(lo_ - sb) + c) == (uint32_t)key;
            }
            bool found = false;
            IDX ans = 0;
            if (c == (uint32_t)(hi_ - lo_)) {        // every candidate here is < key
                sfirst = hi_;
                found = sfirst == slast;
                ans = slast;
                eq = false;
            } else if (c == 0 && lo_ > sfirst) {      // the answer is at or before lo_
                slast = lo_;
                found = sfirst == slast;
                ans = lo_;
                eq = false;
            } else {
                ans = lo_ + c;
                found = true;
            }
            if (found) {
                if (slvl == 0) {
                    if (sarr == 0) {
                        st = ST_COL;                  // proposal index -> col
                        nxt = P.col.a[0] + ans;
                    } else {
                        emit = eq == P.member_accepts;   // u in [T_lo, T_hi): the class decides
                        draw = !emit;
                    }
                } else {                              // descend into block `ans` of level slvl - 1
                    --slvl;
                    const IDX sl = slo >> (lb * slvl);
                    IDX el = shi;
#pragma unroll
                    for (uint32_t q = 0; q < (uint32_t)NL; ++q)
                        if (q < slvl) el = (el - 1) >> lb;
                    sfirst = sl > ans * B ? sl : ans * B;
                    slast = el < ans * B + B ? el : ans * B + B;
                }
            }
        } else if (st == ST_COL) {
            x = pick8(sec, j);
            bool memb = false;
            if (!NODE2VEC || t == kNone) emit = true;
            else if (x == t) emit = u <= P.tp_m1;
            else if (!NEED_MEMBER) emit = u <= P.t1_m1;
            else if (u <= P.lo_m1) emit = true;
            else if (u > P.hi_m1) emit = false;
            else memb = true;
            draw = !emit && !memb;
            if (memb) {
                if (SYM) {
                    st = ST_XNODE;
                    nxt = P.nodes + x;
                } else {
                    sinit = true; sarr = 1; key = (KeyT)x; ilo = tstart; ihi = tstart + tdeg;
                }
            }
        } else if (st == ST_NODE || st == ST_XNODE) {
            const bool hi4 = (j & 4) != 0;
            const uint32_t w0 = hi4 ? sec[4] : sec[0], w1 = hi4 ? sec[5] : sec[1];
            const uint32_t deg = hi4 ? sec[6] : sec[2];
            const uint32_t w32 = hi4 ? sec[7] : sec[3];
            IDX start;
            if constexpr (sizeof(IDX) == 8) start = ((uint64_t)w1 << 32) | w0;
            else start = w0;
            (void)w1;
            if (st == ST_NODE) {
                vstart = start;
                vdeg = deg;
                vW = w32;
                a = 0;
                if (deg == 0) {
                    fin = true;
                } else if (CW64) {
                    st = ST_WV;
                    nxt = P.cw.a[0] + (start + deg - 1);
                } else {
                    draw = true;
                }
            } else {   // GRAPE_SYMMETRIC: search the shorter row, t in N(x) or x in N(t)
                sinit = true;
                sarr = 1;
                if (deg < tdeg) { key = (KeyT)t; ilo = start; ihi = start + deg; }
                else { key = (KeyT)x; ilo = tstart; ihi = tstart + tdeg; }
            }
        } else if (st == ST_WV) {
            const uint32_t jj = j & 6;   // u64 entry: words jj, jj+1
            vW = ((uint64_t)pick8(sec, jj + 1) << 32) | pick8(sec, jj);
            draw = true;
        } else if (st == ST_START) {
            const uint32_t start = pick8(sec, j);
            w.begin(P.out + i * L);
            s = 0;
            t = kNone;
            if (start < P.n) {
                x = start;
                emit = true;   // row[0] = start, then its node record
            } else {
                fin = true;
            }
        }

        // ---- consolidated actions (one call site each), entered by the whole warp at
        // once so that each block is issued once per iteration, not once per lane group
        __syncwarp();
        if (emit) {
            w.put(s, x);
            if (s > 0) {
                ++steps;
                t = v; tstart = vstart; tdeg = vdeg;
            }
            v = x;
            ++s;
            if (s == L) {
                fin = true;
            } else {
                st = ST_NODE;
                nxt = P.nodes + x;
            }
        }
        if (fin) {
            w.pad(s, L);
            w.finish(L);
            i += stride;
            st = i < P.num_walks ? ST_START : ST_DONE;
            nxt = P.starts + (i < P.num_walks ? i : 0);
        }
        __syncwarp();
        if (STATS) {
            cnt[C_ATTEMPT] += draw;
            cnt[C_MEMB] += sinit && sarr == 1;
        }
        if (draw) {
            if (st != ST_NODE && st != ST_WV) ++a;   // a rejected attempt; a new step starts at 0
            const Draw dr = philox_draw_rk(P.rk, P.base + i, s, a);
            u = dr.u;
            if constexpr (WEIGHTED) {
                sinit = true; sarr = 0; key = (KeyT)(bounded64(dr.x64, vW) + 1);   // first cw >= r+1
                ilo = vstart; ihi = vstart + vdeg;
            } else {
                st = ST_COL;
                nxt = P.col.a[0] + (vstart + (IDX)bounded64(dr.x64, vdeg));
            }
        }
        __syncwarp();
        if (sinit) {   // highest level whose range spans > 1 block; its range and first probe
            const uint32_t lb = (CW64 && sarr == 0) ? 2 : 3;
            slo = ilo; shi = ihi;
            IDX sv = ilo, ev = ihi;
            uint32_t l = 0;
#pragma unroll
            for (int q = 0; q < NL; ++q) {
                if (l == (uint32_t)q && (sv >> lb) != ((ev - 1) >> lb)) {
                    sv >>= lb;
                    ev = (ev - 1) >> lb;
                    l = q + 1;
                }
            }
            slvl = l; sfirst = sv; slast = ev;
            st = ST_SEARCH;
        }
        if (st == ST_SEARCH) {   // next probe address
            const IDX mid = sfirst + ((slast - sfirst) >> 1);
            if (sarr) nxt = P.col.a[slvl] + mid;
            else nxt = P.cw.a[slvl] + mid;
        }
    }
    add_steps(P.steps_out, steps);
    if (STATS) {
        cnt[C_STEPS] = (uint32_t)steps;
#pragma unroll
        for (int q = 0; q < kStatsWords; ++q) {
            unsigned long long c = cnt[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if ((threadIdx.x & 31) == 0) atomicAdd(P.stats + q, c);
        }
    }
}

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM, bool STATS>
cudaError_t launch_sm_k(const grape_graph* gg, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    const Params<CW> P = make_params<CW>(gg, a, T);
    // blocks per SM x SMs of the graph's device (cached per kernel and device)
    const int resident = resident_blocks((const void*)walk_sm_kernel<CW, IDX, NODE2VEC, NEED_MEMBER, SYM, STATS>,
                                         kBlock, 0, gg->device);
    uint64_t blocks = (a.num_walks + kBlock - 1) / kBlock;
    if (blocks > (uint64_t)resident) blocks = resident;   // persistent: lanes loop over walks
    walk_sm_kernel<CW, IDX, NODE2VEC, NEED_MEMBER, SYM, STATS><<<(unsigned)blocks, kBlock, 0, stream>>>(P);
    return cudaGetLastError();
}

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
cudaError_t launch_sm(const grape_graph* gg, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    if (a.stats != nullptr) return launch_sm_k<CW, IDX, NODE2VEC, NEED_MEMBER, SYM, true>(gg, a, T, stream);
    return launch_sm_k<CW, IDX, NODE2VEC, NEED_MEMBER, SYM, false>(gg, a, T, stream);
}

template <typename CW, typename IDX>
cudaError_t dispatch(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                     cudaStream_t stream)
{
    const bool all_equal = T.Tp == T.T1 && T.T1 == T.Tq;
    if (!node2vec || all_equal) return launch_sm<CW, IDX, false, false, false>(g, a, T, stream);
    const bool need_member = T.T1 != T.Tq;
    if (!need_member) return launch_sm<CW, IDX, true, false, false>(g, a, T, stream);
    if (g->flags & GRAPE_SYMMETRIC) return launch_sm<CW, IDX, true, true, true>(g, a, T, stream);
    return launch_sm<CW, IDX, true, true, false>(g, a, T, stream);
}

template <typename CW>
cudaError_t dispatch_idx(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                         cudaStream_t stream)
{
    if (g->m < (1ull << 32) - 64) return dispatch<CW, uint32_t>(g, a, node2vec, T, stream);
    return dispatch<CW, uint64_t>(g, a, node2vec, T, stream);
}

}  // namespace

cudaError_t launch_walks_sm(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                            cudaStream_t stream)
{
    switch (g->cw_bytes) {
    case 0: return dispatch_idx<Unweighted>(g, a, node2vec, T, stream);
    case 4: return dispatch_idx<uint32_t>(g, a, node2vec, T, stream);
    default: return dispatch_idx<uint64_t>(g, a, node2vec, T, stream);
    }
}

}  // namespace grape
