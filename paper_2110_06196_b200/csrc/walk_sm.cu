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

// Search over a fenced sorted row (walk_common.cuh Levels): "first i in [lo, hi)
// with A[i] >= key".  State: the level being probed and the candidate range
// [first, last] at that level (last = the default answer).  A probe loads the
// sector holding the range's midpoint and either finds the answer inside it or
// discards it; at levels below the top the range is one block, so one probe.
template <typename IDX>
struct Search {
    IDX lo, hi;          // the row at level 0
    IDX first, last;     // candidate range at level lvl
    uint32_t lvl;
    uint32_t is_col;     // 0: cw row (key = r + 1); 1: col row of t (key = x); 2: col row of x (key = t)
};

template <int LB, typename IDX>
__device__ __forceinline__ IDX e_at(IDX hi, uint32_t l)
{
    IDX e = hi;
#pragma unroll
    for (uint32_t j = 0; j < (uint32_t)NL; ++j)
        if (j < l) e = (e - 1) >> LB;
    return e;
}

// Highest level whose candidate range still spans more than one block, and its range.
template <int LB, typename IDX>
__device__ __forceinline__ void search_init(Search<IDX>& S, IDX lo, IDX hi, uint32_t is_col)
{
    S.lo = lo;
    S.hi = hi;
    S.is_col = is_col;
    IDX s = lo, e = hi;
    uint32_t l = 0;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        if (l == (uint32_t)j && (s >> LB) != ((e - 1) >> LB)) {
            s >>= LB;
            e = (e - 1) >> LB;
            l = j + 1;
        }
    }
    S.lvl = l;
    S.first = s;
    S.last = e;
}

template <typename IDX>
__device__ __forceinline__ IDX search_mid(const Search<IDX>& S)
{
    return S.first + ((S.last - S.first) >> 1);
}

// One probe with the sector w (entries of width 4 or 8 bytes, B = 8 or 4 per
// sector).  Returns true when the search is complete (k = answer at level 0,
// eq = A[k] == key).
template <typename T, int LB, typename IDX>
__device__ __forceinline__ bool search_step(Search<IDX>& S, const uint32_t (&w)[8], T key, IDX& k, bool& eq)
{
    constexpr IDX B = IDX(1) << LB;
    const IDX mid = search_mid(S);
    const IDX sb = mid & ~(B - 1);
    const IDX a = S.first > sb ? S.first : sb;
    const IDX b = S.last < sb + B ? S.last : sb + B;
    const int ja = (int)(a - sb), jb = (int)(b - sb);
    uint32_t c = 0;
    bool e = false;
#pragma unroll
    for (int j = 0; j < (int)B; ++j) {
        T val;
        if constexpr (sizeof(T) == 4) val = w[j];
        else val = ((uint64_t)w[2 * j + 1] << 32) | w[2 * j];
        const bool in = j >= ja && j < jb;
        c += (in && val < key) ? 1u : 0u;
        e |= in && val == key;
    }
    bool found = false;
    IDX ans = 0;
    if (c == (uint32_t)(b - a)) {
        S.first = b;                       // every candidate here is < key
        if (S.first == S.last) { ans = S.last; found = true; e = false; }
    } else if (c == 0 && a > S.first) {
        S.last = a;                        // answer is at or before a
        if (S.first == S.last) { ans = a; found = true; }
        e = false;
    } else {
        ans = a + c;                       // first entry >= key is in this sector
        found = true;
    }
    if (!found) return false;
    if (S.lvl == 0) {
        k = ans;
        eq = e;
        return true;
    }
    // descend: the answer lies in block `ans` of the level below
    const uint32_t l = S.lvl - 1;
    const IDX sl = S.lo >> (LB * l);
    const IDX el = e_at<LB, IDX>(S.hi, l);
    S.lvl = l;
    S.first = sl > ans * B ? sl : ans * B;
    S.last = el < ans * B + B ? el : ans * B + B;
    return false;
}

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
__global__ void __launch_bounds__(kBlock, kMinBlocks) walk_sm_kernel(const __grid_constant__ Params<CW> P)
{
    constexpr bool WEIGHTED = !std::is_same<CW, Unweighted>::value;
    constexpr int CLB = sizeof(CwStore<CW>) == 8 ? 2 : 3;   // log2 entries per sector of cw
    using KeyT = CwStore<CW>;
    __shared__ uint32_t stage[8 * kBlock];
    RowWriter w;
    w.slot = stage + threadIdx.x;
    const uint32_t L = P.L;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t st = i < P.num_walks ? ST_START : ST_DONE;
    unsigned long long steps = 0;

    uint32_t s = 0, a = 0, v = 0, t = kNone, x = 0, u = 0;
    IDX vstart = 0, tstart = 0, ci = 0;
    uint32_t vdeg = 0, tdeg = 0;
    uint64_t vW = 0;
    KeyT key = 0;
    Search<IDX> S{};

    for (;;) {
        const bool active = st != ST_DONE;
        if (!__any_sync(0xffffffffu, active)) break;
        // ---- 1. the one address this lane needs
        const void* ea = P.starts;
        if (st == ST_START) ea = P.starts + i;
        else if (st == ST_NODE) ea = P.nodes + v;
        else if (st == ST_XNODE) ea = P.nodes + x;
        else if (st == ST_COL) ea = P.col.a[0] + ci;
        else if (st == ST_WV) ea = P.cw.a[0] + (vstart + vdeg - 1);
        else if (st == ST_SEARCH) {
            const IDX mid = search_mid(S);
            if (S.is_col) ea = P.col.a[S.lvl] + mid;
            else ea = P.cw.a[S.lvl] + mid;
        }
        // ---- 2. one sector load for every active lane, issued by the whole warp
        // together (independent thread scheduling would otherwise let divergent
        // lane groups issue it one group at a time)
        __syncwarp();
        uint32_t sec[8];
        if (active) ld8(sector_of(ea), sec);
        const uint32_t j = word_of(ea);
        // ---- 3. per-state extraction -> at most one action per lane
        // actions: emit (accept x), draw (new attempt), fin (end of walk), memb (start membership search)
        bool emit = false, draw = false, fin = false, memb = false;
        if (st == ST_SEARCH) {
            IDX k = 0;
            bool eq = false, done = false;
            if (S.is_col) {
                done = search_step<uint32_t, 3, IDX>(S, sec, S.is_col == 1 ? x : t, k, eq);
            } else if constexpr (WEIGHTED) {
                done = search_step<KeyT, CLB, IDX>(S, sec, key, k, eq);
            }
            if (done) {
                if (S.is_col) {
                    emit = eq == P.member_accepts;   // u in [T_lo, T_hi): the class decides
                    draw = !emit;
                } else {
                    ci = k;
                    st = ST_COL;
                }
            }
        } else if (st == ST_COL) {
            x = pick8(sec, j);
            if (!NODE2VEC || t == kNone) emit = true;
            else if (x == t) emit = u <= P.tp_m1;
            else if (!NEED_MEMBER) emit = u <= P.t1_m1;
            else if (u <= P.lo_m1) emit = true;
            else if (u > P.hi_m1) emit = false;
            else memb = true;
            draw = !emit && !memb;
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
                if (deg == 0) fin = true;
                else if (sizeof(KeyT) == 8 && WEIGHTED) st = ST_WV;
                else draw = true;
            } else {   // membership on the shorter row (GRAPE_SYMMETRIC): t in N(x) or x in N(t)
                if (deg < tdeg) search_init<3, IDX>(S, start, start + deg, 2);
                else search_init<3, IDX>(S, tstart, tstart + tdeg, 1);
                st = ST_SEARCH;
            }
        } else if (st == ST_WV) {
            const uint32_t jj = j & 6;   // u64 entry: words jj, jj+1
            vW = ((uint64_t)pick8(sec, jj + 1) << 32) | pick8(sec, jj);
            draw = true;
        } else if (st == ST_START) {
            const uint32_t start = pick8(sec, j);
            w.begin(P.out + i * L);
            s = 0;
            if (start < P.n) {
                x = start;
                v = kNone;
                t = kNone;
                emit = true;   // row[0] = start, then load its node record
            } else {
                fin = true;
            }
        }
        // ---- 4. consolidated actions (each executed once per iteration)
        if (memb) {
            if (SYM) {
                st = ST_XNODE;
            } else {
                search_init<3, IDX>(S, tstart, tstart + tdeg, 1);
                st = ST_SEARCH;
            }
        }
        if (emit) {
            w.put(s, x);
            if (s > 0) {
                ++steps;
                t = v; tstart = vstart; tdeg = vdeg;
            }
            v = x;
            ++s;
            if (s == L) fin = true;
            else st = ST_NODE;
        }
        if (fin) {
            for (uint32_t q = s; q < L; ++q) w.put(q, kPad);
            w.finish(L);
            i += stride;
            st = i < P.num_walks ? ST_START : ST_DONE;
        }
        if (draw) {
            if (st != ST_NODE && st != ST_WV) ++a;   // rejected attempt (a new step starts at a = 0)
            const Draw dr = philox_draw(P.k0, P.k1, P.base + i, s, a);
            u = dr.u;
            if constexpr (WEIGHTED) {
                key = (KeyT)(bounded64(dr.x64, vW) + 1);   // first cw >= r + 1  <=>  cw > r
                search_init<CLB, IDX>(S, vstart, vstart + vdeg, 0);
                st = ST_SEARCH;
            } else {
                ci = vstart + (IDX)bounded64(dr.x64, vdeg);
                st = ST_COL;
            }
        }
    }
    add_steps(P.steps_out, steps);
}

template <typename CW, typename IDX, bool NODE2VEC, bool NEED_MEMBER, bool SYM>
cudaError_t launch_sm(const grape_graph* gg, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    const Params<CW> P = make_params<CW>(gg, a, T);
    static int resident = 0;   // blocks per SM x SMs, queried once per process
    if (resident == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_sm_kernel<CW, IDX, NODE2VEC, NEED_MEMBER, SYM>,
                                                      kBlock, 0);
        resident = sms * (per_sm > 0 ? per_sm : 1);
    }
    uint64_t blocks = (a.num_walks + kBlock - 1) / kBlock;
    if (blocks > (uint64_t)resident) blocks = resident;   // persistent: lanes loop over walks
    walk_sm_kernel<CW, IDX, NODE2VEC, NEED_MEMBER, SYM><<<(unsigned)blocks, kBlock, 0, stream>>>(P);
    return cudaGetLastError();
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
