// walk_tab.cu — the v4 walker: convergent state machine over the sampling
// tables of graph_tables.cu ("v4").  Same rules, same results as
// every other walker (include/grape_walk.h); the oracle decides.
//
// Each lane owns one walk.  Every iteration of the outer loop issues at most
// ONE aligned 32-byte sector load per lane (LDG.E.ENL2.256), whatever the lane
// is doing:
//   ST_START  starts[i]                          -> row[0]
//   ST_NODE   node record of v {start, deg, W_v}
//   ST_GUIDE  guide entry of the draw's bucket    -> first candidate index
//   ST_REC    arc record(s) {x, hi, rlo, rhi}     -> proposal x, and the reverse arc's
//                                                   interval for the next step
//   ST_HASH   one sector of t's edge-hash set     -> "x in N(t)"
// then an ALU-only phase (the inner loop) that may run several draws, emits and
// walk ends without touching memory:
//   * The three acceptance classes (thresholds §8(c) c9) split the
//     u range into bands.  When u accepts all classes or rejects all, x does
//     not matter (§8(c) c12: early accept / early reject).  When the decision
//     hinges only on "x == t", it is settled by comparing r with the interval
//     [tlo, thi) that the proposal index of t occupies in v's row — known from
//     the arc record that brought the walk to v — so the attempt costs a
//     Philox draw and nothing else; an accepted return x = t needs no load
//     either (t's node record is kept in registers, v and t swap).
//   * Only when the class of x matters beyond "x == t" is x read and, if
//     x != t, looked up in t's edge-hash set.
// Counter layout, bounded draws, thresholds and PAD handling are the ABI's;
// every decision above is decision-identical to the oracle's loop (the GPU
// parity tests compare whole walk matrices bit for bit).
#include "walk_common.cuh"

namespace grape {
namespace {
using namespace walk;

enum : uint32_t { ST_START = 0, ST_NODE, ST_GUIDE, ST_REC, ST_HASH, ST_DRAW, ST_DONE };

constexpr uint32_t kEmptySlot = 0xFFFFFFFFu;
// Inner (ALU) rounds per outer iteration before a lane that is still drawing
// yields to the next round of loads (bounds the warp's divergent tail).
#ifndef GRAPE_TAB_ALU_ROUNDS
#define GRAPE_TAB_ALU_ROUNDS 4
#endif
#ifndef GRAPE_TAB_MIN_BLOCKS
#define GRAPE_TAB_MIN_BLOCKS 3
#endif

struct TabParams {
    const NodeRec* nodes;
    const uint32_t* col;      // first-order unweighted proposals
    const void* rec;          // arc records (8 or 16 B)
    const uint32_t* guide;
    const uint32_t* ehash;
    uint32_t n;
    const uint32_t* starts;
    uint64_t num_walks;
    uint64_t base;
    uint32_t L;
    RoundKeys rk;
    uint32_t* out;
    unsigned long long* steps_out;
    unsigned long long* stats;
    uint32_t tp_m1, t1_m1, tq_m1;   // accept iff u <= T_c - 1
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

enum : int { C_LOADS = 0, C_NODE, C_XNODE, C_CWPROBE, C_COLPROBE, C_REC, C_ATTEMPT, C_MEMB, C_START, C_STEPS,
             C_GUIDE, C_HASH, C_ALU };

// REC: 4 = first-order unweighted (col only), 8 = {x, rev}, 16 = {x, hi, rlo, rhi}.
// WSYM: weighted graph whose reverse arcs carry equal weights, so the interval of
// an arc taken forward is known from its reverse's width (needed after a return).
template <int REC, bool NODE2VEC, bool NEED_MEMBER, bool WSYM, bool STATS>
__global__ void __launch_bounds__(kBlock, GRAPE_TAB_MIN_BLOCKS) walk_tab_kernel(const __grid_constant__ TabParams P)
{
    constexpr bool WEIGHTED = REC == 16;
    uint32_t cnt[kStatsWords];
    if (STATS) {
#pragma unroll
        for (int q = 0; q < kStatsWords; ++q) cnt[q] = 0;
    }
    __shared__ uint32_t stage[8 * kBlock];
    RowWriter w;
    w.slot = stage + threadIdx.x;
    const uint32_t L = P.L;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t st = i < P.num_walks ? ST_START : ST_DONE;
    const void* nxt = P.starts + (i < P.num_walks ? i : 0);
    unsigned long long steps = 0;

    uint32_t s = 0, a = 0;
    uint32_t vid = 0, vstart = 0, vdeg = 0, vW = 0;        // current node v
    uint32_t tid = kNone, tstart = 0, tdeg = 0, tW = 0;    // previous node t (kNone: first step)
    uint32_t tlo = 0, thi = 0;    // proposal interval of t in v's row (r units); tlo > thi: unknown
    uint32_t slo = 0, shi = 0;    // proposal interval of v in t's row (for a return v -> t)
    uint32_t u = 0, r = 0;        // pending attempt: acceptance draw, bounded proposal draw
    uint32_t ri = 0;              // row-local record index being read
    bool split = false;           // weighted: the guide bucket holds several candidates
    uint32_t x = 0, nlo = 0, nhi = 0, nslo = 0, nshi = 0;   // proposal and its intervals
    uint32_t hk = 0;              // edge-hash slot (absolute index)

    for (;;) {
        const bool load = st < ST_DRAW;
        if (!__any_sync(0xffffffffu, st != ST_DONE)) break;
        __syncwarp();
        uint32_t sec[8];
        if (load) ld8(sector_of(nxt), sec);
        const uint32_t j = word_of(nxt);
        if (STATS && load) {
            ++cnt[C_LOADS];
            cnt[C_NODE] += st == ST_NODE;
            cnt[C_REC] += st == ST_REC;
            cnt[C_START] += st == ST_START;
            cnt[C_GUIDE] += st == ST_GUIDE;
            cnt[C_HASH] += st == ST_HASH;
        }

        // ---- interpret the sector; at most one action flag per lane
        bool emit = false, fin = false, draw = st == ST_DRAW, decide = false;
        if (st == ST_REC) {
            bool found = true;
            if constexpr (REC == 4) {
                x = pick8(sec, j);
            } else if constexpr (REC == 8) {
                const uint32_t k = j & 6;
                x = pick8(sec, k);
                const uint32_t rev = pick8(sec, k + 1);
                nlo = rev;
                nhi = rev == kNone ? rev : rev + 1;   // [rev, rev+1), or the empty [NONE, NONE)
                nslo = ri;
                nshi = ri + 1;
            } else {
                // records k = 0, 1 of this sector; the target is k0 = j >> 2
                const uint32_t k0 = j >> 2;
                const uint32_t h0 = k0 ? sec[5] : sec[1];
                uint32_t k = k0;
                if (split && r >= h0) {
                    if (k0 == 0 && r < sec[5]) {
                        k = 1;
                        ri += 1;
                    } else {
                        found = false;                 // continue with the next sector
                        ri += 2 - k0;
                        nxt = (const uint4*)P.rec + (vstart + ri);
                    }
                }
                if (found) {
                    const uint32_t b = k ? 4 : 0;
                    x = k ? sec[4] : sec[0];
                    const uint32_t hi = k ? sec[5] : sec[1];
                    nlo = k ? sec[6] : sec[2];
                    nhi = k ? sec[7] : sec[3];
                    (void)b;
                    if (WSYM) {
                        nshi = hi;
                        nslo = hi - (nhi - nlo);
                    } else {
                        nslo = 1;                      // unknown
                        nshi = 0;
                    }
                }
            }
            decide = found;
        } else if (st == ST_NODE) {
            const bool hi4 = (j & 4) != 0;
            vstart = hi4 ? sec[4] : sec[0];
            vdeg = hi4 ? sec[6] : sec[2];
            vW = hi4 ? sec[7] : sec[3];
            a = 0;
            if (vdeg == 0) fin = true;
            else draw = true;
        } else if (st == ST_GUIDE) {
            const uint32_t e = pick8(sec, j);
            ri = e & 0x7FFFFFFFu;
            split = (e >> 31) != 0;
            st = ST_REC;
            nxt = (const uint4*)P.rec + (vstart + ri);
        } else if (st == ST_HASH) {
            // slots [hk, min(sector end, region end)) of t's set
            const uint32_t sb = hk & ~7u;
            const uint32_t rend = 2 * (tstart + tdeg);
            const uint32_t e = rend - sb < 8 ? rend - sb : 8;
            const uint32_t q0 = hk - sb;
            uint32_t fm = 0, em = 0;
#pragma unroll
            for (uint32_t q = 0; q < 8; ++q) {
                fm |= (sec[q] == x ? 1u : 0u) << q;
                em |= (sec[q] == kEmptySlot ? 1u : 0u) << q;
            }
            const uint32_t in = (0xFFu >> (8 - e)) & (0xFFu << q0);
            if ((fm | em) & in) {
                const bool member = (fm & in) != 0;
                emit = member ? u <= P.t1_m1 : u <= P.tq_m1;
                draw = !emit;
                if (draw) ++a;
            } else {
                hk = sb + e == rend ? 2 * tstart : sb + e;
                nxt = P.ehash + hk;
            }
        } else if (st == ST_START) {
            const uint32_t start = pick8(sec, j);
            w.begin(P.out + i * L);
            s = 0;
            tid = kNone;
            if (start < P.n) {
                x = start;
                emit = true;
            } else {
                fin = true;
            }
        }
        if (decide) {   // x is known: the class of x, if it matters
            if (!NODE2VEC || tid == kNone) {
                emit = true;
            } else {
                const bool cp = u <= P.tp_m1, c1 = u <= P.t1_m1, cq = u <= P.tq_m1;
                if (x == tid) emit = cp;
                else if (!NEED_MEMBER || c1 == cq) emit = c1;
                else {
                    if (STATS) ++cnt[C_MEMB];
                    st = ST_HASH;
                    hk = 2 * tstart + (uint32_t)(((uint64_t)fmix32(x) * (2 * tdeg)) >> 32);
                    nxt = P.ehash + hk;
                }
                draw = !emit && st != ST_HASH;
                if (draw) ++a;
            }
        }

        // ---- ALU phase: emits, walk ends and draws until every lane has a load
        // pending (or has drawn GRAPE_TAB_ALU_ROUNDS times)
#pragma unroll 1
        for (int round = 0;; ++round) {
            if (!__any_sync(0xffffffffu, emit || fin || draw)) break;
            __syncwarp();
            if (emit) {   // x becomes row[s]; [nlo,nhi) / [nslo,nshi) are the new T / S
                w.put(s, x);
                if (s > 0) {
                    ++steps;
                    if (x == tid) {   // a return: v and t swap, t's record is in registers
                        uint32_t q;
                        q = vstart; vstart = tstart; tstart = q;
                        q = vdeg; vdeg = tdeg; tdeg = q;
                        q = vW; vW = tW; tW = q;
                        tid = vid;
                        vid = x;
                        tlo = nlo; thi = nhi; slo = nslo; shi = nshi;
                        a = 0;
                        draw = s + 1 < L;
                        st = ST_DRAW;
                    } else {
                        tid = vid; tstart = vstart; tdeg = vdeg; tW = vW;
                        vid = x;
                        tlo = nlo; thi = nhi; slo = nslo; shi = nshi;
                        st = ST_NODE;
                        nxt = P.nodes + x;
                    }
                } else {
                    vid = x;
                    st = ST_NODE;
                    nxt = P.nodes + x;
                }
                ++s;
                fin = s == L;
                emit = false;
            }
            if (fin) {
                for (uint32_t q = s; q < L; ++q) w.put(q, kPad);
                w.finish(L);
                i += stride;
                st = i < P.num_walks ? ST_START : ST_DONE;
                nxt = P.starts + (i < P.num_walks ? i : 0);
                fin = false;
                draw = false;
            }
            __syncwarp();
            if (draw && round >= GRAPE_TAB_ALU_ROUNDS) {
                st = ST_DRAW;   // keep drawing after the next round of loads
                draw = false;
            }
            if (draw) {
                if (STATS) ++cnt[C_ATTEMPT];
                const Draw dr = philox_draw_rk(P.rk, P.base + i, s, a);
                u = dr.u;
                r = (uint32_t)bounded64(dr.x64, vW);   // index (unweighted: vW = deg) or weight point
                bool need_x = true, back = false;
                if (NODE2VEC && tid != kNone) {
                    const bool cp = u <= P.tp_m1, c1 = u <= P.t1_m1, cq = u <= P.tq_m1;
                    if (cp == c1 && c1 == cq) {
                        need_x = cp;
                    } else if (c1 == cq && tlo <= thi) {   // only "x == t" matters, and it is known
                        const bool is_t = r - tlo < thi - tlo;
                        const bool acc = is_t ? cp : c1;
                        need_x = acc && !is_t;
                        back = acc && is_t;
                    }
                    if (STATS) cnt[C_ALU] += !need_x;
                }
                if (back) {   // return to t: x = t, the new T / S are the old S / T
                    x = tid;
                    nlo = slo; nhi = shi; nslo = tlo; nshi = thi;
                    emit = true;
                    draw = false;
                } else if (need_x) {
                    draw = false;
                    if constexpr (REC == 16) {
                        if (vdeg == 1) {
                            ri = 0;
                            split = false;
                            st = ST_REC;
                            nxt = (const uint4*)P.rec + vstart;
                        } else {
                            const uint32_t kb = (uint32_t)__umul64hi(dr.x64, 2ull * vdeg);
                            st = ST_GUIDE;
                            nxt = P.guide + (2ull * vstart + kb);
                        }
                    } else if constexpr (REC == 8) {
                        ri = r;
                        st = ST_REC;
                        nxt = (const uint2*)P.rec + (vstart + r);
                    } else {
                        st = ST_REC;
                        nxt = P.col + (vstart + r);
                    }
                } else {
                    ++a;   // rejected without reading the graph
                }
            }
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

template <int REC, bool NODE2VEC, bool NEED_MEMBER, bool WSYM, bool STATS>
cudaError_t launch_k(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    TabParams P{};
    P.nodes = g->nodes;
    P.col = g->col;
    P.rec = g->rec;
    P.guide = g->guide;
    P.ehash = g->ehash;
    P.n = g->n;
    P.starts = a.starts;
    P.num_walks = a.num_walks;
    P.base = a.walk_id_base;
    P.L = a.L;
    P.rk = philox_round_keys(a.seed);
    P.out = a.out;
    P.steps_out = a.steps_out;
    P.stats = a.stats;
    P.tp_m1 = (uint32_t)(T.Tp - 1);
    P.t1_m1 = (uint32_t)(T.T1 - 1);
    P.tq_m1 = (uint32_t)(T.Tq - 1);
    static int resident = 0;
    if (resident == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_tab_kernel<REC, NODE2VEC, NEED_MEMBER, WSYM, STATS>,
                                                      kBlock, 0);
        resident = sms * (per_sm > 0 ? per_sm : 1);
    }
    uint64_t blocks = (a.num_walks + kBlock - 1) / kBlock;
    if (blocks > (uint64_t)resident) blocks = resident;
    walk_tab_kernel<REC, NODE2VEC, NEED_MEMBER, WSYM, STATS><<<(unsigned)blocks, kBlock, 0, stream>>>(P);
    return cudaGetLastError();
}

template <int REC, bool NODE2VEC, bool NEED_MEMBER, bool WSYM>
cudaError_t launch_s(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    if (a.stats != nullptr) return launch_k<REC, NODE2VEC, NEED_MEMBER, WSYM, true>(g, a, T, stream);
    return launch_k<REC, NODE2VEC, NEED_MEMBER, WSYM, false>(g, a, T, stream);
}

template <int REC, bool WSYM>
cudaError_t dispatch_n2v(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    if (T.T1 != T.Tq) return launch_s<REC, true, true, WSYM>(g, a, T, stream);
    return launch_s<REC, true, false, WSYM>(g, a, T, stream);
}

}  // namespace

cudaError_t launch_walks_tab(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                             cudaStream_t stream)
{
    const bool weighted = g->cw_bytes != 0;
    const bool first_order = !node2vec || (T.Tp == T.T1 && T.T1 == T.Tq);
    if (first_order) {
        if (weighted) return launch_s<16, false, false, false>(g, a, T, stream);
        return launch_s<4, false, false, false>(g, a, T, stream);
    }
    if (!weighted) return dispatch_n2v<8, false>(g, a, T, stream);
    if (g->wsym) return dispatch_n2v<16, true>(g, a, T, stream);
    return dispatch_n2v<16, false>(g, a, T, stream);
}

}  // namespace grape
