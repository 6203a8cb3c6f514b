// walk_tab.cu — the table walker (v4/v5/v6): a convergent state machine over
// the sampling tables of graph_tables.cu.  Same rules, same
// results as every other walker (include/grape_walk.h); the oracle decides.
//
// Each lane owns one walk.  Every iteration of the outer loop issues at most
// ONE aligned 32-byte sector load per lane (LDG.E.ENL2.256), its address
// computed in one place for every state:
//   ST_START  starts[i]                           -> row[0]
//   ST_NODE   node record {start, deg, W}          -> a start node (or, compact
//                                                    records, a taken arc's head)
//   ST_GUIDE  guide entry of the draw's bucket     -> the proposal and its record (fat,
//                                                    unsplit), or the split boundary
//   ST_REC    arc record {x, hi, rlo, rhi, x's node record, lo}
//                                                  -> proposal x, the reverse arc's interval
//                                                    and the pair's no-common-neighbour flags
//   ST_HASH   one bucket of t's edge-hash set      -> "x in N(t)"
//   ST_CAND   (SUSS, weighted) a candidate's record into the lane's scratch
// No load: ST_DRAW (keep drawing), ST_BACK (emit a register-decided return).
// After the load: the decision where x is needed, the walk's advance (emit,
// reading the taken arc's record from the sector in hand), and up to
// GRAPE_TAB_DRAWS draws:
//   * The three acceptance classes (thresholds §8(c) c9) split the
//     u range into bands.  When u accepts all classes or rejects all, x does
//     not matter (§8(c) c12: early accept / early reject).  When the decision
//     hinges only on "x == t" — always so when the pair (t, v) has no common
//     neighbour, since then every x != t is class q — it is settled by
//     comparing r with the interval [tlo, thi) that the proposal index of t
//     occupies in v's row, known from the arc record that brought the walk to
//     v: the attempt costs a Philox draw and nothing else; an accepted return
//     x = t needs no load either (t's node record is in registers, v and t swap).
//   * Only when the class of x matters beyond "x == t" is x read and, if
//     x != t, looked up in t's edge-hash set.
// Walks are assigned round-robin for the first half of the launch, then from a
// warp-aggregated shared counter (balances the tail).  Counter layout, bounded
// draws, thresholds and PAD handling are the ABI's; every decision above is
// decision-identical to the oracle's loop (the GPU parity tests compare whole
// walk matrices bit for bit).
#include "walk_tab.cuh"

namespace grape {
namespace {
using namespace walk;

enum : uint32_t { ST_START = 0, ST_NODE, ST_GUIDE, ST_REC, ST_HASH, ST_CAND, ST_DRAW, ST_BACK, ST_DONE };

#ifndef GRAPE_TAB_DRAWS
#define GRAPE_TAB_DRAWS 2
#endif
#ifndef GRAPE_TAB_DRAW_UNROLL
#define GRAPE_TAB_DRAW_UNROLL 1
#endif
constexpr int kDrawUnroll = GRAPE_TAB_DRAW_UNROLL;
#ifndef GRAPE_SUSS_UNROLL
#define GRAPE_SUSS_UNROLL 1
#endif
constexpr int kSussUnroll = GRAPE_SUSS_UNROLL;
#ifndef GRAPE_SUSS_MIN_BLOCKS
#define GRAPE_SUSS_MIN_BLOCKS GRAPE_TAB_MIN_BLOCKS   // resident blocks per SM of the SUSS kernels
#endif   // candidate pairs per unrolled step of the SUSS burst
#ifndef GRAPE_TAB_EMIT_SPOT
#define GRAPE_TAB_EMIT_SPOT 0    // 1: a register-decided return is emitted inside the draw round when another follows (measured slower: DESIGN.md §7)
#endif
#ifndef GRAPE_TAB_SEL_ADV
#define GRAPE_TAB_SEL_ADV 1      // 1: emit / back update the walk's state through one set of selects (full records)
#endif
#ifndef GRAPE_TAB_ADDR_TABLE
#define GRAPE_TAB_ADDR_TABLE 1   // 1: the load's table base and shift from a per-state parameter table
#endif
#ifndef GRAPE_TAB_SYNC_TOP
#define GRAPE_TAB_SYNC_TOP 0     // explicit reconvergence points (measured: the emit one matters)
#endif
#ifndef GRAPE_TAB_SYNC_EMIT
#define GRAPE_TAB_SYNC_EMIT 1
#endif
#ifndef GRAPE_TAB_SYNC_DRAW
#define GRAPE_TAB_SYNC_DRAW 1
#endif

// WEIGHTED: 32-B records + guide; else 16-B records indexed by the draw.
// WIDE: arc offsets of 34 bits (graphs of 2^32 - 64 .. 2^34 arcs, or the arc-offset bias
// test hook): row starts are u64 in registers, their bits 32-33 come from bits 26-27 of a
// full record's degree word or from the node record's high word.
template <bool WEIGHTED, bool FAT, bool COMPACT, bool NODE2VEC, bool NEED_MEMBER, bool STATS, int MODE,
          bool WIDE = false>
__global__ void __launch_bounds__(kBlock, MODE == 1 ? GRAPE_SUSS_MIN_BLOCKS : GRAPE_TAB_MIN_BLOCKS) walk_tab_kernel(const __grid_constant__ TabParams P)
{
    using off_t_ = typename std::conditional<WIDE, uint64_t, uint32_t>::type;   // a row start
    constexpr uint32_t kDegMask = WIDE ? 0x03FFFFFFu : 0x0FFFFFFFu;                  // degree bits of a record
    constexpr bool SUSS = MODE == 1;   // approximated walks (grape_walks_approx)
    constexpr bool FOLD = MODE == 2;   // outlier-folded rejection (grape_walks_node2vec_folded)
    constexpr bool PARTS = MODE == 3;  // the default rule over partitioned tables (grape_graph_partition)
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
    auto divH = [&](uint32_t v) { return __umulhi(v, P.h_mul) >> P.h_shift; };   // floor(v / H)
    auto divHo = [&](off_t_ t) -> uint32_t {   // floor(row start / H): an edge-hash bucket index
        if constexpr (WIDE) return (uint32_t)(P.h_shift ? __umul64hi(t, 0xAAAAAAAAAAAAAAABull) >> 2 : t >> 2);
        else return divH(t);
    };

    uint32_t idx = 0;   // what the next load reads: NODE node id, GUIDE bucket (REC: ri, HASH: hb)
    uint32_t hb = 0;    // edge-hash bucket (absolute index)
    bool gsrc = false;  // fat guide: the proposal's record is the guide entry idx
    // no common neighbour (graph_tables.cu build_notri): nt for the current (t, v) —
    // every proposal x != t is then in class q — and ntr for (v, t), used after a return
    bool nt = false, ntr = false;
    uint32_t hfl = 0;   // unweighted: x's record flags, kept across its membership test
    unsigned long long steps = 0;

    uint32_t s = 0, a = 0;
    uint32_t vid = 0;                           // current node v
    off_t_ vstart = 0;                          // (its row start)
    uint32_t vdeg = 0, vW = 0;
    uint32_t tid = kNone;                       // previous node t (kNone: first step)
    off_t_ tstart = 0;
    uint32_t tdeg = 0, tW = 0;
#define GRAPE_SWAP_VT()                                        \
    do {                                                       \
        const off_t_ z_ = vstart; vstart = tstart; tstart = z_; \
        uint32_t q_;                                           \
        q_ = vdeg; vdeg = tdeg; tdeg = q_;                     \
        q_ = vW; vW = tW; tW = q_;                             \
        q_ = vid; vid = tid; tid = q_;                         \
    } while (0)
    uint32_t tlo = 0, thi = 0;    // proposal interval of t in v's row (r units; empty if no arc v -> t)
    uint32_t slo = 0, shi = 0;    // proposal interval of v in t's row (for a return v -> t)
    uint32_t u = 0, r = 0;        // pending attempt: acceptance draw, bounded proposal draw
    uint32_t ri = 0;              // row-local index of the proposal (record being read)
    bool scan = false;            // weighted: compare r with the record's hi, advance if past it
    bool acc = false;             // the attempt is accepted; the record is read for x's data
    uint32_t x = 0;               // proposal
    uint32_t hrev = 0;   // unweighted: x's record, kept across its membership test
    off_t_ hxs = 0;
    uint32_t hxd = 0;
    // SUSS (approximated walks, §8(f) f1): at a node with deg > dT the step runs on dT
    // candidates, one uniform pick per bucket [floor(b deg/dT), floor((b+1) deg/dT))
    uint32_t cb = 0;              // weighted: candidates read so far this step (dT: sub-sample in scratch)
    uint32_t bt = kNone;          // weighted: the candidate that is t, if any
    uint32_t wc = 0;              // weighted: running / total candidate weight
    uint32_t clo = 0;             // compact records: cw of the candidate's predecessor
    bool cph = false;             // compact records: reading the predecessor's sector
    const uint64_t gl = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto suss_index = [&](uint32_t b) {   // row-local index of candidate b of this step
        const uint32_t lo = (uint32_t)(((uint64_t)b * vdeg) / P.dT);
        const uint32_t hi = (uint32_t)(((uint64_t)(b + 1) * vdeg) / P.dT);
        const uint4 o = philox_block_rk(P.rk, P.base + i, s, 0x80000000u | (b >> 1));
        const uint64_t h = (b & 1) ? ((uint64_t)o.w << 32 | o.z) : ((uint64_t)o.y << 32 | o.x);
        return lo + bounded32(h, hi - lo);
    };

    for (;;) {
        if (!__any_sync(0xffffffffu, st != ST_DONE)) break;
        const bool load = st < ST_DRAW;
        if (GRAPE_TAB_SYNC_TOP) __syncwarp();
        uint32_t sec[8];
        uint32_t j;
        {   // the one load of this iteration: a single address computation for every state
            const bool rec = st == ST_REC || (SUSS && st == ST_CAND), gd = st == ST_GUIDE, nd = st == ST_NODE;
            uint32_t mul = rec ? 1u : gd ? P.G : 0u;
            if constexpr (GRAPE_TAB_ADDR_TABLE == 2 && !PARTS && !SUSS) mul = P.tbl_mul[st < ST_DRAW ? st : 0u];
            uint64_t e = (uint64_t)mul * vstart + (rec ? ri : st == ST_HASH ? hb : idx);
            const char* b = rec ? (const char*)P.rec : gd ? (const char*)P.guide
                          : nd ? (const char*)P.nodes : (const char*)P.ehash;
            constexpr uint32_t RSH = (WEIGHTED ? 5u : 4u) - (COMPACT ? 1u : 0u);   // log2 record bytes
            uint32_t sh = rec ? RSH : gd ? (FAT ? 5u : 3u) : nd ? 4u : 5u;
            if (st == ST_START) {
                b = (const char*)P.starts;
                e = i;
                sh = 2;
            }
            if constexpr (GRAPE_TAB_ADDR_TABLE && !PARTS && !SUSS) {   // base and shift of the state's table
                const uint32_t k = st < ST_DRAW ? st : 0u;
                b = P.tbl_base[k];
                sh = P.tbl_shift[k];
            }
            const char* addr = b + (e << sh);
            if (PARTS && st != ST_START) {   // part (offset >> k) of table T, at offset mod 2^k
                const uint32_t T = rec ? 0u : gd ? 1u : nd ? 2u : 3u;
                const uint64_t o = e << sh;
                const uint32_t ps = __ldg(&P.pmap->shift[T]);
                addr = (const char*)__ldg((const unsigned long long*)&P.pmap->base[T][o >> ps]) +
                       (o & ((1ull << ps) - 1));
            }
#if GRAPE_CHECKED
            if (load) {
                if (st == ST_START) {
                    GRAPE_DCHECK(i < P.num_walks, "start index < num_walks");
                } else {
                    const uint32_t T = rec ? 0u : gd ? 1u : nd ? 2u : 3u;
                    GRAPE_DCHECK((e << sh) < P.lim[T], "table read within its table");
                    if (rec) GRAPE_DCHECK(ri < vdeg && e < P.m, "arc record within the row");
                    if (gd) GRAPE_DCHECK(idx < P.G * vdeg, "guide bucket within the row");
                    if (nd) GRAPE_DCHECK(idx < P.n, "node record of a node");
                    if (st == ST_HASH)
                        GRAPE_DCHECK(hb >= divHo(tstart) + tid && hb < divHo(tstart) + tid + divH(tdeg) + 1,
                                     "hash bucket within t's buckets");
                }
            }
#endif
            if (load) ld8(sector_of(addr), sec);
            j = word_of(addr);
        }
        if (STATS && st != ST_DONE) {
            ++cnt[C_ITER];
            cnt[C_ITER_DRAW] += st == ST_DRAW;
            cnt[C_ITER_BACK] += st == ST_BACK;
        }
        if (STATS && load) {
            ++cnt[C_LOADS];
            cnt[C_NODE] += st == ST_NODE;
            cnt[C_REC] += st == ST_REC || st == ST_CAND;
            cnt[C_START] += st == ST_START;
            cnt[C_GUIDE] += st == ST_GUIDE;
            cnt[C_HASH] += st == ST_HASH;
        }

        // ---- interpret the sector
        bool emit = false, back = st == ST_BACK, fin = false, draw = st == ST_DRAW, decide = false;
        // when emit: the taken arc's record is in sec (at word j for 8/16-B records) —
        // read by the emit block itself, so no per-branch copies — or, after an
        // unweighted membership test, in the kept registers (kept)
        bool have_rec = false;   // the sector in hand is x's record
        bool kept = false;
        // one attempt of a drawing lane: Philox, the band of u, the decisions that need no
        // read (§8(c) c12); more (GRAPE_TAB_EMIT_SPOT builds only): another draw follows in this
        // iteration and a register-decided return is emitted on the spot; by default the lane
        // goes to ST_BACK and the next iteration's emit block takes it
        auto draw_once = [&](const bool more, const bool sub) {
            if (STATS) ++cnt[C_ATTEMPT];
            Draw dr;
            uint32_t o3 = 0;
            if constexpr (FOLD) {   // all four words: o3 decides the return's excess mass
                const uint4 o = philox_block_rk(P.rk, P.base + i, s, a);
                dr.x64 = (uint64_t)o.y << 32 | o.x;
                dr.u = o.z;
                o3 = o.w;
            } else {
                dr = philox_draw_rk(P.rk, P.base + i, s, a);
            }
            u = dr.u;
            bool known = tlo <= thi;
            uint32_t bs = 0;                 // SUSS: the proposed candidate
            if (SUSS && sub) {
                if constexpr (WEIGHTED) {    // first candidate whose running weight exceeds r
                    r = bounded32(dr.x64, wc);
                    uint32_t lo = 0, hi = P.dT;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (P.scratch[(uint64_t)(2 * mid) * P.lanes + gl] <= r) lo = mid + 1;
                        else hi = mid;
                    }
                    bs = lo;
                    r = bs;                  // "x == t" <=> the candidate is t's
                    known = true;
                } else {                     // uniform candidate; its row index vs t's
                    bs = bounded32(dr.x64, P.dT);
                    r = suss_index(bs);
                }
            } else {
                r = bounded32(dr.x64, vW);   // index (unweighted: vW = deg) or weight point
            }
            bool need_x = true, ret = false;
            bool outlier = false;
            if (FOLD && tid != kNone) {   // o3 * M < N * 2^32, N = w_vt X, M = W_v E + N
                const uint64_t N = known ? (uint64_t)(thi - tlo) * P.fold_x : 0;   // w_vt = width of t's interval
                const uint64_t M = (uint64_t)vW * P.fold_e + N;
                const uint64_t p1 = (uint64_t)o3 * (M >> 32) + (((uint64_t)o3 * (uint32_t)M) >> 32);
                outlier = p1 < N;
            }
            if (outlier) {
                need_x = false;
                ret = true;
                if (STATS) ++cnt[C_ALU];
            } else if (NODE2VEC && tid != kNone) {
                const bool cp = u <= P.tp_m1, cq = u <= P.tq_m1, c1 = nt ? cq : u <= P.t1_m1;
                if (cp == c1 && c1 == cq) {
                    need_x = cp;
                } else if (c1 == cq && known) {   // only "x == t" matters, and it is known
                    const bool is_t = (SUSS && WEIGHTED && sub) ? bs == bt : r - tlo < thi - tlo;
                    const bool ok = is_t ? cp : c1;
                    need_x = ok && !is_t;
                    ret = ok && is_t;
                }
                if (STATS) cnt[C_ALU] += !need_x;
            }
            acc = false;
            scan = false;
            gsrc = false;
            draw = false;
            if (ret) {          // return to t, no read
                if (more && s + 1 < L) {   // emit now; t's row is not empty
                    GRAPE_DCHECK(s < L && tid < P.n, "returned walk entry within the row");
                    w.put(s, tid);
                    ++steps;
                    GRAPE_SWAP_VT();
                    uint32_t q;
                    q = tlo; tlo = slo; slo = q;
                    q = thi; thi = shi; shi = q;
                    const bool b_ = nt; nt = ntr; ntr = b_;
                    ++s;
                    a = 0;
                    cb = 0;
                    draw = true;
                } else {        // emitted next iteration
                    x = tid;
                }
                st = ST_BACK;
            } else if (!need_x) {
                ++a;            // rejected without reading the graph
                st = ST_DRAW;
                draw = true;
            } else if (SUSS && WEIGHTED && sub) {   // x is in scratch: decide, then read its record
                x = P.scratch[(uint64_t)(2 * bs + 1) * P.lanes + gl];
                ri = suss_index(bs);
                bool ok = true, hash = false;
                if (NODE2VEC && tid != kNone) {
                    const bool cp = u <= P.tp_m1, cq = u <= P.tq_m1, c1 = nt ? cq : u <= P.t1_m1;
                    if (x == tid) ok = cp;
                    else if (!NEED_MEMBER || c1 == cq) ok = c1;
                    else hash = true;
                }
                if (hash) {
                    if (STATS) ++cnt[C_MEMB];
                    st = ST_HASH;
                    hb = divHo(tstart) + tid + (uint32_t)(((uint64_t)fmix32(x) * (divH(tdeg) + 1)) >> 32);
                } else if (ok) {
                    acc = true;
                    st = ST_REC;
                } else {
                    ++a;
                    st = ST_DRAW;
                    draw = true;
                }
            } else if constexpr (WEIGHTED) {
                if (vdeg == 1) {
                    ri = 0;
                    st = ST_REC;
                } else {
                    idx = bounded32(dr.x64, P.G * vdeg);   // guide bucket
                    st = ST_GUIDE;
                }
            } else {
                ri = r;
                st = ST_REC;
            }
        };
        const uint32_t st0 = st;   // the state this iteration's load served (the dispatch below)
        if (st0 == ST_REC) {
            have_rec = true;
            bool found = true;
            if constexpr (WEIGHTED && COMPACT) {   // 16-B {x, hi, rlo, rhi} at word j (0 or 4)
                const bool h = (j & 4) != 0;
                const uint32_t hi = h ? sec[5] : sec[1];
                if (scan && r >= hi) {   // past this record's interval: the next one
                    found = false;
                    ++ri;
                }
                x = (h ? sec[4] : sec[0]) & P.xmask;
            } else if constexpr (WEIGHTED) {
                if (scan && r >= sec[1]) {   // past this record's interval: the next one
                    found = false;
                    ++ri;
                }
                x = sec[0];
            } else if constexpr (COMPACT) {   // 8-B {x, rev} at word j (even)
                const uint32_t xr = pick8(sec, j);
                x = xr & P.xmask;
                hfl = P.notri ? xr >> 30 : 0u;
                hrev = pick8(sec, j | 1);
            } else {
                const bool h = (j & 4) != 0;
                x = h ? sec[4] : sec[0];
                hrev = h ? sec[5] : sec[1];
                hxs = h ? sec[6] : sec[2];
                hxd = h ? sec[7] : sec[3];
            }
            if (found) {
                if (acc) emit = true;
                else decide = true;
            }
        } else if (st0 == ST_GUIDE) {
            uint32_t e0, e1;
            bool split;
            if constexpr (FAT) {   // unsplit: a record copy; split: {i_lo, cw[i_lo], .., flags in word 5}
                split = (sec[5] >> 31) != 0;
                e0 = sec[0] | (sec[5] & 0xC0000000u);
                e1 = sec[1];
            } else {
                e0 = pick8(sec, j);   // 8-B entry at word j (even)
                e1 = pick8(sec, j | 1);
                split = (e0 >> 31) != 0;
            }
            if (split) {      // split bucket: r against the upper end of i_lo's interval
                ri = e0 & 0x3FFFFFFFu;
                scan = false;
                if (r >= e1) {
                    ++ri;
                    scan = (e0 >> 30) & 1;   // more boundaries: compare record by record
                }
                acc = false;
                st = ST_REC;
            } else if constexpr (FAT) {   // the bucket's proposal, with its whole record
                have_rec = true;
                gsrc = true;
                x = sec[0];
                if (acc) emit = true;
                else decide = true;
            } else {          // the bucket proposes i_lo = e1 whatever the draw
                ri = e0 & 0x3FFFFFFFu;
                x = e1;
                decide = true;
            }
        } else if (SUSS && WEIGHTED && st0 == ST_CAND) {   // candidate cb's record: its node and weight
            bool done = true;
            uint32_t wgt = 0;
            if constexpr (COMPACT) {
                const bool h = (j & 4) != 0;
                if (cph) {                    // the predecessor (odd index: upper half): hi = cw[c - 1]
                    wgt = clo - (h ? sec[5] : sec[1]);
                    cph = false;
                    ++ri;
                } else {
                    x = (h ? sec[4] : sec[0]) & P.xmask;
                    const uint32_t hi = h ? sec[5] : sec[1];
                    const uint32_t rl = h ? sec[6] : sec[2], rh = h ? sec[7] : sec[3];
                    if (P.wsym && rh > rl) wgt = rh - rl;          // the reverse arc has the same weight
                    else if (ri == 0) wgt = hi;
                    else if (h) wgt = hi - sec[1];                 // predecessor in this sector
                    else { cph = true; clo = hi; --ri; done = false; }   // read the predecessor
                }
            } else {
                x = sec[0];
                wgt = sec[1] - sec[7];        // hi - lo
            }
            if (done) {
                wc += wgt;
                P.scratch[(uint64_t)(2 * cb) * P.lanes + gl] = wc;
                P.scratch[(uint64_t)(2 * cb + 1) * P.lanes + gl] = x;
                if (x == tid) bt = cb;
                ++cb;
                if (cb < P.dT) ri = suss_index(cb);
                else draw = true;
            }
        } else if (st0 == ST_HASH) {   // one bucket (8 slots) of t's set
            // a bucket fills from slot 0 up (graph_tables.cu build_ehash: a slot is only tried
            // after the ones before it were found taken, and nothing is ever removed), so it
            // has an empty slot iff its last slot is empty
            bool found = false;
            const bool empty = sec[7] == kEmptySlot;
#if GRAPE_CHECKED
            {   // the invariant itself: no empty slot before a taken one
                bool gap = false, seen_empty = false;
                for (int q = 0; q < 8; ++q) {
                    gap |= seen_empty && sec[q] != kEmptySlot;
                    seen_empty |= sec[q] == kEmptySlot;
                }
                GRAPE_DCHECK(!gap, "edge-hash bucket filled from slot 0 up");
            }
#endif
#pragma unroll
            for (int q = 0; q < 8; ++q) found |= sec[q] == x;
            if (found || empty) {
                if (found ? u <= P.t1_m1 : u <= P.tq_m1) {
                    if constexpr (WEIGHTED) {
                        acc = true;   // read the record again for x's data
                        scan = false;
                        st = gsrc ? ST_GUIDE : ST_REC;
                    } else {          // the record was kept in registers
                        emit = true;
                        kept = true;
                    }
                } else {
                    draw = true;
                    ++a;
                }
            } else {   // full bucket without x: the next one, cyclically within t's buckets
                const uint32_t base = divHo(tstart) + tid;
                hb = hb + 1 == base + divH(tdeg) + 1 ? base : hb + 1;
            }
        } else if (st0 == ST_NODE) {   // node record: a start node, or (compact records) a taken arc's head
            const bool h = (j & 4) != 0;
            vstart = h ? sec[4] : sec[0];
            if constexpr (WIDE) vstart |= (off_t_)(h ? sec[5] : sec[1]) << 32;   // NodeRec.start is u64
            vdeg = h ? sec[6] : sec[2];
            vW = h ? sec[7] : sec[3];
            a = 0;
            cb = 0;
            if (vdeg == 0) fin = true;
            else draw = true;
        } else if (st0 == ST_START) {
            const uint32_t start = pick8(sec, j);
            w.begin(P.out + i * L);
            s = 0;
            tid = kNone;
            nt = ntr = false;
            if (start < P.n) {
                w.put(0, start);
                vid = start;
                s = 1;
                if (L == 1) {
                    fin = true;
                } else {
                    st = ST_NODE;
                    idx = start;
                }
            } else {
                fin = true;
            }
        }
        if (decide) {   // x is known: its class, if it matters
            bool ok = true, hash = false;
            if (NODE2VEC && tid != kNone) {
                const bool cp = u <= P.tp_m1, cq = u <= P.tq_m1, c1 = nt ? cq : u <= P.t1_m1;
                if (x == tid) ok = cp;
                else if (!NEED_MEMBER || c1 == cq) ok = c1;
                else hash = true;
            }
            if (hash) {
                if (STATS) ++cnt[C_MEMB];
                st = ST_HASH;   // home bucket of x among t's floor(deg t / H) + 1 buckets
                hb = divHo(tstart) + tid + (uint32_t)(((uint64_t)fmix32(x) * (divH(tdeg) + 1)) >> 32);
            } else if (!ok) {
                draw = true;
                ++a;
            } else if (have_rec) {
                emit = true;      // the record is in hand
            } else {              // x came from the guide: read its record
                acc = true;
                scan = false;
                st = ST_REC;
            }
        }

        // ---- the walk advances: from a record (emit) or by a register-decided
        // return to t (back, decided by the previous iteration's draw)
        if (GRAPE_TAB_SYNC_EMIT) __syncwarp();
        if (emit || back) {
            GRAPE_DCHECK(s < L && x < P.n, "walk entry within the row, a node id");
            w.put(s, x);
            ++steps;
            bool need_node = false;
            if constexpr (GRAPE_TAB_SEL_ADV && !COMPACT) {
                // one update for both ways to advance (x == t when back): t <- v; v <- the taken
                // arc's head (emit: from its record) or the old t (back); T, S and the flags from
                // the record, or swapped
                uint32_t fnlo, fnhi, fnslo, fnshi, fxd, fxw, ffl;
                off_t_ fxs;
                if constexpr (WEIGHTED) {
                    fnlo = sec[2]; fnhi = sec[3]; fnslo = sec[7]; fnshi = sec[1];
                    fxs = sec[4]; fxd = sec[5] & kDegMask; fxw = sec[6];
                    if constexpr (WIDE) fxs |= (off_t_)((sec[5] >> 26) & 3u) << 32;
                    ffl = (sec[5] >> 28) & 3u;
                } else {
                    fxs = hxs;
                    if constexpr (WIDE) fxs |= (off_t_)((hxd >> 26) & 3u) << 32;
                    ffl = (hxd >> 28) & 3u;
                    fxd = hxd & kDegMask;
                    fxw = fxd;
                    fnlo = hrev;
                    fnhi = hrev == kNone ? hrev : hrev + 1;
                    fnslo = ri;
                    fnshi = ri + 1;
                }
                const uint32_t ovid = vid, ovdeg = vdeg, ovW = vW, otlo = tlo, othi = thi;
                const off_t_ ovs = vstart;
                const bool ont = nt;
                vid = x;
                vstart = emit ? fxs : tstart; vdeg = emit ? fxd : tdeg; vW = emit ? fxw : tW;
                tid = ovid; tstart = ovs; tdeg = ovdeg; tW = ovW;
                tlo = emit ? fnlo : slo; thi = emit ? fnhi : shi;
                slo = emit ? fnslo : otlo; shi = emit ? fnshi : othi;
                nt = emit ? (ffl >> 1) != 0 : ntr; ntr = emit ? (ffl & 1) != 0 : ont;
            } else
            if (emit) {   // the record of the taken arc: T, S, flags and (full records) x's node record
                uint32_t fnlo, fnhi, fnslo, fnshi, fxd = 0, fxw = 0, ffl;
                off_t_ fxs = 0;
                if constexpr (WEIGHTED && !COMPACT) {   // 32-B record at word 0 (also a fat guide entry)
                    fnlo = sec[2]; fnhi = sec[3]; fnslo = sec[7]; fnshi = sec[1];
                    fxs = sec[4]; fxd = sec[5] & kDegMask; fxw = sec[6];
                    if constexpr (WIDE) fxs |= (off_t_)((sec[5] >> 26) & 3u) << 32;
                    ffl = (sec[5] >> 28) & 3u;
                } else if constexpr (WEIGHTED) {        // 16-B {x, hi, rlo, rhi} at word j
                    const bool h = (j & 4) != 0;
                    const uint32_t hi = h ? sec[5] : sec[1];
                    ffl = P.notri ? (h ? sec[4] : sec[0]) >> 30 : 0u;
                    fnlo = h ? sec[6] : sec[2];
                    fnhi = h ? sec[7] : sec[3];
                    fnshi = P.wsym ? hi : 0u;
                    fnslo = P.wsym ? hi - (fnhi - fnlo) : 1u;   // [1, 0): unknown (asymmetric weights)
                } else {                                 // unweighted: index intervals
                    uint32_t rev;
                    if constexpr (COMPACT) {
                        rev = hrev;
                        ffl = hfl;
                    } else {
                        rev = hrev;
                        fxs = hxs;
                        if constexpr (WIDE) fxs |= (off_t_)((hxd >> 26) & 3u) << 32;
                        ffl = (hxd >> 28) & 3u;
                        fxd = hxd & kDegMask;
                        fxw = fxd;
                    }
                    (void)kept;
                    fnlo = rev;
                    fnhi = rev == kNone ? rev : rev + 1;   // [rev, rev+1), or the empty [NONE, NONE)
                    fnslo = ri;
                    fnshi = ri + 1;
                }
                if (!(COMPACT && x == tid)) {
                    tid = vid; tstart = vstart; tdeg = vdeg; tW = vW;
                    vid = x;
                    if constexpr (COMPACT) need_node = true;   // x's node record: next iteration
                    else { vstart = fxs; vdeg = fxd; vW = fxw; }
                } else {   // compact record of a return: t's node record is in registers
                    GRAPE_SWAP_VT();
                }
                tlo = fnlo; thi = fnhi; slo = fnslo; shi = fnshi;
                nt = (ffl >> 1) != 0; ntr = (ffl & 1) != 0;
            } else {   // x = t: v and t swap, and so do T and S
                const bool b_ = nt; nt = ntr; ntr = b_;
                GRAPE_SWAP_VT();
                uint32_t q;
                q = tlo; tlo = slo; slo = q;
                q = thi; thi = shi; shi = q;
            }
            ++s;
            a = 0;
            cb = 0;
            if (need_node) {
                fin = s == L;
                if (!fin) {
                    st = ST_NODE;
                    idx = x;
                }
            } else {
                fin = s == L || vdeg == 0;
                draw = !fin;
            }
        }
        if (fin) {
            w.pad(s, L);
            w.finish(L);
            // next walk: round-robin over the statically assigned prefix [0, P.nstatic),
            // then from the shared counter (balances the tail across lanes)
            i += stride;
            if (i >= P.nstatic) {
                const unsigned am = __activemask();
                const int leader = __ffs(am) - 1;
                const unsigned rank = __popc(am & ((1u << (threadIdx.x & 31)) - 1));
                unsigned long long b0 = 0;
                if ((int)(threadIdx.x & 31) == leader) b0 = atomicAdd(P.next, (unsigned long long)__popc(am));
                i = P.nstatic + __shfl_sync(am, b0, leader) + rank;
            }
            st = i < P.num_walks ? ST_START : ST_DONE;
            draw = false;
        }

        // ---- draws: Philox, the band of u, and the decisions that need no read
        // (§8(c) c12).  A lane whose attempt is decided from registers draws again
        // in the same iteration, up to GRAPE_TAB_DRAWS draws; a register-decided
        // return x = t ends the lane's draws (ST_BACK: emitted by the next iteration).
#pragma unroll kDrawUnroll
        for (int k = 0; k < GRAPE_TAB_DRAWS; ++k) {
            if (GRAPE_TAB_SYNC_DRAW) __syncwarp();
            if (!__any_sync(0xffffffffu, draw)) break;
            const bool sub = SUSS && vdeg > P.dT;   // this step runs on a SUSS sub-sample
            if (SUSS && WEIGHTED && draw && sub && cb < P.dT) {   // first: read the dT candidates
                wc = 0;
                bt = kNone;
                if constexpr (!COMPACT) {
                    // full records carry both ends of a candidate's interval: all dT records are
                    // read in this iteration, two candidates per Philox block (candidates 2k and
                    // 2k+1 take its two halves, as suss_index does), the row-local bucket bounds
                    // floor(b deg / dT) stepped incrementally (quotient and remainder)
                    const uint32_t dq = vdeg / P.dT, dr = vdeg - dq * P.dT;
                    uint32_t lq = 0, lr = 0;   // floor(b deg / dT), b deg mod dT
                    auto next_bound = [&]() {
                        lq += dq;
                        lr += dr;
                        if (lr >= P.dT) { lr -= P.dT; ++lq; }
                    };
#pragma unroll kSussUnroll
                    for (uint32_t b = 0; b < P.dT; b += 2) {
                        const uint4 o = philox_block_rk(P.rk, P.base + i, s, 0x80000000u | (b >> 1));
                        const bool two = b + 1 < P.dT;
                        const uint32_t l0 = lq;
                        next_bound();
                        const uint32_t l1 = lq;
                        if (two) next_bound();
                        const uint32_t l2 = lq;
                        const uint32_t i0 = l0 + bounded32((uint64_t)o.y << 32 | o.x, l1 - l0);
                        const uint32_t i1 = two ? l1 + bounded32((uint64_t)o.w << 32 | o.z, l2 - l1) : i0;
                        GRAPE_DCHECK(i0 < vdeg && i1 < vdeg, "SUSS candidate within the row");
                        const uint32_t* r0 = (const uint32_t*)P.rec + ((uint64_t)vstart + i0) * 8;
                        const uint32_t* r1 = (const uint32_t*)P.rec + ((uint64_t)vstart + i1) * 8;
                        const uint2 a0 = __ldg((const uint2*)r0), a1 = __ldg((const uint2*)r1);   // {x, hi}
                        const uint32_t z0 = __ldg(r0 + 7), z1 = __ldg(r1 + 7);                 // lo
                        if (STATS) {
                            cnt[C_LOADS] += two ? 2 : 1;
                            cnt[C_REC] += two ? 2 : 1;
                        }
                        wc += a0.y - z0;
                        P.scratch[(uint64_t)(2 * b) * P.lanes + gl] = wc;
                        P.scratch[(uint64_t)(2 * b + 1) * P.lanes + gl] = a0.x;
                        if (a0.x == tid) bt = b;
                        if (two) {
                            wc += a1.y - z1;
                            P.scratch[(uint64_t)(2 * b + 2) * P.lanes + gl] = wc;
                            P.scratch[(uint64_t)(2 * b + 3) * P.lanes + gl] = a1.x;
                            if (a1.x == tid) bt = b + 1;
                        }
                    }
                    cb = P.dT;   // the sub-sample is in scratch: this round draws on it
                } else {   // compact records: one candidate per iteration (ST_CAND; a weight may need
                           // the predecessor's record)
                    draw = false;
                    cph = false;
                    ri = suss_index(0);
                    st = ST_CAND;
                }
            }
            if (draw) draw_once(GRAPE_TAB_EMIT_SPOT && k + 1 < GRAPE_TAB_DRAWS, sub);
        }
        if (draw) st = ST_DRAW;   // still drawing: no load next iteration
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

#undef GRAPE_SWAP_VT

template <bool WEIGHTED, bool FAT, bool COMPACT, bool NODE2VEC, bool NEED_MEMBER, bool STATS, int MODE,
          bool WIDE = false>
cudaError_t launch_k(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    TabParams P = tab_params(g, a, T);
    if (MODE == 2) {   // A_c = ceil(min(T_c, E) 2^32 / E); accept iff u < A_c
        const uint64_t E = T.T1 > T.Tq ? T.T1 : T.Tq;
        auto A = [&](uint64_t tc) {
            const uint64_t m = tc < E ? tc : E;
            return (uint64_t)((((unsigned __int128)m << 32) + E - 1) / E);
        };
        P.tp_m1 = (uint32_t)(A(T.Tp) - 1);
        P.t1_m1 = (uint32_t)(A(T.T1) - 1);
        P.tq_m1 = (uint32_t)(A(T.Tq) - 1);
        P.fold_e = (uint32_t)E;   // < 2^32: T_p > E
        P.fold_x = (uint32_t)(T.Tp - E);
    }
    constexpr bool SUSS = MODE == 1;
    return launch_tab_grid(walk_tab_kernel<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, STATS, MODE, WIDE>, P, g, a,
                           SUSS && WEIGHTED ? 2ull * a.dT : 0ull, stream);
}

template <bool WEIGHTED, bool FAT, bool COMPACT, bool NODE2VEC, bool NEED_MEMBER>
cudaError_t launch_s(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream)
{
    // approximated walks only when some row exceeds the threshold (else they are the exact walks)
    if (a.dT != 0 && a.dT < g->max_degree) {
        if (a.stats != nullptr) return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, true, true, 1>(g, a, T, stream);
        return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, true, false, 1>(g, a, T, stream);
    }
    // outlier folding only when the return class dominates (else it is the default rule)
    if (NODE2VEC && a.sampler == 2 && T.Tp > (T.T1 > T.Tq ? T.T1 : T.Tq)) {
        if (a.stats != nullptr) return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, true, true, 2>(g, a, T, stream);
        return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, true, false, 2>(g, a, T, stream);
    }
    if (g->wide) {   // 34-bit arc offsets: the default rule, contiguous or partitioned tables (capi.cu)
        if (g->parts > 1) {
            if (a.stats != nullptr) return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, true, 3, true>(g, a, T, stream);
            return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, false, 3, true>(g, a, T, stream);
        }
        if (a.stats != nullptr) return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, true, 0, true>(g, a, T, stream);
        return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, false, 0, true>(g, a, T, stream);
    }
    if (g->parts > 1) {   // partitioned tables: the default rule only (capi.cu rejects the other modes)
        if (a.stats != nullptr) return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, true, 3>(g, a, T, stream);
        return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, false, 3>(g, a, T, stream);
    }
    if (a.stats != nullptr) return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, true, 0>(g, a, T, stream);
    return launch_k<WEIGHTED, FAT, COMPACT, NODE2VEC, NEED_MEMBER, false, 0>(g, a, T, stream);
}

template <bool WEIGHTED, bool FAT, bool COMPACT>
cudaError_t dispatch(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                     cudaStream_t stream)
{
    if (!node2vec || (T.Tp == T.T1 && T.T1 == T.Tq))
        return launch_s<WEIGHTED, FAT, COMPACT, false, false>(g, a, T, stream);
    if (T.T1 != T.Tq) return launch_s<WEIGHTED, FAT, COMPACT, true, true>(g, a, T, stream);
    return launch_s<WEIGHTED, FAT, COMPACT, true, false>(g, a, T, stream);
}

}  // namespace

cudaError_t launch_walks_tab(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                             cudaStream_t stream)
{
    if (g->cw_bytes == 0) {
        if (g->compact) return dispatch<false, false, true>(g, a, node2vec, T, stream);
        return dispatch<false, false, false>(g, a, node2vec, T, stream);
    }
    if (g->compact) return dispatch<true, false, true>(g, a, node2vec, T, stream);
    if (g->guide_bytes == 32) return dispatch<true, true, false>(g, a, node2vec, T, stream);
    return dispatch<true, false, false>(g, a, node2vec, T, stream);
}

}  // namespace grape
