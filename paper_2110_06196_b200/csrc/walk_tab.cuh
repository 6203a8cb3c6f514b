// walk_tab.cuh — the table walker's parameters, their host-side fill, the
// persistent-grid launch, and the device helpers (bounded draws, sector loads,
// the edge-hash mix) — kept apart from the state machine (walk_tab.cu) so a
// variant kernel can share them (DESIGN.md §7 lists the variants measured).  Internal.
#pragma once
#include "walk_common.cuh"

#ifndef GRAPE_TAB_MIN_BLOCKS
#define GRAPE_TAB_MIN_BLOCKS 4   // resident blocks per SM the table walkers are compiled for
#endif

namespace grape {
namespace {
using namespace walk;

constexpr uint32_t kEmptySlot = 0xFFFFFFFFu;
struct TabParams {
    const NodeRec* nodes;
    const void* rec;          // arc records (16 or 32 B)
    const uint32_t* guide;    // 8-B entries
    const uint32_t* ehash;
    uint32_t G;               // guide buckets per arc
    uint32_t h_mul, h_shift;  // floor(v / H) = umulhi(v, h_mul) >> h_shift (edge-hash buckets)
    bool wsym;                // weighted: reverse arcs carry equal weights
    bool notri;               // records carry the no-common-neighbour flags
    uint32_t xmask;           // compact records: x without its flag bits
    uint32_t dT;              // approximated walks (SUSS): degree threshold
    uint32_t* scratch;        // SUSS, weighted: per lane 2 dT words, [2 b + {0: running weight, 1: x}][lane]
    uint32_t lanes;           // resident lanes of the launch (scratch stride)
    uint32_t fold_e, fold_x;  // outlier-folded rule: E = max(T_1, T_q), X = T_p - E (thresholds hold A_c)
    uint64_t nstatic;         // walks [0, nstatic) go round-robin to the lanes; the rest via *next
    unsigned long long* next; // shared walk counter (starts at nstatic)
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
    const PartMap* pmap;            // MODE 3 (§8(f) f4 layout, partition.cu): the partition map
    const char* tbl_base[6];        // per load state (ST_START .. ST_CAND): the table it reads
    uint32_t tbl_shift[6];          //   and log2 of its entry size
    uint32_t tbl_mul[6];            //   and how many entries it holds per arc of the row start (0: not per row)
#if GRAPE_CHECKED
    uint64_t lim[4];                // checked build: bytes of records, guide, node records, edge hash
    uint64_t m;
#endif
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

// floor(x64 * w / 2^64) for w < 2^32 (§8(c) c8) from two 32x32 products:
// x64 w = x_hi w 2^32 + x_lo w, and the dropped fraction of x_lo w / 2^32 never
// carries across a multiple of 2^32.
__device__ __forceinline__ uint32_t bounded32(uint64_t x64, uint32_t w)
{
    const uint32_t lo = __umulhi((uint32_t)x64, w);                             // IMAD.HI
    return (uint32_t)(((uint64_t)(uint32_t)(x64 >> 32) * w + lo) >> 32);      // IMAD.WIDE + carry word
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
             C_GUIDE, C_HASH, C_ALU, C_ITER, C_ITER_DRAW, C_ITER_BACK };

// The parameters every table-walker launch shares (tables, thresholds, walk
// arguments); the launcher adds the grid-dependent ones (lanes, nstatic, next,
// scratch).  Thresholds: accept iff u <= T_c - 1 (§8(c) c9).
inline TabParams tab_params(const grape_graph* g, const WalkArgs& a, const Thresholds& T)
{
    TabParams P{};
    P.pmap = g->part_map;
    P.nodes = g->nodes;
    P.rec = g->rec;
    P.guide = g->guide;
    P.ehash = g->ehash;
    P.G = g->guide_factor;
    if (g->arc_bias) {   // test hook (graph_tables.cu): row starts are biased; the bases move back
        const uint64_t b = g->arc_bias;
        P.rec = (const char*)g->rec - b * g->rec_bytes;
        P.guide = (const uint32_t*)((const char*)g->guide - b * g->guide_factor * g->guide_bytes);
        P.ehash = (const uint32_t*)((const char*)g->ehash - (b / g->hash_h) * 32);
    }
    if (g->hash_h == 6) { P.h_mul = 0xAAAAAAABu; P.h_shift = 2; }   // floor(v/6) = umulhi(v, ceil(2^34/6)) >> 2
    else { P.h_mul = 0x40000000u; P.h_shift = 0; }                  // floor(v/4)
    P.wsym = g->wsym;
    P.notri = g->notri;
    P.xmask = (g->notri && g->compact) ? 0x3FFFFFFFu : 0xFFFFFFFFu;
    P.n = g->n;
    P.starts = a.starts;
    P.num_walks = a.num_walks;
    P.base = a.walk_id_base;
    P.L = a.L;
    P.rk = philox_round_keys(a.seed);
    P.out = a.out;
    P.steps_out = a.steps_out;
    P.stats = a.stats;
    auto lg2 = [](uint32_t b) { uint32_t k = 0; while ((1u << k) < b) ++k; return k; };
    P.tbl_base[0] = (const char*)P.starts;  P.tbl_shift[0] = 2;
    P.tbl_base[1] = (const char*)P.nodes;   P.tbl_shift[1] = 4;
    P.tbl_base[2] = (const char*)P.guide;   P.tbl_shift[2] = lg2(g->guide_bytes ? g->guide_bytes : 8);
    P.tbl_base[3] = (const char*)P.rec;     P.tbl_shift[3] = lg2(g->rec_bytes ? g->rec_bytes : 32);
    P.tbl_base[4] = (const char*)P.ehash;   P.tbl_shift[4] = 5;
    P.tbl_base[5] = (const char*)P.rec;     P.tbl_shift[5] = P.tbl_shift[3];
    P.tbl_mul[2] = P.G; P.tbl_mul[3] = 1; P.tbl_mul[5] = 1;   // (P{} zeroed the rest)
    P.tp_m1 = (uint32_t)(T.Tp - 1);
    P.t1_m1 = (uint32_t)(T.T1 - 1);
    P.tq_m1 = (uint32_t)(T.Tq - 1);
    P.dT = a.dT;
#if GRAPE_CHECKED
    P.lim[0] = g->rec_alloc;
    P.lim[1] = g->guide_alloc;
    P.lim[2] = ((uint64_t)g->n * sizeof(NodeRec) + 31) / 32 * 32 + 32;
    P.lim[3] = g->hash_alloc;
    P.m = g->m;
#endif
    return P;
}

#ifndef GRAPE_TAB_DYN_MIN_ROUNDS
#define GRAPE_TAB_DYN_MIN_ROUNDS 2
#endif
#ifndef GRAPE_TAB_STATIC_PCT
#define GRAPE_TAB_STATIC_PCT 50
#endif

// Launch a persistent table-walker grid: resident blocks x SMs of the graph's device
// (cached per kernel and device), at most one lane per walk.  Walk assignment:
// GRAPE_TAB_STATIC_PCT percent of the walks, in whole rounds of the grid, go
// round-robin to the lanes; the rest come from a warp-aggregated shared counter
// (launches of under GRAPE_TAB_DYN_MIN_ROUNDS rounds are all static: no counter to
// allocate).  scratch_words: per-lane u32 scratch (SUSS candidates), stream-ordered.
template <typename Kernel>
cudaError_t launch_tab_grid(Kernel kern, TabParams& P, const grape_graph* g, const WalkArgs& a,
                            uint64_t scratch_words, cudaStream_t stream)
{
    const int resident = resident_blocks((const void*)kern, kBlock, 0, g->device);
    uint64_t blocks = (a.num_walks + kBlock - 1) / kBlock;
    if (blocks > (uint64_t)resident) blocks = resident;
    P.lanes = (uint32_t)(blocks * kBlock);
    const uint64_t rounds = a.num_walks / P.lanes;
    uint64_t srounds = rounds * GRAPE_TAB_STATIC_PCT / 100;
    if (srounds < 1) srounds = 1;
    const bool dyn = rounds >= GRAPE_TAB_DYN_MIN_ROUNDS;
    P.nstatic = dyn ? srounds * P.lanes : ~0ull;   // >= lanes: every lane's first walk is static
    cudaError_t e = cudaSuccess;
    if (dyn) {
        e = cudaMallocAsync((void**)&P.next, 8, stream);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(P.next, 0, 8, stream);
    }
    if (e == cudaSuccess && scratch_words)
        e = cudaMallocAsync((void**)&P.scratch, scratch_words * P.lanes * 4, stream);
    if (e == cudaSuccess) {
        kern<<<(unsigned)blocks, kBlock, 0, stream>>>(P);
        e = cudaGetLastError();
    }
    if (P.scratch) cudaFreeAsync(P.scratch, stream);
    if (P.next) cudaFreeAsync(P.next, stream);
    return e;
}

}  // namespace
}  // namespace grape
