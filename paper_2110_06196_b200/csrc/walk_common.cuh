// walk_common.cuh — device building blocks shared by the walk kernels
// (walk_sm.cu, walk_tab.cu, walk_cdf.cu): the v3 kernel parameters, the staged
// row writer, the step counter.  Internal to libgrape_walk.
#pragma once
#include <cstdint>
#include <type_traits>
#include "internal.h"
#include "philox.cuh"

namespace grape {
namespace walk {


constexpr uint32_t kPad = 0xFFFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
#ifndef GRAPE_BLOCK
#define GRAPE_BLOCK 256
#endif
constexpr int kBlock = GRAPE_BLOCK;   // threads per block of the walk kernels
#ifndef GRAPE_MIN_BLOCKS
#define GRAPE_MIN_BLOCKS 4
#endif
constexpr int kMinBlocks = GRAPE_MIN_BLOCKS;   // 4 x 256 threads/SM -> <= 64 registers
constexpr int NL = kFenceLevels;

struct Unweighted {};

template <typename T>
struct Levels {
    const T* a[NL + 1];   // a[0] = the array itself, a[1..NL] = its fence levels
};

template <typename CW>
using CwStore = typename std::conditional<std::is_same<CW, Unweighted>::value, uint32_t, CW>::type;

// Kernel parameters (constant bank; nothing here occupies registers until used).
template <typename CW>
struct Params {
    const NodeRec* nodes;
    Levels<uint32_t> col;
    Levels<CwStore<CW>> cw;
    uint32_t n;
    const uint32_t* starts;
    uint64_t num_walks;
    uint64_t base;
    uint32_t L;
    uint32_t k0, k1;
    RoundKeys rk;          // Philox round keys of the seed
    uint32_t* out;
    unsigned long long* steps_out;
    unsigned long long* stats;   // diagnostics counters (grape_walks_stats) or NULL
    // acceptance: u < T  <=>  u <= T - 1  (T in [1, 2^32], so T - 1 fits u32)
    uint32_t tp_m1, t1_m1, lo_m1, hi_m1;
    bool member_accepts;   // for u in [T_lo, T_hi): accepted iff (x in N(t)) == (T_1 > T_q)
};

__device__ __forceinline__ void st_cs_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Per-thread output staging: 8 u32 slots in shared memory (transposed, so the
// 32 lanes of a warp hit 32 banks), flushed as one aligned 32-B sector.  Entry
// s of a row goes to slot (phase + s) & 7, phase = the row's 4-B offset within
// its 32-B sector, so a flush at slot 7 always ends a real sector of `out`.
#ifndef GRAPE_ROW_OUTLINE
#define GRAPE_ROW_OUTLINE 0   // the partial-sector flush as a call (keeps its loop out of the walkers' hot code)
#endif
// entries [first, end) of a row from their staging slots, one by one (a row's partial
// first or last sector)
#if GRAPE_ROW_OUTLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void flush_entries(uint32_t* row, const uint32_t* slot, uint32_t phase, uint32_t first, uint32_t end)
{
    for (uint32_t q = first; q < end; ++q) row[q] = slot[((phase + q) & 7) * kBlock];
}

struct RowWriter {
    uint32_t* slot;     // &smem[tid]; slot j at slot[j * kBlock]
    uint32_t* row;      // &out[i * L]
    uint32_t phase;     // (row address / 4) & 7
    uint32_t first;     // first unflushed entry of the row

    __device__ __forceinline__ void begin(uint32_t* row_)
    {
        row = row_;
        phase = (uint32_t)(((uintptr_t)row_ >> 2) & 7);
        first = 0;
    }
    __device__ __forceinline__ void put(uint32_t s, uint32_t x)
    {
        const uint32_t j = (phase + s) & 7;
        slot[j * kBlock] = x;
        if (j == 7) {
            if (s >= first + 7) {   // the whole sector belongs to this row
                uint32_t* p = row + s - 7;
                st_cs_v4(p, slot[0], slot[kBlock], slot[2 * kBlock], slot[3 * kBlock]);
                st_cs_v4(p + 4, slot[4 * kBlock], slot[5 * kBlock], slot[6 * kBlock], slot[7 * kBlock]);
            } else {
                flush_entries(row, slot, phase, first, s + 1);
            }
            first = s + 1;
        }
    }
    // entries [s, end) = PAD (a dead end or the end of an early-ending walk): the staged
    // entries [first, s) are written out, then PAD with 16-B stores where aligned
    __device__ __forceinline__ void pad(uint32_t s, uint32_t end)
    {
        finish(s);
        uint32_t q = s;
        for (; q < end && (((uintptr_t)(row + q)) & 15) != 0; ++q) row[q] = kPad;
        for (; q + 4 <= end; q += 4) st_cs_v4(row + q, kPad, kPad, kPad, kPad);
        for (; q < end; ++q) row[q] = kPad;
        first = end;
    }
    __device__ __forceinline__ void finish(uint32_t end)   // flush [first, end)
    {
        flush_entries(row, slot, phase, first, end);
    }
};

__device__ __forceinline__ void add_steps(unsigned long long* steps_out, unsigned long long mine)
{
    if (steps_out == nullptr) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(steps_out, mine);
}

template <typename T>
Levels<T> levels_of(const void* base, void* const* fences)
{
    Levels<T> lv;
    lv.a[0] = (const T*)base;
    for (int l = 0; l < NL; ++l) lv.a[l + 1] = (const T*)fences[l];
    return lv;
}

template <typename CW>
Params<CW> make_params(const grape_graph* gg, const WalkArgs& a, const Thresholds& T)
{
    Params<CW> P{};
    P.nodes = gg->nodes;
    P.col = levels_of<uint32_t>(gg->col, (void* const*)gg->col_fence);
    if constexpr (!std::is_same<CW, Unweighted>::value) P.cw = levels_of<CW>(gg->cw, gg->cw_fence);
    P.n = gg->n;
    P.starts = a.starts;
    P.num_walks = a.num_walks;
    P.base = a.walk_id_base;
    P.L = a.L;
    P.k0 = (uint32_t)a.seed;
    P.k1 = (uint32_t)(a.seed >> 32);
    P.rk = philox_round_keys(a.seed);
    P.out = a.out;
    P.steps_out = a.steps_out;
    P.stats = a.stats;
    const uint64_t lo = T.T1 < T.Tq ? T.T1 : T.Tq, hi = T.T1 < T.Tq ? T.Tq : T.T1;
    P.tp_m1 = (uint32_t)(T.Tp - 1);
    P.t1_m1 = (uint32_t)(T.T1 - 1);
    P.lo_m1 = (uint32_t)(lo - 1);
    P.hi_m1 = (uint32_t)(hi - 1);
    P.member_accepts = T.T1 > T.Tq;
    return P;
}

}  // namespace walk
}  // namespace grape
