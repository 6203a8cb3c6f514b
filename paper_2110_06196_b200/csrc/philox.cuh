// philox.cuh — device Philox4x32-10 and the bounded-integer map (§8(c) c7, c8).
//
// Philox4x32-10 (Salmon et al., SC'11): ten rounds of
//   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;  c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0)
// with the key bumped by (W0, W1) between rounds.  Counter = (wid lo, wid hi,
// step, attempt), key = seed (include/grape_walk.h).  Written for the GPU:
// __umulhi + IMAD for the 32x32->64 products, fully unrolled, state in
// registers; round keys are seed + r*W (one add each, hoisted by ptxas).
#pragma once
#include <cstdint>

namespace grape {

struct Draw {
    uint64_t x64;   // o1 << 32 | o0  — proposal draw
    uint32_t u;     // o2             — acceptance draw
};

__device__ __forceinline__ Draw philox_draw(uint32_t k0, uint32_t k1, uint64_t wid,
                                            uint32_t step, uint32_t attempt)
{
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = (uint32_t)wid, c1 = (uint32_t)(wid >> 32), c2 = step, c3 = attempt;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
        const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    Draw d;
    d.x64 = ((uint64_t)c1 << 32) | c0;
    d.u = c2;
    return d;
}

// Round keys of Philox4x32-10 for a seed: rk[2r], rk[2r+1] = key + r * (W0, W1)
// (mod 2^32), r = 0..9 — computed once on the host and passed in the kernel
// parameters, so every round's XOR takes its key straight from the constant bank.
struct RoundKeys {
    uint32_t k[20];
};

inline RoundKeys philox_round_keys(uint64_t seed)
{
    RoundKeys rk;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = k0;
        rk.k[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return rk;
}

__device__ __forceinline__ Draw philox_draw_rk(const RoundKeys& rk, uint64_t wid, uint32_t step, uint32_t attempt)
{
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t c0 = (uint32_t)wid, c1 = (uint32_t)(wid >> 32), c2 = step, c3 = attempt;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;   // IMAD.WIDE.U32
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    Draw d;
    d.x64 = ((uint64_t)c1 << 32) | c0;
    d.u = c2;
    return d;
}

// All four output words (c0, c1, c2, c3) of the block for counter (wid, step, word3).
__device__ __forceinline__ uint4 philox_block_rk(const RoundKeys& rk, uint64_t wid, uint32_t step, uint32_t word3)
{
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t c0 = (uint32_t)wid, c1 = (uint32_t)(wid >> 32), c2 = step, c3 = word3;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

// floor(x64 * W / 2^64): the high word of the 128-bit product (§8(c) c8).
__device__ __forceinline__ uint64_t bounded64(uint64_t x64, uint64_t W)
{
    return __umul64hi(x64, W);
}

}  // namespace grape
