// Pin for the oracle's Philox4x32-10 (oracle/grape_oracle.c): compare it, on
// the HOST, with the CUDA toolkit's own independent implementation
// curand_Philox4x32_10 (/usr/local/cuda/include/curand_philox4x32_x.h), over
// N pseudo-random (counter, key) pairs plus edge patterns.  The header's
// QUALIFIERS macro is redefined so its functions compile as host code; its
// mulhilo32 has an explicit host branch.  Test infrastructure only.
#define QUALIFIERS static inline __host__ __device__
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

extern "C" void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

static uint64_t sm64(uint64_t& s) {  // splitmix64 stream for test inputs
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int main(int argc, char** argv) {
    long n = argc > 1 ? atol(argv[1]) : 1000000;
    uint64_t s = argc > 2 ? strtoull(argv[2], 0, 0) : 1;
    long bad = 0;
    for (long i = 0; i < n + 4; i++) {
        uint32_t c[4], k[2], o[4];
        if (i < n) {
            uint64_t a = sm64(s), b = sm64(s), d = sm64(s);
            c[0] = (uint32_t)a; c[1] = (uint32_t)(a >> 32); c[2] = (uint32_t)b; c[3] = (uint32_t)(b >> 32);
            k[0] = (uint32_t)d; k[1] = (uint32_t)(d >> 32);
            if (i % 7 == 0) { c[1] = 0; c[3] = (uint32_t)(i & 0xFF); }   // walk-like counters
        } else {  // edge patterns: all-zero, all-one words
            uint32_t v = (i - n) & 1 ? 0xFFFFFFFFu : 0u, kv = (i - n) & 2 ? 0xFFFFFFFFu : 0u;
            c[0] = c[1] = c[2] = c[3] = v; k[0] = k[1] = kv;
        }
        uint4 cc = make_uint4(c[0], c[1], c[2], c[3]);
        uint2 kk = make_uint2(k[0], k[1]);
        uint4 r = curand_Philox4x32_10(cc, kk);
        oracle_philox4x32_10(c, k, o);
        if (r.x != o[0] || r.y != o[1] || r.z != o[2] || r.w != o[3]) {
            if (bad < 5)
                printf("MISMATCH ctr=%08x %08x %08x %08x key=%08x %08x curand=%08x %08x %08x %08x oracle=%08x %08x %08x %08x\n",
                       c[0], c[1], c[2], c[3], k[0], k[1], r.x, r.y, r.z, r.w, o[0], o[1], o[2], o[3]);
            bad++;
        }
    }
    printf("checked=%ld mismatches=%ld\n", n + 4, bad);
    return bad != 0;
}
