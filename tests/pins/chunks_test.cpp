// Host-side check of the chunked table layout shared by grape_graph_partition and the
// distributed build (paper_2110_06196_b200/csrc/internal.h: chunk_shift, owner_range,
// map_chunks): owners' byte ranges tile the table exactly, differ by at most one chunk,
// start on chunk boundaries, and map_chunks resolves every byte offset to the owner's
// allocation at the right place.  Built and run by tests/test_capi_host.py (no GPU).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2110_06196_b200/csrc/internal.h"

using namespace grape;

static int fails = 0;
#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

int main()
{
    const uint64_t sizes[] = {1, 31, 32, 2097152, 2097153, 123456789, 1ull << 30, (1ull << 30) + 96,
                              22000000032ull, 68000000000ull, 250000000000ull};
    for (uint64_t bytes : sizes) {
        const uint32_t k = chunk_shift(bytes);
        CHECK(k >= 21 && (1ull << k) * kChunks >= bytes);
        CHECK(k == 21 || (1ull << (k - 1)) * kChunks < bytes);   // the smallest such k
        const uint64_t C = chunk_count(bytes, k);
        CHECK(C <= (uint64_t)kChunks && C >= 1);
        for (uint32_t parts = 1; parts <= 8; ++parts) {
            uint64_t prev = 0, mn = ~0ull, mx = 0;
            std::vector<char*> owner(8, nullptr);
            std::vector<uint64_t> lo(parts), hi(parts);
            for (uint32_t j = 0; j < parts; ++j) {
                owner_range(bytes, k, j, parts, &lo[j], &hi[j]);
                CHECK(lo[j] == prev);                           // contiguous, in order
                CHECK(lo[j] % (1ull << k) == 0 || lo[j] == bytes);   // chunk-aligned starts
                prev = hi[j];
                const uint64_t chunks = ((hi[j] - lo[j]) + (1ull << k) - 1) >> k;
                if (chunks < mn) mn = chunks;
                if (chunks > mx) mx = chunks;
                owner[j] = reinterpret_cast<char*>(0x100000000ull * (j + 1));   // fake, distinct bases
            }
            CHECK(prev == bytes);                               // the ranges tile the table
            CHECK(mx - mn <= 1);                                // balanced to one chunk
            char* map[kChunks];
            map_chunks(owner.data(), bytes, k, parts, map);
            // every probed offset lands in its owner's allocation at offset - lo
            const uint64_t probes[] = {0, bytes / 3, bytes / 2, bytes - 1, (1ull << k) - 1, 1ull << k};
            for (uint64_t off : probes) {
                if (off >= bytes) continue;
                uint32_t j = 0;
                while (!(off >= lo[j] && off < hi[j])) ++j;
                char* got = map[off >> k] + (off & ((1ull << k) - 1));
                CHECK(got == owner[j] + (off - lo[j]));
            }
        }
    }
    if (fails == 0) std::printf("chunks_test: ok\n");
    return fails ? 1 : 0;
}
