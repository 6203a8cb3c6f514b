// build_common.cuh — work distribution of the one-off graph-build kernels
// (graph.cu, graph_tables.cu; not on the timed path).
//
// The build kernels answer per-arc questions (is the reverse arc there, where is
// it, do t and v share a neighbour, which slot holds x).  Distributing them one
// warp per row left hub rows (10^5-10^6 arcs) to a single warp each: the launch
// ended with a few warps grinding through hubs (build).  Here the
// unit is the arc: thread i of the grid takes arcs i, i + stride, ...; the source
// row of arc e comes from a binary search of off[] (consecutive lanes search
// neighbouring values, so the search path is shared in L1).
#pragma once
#include <cstdint>

namespace grape {
namespace build {

// The row v holding arc e: off[v] <= e < off[v + 1] (e < off[n]).  Of equal offsets
// (empty rows) the largest index is taken, which is the non-empty row.
__device__ __forceinline__ uint32_t row_of(const uint64_t* __restrict__ off, uint32_t n, uint64_t e)
{
    uint32_t lo = 0, hi = n - 1;   // off[lo] <= e < off[hi + 1]
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo + 1) >> 1);
        if (__ldg(off + mid) <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Grid for a per-item grid-stride kernel of 256 threads: 8 blocks per SM of the
// current device, at most enough for the items.
inline int item_grid(uint64_t items, int sms)
{
    uint64_t blocks = (items + 255) / 256;
    const uint64_t cap = (uint64_t)(sms > 0 ? sms : 148) * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

}  // namespace build
}  // namespace grape
