// partition.cu — the §8(f) f4 table layout: the sampling tables of
// a built graph split into chunks of 2^k bytes (at most kChunks per table), owner j
// of `parts` holding a contiguous range of chunks on device devices[j], read by
// the walker over NVLink peer access.  The walker's single address computation
// resolves base[T][offset >> k] + (offset & (2^k - 1)) (walk_tab.cu, MODE 3), so
// every walk is the one the contiguous tables give.
//
// This first form partitions a graph that was built on one GPU (the build itself is
// not distributed): it places the tables of a graph over several GPUs' memory and
// measures the addressing; a graph larger than one HBM additionally needs the
// build to write each part on its owner.
#include "internal.h"

namespace grape {
namespace {

struct Split {
    void* mem[8] = {};    // owner j's contiguous range (chunks [C j / parts, C (j+1) / parts))
    uint32_t shift = 63;  // chunk size 2^shift
};

// copy table bytes at src (on the graph's device) into owner ranges of 2^k-byte chunks
cudaError_t split(const grape_graph* g, const void* src, uint64_t bytes, uint32_t parts, const int* devices,
                  Split& out)
{
    const uint32_t k = chunk_shift(bytes);
    out.shift = k;
    cudaError_t e = cudaSuccess;
    for (uint32_t j = 0; j < parts && e == cudaSuccess; ++j) {
        uint64_t lo, hi;
        owner_range(bytes, k, j, parts, &lo, &hi);
        if (hi == lo) continue;   // (fewer chunks than owners) never addressed
        {   // whole 2 MB pages (see dist.cu: ragged last pages of shared allocations were slow)
            DeviceGuard on(devices[j]);
            e = cudaMalloc(&out.mem[j], ((hi - lo) + (2ull << 20) - 1) & ~((2ull << 20) - 1));
        }
        if (e == cudaSuccess) e = cudaMemcpyPeer(out.mem[j], devices[j], (const char*)src + lo, g->device, hi - lo);
    }
    return e;
}

void release(Split& s, uint32_t parts)
{
    for (uint32_t j = 0; j < parts; ++j) {
        if (s.mem[j]) cudaFree(s.mem[j]);
        s.mem[j] = nullptr;
    }
}

}  // namespace
}  // namespace grape

using namespace grape;

extern "C" grape_status grape_graph_partition(grape_graph* g, uint32_t parts, const int* devices)
{
    if (g == nullptr || parts < 2 || parts > 8 || devices == nullptr) {
        set_error("grape_graph_partition: need a graph, 2 <= parts <= 8 and a device list");
        return GRAPE_EINVAL;
    }
    if (!g->tables || g->parts != 1 || g->arc_bias != 0) {
        set_error("grape_graph_partition: the graph has no sampling tables, or is already partitioned");
        return GRAPE_EINVAL;
    }
    // every step below (peer access, synchronisation, the device partition map) on the
    // graph's device, whatever device the caller has current
    DeviceGuard guard(g->device);
    if (!guard.ok) {
        set_error("grape_graph_partition: cannot make the graph's device %d current", g->device);
        return GRAPE_ECUDA;
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    for (uint32_t j = 0; j < parts; ++j) {
        if (devices[j] < 0 || devices[j] >= ndev) {
            set_error("grape_graph_partition: device %d does not exist", devices[j]);
            return GRAPE_EINVAL;
        }
        if (devices[j] == g->device) continue;
        int ok = 0;   // the walker on g->device reads part j over NVLink
        cudaDeviceCanAccessPeer(&ok, g->device, devices[j]);
        if (!ok) {
            set_error("grape_graph_partition: device %d cannot access device %d", g->device, devices[j]);
            return GRAPE_EINVAL;
        }
        e = cudaDeviceEnablePeerAccess(devices[j], 0);   // (the graph's device is current)
        if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
        cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
    e = cudaDeviceSynchronize();
    // copy every table into its parts first; the graph changes only if all succeed
    const void* src[4] = {g->rec, g->guide, g->nodes, g->ehash};
    const uint64_t bytes[4] = {g->rec_alloc, g->guide ? g->guide_alloc : 0, (uint64_t)g->n * sizeof(NodeRec),
                               g->hash_alloc};
    Split sp[4];
    for (int t = 0; t < 4 && e == cudaSuccess; ++t)
        if (src[t] != nullptr && bytes[t] != 0) e = split(g, src[t], bytes[t], parts, devices, sp[t]);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    PartMap pm{};
    for (int t = 0; t < 4; ++t) {
        map_chunks((char* const*)sp[t].mem, bytes[t], sp[t].shift, parts, (char**)pm.base[t]);
        pm.shift[t] = sp[t].shift;
    }
    PartMap* dmap = nullptr;
    if (e == cudaSuccess) e = cudaMalloc((void**)&dmap, sizeof(PartMap));
    if (e == cudaSuccess) e = cudaMemcpy(dmap, &pm, sizeof(PartMap), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        for (int t = 0; t < 4; ++t) release(sp[t], parts);
        cudaFree(dmap);
        return cuda_fail(e, "grape_graph_partition (the graph is unchanged)");
    }
    cudaFree(g->rec);
    cudaFree(g->guide);
    cudaFree(g->nodes);
    cudaFree(g->ehash);
    g->rec = nullptr;
    g->guide = nullptr;
    g->nodes = nullptr;
    g->ehash = nullptr;
    for (int t = 0; t < 4; ++t) {
        for (uint32_t j = 0; j < parts; ++j) g->part_mem[t][j] = sp[t].mem[j];
        g->part_shift[t] = sp[t].shift;
    }
    g->part_map = dmap;
    g->parts = parts;
    // the same table bytes, now spread over the parts' devices (device_bytes counts the
    // graph's bytes on every device it uses), plus the map
    g->device_bytes += sizeof(PartMap);
    return GRAPE_OK;
}
