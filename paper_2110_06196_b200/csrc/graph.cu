// graph.cu — grape_graph_from_csr: copy, validate and prefix-sum the CSR on the device.
//
// Layout in HBM:
//   off u64[n+1]   the paper's "explicit out-bound degrees vector" as offsets
//   col u32[m]     the "explicit destinations vector", rows sorted
//   cw  u32|u64[m] row-local inclusive prefix of the u32 weights ("un-normalized
//                  cumulative distribution", built once instead of per step);
//                  u32 when every row sum < 2^32, else u64.
// All kernels here run once per graph (not on the timed path): streaming passes
// one warp per row (a hub row is scanned by a whole warp, coalesced); the
// symmetric check, a search per arc, is distributed per arc (build_common.cuh).
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include "internal.h"
#include "build_common.cuh"

namespace grape {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;

enum : unsigned {
    BAD_OFF0 = 1u << 0,        // off[0] != 0
    BAD_OFFN = 1u << 1,        // off[n] != m
    BAD_MONO = 1u << 2,        // off[v] > off[v+1]
    BAD_COL = 1u << 3,         // col >= n
    BAD_SORT = 1u << 4,        // row not strictly increasing
    BAD_W = 1u << 5,           // weight == 0
    BAD_SYM = 1u << 6,         // GRAPE_SYMMETRIC asserted but an arc has no reverse
    SELF_LOOP = 1u << 7,       // (not an error) some row holds its own node
    BAD_MASK = 0x7Fu,
};

__global__ void check_offsets(const uint64_t* __restrict__ off, uint32_t n, uint64_t m,
                              unsigned* __restrict__ bad)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += stride) {
        const uint64_t a = off[v];
        if (v == 0 && a != 0) atomicOr(bad, BAD_OFF0);
        if (v == n && a != m) atomicOr(bad, BAD_OFFN);
        if (v < n && a > off[v + 1]) atomicOr(bad, BAD_MONO);
    }
}

__global__ void check_rows(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col,
                           const uint32_t* __restrict__ w, uint32_t n, unsigned* __restrict__ bad)
{
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned mine = 0;
    for (uint64_t v = warp; v < n; v += nwarps) {
        const uint64_t lo = off[v], hi = off[v + 1];
        for (uint64_t e = lo + lane; e < hi; e += 32) {
            const uint32_t c = col[e];
            if (c >= n) mine |= BAD_COL;
            if (e > lo && col[e - 1] >= c) mine |= BAD_SORT;
            if (c == (uint32_t)v) mine |= SELF_LOOP;
            if (w != nullptr && w[e] == 0) mine |= BAD_W;
        }
    }
    if (mine) atomicOr(bad, mine);
}

// Every arc v -> u needs u -> v: binary search of v in row u, one thread per arc.
__global__ void check_symmetric(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col,
                                uint32_t n, uint64_t m, unsigned* __restrict__ bad)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool ok = true;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const uint32_t v = build::row_of(off, n, e);
        const uint32_t u = col[e];
        uint64_t a = off[u], b = off[u + 1];
        const uint64_t end = b;
        while (a < b) {
            const uint64_t mid = a + ((b - a) >> 1);
            if (col[mid] < v) a = mid + 1; else b = mid;
        }
        if (a == end || col[a] != v) ok = false;
    }
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, BAD_SYM);
}

// Row sums (W_v) and degrees -> maxima.
__global__ void row_stats(const uint64_t* __restrict__ off, const uint32_t* __restrict__ w, uint32_t n,
                          unsigned long long* __restrict__ max_w, unsigned* __restrict__ max_deg)
{
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long wmax = 0;
    unsigned dmax = 0;
    for (uint64_t v = warp; v < n; v += nwarps) {
        const uint64_t lo = off[v], hi = off[v + 1];
        unsigned long long s = 0;
        if (w != nullptr)
            for (uint64_t e = lo + lane; e < hi; e += 32) s += w[e];
        else if (lane == 0)
            s = hi - lo;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (s > wmax) wmax = s;
        const uint64_t d = hi - lo;
        if (d > dmax) dmax = (unsigned)(d > 0xFFFFFFFFull ? 0xFFFFFFFFull : d);
    }
    if (lane == 0) {
        atomicMax(max_w, wmax);
        atomicMax(max_deg, dmax);
    }
}

// Row-local inclusive prefix sums: one warp per row, 32 arcs per iteration,
// shuffle scan + running carry.
template <typename CW>
__global__ void row_prefix(const uint64_t* __restrict__ off, const uint32_t* __restrict__ w, uint32_t n,
                           CW* __restrict__ cw)
{
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < n; v += nwarps) {
        const uint64_t lo = off[v], hi = off[v + 1];
        uint64_t carry = 0;
        for (uint64_t b = lo; b < hi; b += 32) {
            const uint64_t e = b + lane;
            uint64_t x = e < hi ? (uint64_t)w[e] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if ((int)lane >= o) x += y;
            }
            if (e < hi) cw[e] = (CW)(carry + x);
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}

// Node records: {row start, degree, W_v if it fits 32 bits}.
template <typename CW>
__global__ void build_nodes(const uint64_t* __restrict__ off, const CW* __restrict__ cw, uint32_t n,
                            NodeRec* __restrict__ nodes)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const uint64_t a = off[v], d = off[v + 1] - a;
        NodeRec r;
        r.start = a;
        r.deg = (uint32_t)d;
        if (cw == nullptr) r.w32 = (uint32_t)d;
        else if (sizeof(CW) == 4) r.w32 = d ? (uint32_t)cw[a + d - 1] : 0u;
        else r.w32 = 0u;
        nodes[v] = r;
    }
}

// Fence level: dst[k] = src[k*B + B - 1] for every full 32-byte block k of src.
template <typename T>
__global__ void build_fence(const T* __restrict__ src, uint64_t nsrc, T* __restrict__ dst)
{
    constexpr uint64_t B = 32 / sizeof(T);
    const uint64_t nd = nsrc / B;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nd; k += stride)
        dst[k] = src[k * B + B - 1];
}

int grid_for(uint64_t items_per_warp_rows)
{
    uint64_t blocks = (items_per_warp_rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 32) blocks = 148 * 32;
    return (int)blocks;
}

// Allocation size rounded up to whole 32-byte sectors plus one spare sector, so
// an aligned sector load of the last (partial) block never leaves the buffer.
uint64_t padded(uint64_t bytes) { return ((bytes + 31) / 32) * 32 + 32; }

}  // namespace

void destroy_graph(grape_graph* g)
{
    if (!g) return;
    cudaFree(g->off);
    cudaFree(g->col);
    cudaFree(g->cw);
    cudaFree(g->nodes);
    destroy_tables(g);
    cudaFree(g->stage_buf);
    cudaFree(g->node_guide);
    cudaFree(g->part_map);
    // partitioned tables (the contiguous pointers are NULL then): parts this process
    // allocated are freed; parts opened from another process (distributed build,
    // dist.cu) are closed; aliases of an earlier part are skipped
    static const int ipc_t[4] = {0, 1, -1, 2};   // PartMap table -> dist.cu exchange index
    for (int t = 0; t < 4; ++t)
        for (int j = 0; j < (int)g->parts && g->parts > 1; ++j) {
            bool dup = g->part_mem[t][j] == nullptr;
            for (int q = 0; q < j; ++q) dup |= g->part_mem[t][q] == g->part_mem[t][j];
            if (dup) continue;
            if (ipc_t[t] >= 0 && g->part_ipc[ipc_t[t]][j]) cudaIpcCloseMemHandle(g->part_mem[t][j]);
            else cudaFree(g->part_mem[t][j]);
        }
    for (int j = 0; j < (int)g->parts && g->dist; ++j) {   // the build's flag parts
        bool dup = g->notri_mem[j] == nullptr;
        for (int q = 0; q < j; ++q) dup |= g->notri_mem[q] == g->notri_mem[j];
        if (dup) continue;
        if (g->part_ipc[3][j]) cudaIpcCloseMemHandle(g->notri_mem[j]);
        else cudaFree(g->notri_mem[j]);
    }
    for (int l = 0; l < kFenceLevels; ++l) {
        cudaFree(g->col_fence[l]);
        cudaFree(g->cw_fence[l]);
    }
    delete g;
}

grape_status build_graph(uint32_t n, uint64_t m, const uint64_t* off_in, const uint32_t* col_in,
                         const uint32_t* w_in, int device, uint32_t flags, const grape_table_options& opts,
                         grape_graph** out)
{
    DeviceGuard guard(device);
    cudaError_t e = cudaGetLastError();  // clear stale errors
    grape_graph* g = new grape_graph();   // value-initialised (pointers null, counts 0)
    g->device = device;
    g->n = n;
    g->m = m;
    g->flags = flags & (GRAPE_SYMMETRIC | GRAPE_NO_TABLES);
    uint32_t* w = nullptr;
    unsigned* d_bad = nullptr;
    unsigned long long* d_maxw = nullptr;
    unsigned* d_maxdeg = nullptr;
    grape_status st = GRAPE_OK;
    uint64_t fence_bytes = 0;
    auto fail = [&](grape_status s) {
        cudaFree(w);
        cudaFree(d_bad);
        cudaFree(d_maxw);
        cudaFree(d_maxdeg);
        destroy_graph(g);
        *out = nullptr;
        return s;
    };
#define GRAPE_TRY_ALLOC(ptr, bytes)                                                        \
    do {                                                                                    \
        e = cudaMalloc((void**)&(ptr), (bytes) ? (bytes) : 4);                              \
        if (e != cudaSuccess) {                                                             \
            cudaGetLastError();                                                             \
            set_error("cudaMalloc of %llu bytes failed: %s", (unsigned long long)(bytes),   \
                      cudaGetErrorString(e));                                               \
            return fail(GRAPE_ENOMEM);                                                      \
        }                                                                                   \
    } while (0)
#define GRAPE_TRY_CUDA(call, what)                                                         \
    do {                                                                                    \
        e = (call);                                                                         \
        if (e != cudaSuccess) return fail(cuda_fail(e, what));                              \
    } while (0)

    GRAPE_TRY_ALLOC(g->off, (n + 1ull) * 8);
    GRAPE_TRY_ALLOC(g->col, padded(m * 4));
    GRAPE_TRY_CUDA(cudaMemset(g->col, 0, padded(m * 4)), "memset");
    GRAPE_TRY_ALLOC(d_bad, 4);
    GRAPE_TRY_ALLOC(d_maxw, 8);
    GRAPE_TRY_ALLOC(d_maxdeg, 4);
    GRAPE_TRY_CUDA(cudaMemcpy(g->off, off_in, (n + 1ull) * 8, cudaMemcpyDefault), "copy row_offsets");
    if (m) GRAPE_TRY_CUDA(cudaMemcpy(g->col, col_in, m * 4, cudaMemcpyDefault), "copy col_indices");
    if (w_in) {
        GRAPE_TRY_ALLOC(w, m * 4);
        if (m) GRAPE_TRY_CUDA(cudaMemcpy(w, w_in, m * 4, cudaMemcpyDefault), "copy weights");
    }
    GRAPE_TRY_CUDA(cudaMemset(d_bad, 0, 4), "memset");
    GRAPE_TRY_CUDA(cudaMemset(d_maxw, 0, 8), "memset");
    GRAPE_TRY_CUDA(cudaMemset(d_maxdeg, 0, 4), "memset");

    const int rows_grid = grid_for(n);
    unsigned bad = 0;
    if (!(flags & GRAPE_SKIP_VALIDATION)) {
        int g1 = (int)((n + 1ull + kThreads - 1) / kThreads);
        if (g1 > 148 * 32) g1 = 148 * 32;
        check_offsets<<<g1, kThreads>>>(g->off, n, m, d_bad);
        GRAPE_TRY_CUDA(cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost), "validate offsets");
        if (!bad) {
            check_rows<<<rows_grid, kThreads>>>(g->off, g->col, w, n, d_bad);
            // GRAPE_SYMMETRIC: when the tables will be built, their record kernel finds every
            // reverse arc anyway and checks it there (build_tables); else check here
            g->sym_checked_by_tables = (flags & GRAPE_SYMMETRIC) && !(flags & GRAPE_NO_TABLES);
            if ((flags & GRAPE_SYMMETRIC) && m && !g->sym_checked_by_tables) {
                int sms = 0;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
                check_symmetric<<<build::item_grid(m, sms), kThreads>>>(g->off, g->col, n, m, d_bad);
            }
            GRAPE_TRY_CUDA(cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost), "validate rows");
            g->validated = true;
            g->self_loops = (bad & SELF_LOOP) != 0;
            bad &= BAD_MASK;
        }
        if (bad) {
            const char* what = (bad & BAD_OFF0)   ? "row_offsets[0] != 0"
                               : (bad & BAD_OFFN) ? "row_offsets[num_nodes] != num_arcs"
                               : (bad & BAD_MONO) ? "row_offsets decrease"
                               : (bad & BAD_COL)  ? "a col_indices value >= num_nodes"
                               : (bad & BAD_SORT) ? "a row of col_indices is not strictly increasing (unsorted or duplicate arc)"
                               : (bad & BAD_W)    ? "a weight is 0 (weights must be >= 1)"
                                                  : "GRAPE_SYMMETRIC asserted but an arc has no reverse arc";
            set_error("invalid CSR: %s", what);
            return fail(GRAPE_EINVAL);
        }
    }
    row_stats<<<rows_grid, kThreads>>>(g->off, w, n, d_maxw, d_maxdeg);
    unsigned long long maxw = 0;
    unsigned maxdeg = 0;
    GRAPE_TRY_CUDA(cudaMemcpy(&maxw, d_maxw, 8, cudaMemcpyDeviceToHost), "row stats");
    GRAPE_TRY_CUDA(cudaMemcpy(&maxdeg, d_maxdeg, 4, cudaMemcpyDeviceToHost), "row stats");
    g->max_row_weight = maxw;
    g->max_degree = maxdeg;
    if (w) {
        if (maxw < (1ull << 32)) {
            g->cw_bytes = 4;
            GRAPE_TRY_ALLOC(g->cw, padded(m * 4));
            GRAPE_TRY_CUDA(cudaMemset(g->cw, 0, padded(m * 4)), "memset");
            row_prefix<uint32_t><<<rows_grid, kThreads>>>(g->off, w, n, (uint32_t*)g->cw);
        } else {
            g->cw_bytes = 8;
            GRAPE_TRY_ALLOC(g->cw, padded(m * 8));
            GRAPE_TRY_CUDA(cudaMemset(g->cw, 0, padded(m * 8)), "memset");
            row_prefix<uint64_t><<<rows_grid, kThreads>>>(g->off, w, n, (uint64_t*)g->cw);
        }
        GRAPE_TRY_CUDA(cudaGetLastError(), "prefix kernel launch");
    }
    {
        int gn = (int)((n + 255ull) / 256);
        if (gn > 148 * 32) gn = 148 * 32;
        if (gn < 1) gn = 1;
        // whole 32-B sectors plus one (the walker reads a node record as part of an
        // aligned sector), zeroed: every byte a sector load can touch is initialised
        GRAPE_TRY_ALLOC(g->nodes, padded((uint64_t)n * sizeof(NodeRec)));
        GRAPE_TRY_CUDA(cudaMemset(g->nodes, 0, padded((uint64_t)n * sizeof(NodeRec))), "memset");
        if (g->cw_bytes == 4)
            build_nodes<uint32_t><<<gn, 256>>>(g->off, (const uint32_t*)g->cw, n, g->nodes);
        else if (g->cw_bytes == 8)
            build_nodes<uint64_t><<<gn, 256>>>(g->off, (const uint64_t*)g->cw, n, g->nodes);
        else
            build_nodes<uint32_t><<<gn, 256>>>(g->off, nullptr, n, g->nodes);
        GRAPE_TRY_CUDA(cudaGetLastError(), "node records");
    }
    GRAPE_TRY_CUDA(cudaDeviceSynchronize(), "graph build");
    cudaFree(w);   // the prefix sums hold everything the walkers need from the weights
    w = nullptr;
    if (flags & kCsrOnly) {   // dist.cu builds the tables; keep col / cw for it
        cudaFree(d_bad);
        cudaFree(d_maxw);
        cudaFree(d_maxdeg);
        g->device_bytes = (n + 1ull) * 8 + (uint64_t)n * sizeof(NodeRec) + padded(m * 4) +
                          (g->cw_bytes ? padded(m * g->cw_bytes) : 0);
        *out = g;
        return GRAPE_OK;
    }
    if (!(flags & GRAPE_NO_TABLES)) {
        st = build_tables(g, opts);
        if (st != GRAPE_OK) return fail(st);
        GRAPE_TRY_CUDA(cudaDeviceSynchronize(), "table build");
    }
    if (g->sym_checked_by_tables && !g->tables && m) {   // no tables after all: check GRAPE_SYMMETRIC here
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        GRAPE_TRY_CUDA(cudaMemset(d_bad, 0, 4), "memset");
        check_symmetric<<<build::item_grid(m, sms), kThreads>>>(g->off, g->col, n, m, d_bad);
        GRAPE_TRY_CUDA(cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost), "validate symmetry");
        if (bad) {
            set_error("invalid CSR: GRAPE_SYMMETRIC asserted but an arc has no reverse arc");
            return fail(GRAPE_EINVAL);
        }
    }
    if (g->tables) {   // the table walker reads only nodes / rec / guide / ehash
        cudaFree(g->col);
        cudaFree(g->cw);
        g->col = nullptr;
        g->cw = nullptr;
    } else {           // fence levels for the v3 walker
        fence_bytes = 0;
        uint64_t len = m;
        for (int l = 0; l < kFenceLevels; ++l) {
            len /= 8;
            GRAPE_TRY_ALLOC(g->col_fence[l], padded(len * 4));
            GRAPE_TRY_CUDA(cudaMemset(g->col_fence[l], 0, padded(len * 4)), "memset");
            fence_bytes += padded(len * 4);
            const uint32_t* src = l == 0 ? g->col : g->col_fence[l - 1];
            build_fence<uint32_t><<<grid_for(len / 8 + 1), kThreads>>>(src, len * 8, g->col_fence[l]);
        }
        if (g->cw_bytes) {
            const uint64_t B = 32 / g->cw_bytes;
            len = m;
            for (int l = 0; l < kFenceLevels; ++l) {
                len /= B;
                GRAPE_TRY_ALLOC(g->cw_fence[l], padded(len * g->cw_bytes));
                GRAPE_TRY_CUDA(cudaMemset(g->cw_fence[l], 0, padded(len * g->cw_bytes)), "memset");
                fence_bytes += padded(len * g->cw_bytes);
                if (g->cw_bytes == 4)
                    build_fence<uint32_t><<<grid_for(len / 8 + 1), kThreads>>>(
                        l == 0 ? (const uint32_t*)g->cw : (const uint32_t*)g->cw_fence[l - 1], len * B,
                        (uint32_t*)g->cw_fence[l]);
                else
                    build_fence<uint64_t><<<grid_for(len / 8 + 1), kThreads>>>(
                        l == 0 ? (const uint64_t*)g->cw : (const uint64_t*)g->cw_fence[l - 1], len * B,
                        (uint64_t*)g->cw_fence[l]);
            }
        }
        GRAPE_TRY_CUDA(cudaGetLastError(), "fence levels");
        GRAPE_TRY_CUDA(cudaDeviceSynchronize(), "fence levels");
    }
    cudaFree(d_bad);
    cudaFree(d_maxw);
    cudaFree(d_maxdeg);
    d_bad = nullptr; d_maxw = nullptr; d_maxdeg = nullptr;
    g->device_bytes = (n + 1ull) * 8 + (uint64_t)n * sizeof(NodeRec) + g->table_bytes +
                      (g->tables ? 0 : padded(m * 4) + (g->cw_bytes ? padded(m * g->cw_bytes) : 0) + fence_bytes);
    *out = g;
    return GRAPE_OK;
#undef GRAPE_TRY_ALLOC
#undef GRAPE_TRY_CUDA
}

}  // namespace grape
