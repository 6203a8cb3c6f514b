// internal.h — structures shared by the CUDA translation units of libgrape_walk.
// Not part of the ABI (the ABI is include/grape_walk.h).
#pragma once
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>
#include "grape_walk.h"

// Bounds-checked build (make checked -> libgrape_walk_checked.so, -DGRAPE_CHECKED=1):
// every table read, row write and index the kernels derive is checked against the
// allocation it belongs to; a failed check prints the condition and traps (the
// launch fails with an error the caller sees).  compute-sanitizer is closed on the
// GPU pool this was developed on; the checked build plus the oracle comparison is
// what stands in for it (tests/test_gpu_checked.py).  The product
// build compiles every check away.
#ifndef GRAPE_CHECKED
#define GRAPE_CHECKED 0
#endif
#if GRAPE_CHECKED
#include <cstdio>
#define GRAPE_DCHECK(cond, what)                                                                    \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("GRAPE_CHECKED: %s failed at %s:%d (block %d thread %d)\n", what, __FILE__,       \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                    \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define GRAPE_DCHECK(cond, what) \
    do {                         \
    } while (0)
#endif

namespace grape {
// Fence levels over col and cw: level l+1 holds the last entry of
// every full 32-byte block of level l, so a search reads one sector per level
// below a short binary search on the (small, L2-resident) top level.
constexpr int kFenceLevels = 3;

// Per-node record, one 16-byte load per visited node: row start, degree and the
// row's total weight W_v when it fits 32 bits (else w32 = 0 and W_v is read
// from the u64 prefix row).
struct alignas(16) NodeRec {
    uint64_t start;
    uint32_t deg;
    uint32_t w32;
};

// §8(f) f4 layout (partition.cu, dist.cu): table T (0 records, 1 guide, 2 node
// records, 3 edge hash) in chunks of 2^shift[T] bytes, chunk c at base[T][c].  A
// table has at most kChunks chunks; owner j of `parts` holds the contiguous chunk
// range [floor(C j / parts), floor(C (j+1) / parts)) of its C chunks (one
// allocation per owner), so owners differ by at most one chunk.
constexpr int kChunks = 64;
struct PartMap {
    const char* base[4][kChunks];
    uint32_t shift[4];
};
inline uint32_t chunk_shift(uint64_t bytes)   // >= 2 MB chunks (a multiple of every entry size)
{
    uint32_t k = 21;
    while ((1ull << k) * kChunks < bytes) ++k;
    return k;
}
inline uint64_t chunk_count(uint64_t bytes, uint32_t k) { return (bytes + (1ull << k) - 1) >> k; }
// owner j's byte range [*lo, *hi) of a table of `bytes` bytes in chunks of 2^k
inline void owner_range(uint64_t bytes, uint32_t k, uint32_t j, uint32_t parts, uint64_t* lo, uint64_t* hi)
{
    const uint64_t C = chunk_count(bytes, k);
    const uint64_t a = (C * j / parts) << k, b = (C * (j + 1) / parts) << k;
    *lo = a < bytes ? a : bytes;
    *hi = b < bytes ? b : bytes;
}

// Chunk c of a table at owner_base[owner(c)] + (c's offset within that owner's range)
inline void map_chunks(char* const* owner_base, uint64_t bytes, uint32_t k, uint32_t parts, char** out)
{
    const uint64_t C = chunk_count(bytes, k);
    for (uint32_t j = 0; j < parts; ++j) {
        uint64_t lo, hi;
        owner_range(bytes, k, j, parts, &lo, &hi);
        for (uint64_t c = lo >> k; (c << k) < hi; ++c) out[c] = owner_base[j] + ((c << k) - lo);
    }
    for (uint64_t c = C; c < (uint64_t)kChunks; ++c) out[c] = C ? out[0] : nullptr;   // never addressed
}

// A table as the build kernels address it: contiguous (shift = 63: everything at
// base[0]) or in parts of 2^shift bytes, part j at base[j] (local, on a peer GPU,
// or opened from another process by CUDA IPC; graph_tables.cu, dist.cu).
struct TabRef {
    char* base[kChunks];
    uint32_t shift;
    uint64_t bytes;   // table size (checked builds compare every access with it)
    __host__ __device__ char* at(uint64_t byte) const
    {
#if GRAPE_CHECKED && defined(__CUDA_ARCH__)
        GRAPE_DCHECK(byte < bytes && (byte >> shift) < (uint64_t)kChunks && base[byte >> shift] != nullptr,
                     "table access within the table (TabRef)");
#endif
        return base[byte >> shift] + (byte & ((1ull << shift) - 1));
    }
};

// The share of the table build one builder runs (the whole graph, or one rank's
// parts in a distributed build, dist.cu): arc records and no-common-neighbour
// flags of arcs [e_lo, e_hi), edge-hash sets of the rows whose arcs are
// [h_lo, h_hi) (row-aligned), guide buckets [b_lo, b_hi).
struct TableJob {
    uint64_t e_lo, e_hi, h_lo, h_hi, b_lo, b_hi;
    TabRef rec, guide, ehash, notri;   // notri.base[0] == nullptr: no flags
};
}  // namespace grape

struct grape_graph {
    int device;
    uint32_t n;
    uint64_t m;
    uint64_t* off;        // u64[n+1]
    uint32_t* col;        // u32[m], rows strictly increasing (allocation padded to whole sectors)
    void* cw;             // row-local inclusive weight prefix: u32[m] or u64[m]; NULL if unweighted
    uint32_t cw_bytes;    // 0, 4 or 8
    grape::NodeRec* nodes;                       // [n]
    uint32_t* col_fence[grape::kFenceLevels];    // col fence levels 1..3
    void* cw_fence[grape::kFenceLevels];         // cw fence levels 1..3 (cw_bytes each)
    uint32_t flags;       // GRAPE_SYMMETRIC ...
    // Sampling tables (graph_tables.cu), absent with GRAPE_NO_TABLES
    // or when the graph exceeds their index ranges (then the v3 walker runs):
    bool tables;          // rec / guide / ehash below are built
    bool wsym;            // every arc with a reverse arc has the reverse's weight
    uint32_t rec_bytes;   // 32 / 16 (weighted: full / compact), 16 / 8 (unweighted), graph_tables.cu
    void* rec;            // per-arc records, arc order
    uint32_t* guide;      // weighted: G*deg(v) guide entries per row at G*off[v] (guide_bytes each: 32 fat / 8 slim)
    uint32_t guide_factor;   // G (buckets per arc) of the guide
    uint32_t guide_bytes;    // 32 (fat: unsplit buckets hold a record copy) or 8 (slim)
    uint32_t hash_h;         // edge-hash buckets: floor(deg / H) + 1 per row (H = 4 or 6)
    bool compact;            // records without the head's node record (16 B weighted / 8 B)
    bool notri;              // records carry the no-common-neighbour flags (graph_tables.cu)
    // 34-bit arc offsets (m >= 2^32 - 64; graph_tables.cu tables_in_range): the walker keeps
    // row starts in 64 bits, records carry bits 32-33 of the head's row start in bits 26-27
    // of the degree word (degrees < 2^26).  arc_bias: test hook (GRAPE_TEST_ARC_BIAS) —
    // every row start in the node records and records is offset by it and the walker's
    // table bases are moved back, so offsets past 2^32 run on a small graph
    bool wide = false;
    uint64_t arc_bias = 0;
    uint32_t* ehash;      // per-row bucketised sets of N(v): floor(deg/H)+1 buckets of 8 u32 slots from bucket floor(off[v]/H)+v
    uint64_t table_bytes;
    uint64_t rec_alloc = 0, guide_alloc = 0, hash_alloc = 0;   // table allocation bytes
    // §8(f) f4 layout (partition.cu, grape_graph_partition): every table split into
    // chunks of 2^part_shift[T] bytes, owner j's contiguous range of table T at
    // part_mem[T][j] (possibly on a peer GPU, or opened from another process);
    // T = 0 arc records, 1 guide, 2 node records, 3 edge hash
    uint32_t parts = 1;
    void* part_mem[4][8] = {};
    uint32_t part_shift[4] = {63, 63, 63, 63};
    grape::PartMap* part_map = nullptr;   // device copy of {part_mem, part_shift} for the walker
    // distributed build (dist.cu): this process owns part dist_part of every table; the
    // others were opened by CUDA IPC (closed, not freed, by destroy_graph); the
    // no-common-neighbour flags live in parts of 2^notri_shift bytes while building
    // validation state (graph.cu): the CSR was validated; some row holds its own node;
    // GRAPE_SYMMETRIC is checked by the table build (its record kernel finds every
    // reverse arc) instead of a separate pass
    bool validated = false;
    bool self_loops = true;
    bool sym_checked_by_tables = false;
    bool dist = false;
    uint32_t dist_part = 0;
    bool part_ipc[5][8] = {};
    void* notri_mem[8] = {};
    uint64_t part_len[5] = {};            // bytes of this process's part of table T (T = 4: flags)
    // host-buffer staging (capi.cu walks_host): device buffers kept between calls;
    // a call that finds the mutex taken (a concurrent host-buffer call) allocates its own
    std::mutex stage_mu;
    void* stage_buf = nullptr;
    uint64_t stage_bytes = 0;
    // SkipGram negatives (skipgram.cu): node guide (16-B entries) over arc-index buckets of
    // 2^node_guide_shift arcs, built on the first grape_skipgram_pairs call
    std::mutex node_guide_mu;
    uint4* node_guide = nullptr;
    uint32_t node_guide_shift = 0;
    uint32_t max_degree;
    uint64_t max_row_weight;
    uint64_t device_bytes;
};

namespace grape {

// build_graph flag (internal, above the ABI's flags): stop after the CSR, its prefix
// sums and the node records (no tables, no fence levels) — dist.cu builds the tables.
constexpr uint32_t kCsrOnly = 1u << 30;

// Makes `dev` current for a scope (restores the caller's device on exit).
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; ok = false; cudaGetLastError(); return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) { ok = false; cudaGetLastError(); }
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Resident blocks of `kernel` (block threads, dynamic smem bytes) on the whole of
// `device`: SMs x blocks per SM, cached per (kernel, device) (capi.cu).  A process
// that walks graphs on GPUs of different SM counts sizes each grid for its own GPU.
int resident_blocks(const void* kernel, int block, size_t smem, int device);

// Thread-local error message (capi.cu).
void set_error(const char* fmt, ...);
grape_status cuda_fail(cudaError_t e, const char* what);

// Node2vec acceptance thresholds (T_p, T_1, T_q), computed on the host (capi.cu).
struct Thresholds {
    uint64_t Tp, T1, Tq;
};

struct WalkArgs {
    const uint32_t* starts;
    uint64_t num_walks;
    uint64_t walk_id_base;
    uint32_t L;
    uint64_t seed;
    uint32_t* out;
    unsigned long long* steps_out;   // device, may be NULL
    unsigned long long* stats;       // device grape_walk_stats (as u64[kStatsWords]) or NULL
    uint32_t dT;                     // approximated walks: SUSS degree threshold (0: exact walks)
    uint32_t sampler;                // 0: rejection (the default rules), 1: the paper's CDF sampler (walk_cdf.cu)
};
constexpr int kStatsWords = 16;

// walk.cu: launch one walk kernel (device buffers) on `stream`.
// node2vec == false -> first order.  Returns cudaGetLastError() of the launch.
cudaError_t launch_walks(const grape_graph* g, const WalkArgs& a, bool node2vec,
                         const Thresholds& T, cudaStream_t stream);
cudaError_t launch_walks_cdf(const grape_graph* g, const WalkArgs& a, const Thresholds& T, cudaStream_t stream);
// SkipGram consumer (skipgram.cu, §8(f) f3)
cudaError_t ensure_node_guide(grape_graph* g, cudaStream_t stream);
cudaError_t launch_skipgram(const grape_graph* g, const uint32_t* walks, uint64_t num_walks, uint64_t base,
                            uint32_t L, uint32_t window, uint32_t K, uint64_t seed, uint32_t* centers,
                            uint32_t* contexts, uint32_t* negs, cudaStream_t stream);
// skipgram.cu: walks streamed chunk by chunk into the SkipGram consumer (grape_walks_skipgram)
cudaError_t launch_walks_skipgram(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                                  uint32_t window, uint32_t K, uint64_t pair_seed, uint32_t* centers,
                                  uint32_t* contexts, uint32_t* negs, uint64_t chunk_walks, cudaStream_t stream);
cudaError_t launch_walks_tab(const grape_graph* g, const WalkArgs& a, bool node2vec,
                             const Thresholds& T, cudaStream_t stream);
cudaError_t launch_walks_sm(const grape_graph* g, const WalkArgs& a, bool node2vec,
                            const Thresholds& T, cudaStream_t stream);

// capi.cu: the argument checks of grape_graph_from_csr_opts (pointers, n, flags,
// device, table option values)
grape_status check_build_args(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* col, const uint32_t* w,
                              int device, uint32_t flags, const grape_table_options* opts);
// graph.cu
grape_status build_graph(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* col,
                         const uint32_t* w, int device, uint32_t flags, const grape_table_options& opts,
                         grape_graph** out);
void destroy_graph(grape_graph* g);
// graph_tables.cu: build rec / guide / ehash for a validated graph whose off,
// col (and cw when weighted) are on the device.  Leaves g->tables false (and
// returns GRAPE_OK) when the graph is outside the tables' index ranges.
grape_status build_tables(grape_graph* g, const grape_table_options& opts);
void destroy_tables(grape_graph* g);
// graph_tables.cu: the layout (record / guide / hash sizes) whose tables fit `budget`
// bytes; sets g->rec_bytes, compact, guide_factor, guide_bytes, hash_h and the
// table sizes g->rec_alloc, guide_alloc, hash_alloc.  1: chosen, 0: none fits
// (automatic layout: the caller keeps the v3 walker), -1: a forced layout does not
// fit (error message set).  in_range: the graph is inside the tables' index ranges.
bool tables_in_range(const grape_graph* g);
int choose_layout(grape_graph* g, const grape_table_options& o, double budget);
// graph_tables.cu: one stage of the table build over a job's share (0 edge hash,
// 1 no-common-neighbour flags, 2 arc records, 3 guide); asynchronous on the
// default stream; *asym (device) gets bit 0 when a reverse arc's weight differs.
cudaError_t run_table_stage(const grape_graph* g, const TableJob& j, int stage, unsigned* asym);

}  // namespace grape
