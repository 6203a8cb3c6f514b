// dist.cu — the §8(f) f4 row, distributed: sampling tables
// larger than one GPU, built by one process per GPU, each owning one part.
//
// The tables (arc records, guide, edge hash) are laid out as in
// grape_graph_partition: table T in chunks of 2^k_T bytes (at most kChunks),
// rank j owning a contiguous range of chunks (its "part").  Every rank holds the whole CSR (col, prefix sums,
// off: 8 bytes per arc against the tables' 30-550) and its node records; it
// allocates only its own part of each table.  The ranks exchange CUDA IPC handles
// of their parts (the caller all-gathers them, e.g. over torch.distributed), open
// each other's, and then build in four stages with a barrier between stages,
// each rank building the entries that land in its own part:
//   0 edge-hash sets of the rows whose first bucket is in its part (a row's last
//     buckets may lie in the next part: written there through the IPC mapping; one
//     rank owns each row, so no two ranks probe the same buckets)
//   1 no-common-neighbour flags of its arcs (reading any rank's hash sets)
//   2 arc records of its arcs (reading the flags of the reverse arcs, anywhere)
//   3 guide buckets of its part (fat entries copy records, anywhere)
// The build kernels are the single-GPU ones (graph_tables.cu) over TabRef
// addressing; the walker reads the parts through the partition map (walk_tab.cu
// MODE 3), so every walk is the one the contiguous tables give.  The host runs
// no collective: the ABI is a sequence of synchronous calls, and the caller
// supplies the exchange and the barriers (paper_2110_06196_b200.graph_from_csr_dist).
#include <cstring>
#include "internal.h"

namespace grape {
namespace {

// Table indices of the exchange: 0 records, 1 guide, 2 edge hash, 3 flags (build only)
constexpr int kDistTables = 4;

__global__ void first_row_with_bucket(const uint64_t* __restrict__ off, uint32_t n, uint32_t H, uint64_t bucket,
                                      uint32_t* __restrict__ out)
{
    // smallest v in [0, n] with floor(off[v] / H) + v >= bucket (n: none); monotone in v
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (off[mid] / H + mid >= bucket) hi = mid;
        else lo = mid + 1;
    }
    *out = lo;
}

}  // namespace
}  // namespace grape

using namespace grape;

namespace {

struct Layout {   // byte sizes and chunk shifts of the exchanged tables
    uint64_t bytes[kDistTables];
    uint32_t shift[kDistTables];
};

Layout layout_of(const grape_graph* g)
{
    Layout L{};
    L.bytes[0] = g->rec_alloc;
    L.bytes[1] = g->guide_alloc;
    L.bytes[2] = g->hash_alloc;
    L.bytes[3] = g->notri ? g->m : 0;   // one byte per arc
    for (int t = 0; t < 3; ++t) L.shift[t] = chunk_shift(L.bytes[t]);
    // flags in the chunks of the records they belong to: the same chunk indices, so an
    // owner's flag range covers exactly the arcs of its record range
    uint32_t lg = 0;
    while ((1u << lg) < g->rec_bytes) ++lg;
    L.shift[3] = L.shift[0] - lg;
    return L;
}

// owner j's byte range of exchange table t
void range_of(const grape_graph* g, const Layout& L, int t, uint32_t j, uint64_t* lo, uint64_t* hi)
{
    if (t == 3) {   // the flag range = the record range / record bytes (clamped to m)
        uint64_t a, b;
        owner_range(L.bytes[0], L.shift[0], j, g->parts, &a, &b);
        a /= g->rec_bytes;
        b /= g->rec_bytes;
        *lo = a < g->m ? a : g->m;
        *hi = b < g->m ? b : g->m;
        if (L.bytes[3] == 0) *lo = *hi = 0;
        return;
    }
    owner_range(L.bytes[t], L.shift[t], j, g->parts, lo, hi);
}

void** part_slot(grape_graph* g, int t, uint32_t j)
{
    static const int map_t[3] = {0, 1, 3};   // exchange index -> PartMap table (0 rec, 1 guide, 3 hash)
    if (t == 3) return &g->notri_mem[j];
    return &g->part_mem[map_t[t]][j];
}

TabRef tab_of(grape_graph* g, const Layout& L, int t)
{
    char* owners[8] = {};
    for (uint32_t j = 0; j < g->parts; ++j) owners[j] = (char*)*part_slot(g, t, j);
    TabRef r{};
    r.shift = L.shift[t];
    // flags: chunk c of the flags = the arcs of record chunk c; its bytes start at
    // (c << shift[3]) within the owner's flag range
    uint64_t bytes = L.bytes[t];
    if (t == 3) bytes = L.bytes[0] >> (L.shift[0] - L.shift[3]);
    map_chunks(owners, bytes, r.shift, g->parts, r.base);
    r.bytes = t == 3 ? L.bytes[3] : bytes;
    return r;
}

}  // namespace

extern "C" {

grape_status grape_graph_dist_create(uint32_t num_nodes, uint64_t num_arcs, const uint64_t* row_offsets,
                                     const uint32_t* col_indices, const uint32_t* weights, int device,
                                     uint32_t flags, const grape_table_options* opts, uint32_t part, uint32_t parts,
                                     grape_graph** out)
{
    if (out == nullptr) {
        set_error("out must be non-NULL");
        return GRAPE_EINVAL;
    }
    *out = nullptr;
    if (parts < 2 || parts > 8 || part >= parts) {
        set_error("grape_graph_dist_create: need 2 <= parts <= 8 and part < parts (got part %u of %u)", part, parts);
        return GRAPE_EINVAL;
    }
    if (opts == nullptr || opts->table_budget_bytes == 0) {
        set_error("grape_graph_dist_create: opts->table_budget_bytes (bytes of tables per part, the same on every "
                  "rank) is required: the layout must come out the same on every rank");
        return GRAPE_EINVAL;
    }
    if (flags & (GRAPE_NO_TABLES | kCsrOnly)) {
        set_error("grape_graph_dist_create: a distributed graph always has tables");
        return GRAPE_EINVAL;
    }
    const grape_table_options o = *opts;
    grape_status st = check_build_args(num_nodes, num_arcs, row_offsets, col_indices, weights, device, flags, &o);
    if (st != GRAPE_OK) return st;
    grape_graph* g = nullptr;   // the CSR, validated (unless skipped), its prefix sums and node records
    st = build_graph(num_nodes, num_arcs, row_offsets, col_indices, weights, device, flags | kCsrOnly, o, &g);
    if (st != GRAPE_OK) return st;
    DeviceGuard guard(device);
    auto fail = [&](grape_status s) {
        destroy_graph(g);
        return s;
    };
    if (!tables_in_range(g)) {
        set_error("grape_graph_dist_create: the graph is outside the tables' index ranges");
        return fail(GRAPE_EINVAL);
    }
    const int ch = choose_layout(g, o, (double)o.table_budget_bytes * parts);
    if (ch <= 0) {
        if (ch == 0)
            set_error("grape_graph_dist_create: no table layout fits %u parts of %llu bytes", parts,
                      (unsigned long long)o.table_budget_bytes);
        return fail(GRAPE_ENOMEM);
    }
    g->wide = num_arcs >= (1ull << 32) - 64;
    g->dist = true;
    g->dist_part = part;
    g->parts = parts;
    g->notri = !(g->compact && num_nodes >= (1u << 30));
    const Layout L = layout_of(g);
    for (int t = 0; t < kDistTables; ++t) {
        uint64_t lo, hi;
        range_of(g, L, t, part, &lo, &hi);
        const uint64_t len = hi - lo;
        g->part_len[t] = len;
        if (len == 0) continue;
        // whole 2 MB pages: a CUDA IPC mapping of an allocation with a ragged last page was
        // measured 150x slower for random reads from the importing process (the last rank's
        // part, whose length is the table's remainder; tools/dist_probe.py)
        const uint64_t alloc = (len + (2ull << 20) - 1) & ~((2ull << 20) - 1);
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, alloc);
        if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc of this rank's table part"));
        *part_slot(g, t, part) = p;
        e = cudaMemset(p, t == 2 ? 0xFF : 0, alloc);   // empty hash slots = 0xFFFFFFFF
        if (e != cudaSuccess) return fail(cuda_fail(e, "memset of a table part"));
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(cuda_fail(e, "grape_graph_dist_create"));
    *out = g;
    return GRAPE_OK;
}

grape_status grape_graph_dist_export(const grape_graph* g, grape_part_export* out)
{
    if (g == nullptr || out == nullptr || !g->dist) {
        set_error("grape_graph_dist_export: need a graph from grape_graph_dist_create and an output");
        return GRAPE_EINVAL;
    }
    memset(out, 0, sizeof(*out));
    out->part = g->dist_part;
    out->device = g->device;
    DeviceGuard guard(g->device);
    grape_graph* gm = const_cast<grape_graph*>(g);
    for (int t = 0; t < kDistTables; ++t) {
        out->bytes[t] = g->part_len[t];
        if (g->part_len[t] == 0) continue;
        cudaIpcMemHandle_t h;
        cudaError_t e = cudaIpcGetMemHandle(&h, *part_slot(gm, t, g->dist_part));
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
        static_assert(sizeof(h) == sizeof(out->handle[0].bytes), "IPC handle size");
        memcpy(out->handle[t].bytes, &h, sizeof(h));
    }
    return GRAPE_OK;
}

grape_status grape_graph_dist_import(grape_graph* g, const grape_part_export* exports)
{
    if (g == nullptr || exports == nullptr || !g->dist) {
        set_error("grape_graph_dist_import: need a graph from grape_graph_dist_create and the exports");
        return GRAPE_EINVAL;
    }
    DeviceGuard guard(g->device);
    const Layout L = layout_of(g);
    for (uint32_t j = 0; j < g->parts; ++j) {
        const grape_part_export& x = exports[j];
        if (x.part != j) {
            set_error("grape_graph_dist_import: exports[%u] is part %u (index the array by part)", j, x.part);
            return GRAPE_EINVAL;
        }
        for (int t = 0; t < kDistTables; ++t) {
            uint64_t lo, hi;
            range_of(g, L, t, j, &lo, &hi);
            if (x.bytes[t] != hi - lo) {
                set_error("grape_graph_dist_import: part %u of table %d has %llu bytes, this rank expects %llu "
                          "(different graphs or layouts across ranks)", j, t, (unsigned long long)x.bytes[t],
                          (unsigned long long)(hi - lo));
                return GRAPE_EINVAL;
            }
        }
    }
    for (uint32_t j = 0; j < g->parts; ++j) {
        if (j == g->dist_part) continue;
        for (int t = 0; t < kDistTables; ++t) {
            if (exports[j].bytes[t] == 0 || *part_slot(g, t, j) != nullptr) continue;
            cudaIpcMemHandle_t h;
            memcpy(&h, exports[j].handle[t].bytes, sizeof(h));
            void* p = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle of a peer's table part");
            *part_slot(g, t, j) = p;
            g->part_ipc[t][j] = true;
        }
    }
    // the walker's partition map: records, guide and hash in chunks; node records local
    PartMap pm{};
    const TabRef tr[3] = {tab_of(g, L, 0), tab_of(g, L, 1), tab_of(g, L, 2)};
    for (int c = 0; c < kChunks; ++c) {
        pm.base[0][c] = tr[0].base[c];
        pm.base[1][c] = tr[1].base[c];
        pm.base[2][c] = (const char*)g->nodes;
        pm.base[3][c] = tr[2].base[c];
    }
    pm.shift[0] = L.shift[0];
    pm.shift[1] = L.shift[1];
    pm.shift[2] = 63;
    pm.shift[3] = L.shift[2];
    for (int t = 0; t < 4; ++t) g->part_shift[t] = pm.shift[t];
    cudaError_t e = cudaSuccess;
    if (g->part_map == nullptr) e = cudaMalloc((void**)&g->part_map, sizeof(PartMap));
    if (e == cudaSuccess) e = cudaMemcpy(g->part_map, &pm, sizeof(PartMap), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "partition map");
    return GRAPE_OK;
}

grape_status grape_graph_dist_build(grape_graph* g, uint32_t stage, uint32_t* flags_out)
{
    if (g == nullptr || !g->dist || g->part_map == nullptr || stage > 3 || g->col == nullptr) {
        set_error("grape_graph_dist_build: need an imported distributed graph (before finish) and stage 0..3");
        return GRAPE_EINVAL;
    }
    DeviceGuard guard(g->device);
    const Layout L = layout_of(g);
    const uint32_t r = g->dist_part;
    const uint64_t m = g->m;
    TableJob j{};
    uint64_t lo, hi;
    // records and flags: the arcs whose records are in this rank's part
    owner_range(L.bytes[0], L.shift[0], r, g->parts, &lo, &hi);
    j.e_lo = lo / g->rec_bytes < m ? lo / g->rec_bytes : m;
    j.e_hi = hi / g->rec_bytes < m ? hi / g->rec_bytes : m;
    // guide: the buckets whose entries are in this rank's part
    if (g->guide_bytes) {
        const uint64_t nb = (uint64_t)g->guide_factor * m;
        owner_range(L.bytes[1], L.shift[1], r, g->parts, &lo, &hi);
        j.b_lo = lo / g->guide_bytes < nb ? lo / g->guide_bytes : nb;
        j.b_hi = hi / g->guide_bytes < nb ? hi / g->guide_bytes : nb;
    }
    j.rec = tab_of(g, L, 0);
    j.guide = tab_of(g, L, 1);
    j.ehash = tab_of(g, L, 2);
    j.notri = g->notri ? tab_of(g, L, 3) : TabRef{};
    cudaError_t e = cudaSuccess;
    unsigned* d = nullptr;
    uint32_t* dv = nullptr;
    if ((e = cudaMalloc((void**)&d, 8)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    dv = (uint32_t*)(d + 1);
    e = cudaMemset(d, 0, 8);
    if (e == cudaSuccess && stage == 0) {   // hash rows: those whose first bucket is in this rank's part
        owner_range(L.bytes[2], L.shift[2], r, g->parts, &lo, &hi);
        const uint64_t bk[2] = {lo / 32, hi == L.bytes[2] ? ~0ull : hi / 32};   // the last owner: every row left
        uint32_t v[2] = {0, 0};
        for (int s = 0; s < 2 && e == cudaSuccess; ++s) {
            first_row_with_bucket<<<1, 1>>>(g->off, g->n, g->hash_h, bk[s], dv);
            e = cudaMemcpy(&v[s], dv, 4, cudaMemcpyDeviceToHost);
        }
        uint64_t a = 0, b = 0;
        if (e == cudaSuccess) e = cudaMemcpy(&a, g->off + v[0], 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(&b, g->off + v[1], 8, cudaMemcpyDeviceToHost);
        j.h_lo = a;
        j.h_hi = b;
    }
    if (e == cudaSuccess) e = run_table_stage(g, j, (int)stage, d);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned asym = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&asym, d, 4, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "grape_graph_dist_build");
    if (flags_out) *flags_out = asym;   // bit 0: asymmetric weights; bit 1: GRAPE_SYMMETRIC violated
    return GRAPE_OK;
}

grape_status grape_graph_dist_finish(grape_graph* g, uint32_t flags_all)
{
    if (g == nullptr || !g->dist || g->part_map == nullptr || g->col == nullptr) {
        set_error("grape_graph_dist_finish: need a built distributed graph (once)");
        return GRAPE_EINVAL;
    }
    DeviceGuard guard(g->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "grape_graph_dist_finish");
    if (flags_all & 2u) {
        set_error("invalid CSR: GRAPE_SYMMETRIC asserted but an arc has no reverse arc");
        return GRAPE_EINVAL;
    }
    g->wsym = g->cw_bytes == 0 || (flags_all & 1u) == 0;
    // the walker reads only the node records and the table parts: drop the CSR copy
    cudaFree(g->col);
    cudaFree(g->cw);
    g->col = nullptr;
    g->cw = nullptr;
    g->tables = true;
    g->table_bytes = g->part_len[0] + g->part_len[1] + g->part_len[2];
    g->device_bytes = (g->n + 1ull) * 8 + (uint64_t)g->n * sizeof(NodeRec) + g->table_bytes + g->part_len[3] +
                      sizeof(PartMap);
    return GRAPE_OK;
}

}  // extern "C"
