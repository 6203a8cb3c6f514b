// capi.cu — the extern "C" boundary (include/grape_walk.h): argument checks,
// node2vec thresholds, device / host-buffer walk calls, error reporting.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "internal.h"

namespace grape {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

grape_status cuda_fail(cudaError_t e, const char* what)
{
    set_error("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? GRAPE_ENOMEM : GRAPE_ECUDA;
}

int resident_blocks(const void* kernel, int block, size_t smem, int device)
{
    struct Entry { const void* k; int block; size_t smem; int dev; int blocks; };
    static std::mutex mu;
    static Entry cache[256];
    static int used = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (int i = 0; i < used; ++i)
            if (cache[i].k == kernel && cache[i].block == block && cache[i].smem == smem && cache[i].dev == device)
                return cache[i].blocks;
    }
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    cudaGetLastError();
    const int r = (sms > 0 ? sms : 1) * (per_sm > 0 ? per_sm : 1);
    std::lock_guard<std::mutex> lk(mu);
    if (used < 256) cache[used++] = Entry{kernel, block, smem, device, r};
    return r;
}

namespace {

// T_c = floor(2^32 * min(p,1,q) / c) for c in (p, 1, q), IEEE binary64
// (include/grape_walk.h; §8(c) c9-c10).  Host code: one division and one exact
// power-of-two scaling per class.
bool node2vec_thresholds(double p, double q, Thresholds* T)
{
    if (!std::isfinite(p) || !std::isfinite(q) || !(p > 0.0) || !(q > 0.0)) {
        set_error("p and q must be finite and > 0 (got p=%g, q=%g)", p, q);
        return false;
    }
    const double lo = std::fmin(std::fmin(p, 1.0), q);
    const double hi = std::fmax(std::fmax(p, 1.0), q);
    if (hi / lo > 16777216.0) {
        set_error("max(p,1,q)/min(p,1,q) = %g exceeds 2^24", hi / lo);
        return false;
    }
    T->Tp = (uint64_t)std::floor(std::ldexp(lo / p, 32));
    T->T1 = (uint64_t)std::floor(std::ldexp(lo, 32));
    T->Tq = (uint64_t)std::floor(std::ldexp(lo / q, 32));
    return true;
}

enum class Mem { Device, Host, Invalid };

Mem classify(const void* ptr)
{
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return Mem::Host;
    }
    switch (at.type) {
    case cudaMemoryTypeDevice:
    case cudaMemoryTypeManaged: return Mem::Device;
    default: return Mem::Host;   // unregistered (pageable) or pinned host
    }
}

#ifndef GRAPE_HOST_CHUNK_MB
#define GRAPE_HOST_CHUNK_MB 256        // smallest default chunk of the walk matrix
#endif
#ifndef GRAPE_HOST_CHUNK_MAX_MB
#define GRAPE_HOST_CHUNK_MAX_MB 1024
#endif
#ifndef GRAPE_HOST_NBUF
#define GRAPE_HOST_NBUF 4
#endif

// Host buffers: stage chunks through device memory.  Chunk k runs on the
// caller's stream (H2D starts -> kernel), its D2H runs on an internal copy
// stream, so the copy of chunk k overlaps the kernels of chunks k+1 ..; with
// NBUF staging buffers the kernels run ahead of the (PCIe-bound) copies.
// Chunk size: ~1/32 of the walk matrix within [256 MB, 1 GB] (measured, DESIGN.md
// §9: small chunks cost per-launch tails on slow-per-walk workloads, large ones
// leave the first kernel and the last copy unoverlapped); halved while the
// staging allocation fails; GRAPE_HOST_CHUNK_MB in the environment overrides it.
grape_status walks_host(const grape_graph* g, const WalkArgs& a, bool n2v, const Thresholds& T,
                        cudaStream_t stream, uint64_t* steps_host)
{
    constexpr int NB = GRAPE_HOST_NBUF;
    const uint64_t L = a.L;
    uint64_t chunk_mb = (a.num_walks * L * 4 >> 20) / 32;
    if (chunk_mb < GRAPE_HOST_CHUNK_MB) chunk_mb = GRAPE_HOST_CHUNK_MB;
    if (chunk_mb > GRAPE_HOST_CHUNK_MAX_MB) chunk_mb = GRAPE_HOST_CHUNK_MAX_MB;
    if (const char* env = getenv("GRAPE_HOST_CHUNK_MB")) {   // tuning knob (bench A/B)
        const long v = atol(env);
        if (v > 0) chunk_mb = (uint64_t)v;
    }
    uint32_t* d_starts[NB] = {};
    uint32_t* d_out[NB] = {};
    unsigned long long* d_steps = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_kernel[NB] = {}, ev_copied[NB] = {};
    grape_status st = GRAPE_OK;
    cudaError_t e = cudaSuccess;
    grape_graph* gm = const_cast<grape_graph*>(g);
    std::unique_lock<std::mutex> lk(gm->stage_mu, std::try_to_lock);
    char* base = nullptr;
    bool own = false;
    uint64_t chunk, nchunks, per;
    int nbuf;
    for (;;) {
        chunk = (chunk_mb << 20) / (4 * L);   // walks per chunk, >= 1
        if (chunk < 1) chunk = 1;
        if (chunk > a.num_walks) chunk = a.num_walks;
        nchunks = (a.num_walks + chunk - 1) / chunk;
        nbuf = nchunks < (uint64_t)NB ? (int)nchunks : NB;
        // one device allocation for all staging buffers: the graph's cached one when free
        per = ((chunk * 4 + 255) & ~255ull) + ((chunk * L * 4 + 255) & ~255ull);
        const uint64_t need = per * nbuf + 256;
        if (lk.owns_lock()) {
            e = cudaSuccess;
            if (gm->stage_bytes < need) {
                cudaFree(gm->stage_buf);
                gm->stage_buf = nullptr;
                gm->stage_bytes = 0;
                e = cudaMalloc(&gm->stage_buf, need);
                if (e == cudaSuccess) gm->stage_bytes = need;
            }
            base = (char*)gm->stage_buf;
        } else {
            e = cudaMalloc((void**)&base, need);
            own = e == cudaSuccess;
        }
        if (e != cudaErrorMemoryAllocation || chunk_mb <= 16 || chunk == 1) break;
        cudaGetLastError();   // clear the allocation failure and retry smaller
        chunk_mb /= 2;
    }
    const bool single = nchunks == 1;   // one chunk: everything on the caller's stream, nothing to overlap
    for (int b = 0; b < nbuf && e == cudaSuccess; ++b) {
        d_starts[b] = (uint32_t*)(base + b * per);
        d_out[b] = (uint32_t*)(base + b * per + ((chunk * 4 + 255) & ~255ull));
        if (single) continue;
        e = cudaEventCreateWithFlags(&ev_kernel[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_copied[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) d_steps = (unsigned long long*)(base + per * nbuf);
    if (e == cudaSuccess && !single) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_steps, 0, 8, stream);
    if (e == cudaSuccess && single) {
        WalkArgs c = a;
        c.starts = d_starts[0];
        c.out = d_out[0];
        c.steps_out = d_steps;
        unsigned long long steps = 0;
        e = cudaMemcpyAsync(d_starts[0], a.starts, a.num_walks * 4, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) e = launch_walks(g, c, n2v, T, stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(a.out, d_out[0], a.num_walks * L * 4, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&steps, d_steps, 8, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) st = cuda_fail(e, "host-buffer walks");
        else if (steps_host) *steps_host += steps;
        cudaStreamSynchronize(stream);
        if (own) cudaFree(base);
        return st;
    }
    if (e != cudaSuccess) {
        st = cuda_fail(e, "host-buffer staging setup");
    } else {
        uint64_t k = 0;
        for (uint64_t lo = 0; lo < a.num_walks && e == cudaSuccess; lo += chunk, ++k) {
            const int b = (int)(k % nbuf);
            const uint64_t cnt = (a.num_walks - lo < chunk) ? a.num_walks - lo : chunk;
            if (k >= (uint64_t)nbuf) e = cudaStreamWaitEvent(stream, ev_copied[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(d_starts[b], a.starts + lo, cnt * 4, cudaMemcpyHostToDevice, stream);
            if (e != cudaSuccess) break;
            WalkArgs c = a;
            c.starts = d_starts[b];
            c.num_walks = cnt;
            c.walk_id_base = a.walk_id_base + lo;
            c.out = d_out[b];
            c.steps_out = d_steps;
            e = launch_walks(g, c, n2v, T, stream);
            if (e == cudaSuccess) e = cudaEventRecord(ev_kernel[b], stream);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev_kernel[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(a.out + lo * L, d_out[b], cnt * L * 4, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaEventRecord(ev_copied[b], cs);
        }
        unsigned long long steps = 0;
        if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&steps, d_steps, 8, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) st = cuda_fail(e, "host-buffer walks");
        else if (steps_host) *steps_host += steps;
    }
    if (cs) { cudaStreamSynchronize(cs); cudaStreamDestroy(cs); }
    cudaStreamSynchronize(stream);
    for (int b = 0; b < NB; ++b) {
        if (ev_kernel[b]) cudaEventDestroy(ev_kernel[b]);
        if (ev_copied[b]) cudaEventDestroy(ev_copied[b]);
    }
    if (own) cudaFree(base);
    return st;
}

grape_status walks_common(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                          uint64_t base, uint32_t L, bool n2v, double p, double q, uint64_t seed,
                          uint32_t* out, uint64_t* steps_out, cudaStream_t stream, uint32_t dT = 0,
                          uint32_t sampler = 0)
{
    g_err[0] = 0;
    if (g == nullptr || (num_walks > 0 && (starts == nullptr || out == nullptr))) {
        set_error("graph, starts and out must be non-NULL");
        return GRAPE_EINVAL;
    }
    if (L == 0) {
        set_error("walk_length must be >= 1");
        return GRAPE_EINVAL;
    }
    if (num_walks > (~0ull) / L / 4) {
        set_error("num_walks * walk_length overflows");
        return GRAPE_EINVAL;
    }
    Thresholds T{1ull << 32, 1ull << 32, 1ull << 32};
    if (n2v && !node2vec_thresholds(p, q, &T)) return GRAPE_EINVAL;
    if (dT >= g->max_degree) dT = 0;   // no row exceeds the threshold: the exact walks
    if ((sampler == 1 || sampler == 2) && !g->tables) {
        set_error("the %s sampler needs the sampling tables (graph built with GRAPE_NO_TABLES "
                  "or outside their index ranges)", sampler == 1 ? "CDF" : "outlier-folded");
        return GRAPE_EINVAL;
    }
    if (sampler == 2 && g->cw_bytes != 0 && g->compact && !g->wsym) {
        set_error("the outlier-folded sampler needs each return arc's weight: rebuild this graph "
                  "(asymmetric weights) with grape_table_options.record_bytes = 32");
        return GRAPE_EINVAL;
    }
    if (dT != 0 && !g->tables) {
        set_error("approximated walks need the sampling tables (graph built with GRAPE_NO_TABLES "
                  "or outside their index ranges)");
        return GRAPE_EINVAL;
    }
    if (g->parts > 1 && (dT != 0 || sampler != 0)) {
        set_error("a partitioned graph (grape_graph_partition) serves the default walk rules only");
        return GRAPE_EINVAL;
    }
    if (g->dist && !g->tables) {
        set_error("a distributed graph walks after grape_graph_dist_finish");
        return GRAPE_EINVAL;
    }
    if (g->wide && (dT != 0 || sampler != 0)) {
        set_error("a graph with 2^32 - 64 or more arcs serves the default walk rules only");
        return GRAPE_EINVAL;
    }
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) { cudaGetLastError(); cur = -1; }
    if (cur != g->device) {
        set_error("current device %d is not the graph's device %d", cur, g->device);
        return GRAPE_EINVAL;
    }
    if (num_walks == 0) return GRAPE_OK;
    const Mem ms = classify(starts), mo = classify(out);
    if (ms != mo) {
        set_error("starts and out must both be device or both be host memory");
        return GRAPE_EINVAL;
    }
    WalkArgs a{};
    a.starts = starts;
    a.num_walks = num_walks;
    a.walk_id_base = base;
    a.L = L;
    a.seed = seed;
    a.out = out;
    a.steps_out = nullptr;
    a.dT = dT;
    a.sampler = sampler;
    if (ms == Mem::Host) return walks_host(g, a, n2v, T, stream, steps_out);
    if (steps_out != nullptr && classify(steps_out) != Mem::Device) {
        set_error("with device buffers, steps_out must be device memory (or NULL)");
        return GRAPE_EINVAL;
    }
    a.steps_out = (unsigned long long*)steps_out;
    cudaError_t e = launch_walks(g, a, n2v, T, stream);
    if (e != cudaSuccess) return cuda_fail(e, "walk kernel launch");
    return GRAPE_OK;
}

}  // namespace
}  // namespace grape

using namespace grape;

extern "C" {

}  // extern "C"

namespace grape {
grape_status check_build_args(uint32_t num_nodes, uint64_t num_arcs, const uint64_t* row_offsets,
                              const uint32_t* col_indices, const uint32_t* weights, int device, uint32_t flags,
                              const grape_table_options* opts)
{
    if (row_offsets == nullptr || (num_arcs > 0 && col_indices == nullptr)) {
        set_error("row_offsets and col_indices must be non-NULL");
        return GRAPE_EINVAL;
    }
    if (num_nodes >= 0xFFFFFFFFu) {
        set_error("num_nodes must be < 2^32 - 1 (0xFFFFFFFF is GRAPE_PAD)");
        return GRAPE_EINVAL;
    }
    if (flags & ~(uint32_t)(GRAPE_SYMMETRIC | GRAPE_SKIP_VALIDATION | GRAPE_NO_TABLES)) {
        set_error("unknown flags 0x%x", flags);
        return GRAPE_EINVAL;
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) {
        set_error("device %d out of range (%d devices)", device, ndev);
        return GRAPE_EINVAL;
    }
    grape_table_options o{};
    if (opts != nullptr) {
        o = *opts;
        const bool w = weights != nullptr;
        const uint32_t rb = o.record_bytes;
        const bool rec_ok = rb == 0 || (w ? (rb == 32 || rb == 16) : (rb == 16 || rb == 8));
        const bool gb_ok = o.guide_bytes == 0 || o.guide_bytes == 32 || o.guide_bytes == 8;
        const bool g_ok = o.guide_factor == 0 || o.guide_factor == 1 || o.guide_factor == 2 || o.guide_factor == 4 ||
                          o.guide_factor == 8 || o.guide_factor == 16;
        const bool h_ok = o.hash_h == 0 || o.hash_h == 4 || o.hash_h == 6;
        if (!rec_ok || !gb_ok || !g_ok || !h_ok || (!w && (o.guide_bytes || o.guide_factor)) ||
            (o.guide_bytes == 32 && rb == 16)) {
            set_error("grape_table_options: a field is outside its allowed values for this graph");
            return GRAPE_EINVAL;
        }
    }
    return GRAPE_OK;
}
}  // namespace grape

extern "C" {

grape_status grape_graph_from_csr_opts(uint32_t num_nodes, uint64_t num_arcs, const uint64_t* row_offsets,
                                       const uint32_t* col_indices, const uint32_t* weights, int device,
                                       uint32_t flags, const grape_table_options* opts, grape_graph** out)
{
    g_err[0] = 0;
    if (out == nullptr) {
        set_error("out must be non-NULL");
        return GRAPE_EINVAL;
    }
    *out = nullptr;
    const grape_status st = check_build_args(num_nodes, num_arcs, row_offsets, col_indices, weights, device, flags,
                                             opts);
    if (st != GRAPE_OK) return st;
    grape_table_options o{};
    if (opts != nullptr) o = *opts;
    return build_graph(num_nodes, num_arcs, row_offsets, col_indices, weights, device, flags, o, out);
}

grape_status grape_graph_from_csr(uint32_t num_nodes, uint64_t num_arcs, const uint64_t* row_offsets,
                                  const uint32_t* col_indices, const uint32_t* weights, int device,
                                  uint32_t flags, grape_graph** out)
{
    return grape_graph_from_csr_opts(num_nodes, num_arcs, row_offsets, col_indices, weights, device, flags,
                                     nullptr, out);
}

grape_status grape_graph_free(grape_graph* g)
{
    g_err[0] = 0;
    if (g == nullptr) return GRAPE_OK;
    DeviceGuard guard(g->device);
    cudaError_t e = cudaDeviceSynchronize();
    destroy_graph(g);
    if (e != cudaSuccess) return cuda_fail(e, "grape_graph_free synchronize");
    return GRAPE_OK;
}

grape_status grape_graph_get_info(const grape_graph* g, grape_graph_info* info)
{
    if (g == nullptr || info == nullptr) {
        set_error("graph and info must be non-NULL");
        return GRAPE_EINVAL;
    }
    info->num_nodes = g->n;
    info->num_arcs = g->m;
    info->weighted = g->cw_bytes != 0;
    info->flags = g->flags;
    info->cw_bytes = g->cw_bytes;
    info->max_degree = g->max_degree;
    info->max_row_weight = g->max_row_weight;
    info->device_bytes = g->device_bytes;
    info->device = g->device;
    info->tables = g->tables ? 1u : 0u;
    info->weights_symmetric = g->wsym ? 1u : 0u;
    info->table_bytes = g->table_bytes;
    info->guide_factor = g->guide_factor;
    info->guide_bytes = g->guide_bytes;
    info->record_bytes = g->tables ? g->rec_bytes : 0;
    info->hash_h = g->hash_h;
    info->notri = g->notri ? 1u : 0u;
    info->parts = g->parts;
    info->wide = g->wide ? 1u : 0u;
    return GRAPE_OK;
}

grape_status grape_walks_first_order(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                     uint64_t walk_id_base, uint32_t walk_length, uint64_t seed,
                                     uint32_t* out, uint64_t* steps_out, cudaStream_t stream)
{
    return walks_common(g, starts, num_walks, walk_id_base, walk_length, false, 1.0, 1.0, seed, out,
                        steps_out, stream);
}

grape_status grape_walks_node2vec(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, double p, double q,
                                  uint64_t seed, uint32_t* out, uint64_t* steps_out, cudaStream_t stream)
{
    return walks_common(g, starts, num_walks, walk_id_base, walk_length, true, p, q, seed, out,
                        steps_out, stream);
}

grape_status grape_walks_approx(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                uint64_t walk_id_base, uint32_t walk_length, int node2vec, double p, double q,
                                uint32_t degree_threshold, uint64_t seed, uint32_t* out, uint64_t* steps_out,
                                cudaStream_t stream)
{
    if (!node2vec) { p = 1.0; q = 1.0; }
    return walks_common(g, starts, num_walks, walk_id_base, walk_length, node2vec != 0, p, q, seed, out,
                        steps_out, stream, degree_threshold);
}

grape_status grape_walks_node2vec_cdf(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                      uint64_t walk_id_base, uint32_t walk_length, double p, double q,
                                      uint64_t seed, uint32_t* out, uint64_t* steps_out, cudaStream_t stream)
{
    return walks_common(g, starts, num_walks, walk_id_base, walk_length, true, p, q, seed, out, steps_out,
                        stream, 0, 1);
}

grape_status grape_walks_node2vec_folded(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                         uint64_t walk_id_base, uint32_t walk_length, double p, double q,
                                         uint64_t seed, uint32_t* out, uint64_t* steps_out, cudaStream_t stream)
{
    return walks_common(g, starts, num_walks, walk_id_base, walk_length, true, p, q, seed, out, steps_out,
                        stream, 0, 2);
}

grape_status grape_skipgram_pairs(const grape_graph* g, const uint32_t* walks, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, uint32_t window,
                                  uint32_t num_negatives, uint64_t seed, uint32_t* centers, uint32_t* contexts,
                                  uint32_t* negatives, cudaStream_t stream)
{
    g_err[0] = 0;
    if (g == nullptr || (num_walks > 0 && (walks == nullptr || centers == nullptr || contexts == nullptr ||
                                           (num_negatives > 0 && negatives == nullptr)))) {
        set_error("graph, walks, centers, contexts (and negatives when num_negatives > 0) must be non-NULL");
        return GRAPE_EINVAL;
    }
    if (walk_length == 0 || window == 0 || window > 1024 || num_negatives > 1024) {
        set_error("need walk_length >= 1, 1 <= window <= 1024, num_negatives <= 1024");
        return GRAPE_EINVAL;
    }
    const uint64_t slots_per_walk = (uint64_t)walk_length * 2 * window;
    if (slots_per_walk * (num_negatives > 0 ? num_negatives : 1) >= (1ull << 32)) {
        set_error("walk_length * 2 * window * num_negatives must be < 2^32 (one row's output words)");
        return GRAPE_EINVAL;
    }
    const uint64_t max_wid = (~0ull) / slots_per_walk;   // global slot ids must fit 64 bits
    if (num_walks > (~0ull) / slots_per_walk / 4 / (num_negatives + 1) || num_walks > max_wid ||
        walk_id_base > max_wid - num_walks) {
        set_error("the slot count (num_walks * walk_length * 2 * window * (1 + num_negatives)) overflows");
        return GRAPE_EINVAL;
    }
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) { cudaGetLastError(); cur = -1; }
    if (cur != g->device) {
        set_error("current device %d is not the graph's device %d", cur, g->device);
        return GRAPE_EINVAL;
    }
    if (num_walks == 0) return GRAPE_OK;
    if (classify(walks) != Mem::Device || classify(centers) != Mem::Device || classify(contexts) != Mem::Device ||
        (num_negatives > 0 && classify(negatives) != Mem::Device)) {
        set_error("grape_skipgram_pairs needs device buffers (walks, centers, contexts, negatives)");
        return GRAPE_EINVAL;
    }
    cudaError_t e = ensure_node_guide(const_cast<grape_graph*>(g), stream);
    if (e != cudaSuccess) return cuda_fail(e, "node guide for the negatives");
    e = launch_skipgram(g, walks, num_walks, walk_id_base, walk_length, window, num_negatives, seed, centers,
                        contexts, negatives, stream);
    if (e != cudaSuccess) return cuda_fail(e, "skipgram kernel launch");
    return GRAPE_OK;
}

grape_status grape_walks_skipgram(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, int node2vec, double p, double q,
                                  uint64_t walk_seed, uint32_t window, uint32_t num_negatives, uint64_t pair_seed,
                                  uint32_t* centers, uint32_t* contexts, uint32_t* negatives, uint64_t* steps_out,
                                  uint64_t chunk_walks, cudaStream_t stream)
{
    g_err[0] = 0;
    if (g == nullptr || (num_walks > 0 && (starts == nullptr || centers == nullptr || contexts == nullptr ||
                                           (num_negatives > 0 && negatives == nullptr)))) {
        set_error("graph, starts, centers, contexts (and negatives when num_negatives > 0) must be non-NULL");
        return GRAPE_EINVAL;
    }
    if (walk_length == 0 || window == 0 || window > 1024 || num_negatives > 1024) {
        set_error("need walk_length >= 1, 1 <= window <= 1024, num_negatives <= 1024");
        return GRAPE_EINVAL;
    }
    const uint64_t slots_per_walk = (uint64_t)walk_length * 2 * window;
    if (slots_per_walk * (num_negatives > 0 ? num_negatives : 1) >= (1ull << 32)) {
        set_error("walk_length * 2 * window * num_negatives must be < 2^32 (one row's output words)");
        return GRAPE_EINVAL;
    }
    const uint64_t max_wid = (~0ull) / slots_per_walk;
    if (num_walks > (~0ull) / slots_per_walk / 4 / (num_negatives + 1) || num_walks > max_wid ||
        walk_id_base > max_wid - num_walks) {
        set_error("the slot count (num_walks * walk_length * 2 * window * (1 + num_negatives)) overflows");
        return GRAPE_EINVAL;
    }
    Thresholds T{1ull << 32, 1ull << 32, 1ull << 32};
    if (node2vec && !node2vec_thresholds(p, q, &T)) return GRAPE_EINVAL;
    if (g->dist && !g->tables) {
        set_error("a distributed graph walks after grape_graph_dist_finish");
        return GRAPE_EINVAL;
    }
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) { cudaGetLastError(); cur = -1; }
    if (cur != g->device) {
        set_error("current device %d is not the graph's device %d", cur, g->device);
        return GRAPE_EINVAL;
    }
    if (num_walks == 0) return GRAPE_OK;
    if (classify(starts) != Mem::Device || classify(centers) != Mem::Device || classify(contexts) != Mem::Device ||
        (num_negatives > 0 && classify(negatives) != Mem::Device) ||
        (steps_out != nullptr && classify(steps_out) != Mem::Device)) {
        set_error("grape_walks_skipgram needs device buffers (starts, centers, contexts, negatives, steps_out)");
        return GRAPE_EINVAL;
    }
    cudaError_t e = ensure_node_guide(const_cast<grape_graph*>(g), stream);
    if (e != cudaSuccess) return cuda_fail(e, "node guide for the negatives");
    WalkArgs a{};
    a.starts = starts;
    a.num_walks = num_walks;
    a.walk_id_base = walk_id_base;
    a.L = walk_length;
    a.seed = walk_seed;
    a.steps_out = (unsigned long long*)steps_out;
    if (chunk_walks == 0) {
        // Automatic chunk: 4 rounds of the walker's resident lanes (1024 per SM), so each
        // walker launch has few partial waves, and at least two chunks so that the walker
        // of chunk k+1 overlaps the pair kernel of chunk k (measured: chunks of 24 MB of
        // rows, ~half a wave each, ran 0.87x the two separate calls on configs[1]; the
        // rows' HBM round trip, 4L bytes written and read per walk, is small next to the
        // pair kernel's 4 (2 + K) 2wL bytes of output per walk).
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
        chunk_walks = 4ull * 1024 * (uint64_t)(sms > 0 ? sms : 148);
        if (chunk_walks > (num_walks + 1) / 2) chunk_walks = (num_walks + 1) / 2;
        if (chunk_walks < 1) chunk_walks = 1;
    }
    e = launch_walks_skipgram(g, a, node2vec != 0, T, window, num_negatives, pair_seed, centers, contexts,
                              num_negatives ? negatives : nullptr, chunk_walks, stream);
    if (e != cudaSuccess) return cuda_fail(e, "grape_walks_skipgram");
    return GRAPE_OK;
}

grape_status grape_walks_stats(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                               uint64_t walk_id_base, uint32_t walk_length, int node2vec, double p,
                               double q, uint64_t seed, uint32_t* out, grape_walk_stats* stats,
                               cudaStream_t stream)
{
    return grape_walks_stats_ex(g, starts, num_walks, walk_id_base, walk_length, node2vec, p, q, 0, 0, seed,
                                out, stats, stream);
}

grape_status grape_walks_stats_ex(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, int node2vec, double p,
                                  double q, uint32_t degree_threshold, int sampler, uint64_t seed, uint32_t* out,
                                  grape_walk_stats* stats, cudaStream_t stream)
{
    g_err[0] = 0;
    if (g == nullptr || stats == nullptr || (num_walks > 0 && (starts == nullptr || out == nullptr))) {
        set_error("graph, stats, starts and out must be non-NULL");
        return GRAPE_EINVAL;
    }
    if (walk_length == 0) {
        set_error("walk_length must be >= 1");
        return GRAPE_EINVAL;
    }
    if (num_walks > (~0ull) / walk_length / 4) {
        set_error("num_walks * walk_length overflows");
        return GRAPE_EINVAL;
    }
    Thresholds T{1ull << 32, 1ull << 32, 1ull << 32};
    if (node2vec && !node2vec_thresholds(p, q, &T)) return GRAPE_EINVAL;
    uint32_t dT = degree_threshold >= g->max_degree ? 0 : degree_threshold;
    if (dT != 0 && !g->tables) {
        set_error("approximated walks need the sampling tables");
        return GRAPE_EINVAL;
    }
    if (g->parts > 1 && (dT != 0 || sampler != 0)) {
        set_error("a partitioned graph (grape_graph_partition) serves the default walk rules only");
        return GRAPE_EINVAL;
    }
    if (g->dist && !g->tables) {
        set_error("a distributed graph walks after grape_graph_dist_finish");
        return GRAPE_EINVAL;
    }
    if (g->wide && (dT != 0 || sampler != 0)) {
        set_error("a graph with 2^32 - 64 or more arcs serves the default walk rules only");
        return GRAPE_EINVAL;
    }
    if (sampler != 0 && (sampler != 2 || !g->tables || dT != 0 || !node2vec ||
                         (g->cw_bytes != 0 && g->compact && !g->wsym))) {
        set_error("grape_walks_stats_ex: sampler %d is not available with these arguments / this graph "
                  "(counting builds exist for the default and the outlier-folded samplers)", sampler);
        return GRAPE_EINVAL;
    }
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) { cudaGetLastError(); cur = -1; }
    if (cur != g->device) {
        set_error("current device %d is not the graph's device %d", cur, g->device);
        return GRAPE_EINVAL;
    }
    memset(stats, 0, sizeof(*stats));
    if (num_walks == 0) return GRAPE_OK;
    if (classify(starts) != Mem::Device || classify(out) != Mem::Device) {
        set_error("grape_walks_stats needs device starts and out");
        return GRAPE_EINVAL;
    }
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long) * kStatsWords);
    if (e != cudaSuccess) return cuda_fail(e, "stats buffer");
    WalkArgs a{};
    a.starts = starts;
    a.num_walks = num_walks;
    a.walk_id_base = walk_id_base;
    a.L = walk_length;
    a.seed = seed;
    a.out = out;
    a.stats = d;
    a.dT = dT;
    a.sampler = (uint32_t)sampler;
    e = cudaMemsetAsync(d, 0, sizeof(unsigned long long) * kStatsWords, stream);
    if (e == cudaSuccess) e = launch_walks(g, a, node2vec != 0, T, stream);
    unsigned long long h[kStatsWords] = {0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "grape_walks_stats");
    stats->sector_loads = h[0];
    stats->node_loads = h[1];
    stats->xnode_loads = h[2];
    stats->cw_probes = h[3];
    stats->col_probes = h[4];
    stats->col_loads = h[5];
    stats->attempts = h[6];
    stats->membership_tests = h[7];
    stats->start_loads = h[8];
    stats->steps = h[9];
    stats->guide_loads = h[10];
    stats->hash_probes = h[11];
    stats->alu_decisions = h[12];
    stats->iterations = h[13];
    stats->draw_iterations = h[14];
    stats->back_iterations = h[15];
    return GRAPE_OK;
}

const char* grape_status_string(grape_status s)
{
    switch (s) {
    case GRAPE_OK: return "GRAPE_OK";
    case GRAPE_EINVAL: return "GRAPE_EINVAL: invalid argument";
    case GRAPE_ENOMEM: return "GRAPE_ENOMEM: out of device memory";
    case GRAPE_ECUDA: return "GRAPE_ECUDA: CUDA error";
    default: return "GRAPE_UNKNOWN";
    }
}

const char* grape_last_error(void) { return g_err; }

const char* grape_version(void) { return "grape-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
