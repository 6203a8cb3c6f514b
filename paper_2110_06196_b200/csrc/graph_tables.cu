// graph_tables.cu — sampling tables for the v4 walker, built
// once per graph next to the CSR (not on the timed path).
//
// The rules of a walk (include/grape_walk.h) touch the graph in three ways per
// attempt: the proposal index i = min{i : cw[off_v + i] > r}, the
// proposal x = col[off_v + i], and the class of x — p if x == t,
// 1 if x in N(t), q otherwise.  The tables answer each with one
// sector read instead of a search, and never change a result:
//
//   rec    per arc e = (v -> x), arc order, one aligned sector or half of one:
//            weighted (32 B)   {x, hi = cw[e], rlo, rhi, off[x], deg x, W_x, lo = cw[e-1]}
//                              [rlo, rhi) = the r-interval of the reverse arc (x -> v)
//                              inside x's row, [0,0) if there is none
//            unweighted (16 B) {x, rev, off[x], deg x}  rev = index of v in N(x) or NONE
//          With it the walker knows, at x coming from v, which draws propose
//          x' == v (the "return" class p) without reading anything, and
//          it has x's node record without a second read.
//   guide  weighted rows only, B_v = G deg(v) entries at G off[v] (G = 16, 8, 4, 2 or 1,
//          32-B "fat" or 8-B "slim" entries, by free memory; a fat entry of an
//          unsplit bucket is a copy of the record): entry kb covers the x64 draws with
//          floor(x64 * B_v / 2^64) = kb; it holds i_lo = the proposal index of
//          the smallest such draw, and either the proposal col[i_lo] itself
//          (every draw of the bucket proposes i_lo) or, for a "split" bucket,
//          cw[i_lo] to settle i_lo vs i_lo + 1 by one compare (and a MULTI bit
//          when the bucket spans more boundaries: the walker then scans the
//          records comparing r with hi).  A guide table (Chen & Asau) for the
//          inverse-CDF search of P:509-511.
//   ehash  per-row set of N(v) for "x in N(t)": floor(deg v / 4) + 1 buckets of
//          8 u32 slots (one sector each) from bucket floor(off[v] / 4) + v;
//          bucketised linear probing from bucket floor(fmix32(x) nb / 2^32);
//          empty = 0xFFFFFFFF (never a node id).  Load factor <= 1/2, so a
//          lookup reads one sector unless its home bucket is full.
// Index ranges: m < 2^34 - 64 (row starts of 32 bits, or 34 bits in "wide" graphs: the high
// bits in bits 26-27 of a record's degree word), m/4 + n < 2^32 (u32 edge-hash bucket
// indices), max degree < 2^28 (2^26 when wide; flag bits, guide bits 30-31, G deg < 2^32),
// row sums < 2^32 (u32 prefix).  When the tables are
// built, col / cw / fences are released (graph.cu): nothing reads them after.  Outside them the tables are not built and
// the v3 walker (fenced searches) runs.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "internal.h"
#include "build_common.cuh"

namespace grape {
namespace {

constexpr int kThreads = 256;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__host__ __device__ inline uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

// First index in [a, b) with col[j] >= key (b if none).
__device__ inline uint64_t lower_bound_u32(const uint32_t* __restrict__ col, uint64_t a, uint64_t b, uint32_t key)
{
    while (a < b) {
        const uint64_t mid = a + ((b - a) >> 1);
        if (col[mid] < key) a = mid + 1; else b = mid;
    }
    return a;
}

// First index in [a, b) with cw[j] > key (b if none).
__device__ inline uint64_t upper_bound_u32(const uint32_t* __restrict__ cw, uint64_t a, uint64_t b, uint32_t key)
{
    while (a < b) {
        const uint64_t mid = a + ((b - a) >> 1);
        if (cw[mid] <= key) a = mid + 1; else b = mid;
    }
    return a;
}

// One thread per arc of [e_lo, e_hi) (build_common.cuh: hub rows do not leave a
// tail).  Each record also carries the node record of its head x (start, degree,
// W_x), so a walk that takes the arc needs no separate node load.
// Flags of arc e = (v -> x) (rev = its reverse arc): NOTRI_SELF = notri[e] (used on
// arriving at x through e), NOTRI_REV = notri[rev] (used on a register-decided return
// x -> v).  Full records keep them in bits 29 / 28 of the degree word, compact records
// in bits 31 / 30 of x (only when n < 2^30; else never set).
// sym_half: the flags were computed for arcs t -> v with t < v only (build_notri) and
// are read from that canonical arc for both directions.  need_rev: every arc must
// have its reverse (GRAPE_SYMMETRIC, checked here instead of a separate pass;
// bit 1 of *asym when one has none).
// Full records keep the head's row start xa (+ the arc-offset test bias): bits 0-31 in
// their own word, bits 32-33 in bits 26-27 of the degree word (tables past 2^32 arcs).
template <bool WEIGHTED, bool COMPACT>
__global__ void build_records(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col,
                              const uint32_t* __restrict__ cw, uint32_t n, uint64_t e_lo, uint64_t e_hi,
                              const TabRef rec, unsigned* __restrict__ asym, const TabRef notri, bool sym_half,
                              bool need_rev, uint64_t bias)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const bool flags = notri.base[0] != nullptr;
    bool bad = false, norev = false;
    for (uint64_t e = e_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e_hi; e += stride) {
        const uint32_t v = build::row_of(off, n, e);
        const uint64_t lo = off[v];
        const uint32_t x = col[e];
        const uint64_t xa = off[x], xb = off[x + 1];
        const uint64_t j = lower_bound_u32(col, xa, xb, v);
        const bool found = j < xb && col[j] == v;
        norev |= !found;
        uint32_t fl = 0;   // flag bits (0: self, 1: reverse)
        if (flags && sym_half && found) {   // one flag per undirected edge, on the arc from the smaller id
            fl = *notri.at(v < x ? e : j) ? 3u : 0u;
        } else if (flags) {
            fl = (*notri.at(e) ? 1u : 0u) | (found && *notri.at(j) ? 2u : 0u);
        }
        const uint32_t xf = COMPACT ? (x | (fl & 1) << 31 | (fl >> 1) << 30) : x;   // compact: bits 31 (self), 30 (rev)
        const uint64_t xs = xa + bias;   // the head's row start as the walker sees it
        const uint32_t df = COMPACT ? 0u : ((fl & 1) << 29 | (fl >> 1) << 28 | (uint32_t)((xs >> 32) & 3u) << 26);
        if (WEIGHTED) {
            const uint32_t own_hi = cw[e];
            const uint32_t own_lo = e > lo ? cw[e - 1] : 0u;
            uint32_t rlo = 0, rhi = 0;
            if (found) {
                rlo = j > xa ? cw[j - 1] : 0u;
                rhi = cw[j];
                bad |= (rhi - rlo) != own_hi - own_lo;
            }
            if (COMPACT) {
                *reinterpret_cast<uint4*>(rec.at(16 * e)) = make_uint4(xf, own_hi, rlo, rhi);
            } else {
                const uint32_t xW = xb > xa ? cw[xb - 1] : 0u;
                uint4* r = reinterpret_cast<uint4*>(rec.at(32 * e));   // one sector: never split by a part
                r[0] = make_uint4(x, own_hi, rlo, rhi);
                r[1] = make_uint4((uint32_t)xs, (uint32_t)(xb - xa) | df, xW, own_lo);
            }
        } else {
            const uint32_t rev = found ? (uint32_t)(j - xa) : kNone;
            if (COMPACT)
                *reinterpret_cast<uint2*>(rec.at(8 * e)) = make_uint2(xf, rev);
            else
                *reinterpret_cast<uint4*>(rec.at(16 * e)) = make_uint4(x, rev, (uint32_t)xs, (uint32_t)(xb - xa) | df);
        }
    }
    if (WEIGHTED && bad) atomicOr(asym, 1u);
    if (need_rev && norev) atomicOr(asym, 2u);
}

// Guide entries, one thread per bucket of [b_lo, b_hi) (global bucket gb = G off[v]
// + kb, so v = row_of(gb / G)): bucket kb of B = G deg covers the draws x64 in
// [ceil(kb 2^64 / B), ceil((kb+1) 2^64 / B)).  With 2^64 = Q B + R:
// ceil(kb 2^64 / B) = kb Q + ceil(kb R / B)  (kb R < B^2 < 2^64).
// i_lo = the proposal index of the bucket's smallest draw; the bucket is "split"
// when its largest draw proposes a later index (MULTI: more than one later).
struct Bucket {
    uint64_t lo;   // off[v]
    uint32_t i;    // i_lo
    bool split, multi;
};

__device__ __forceinline__ Bucket guide_bucket(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cw,
                                               uint32_t n, uint32_t G, uint64_t gb)
{
    const uint32_t v = build::row_of(off, n, gb >> (31 - __clz(G)));   // G is a power of two
    const uint64_t lo = off[v], hi = off[v + 1], deg = hi - lo;
    const uint64_t B = G * deg, kb = gb - G * lo;
    const uint64_t W = cw[hi - 1];
    uint64_t Q = ~0ull / B, R = ~0ull % B + 1;   // 2^64 = Q B + R, 0 <= R < B
    if (R == B) { ++Q; R = 0; }
    const uint64_t xmin = kb * Q + (kb * R + B - 1) / B;
    const uint64_t xmax = kb + 1 == B ? ~0ull : (kb + 1) * Q + ((kb + 1) * R + B - 1) / B - 1;
    const uint32_t rmin = (uint32_t)__umul64hi(xmin, W), rmax = (uint32_t)__umul64hi(xmax, W);
    Bucket b;
    b.lo = lo;
    b.i = (uint32_t)(upper_bound_u32(cw, lo, hi, rmin) - lo);   // < deg since cw[hi-1] = W > rmin
    b.split = cw[lo + b.i] <= rmax;
    b.multi = b.split && cw[lo + b.i + 1] <= rmax;              // i + 1 < deg when split
    return b;
}

// Slim guide (8-B entries) {e0, e1}: e0 = i_lo | SPLIT (bit 31) | MULTI (bit 30);
// unsplit: e1 = col[i_lo] (the proposal itself); split: e1 = cw[i_lo], the upper end
// of i_lo's interval (r < e1 -> i_lo, else i_lo + 1 unless MULTI: then scan the records).
__global__ void build_guide(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col,
                            const uint32_t* __restrict__ cw, uint32_t n, uint64_t b_lo, uint64_t b_hi, uint32_t G,
                            const TabRef guide)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t gb = b_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gb < b_hi; gb += stride) {
        const Bucket b = guide_bucket(off, cw, n, G, gb);
        *reinterpret_cast<uint2*>(guide.at(8 * gb)) =
            make_uint2(b.i | (b.split ? 0x80000000u : 0u) | (b.multi ? 0x40000000u : 0u),
                       b.split ? cw[b.lo + b.i] : col[b.lo + b.i]);
    }
}

// Fat guide (32-B entries, one sector): an unsplit bucket holds a copy of the
// record of its proposal i_lo (so a proposal from it needs no other read), with
// bits 30-31 of word 5 (the degree of x, < 2^29) clear; a split bucket holds
// {i_lo, cw[i_lo], 0, 0, 0, SPLIT | MULTI<<30, 0, 0}.
__global__ void build_guide_fat(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cw, uint32_t n,
                                uint64_t b_lo, uint64_t b_hi, uint32_t G, const TabRef rec, const TabRef guide)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t gb = b_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gb < b_hi; gb += stride) {
        const Bucket b = guide_bucket(off, cw, n, G, gb);
        uint4* d = reinterpret_cast<uint4*>(guide.at(32 * gb));
        if (b.split) {
            d[0] = make_uint4(b.i, cw[b.lo + b.i], 0u, 0u);
            d[1] = make_uint4(0u, 0x80000000u | (b.multi ? 0x40000000u : 0u), 0u, 0u);
        } else {
            const uint4* r = reinterpret_cast<const uint4*>(rec.at(32 * (b.lo + b.i)));
            d[0] = r[0];
            d[1] = r[1];
        }
    }
}

// Bucketised sets: row v owns the 8-slot buckets [B_v, B_v + nb_v), B_v =
// floor(off[v] / H) + v, nb_v = floor(deg v / H) + 1, H = 4 (load <= 1/2) or 6
// (<= 3/4): disjoint across rows since floor((a + d) / H) - floor(a / H) >=
// floor(d / H), and derivable from the node record.  x goes to the first empty slot
// of bucket B_v + floor(fmix32(x) nb_v / 2^32), or of the next non-full bucket
// (cyclically): a bucket that an item skipped is full forever (no deletions),
// so a lookup may stop at the first bucket holding x or an empty slot.  One
// thread per arc of [h_lo, h_hi) (whole rows: one builder owns a row's buckets).
__global__ void build_ehash(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col, uint32_t n,
                            uint64_t h_lo, uint64_t h_hi, uint32_t H, const TabRef ehash)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = h_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < h_hi; e += stride) {
        const uint32_t v = build::row_of(off, n, e);
        const uint64_t lo = off[v], hi = off[v + 1];
        const uint64_t base = lo / H + v, nb = (hi - lo) / H + 1;
        const uint32_t x = col[e];
        uint64_t b = ((uint64_t)fmix32(x) * nb) >> 32;
        for (uint64_t tries = 0; tries < nb; ++tries) {   // nb * 8 slots >= deg + 1 > items: ends
            uint32_t* slot = reinterpret_cast<uint32_t*>(ehash.at(32 * (base + b)));   // a bucket is one sector
            // slot q is tried only after slots 0 .. q-1 were found taken and nothing is removed, so
            // a bucket's taken slots are always a prefix: the walker (walk_tab.cu, ST_HASH) reads
            // "has an empty slot" from slot 7 alone and the checked build asserts the prefix
            int q = 0;
            while (q < 8 && atomicCAS(slot + q, kEmpty, x) != kEmpty) ++q;
            if (q < 8) break;
            b = b + 1 == nb ? 0 : b + 1;
        }
    }
}

// notri[e] for arc e = (t -> v): 1 iff no x != t in N(v) lies in N(t), i.e. at v
// coming from t every proposal other than t itself is in class q (P:453-470:
// X_beta = N(v) \ N(t) is all of N(v) \ {t}).  The shorter of N(t), N(v) is scanned
// and each entry probed in the other's edge-hash set, stopping at the first common
// neighbour.  One thread per arc; an arc whose shorter row exceeds kCoopLen entries
// is scanned by its whole warp instead (the lanes stride over the row, the warp
// stops as soon as any lane finds a common neighbour), so the work of a warp is
// bounded by kCoopLen sequential probes per lane plus 1/32 of its long scans.
__device__ inline bool hash_has(const TabRef& ehash, uint64_t base, uint64_t nb, uint32_t x)
{
    uint64_t b = ((uint64_t)fmix32(x) * nb) >> 32;
    for (uint64_t tries = 0; tries < nb; ++tries) {
        const uint32_t* slot = reinterpret_cast<const uint32_t*>(ehash.at(32 * (base + b)));
        bool empty = false;
        for (int q = 0; q < 8; ++q) {
            const uint32_t y = slot[q];
            if (y == x) return true;
            empty |= y == kEmpty;
        }
        if (empty) return false;
        b = b + 1 == nb ? 0 : b + 1;
    }
    return false;
}

constexpr uint64_t kCoopLen = 32;
// Scans of more than kNotriScanCap entries stop there with the flag clear ("may share a
// neighbour": the walker then tests membership as usual).  The flag only enables a
// shortcut, so clearing it never changes a walk; it bounds the build's cost on pairs
// of high-degree nodes with no common neighbour (full scans of long rows).  256
// measured (round 2, tools/ab_build.sh): configs[2] build 710 -> 442 ms, configs[3]
// 1608 -> 1386 ms, walks unchanged (configs[3] +0.4%); 64 costs walk time (+3%).
#ifndef GRAPE_NOTRI_SCAN_CAP
#define GRAPE_NOTRI_SCAN_CAP 256
#endif
constexpr uint64_t kNotriScanCap = GRAPE_NOTRI_SCAN_CAP;

// sym_half (a symmetric graph without self-loops): the common neighbours of t and v
// other than t are those other than v (t is not in N(t), v is not in N(v)), so the
// flag of t -> v equals that of v -> t: only arcs with t < v are computed.
__global__ void build_notri(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col, uint32_t n,
                            uint64_t e_lo, uint64_t e_hi, uint32_t H, const TabRef ehash, const TabRef notri,
                            bool sym_half)
{
    const unsigned lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // every lane of a warp runs the same number of rounds (the warp-cooperative scans
    // below need all 32 lanes): rounds over [e_lo, e_hi) rounded up to whole warps
    const uint64_t span = ((e_hi - e_lo) + 31) & ~31ull;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < span; k += stride) {
        const uint64_t e = e_lo + k;
        const bool valid = e < e_hi;
        uint32_t t = 0;
        uint64_t sa = 0, sb = 0;          // the scanned (shorter) row
        uint64_t hbase = 0, hnb = 0;      // the probed row's hash buckets
        bool skip = false;
        if (valid) {
            t = build::row_of(off, n, e);
            const uint32_t v = col[e];
            skip = sym_half && v < t;   // the reverse arc carries this edge's flag
            const uint64_t ta = off[t], tb = off[t + 1], va = off[v], vb = off[v + 1];
            if (vb - va <= tb - ta) {   // x in N(v), x != t: in N(t)?
                sa = va; sb = vb;
                hbase = ta / H + t; hnb = (tb - ta) / H + 1;
            } else {                    // x in N(t), x != t: in N(v)?
                sa = ta; sb = tb;
                hbase = va / H + v; hnb = (vb - va) / H + 1;
            }
        }
        const bool capped = sb - sa > kNotriScanCap;   // too long to scan: the flag stays clear
        if (capped) sb = sa;
        bool common = false;
        if (skip) sa = sb = 0;   // nothing to scan
        const bool coop = valid && !skip && sb - sa > kCoopLen;
        if (valid && !skip && !coop)
            for (uint64_t f = sa; f < sb && !common; ++f) {
                const uint32_t x = col[f];
                common = x != t && hash_has(ehash, hbase, hnb, x);
            }
        unsigned big = __ballot_sync(0xffffffffu, coop);
        while (big) {   // the long scans, one at a time, by the whole warp
            const int src = __ffs(big) - 1;
            big &= big - 1;
            const uint64_t a = __shfl_sync(0xffffffffu, sa, src), b = __shfl_sync(0xffffffffu, sb, src);
            const uint64_t hb0 = __shfl_sync(0xffffffffu, hbase, src), hn = __shfl_sync(0xffffffffu, hnb, src);
            const uint32_t tt = __shfl_sync(0xffffffffu, t, src);
            bool found = false;
            for (uint64_t f0 = a; f0 < b; f0 += 32) {   // uniform trip count across the warp
                const uint64_t f = f0 + lane;
                bool c = false;
                if (f < b) {
                    const uint32_t x = col[f];
                    c = x != tt && hash_has(ehash, hb0, hn, x);
                }
                if (__any_sync(0xffffffffu, c)) { found = true; break; }
            }
            if ((int)lane == src) common = found;
        }
        if (valid && !skip) *reinterpret_cast<uint8_t*>(notri.at(e)) = (common || capped) ? 0 : 1;
    }
}

uint64_t padded(uint64_t bytes) { return ((bytes + 31) / 32) * 32 + 32; }

__global__ void bias_node_starts(NodeRec* __restrict__ nodes, uint32_t n, uint64_t bias)
{
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) nodes[v].start += bias;
}

TabRef flat(void* p, uint64_t bytes)
{
    TabRef t{};
    t.base[0] = (char*)p;
    t.shift = 63;
    t.bytes = p ? bytes : 0;
    return t;
}

}  // namespace

void destroy_tables(grape_graph* g)
{
    cudaFree(g->rec);
    cudaFree(g->guide);
    cudaFree(g->ehash);
    g->rec = nullptr;
    g->guide = nullptr;
    g->ehash = nullptr;
    g->guide_factor = 0;
    g->guide_bytes = 0;
    g->hash_h = 0;
    g->compact = false;
    g->notri = false;
    g->tables = false;
    g->table_bytes = 0;
}

// Random-sector gather rate falls off a cliff once the randomly read footprint
// exceeds ~68 GB on B200 (36 G sectors/s up to 68 GB, 28 at 80 GB, 10.5 at 128 GB;
// tools/gather_footprint.cu, profiles/gather_footprint.txt; page size does not
// move it, tools/gather_vmm.cu).  The automatic layout stays below it.
constexpr double kReachBytes = 68e9;

bool tables_in_range(const grape_graph* g)
{
    const uint64_t m = g->m, n = g->n;
    // arc offsets (node records, the records' copy of off[x]) are u32 in the walker; edge-hash
    // bucket indices floor(off / H) + v are u32; degrees leave 4 flag bits in their word;
    // the guide's per-row bucket index G deg is u32; row sums are u32 prefix values
    // (34-bit offsets, "wide", past 2^32 - 64 arcs: bits 32-33 of a row start ride in bits 26-27
    // of a record's degree word, so degrees stay below 2^26 there)
    const bool wide = m >= (1ull << 32) - 64;
    return !(m >= (1ull << 34) - 64 || (m >> 2) + n + 2 >= (1ull << 32) ||
             g->max_degree >= (wide ? (1u << 26) : (1u << 28)) || g->cw_bytes == 8);
}

// Layout, in order of preference (fewest reads per step first): records with the
// head's node record (32 / 16 B) or compact (16 / 8 B, the head's node record read
// separately); fat (32-B) or slim (8-B) guide entries with G = 16 / 8 / 4 / 2 / 1
// buckets per arc; edge-hash load 1/2 (H = 4) or 3/4 (H = 6).  The first that fits
// `budget` wins (grape_table_options may force any part).  Results do not depend
// on the choice; the number and spread of the reads do.
int choose_layout(grape_graph* g, const grape_table_options& o, double budget)
{
    const uint64_t m = g->m, n = g->n;
    const bool weighted = g->cw_bytes != 0;
    struct Choice { uint32_t rec, gb, G, H; };
    Choice c{0, 0, 0, 0};
    auto size_of = [&](const Choice& k) {
        return (double)padded(m * k.rec) + (double)padded(((m / k.H) + n + 1) * 32) +
               (weighted ? (double)padded((uint64_t)k.G * m * k.gb) : 0.0);
    };
    auto allowed = [&](const Choice& k) {
        return (!o.record_bytes || o.record_bytes == k.rec) && (!o.guide_bytes || o.guide_bytes == k.gb) &&
               (!o.guide_factor || o.guide_factor == k.G) && (!o.hash_h || o.hash_h == k.H);
    };
    bool found = false, any_allowed = false;
    const uint32_t recs_w[2] = {32u, 16u}, recs_u[2] = {16u, 8u};
    const uint32_t gbs_w[2] = {32u, 8u}, gbs_u[1] = {0u};
    const uint32_t Gs_w[5] = {16u, 8u, 4u, 2u, 1u}, Gs_u[1] = {0u};
    const uint32_t Hs[2] = {4u, 6u};
    const uint32_t* recs = weighted ? recs_w : recs_u;
    const uint32_t* gbs = weighted ? gbs_w : gbs_u;
    const uint32_t* Gs = weighted ? Gs_w : Gs_u;
    const int ngb = weighted ? 2 : 1, nG = weighted ? 5 : 1;
    for (int hi = 0; hi < 2; ++hi) {
        for (int ri = 0; ri < 2; ++ri) {
            for (int gi = 0; gi < ngb; ++gi) {
                if (gbs[gi] == 32 && recs[ri] != 32) continue;   // fat entries copy full records
                for (int fi = 0; fi < nG; ++fi) {
                    const Choice k{recs[ri], gbs[gi], Gs[fi], Hs[hi]};
                    if (found || !allowed(k)) continue;
                    any_allowed = true;
                    if ((!weighted || (uint64_t)k.G * g->max_degree < (1ull << 32)) &&
                        size_of(k) <= budget) {
                        c = k;
                        found = true;
                    }
                }
            }
        }
    }
    const bool forced = o.record_bytes || o.guide_bytes || o.guide_factor || o.hash_h;
    if (!found) {
        if (forced && any_allowed) {
            set_error("the requested table layout does not fit (%.3g bytes available)", budget);
            return -1;
        }
        return 0;
    }
    g->rec_bytes = c.rec;
    g->compact = weighted ? c.rec == 16 : c.rec == 8;
    g->guide_factor = c.G;
    g->guide_bytes = c.gb;
    g->hash_h = c.H;
    g->rec_alloc = padded(m * c.rec);
    g->hash_alloc = padded(((m / c.H) + n + 1) * 32);
    g->guide_alloc = weighted ? padded((uint64_t)c.G * m * c.gb) : 0;
    return 1;
}

cudaError_t run_table_stage(const grape_graph* g, const TableJob& j, int stage, unsigned* asym)
{
    const bool weighted = g->cw_bytes != 0;
    // one no-common-neighbour flag per undirected edge: a symmetric graph (validated, or
    // validated by this very build: need_rev) without self-loops
    const bool sym_half = (g->flags & GRAPE_SYMMETRIC) && g->validated && !g->self_loops;
    const bool need_rev = g->sym_checked_by_tables;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const uint32_t* cw = (const uint32_t*)g->cw;
    switch (stage) {
    case 0:
        if (j.h_hi > j.h_lo)
            build_ehash<<<build::item_grid(j.h_hi - j.h_lo, sms), kThreads>>>(g->off, g->col, g->n, j.h_lo, j.h_hi,
                                                                              g->hash_h, j.ehash);
        break;
    case 1:
        if (j.notri.base[0] != nullptr && j.e_hi > j.e_lo)
            build_notri<<<build::item_grid(j.e_hi - j.e_lo, sms), kThreads>>>(g->off, g->col, g->n, j.e_lo, j.e_hi,
                                                                              g->hash_h, j.ehash, j.notri, sym_half);
        break;
    case 2: {
        if (j.e_hi <= j.e_lo) break;
        const int grid = build::item_grid(j.e_hi - j.e_lo, sms);
        if (weighted && g->compact)
            build_records<true, true><<<grid, kThreads>>>(g->off, g->col, cw, g->n, j.e_lo, j.e_hi, j.rec, asym, j.notri, sym_half,
                                                          need_rev, g->arc_bias);
        else if (weighted)
            build_records<true, false><<<grid, kThreads>>>(g->off, g->col, cw, g->n, j.e_lo, j.e_hi, j.rec, asym, j.notri, sym_half,
                                                          need_rev, g->arc_bias);
        else if (g->compact)
            build_records<false, true><<<grid, kThreads>>>(g->off, g->col, nullptr, g->n, j.e_lo, j.e_hi, j.rec, asym,
                                                           j.notri, sym_half, need_rev, g->arc_bias);
        else
            build_records<false, false><<<grid, kThreads>>>(g->off, g->col, nullptr, g->n, j.e_lo, j.e_hi, j.rec, asym,
                                                            j.notri, sym_half, need_rev, g->arc_bias);
        break;
    }
    case 3:
        if (!weighted || j.b_hi <= j.b_lo) break;
        if (g->guide_bytes == 32)
            build_guide_fat<<<build::item_grid(j.b_hi - j.b_lo, sms), kThreads>>>(g->off, cw, g->n, j.b_lo, j.b_hi,
                                                                                  g->guide_factor, j.rec, j.guide);
        else
            build_guide<<<build::item_grid(j.b_hi - j.b_lo, sms), kThreads>>>(g->off, g->col, cw, g->n, j.b_lo, j.b_hi,
                                                                              g->guide_factor, j.guide);
        break;
    default: break;
    }
    return cudaGetLastError();
}

grape_status build_tables(grape_graph* g, const grape_table_options& o)
{
    const uint64_t m = g->m, n = g->n;
    const bool weighted = g->cw_bytes != 0;
    if (!tables_in_range(g)) return GRAPE_OK;
    cudaError_t e = cudaSuccess;
    unsigned* d_asym = nullptr;
    uint8_t* d_notri = nullptr;
    auto fail = [&](cudaError_t err, const char* what) {
        cudaFree(d_asym);
        cudaFree(d_notri);
        destroy_tables(g);
        return cuda_fail(err, what);
    };
    // The layout must fit the device (leaving 10% free: the caller still needs its walk
    // matrices) and the gather reach, or table_budget_bytes when given.
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const double base_b = (double)(n + 1) * 8 + (double)n * sizeof(NodeRec);
    const double cap = o.table_budget_bytes ? (double)o.table_budget_bytes : kReachBytes - base_b;
    const double budget = std::min((double)free_b - 0.1 * (double)total_b, cap);
    const int ch = choose_layout(g, o, budget);
    if (ch < 0) return GRAPE_ENOMEM;
    if (ch == 0) return GRAPE_OK;   // does not fit: v3 walker
    g->wide = m >= (1ull << 32) - 64;
    // Test hook: GRAPE_TEST_ARC_BIAS=b (rounded down to a multiple of 12, so divisible by
    // both edge-hash H) offsets every row start the walker sees by b, so a small graph
    // exercises the wide walker's 34-bit offset arithmetic end to end (tests/test_gpu_wide.py)
    if (const char* env = getenv("GRAPE_TEST_ARC_BIAS")) {
        const uint64_t b = strtoull(env, nullptr, 0) / 12 * 12;
        if (b != 0 && b + m < (1ull << 34) - 64 && g->max_degree < (1u << 26)) {
            g->arc_bias = b;
            g->wide = true;
        }
    }
    if ((e = cudaMalloc(&g->rec, g->rec_alloc)) != cudaSuccess) return fail(e, "cudaMalloc arc records");
    if (weighted && (e = cudaMalloc((void**)&g->guide, g->guide_alloc)) != cudaSuccess)
        return fail(e, "cudaMalloc guide");
    if ((e = cudaMalloc((void**)&g->ehash, g->hash_alloc)) != cudaSuccess) return fail(e, "cudaMalloc edge hash");
    if ((e = cudaMalloc((void**)&d_asym, 4)) != cudaSuccess) return fail(e, "cudaMalloc");
    cudaMemset(d_asym, 0, 4);
    cudaMemset(g->rec, 0, g->rec_alloc);
    cudaMemset(g->ehash, 0xFF, g->hash_alloc);
    if (weighted) cudaMemset(g->guide, 0, g->guide_alloc);
    // no-common-neighbour flags (a temporary byte per arc); compact records need n < 2^30
    const bool flags_ok = !(g->compact && n >= (1u << 30));
    if (flags_ok && cudaMalloc((void**)&d_notri, m ? m : 1) != cudaSuccess) {
        cudaGetLastError();
        d_notri = nullptr;
    }
    TableJob j{};
    j.e_lo = j.h_lo = j.b_lo = 0;
    j.e_hi = j.h_hi = m;
    j.b_hi = weighted ? (uint64_t)g->guide_factor * m : 0;
    j.rec = flat(g->rec, g->rec_alloc);
    j.guide = flat(g->guide, g->guide_alloc);
    j.ehash = flat(g->ehash, g->hash_alloc);
    j.notri = flat(d_notri, m);
    for (int stage = 0; stage < 4 && e == cudaSuccess; ++stage) e = run_table_stage(g, j, stage, d_asym);
    if (e != cudaSuccess) return fail(e, "table kernels");
    g->notri = d_notri != nullptr;
    if (g->arc_bias && n) bias_node_starts<<<(unsigned)((n + 255) / 256), 256>>>(g->nodes, n, g->arc_bias);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e, "node-record bias");
    unsigned asym = 0;
    if ((e = cudaMemcpy(&asym, d_asym, 4, cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e, "table build");
    if (asym & 2u) {   // GRAPE_SYMMETRIC asserted, checked by the record kernel
        cudaFree(d_asym);
        cudaFree(d_notri);
        d_asym = nullptr;
        d_notri = nullptr;
        destroy_tables(g);
        set_error("invalid CSR: GRAPE_SYMMETRIC asserted but an arc has no reverse arc");
        return GRAPE_EINVAL;
    }
    cudaFree(d_asym);
    cudaFree(d_notri);
    g->wsym = !weighted || asym == 0;
    g->table_bytes = g->rec_alloc + g->guide_alloc + g->hash_alloc;
    g->tables = true;
    return GRAPE_OK;
}

}  // namespace grape
