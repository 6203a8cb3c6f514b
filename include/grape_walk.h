/*
 * grape_walk.h — C-ABI of the B200-native GRAPE random-walk engine.
 *
 * The hot path of GRAPE (arxiv 2110.06196) that this library implements:
 * bulk first-order and second-order (node2vec p/q) random walks over a large
 * sparse graph (§4.3).  Plain C types
 * only: pointers, sizes, a CUDA stream handle.  Every call returns a
 * grape_status; nothing throws across the ABI.  On failure a thread-local
 * message is available from grape_last_error().
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * §8(x) = /root/repo/SURVEY.md §8(x); DESIGN.md §k = /root/repo/DESIGN.md.
 *
 * ---------------------------------------------------------------- the rules
 * Walk matrix: row i (L entries, u32, row-major) is the walk with id
 * wid = walk_id_base + i, starting at starts[i].  L counts nodes including the
 * start, so a full walk makes L-1 transitions ("steps") (§8(c) c1).
 *   - start >= num_nodes  -> the whole row is GRAPE_PAD (§8(c) c14);
 *   - a node with out-degree 0 ends the walk; the rest of the row is
 *     GRAPE_PAD (§8(c) c3; the paper is silent, SPEC S:233 truncates).
 * Random draws: Philox4x32-10 with counter (wid & 0xffffffff, wid >> 32,
 * step s, attempt a) and key (seed & 0xffffffff, seed >> 32); output words
 * o0,o1 form x64 = o1<<32 | o0, o2 is the acceptance draw u (§8(c) c7).
 * Proposal from v (§4.3.2 steps 2-4): r = (x64 * W_v) >> 64 with
 * W_v = sum of v's weights; the neighbour is col[off[v] + i] for the smallest
 * i whose row-local prefix sum exceeds r; unweighted: i = (x64 * deg v) >> 64
 * (P:411).  Node2vec (Eq.1-3): from v, coming from t, attempt
 * a = 0,1,...: propose x with draw (wid, s, a); accept iff u < T_class where
 * class = p if x == t, 1 if x in N(t), q otherwise, and
 *   T_c = floor(2^32 * min(p,1,q) / c)      (IEEE binary64, §8(c) c9)
 * so x is taken with probability proportional to alpha_pq(t,x) * w_vx.
 * The first step of a node2vec walk (no t yet) is a first-order step with
 * attempt 0 (§8(c) c2), hence node2vec with p = q = 1 is bit-identical to
 * first order.  Results are bit-identical to the CPU oracle (oracle/).
 */
#ifndef GRAPE_WALK_H
#define GRAPE_WALK_H

#include <stdint.h>
#include <cuda_runtime_api.h>   /* cudaStream_t only */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct grape_graph grape_graph;   /* opaque, device-resident, immutable */

typedef enum {
    GRAPE_OK = 0,
    GRAPE_EINVAL = 1,    /* bad argument or invalid graph; nothing was launched */
    GRAPE_ENOMEM = 2,    /* device allocation failed */
    GRAPE_ECUDA = 3      /* a CUDA runtime call or launch failed */
} grape_status;

#define GRAPE_PAD 0xFFFFFFFFu

/* Flags for grape_graph_from_csr. */
enum {
    /* Caller asserts arc (u,v) exists iff arc (v,u) exists (undirected graph).
     * Checked on the device unless GRAPE_SKIP_VALIDATION.  Without sampling
     * tables it lets the v3 walker evaluate "x in N(t)" as "t in N(x)" on the
     * shorter row — the same predicate (§8(c) c12); with tables the edge-hash
     * sets answer it either way. */
    GRAPE_SYMMETRIC = 1u << 0,
    /* Skip the O(m) device validation of the CSR (trusted input). */
    GRAPE_SKIP_VALIDATION = 1u << 1,
    /* Do not build the sampling tables (per-arc records with the
     * reverse arc's interval, the head's node record and no-common-neighbour
     * flags; per-row guide tables; per-row edge-hash sets — between ~16 and
     * ~550 bytes per arc depending on the layout grape_table_options selects;
     * the CSR arrays are released once the tables exist).  Without them walks
     * run on the fenced-search walker (v3), and grape_walks_approx (when a row
     * exceeds its threshold) and grape_walks_node2vec_cdf are unavailable.
     * Results are identical either way. */
    GRAPE_NO_TABLES = 1u << 2
};

/*
 * Sampling-table layout for grape_graph_from_csr_opts.  Every
 * field 0 = automatic.  The automatic choice takes the first layout, in order
 * of fewest reads per step, whose tables fit both the free device memory
 * (leaving 10% of it) and table_budget_bytes (default 68e9 minus the node
 * records: B200's random-gather rate collapses beyond ~68 GB of randomly read
 * memory).  Forced values that do not fit give GRAPE_ENOMEM.
 * The layout never changes a walk.
 */
typedef struct {
    uint64_t table_budget_bytes; /* cap on rec + guide + hash bytes; 0 = automatic */
    uint32_t record_bytes;       /* weighted: 32 (with the head's node record) or 16;
                                    unweighted: 16 or 8 */
    uint32_t guide_bytes;        /* weighted: 32 (unsplit buckets hold the record; needs
                                    32-B records) or 8 */
    uint32_t guide_factor;       /* weighted: guide buckets per arc, 1, 2, 4, 8 or 16 */
    uint32_t hash_h;             /* edge-hash: one 8-slot bucket per H arcs (+1 per row), 4 or 6 */
} grape_table_options;

typedef struct {
    uint32_t num_nodes;
    uint64_t num_arcs;
    uint32_t weighted;        /* 1 if built with weights */
    uint32_t flags;           /* GRAPE_SYMMETRIC / ... as accepted */
    uint32_t cw_bytes;        /* bytes per stored prefix-sum entry: 0 (unweighted), 4 or 8 */
    uint32_t max_degree;
    uint64_t max_row_weight;  /* max_v W_v (deg for unweighted) */
    uint64_t device_bytes;    /* device memory owned by the handle */
    int device;
    uint32_t tables;          /* 1 if the sampling tables were built (table walker) */
    uint32_t weights_symmetric; /* 1 if every arc with a reverse arc has its weight */
    uint64_t table_bytes;     /* part of device_bytes held by the tables */
    uint32_t guide_factor;    /* weighted tables: guide buckets per arc (16 ... 1) */
    uint32_t guide_bytes;     /* weighted tables: 32 (entries of unsplit buckets hold the record) or 8 */
    uint32_t record_bytes;    /* tables: bytes per arc record */
    uint32_t hash_h;          /* tables: arcs per edge-hash bucket (4 or 6) */
    uint32_t notri;           /* tables: records carry the no-common-neighbour flags */
    uint32_t parts;           /* 1, or the number of parts after grape_graph_partition */
    uint32_t wide;            /* 1: 34-bit arc offsets (m >= 2^32 - 64; the default walk rules only) */
} grape_graph_info;

/*
 * grape_graph_from_csr — build the device CSR (§8(a) a1; the paper's
 * "explicit destinations vector" + "explicit out-bound degrees vector",
 * P:368-374, plus the per-row cumulative weights of P:509).
 *
 *   num_nodes    n, node ids are [0, n); n < 2^32 - 1 so no id equals GRAPE_PAD.
 *   num_arcs     m (an undirected edge counts twice).
 *   row_offsets  u64[n+1]: off[0] = 0, off[n] = m, non-decreasing.
 *   col_indices  u32[m]: every value < n, strictly increasing within a row
 *                (sorted, no duplicate arcs; "sorted vectors").
 *   weights      u32[m], every value >= 1, or NULL for an unweighted graph.
 *   device       CUDA device ordinal that will own the graph.
 *   flags        GRAPE_SYMMETRIC | GRAPE_SKIP_VALIDATION | GRAPE_NO_TABLES.
 *   out          receives the handle.
 * The three arrays may be host (pageable or pinned) or device pointers; they
 * are copied, and the call is synchronous: the caller may free them on return.
 * The handle stores off (u64[n+1]), the node records and, by default, the
 * sampling tables (built from col and the row-local inclusive
 * prefix sums of the weights, then those are released); graphs built with
 * GRAPE_NO_TABLES, or outside the tables' index ranges (m >= 2^34 - 64, a degree
 * >= 2^28, a row sum >= 2^32), keep col (u32[m]), the prefix sums (u32[m] when
 * every row sum fits in 32 bits, else u64[m]) and their fence levels instead.
 * grape_graph_from_csr = grape_graph_from_csr_opts with automatic layout.
 * Errors: GRAPE_EINVAL for null pointers, n >= 2^32-1, or a CSR that fails
 * validation (message names the first check that failed); GRAPE_ENOMEM;
 * GRAPE_ECUDA.  On error *out is set to NULL and nothing is leaked.
 */
grape_status grape_graph_from_csr(uint32_t num_nodes, uint64_t num_arcs,
                                  const uint64_t* row_offsets, const uint32_t* col_indices,
                                  const uint32_t* weights, int device, uint32_t flags,
                                  grape_graph** out);

/* As grape_graph_from_csr, with the sampling-table layout given by *opts
 * (NULL = automatic).  EINVAL for a field outside its listed values. */
grape_status grape_graph_from_csr_opts(uint32_t num_nodes, uint64_t num_arcs,
                                       const uint64_t* row_offsets, const uint32_t* col_indices,
                                       const uint32_t* weights, int device, uint32_t flags,
                                       const grape_table_options* opts, grape_graph** out);

/* Synchronises the owning device, then frees the handle.  NULL is a no-op. */
grape_status grape_graph_free(grape_graph* g);

/* Fills *info.  EINVAL on NULL arguments. */
grape_status grape_graph_get_info(const grape_graph* g, grape_graph_info* info);

/*
 * grape_walks_first_order — first-order walks (DeepWalk; P:394, P:411 unweighted
 * uniform, P:509-511 weighted), one per start.
 *
 *   g             graph handle; the current device must be g's device.
 *   starts        u32[num_walks] start nodes (device, or host — see below).
 *   num_walks     W; 0 returns GRAPE_OK without launching.
 *   walk_id_base  wid of row 0 (sharding: rank r passes its first global wid).
 *   walk_length   L >= 1 (nodes per row, including the start).
 *   seed          64-bit Philox key.
 *   out           u32[num_walks * L], row-major (device, or host).
 *   steps_out     NULL, or one u64 to which the number of realised
 *                 transitions is ADDED (device pointer, or host pointer).
 *   stream        stream for all work (0 = legacy default stream).
 * Device buffers: the call is asynchronous on `stream`; buffers must stay
 * alive until the stream reaches this work; faults surface at the caller's
 * next synchronisation.  Host buffers (starts and out both host memory;
 * pinned memory gives copy/compute overlap): the library stages chunks
 * through device memory, overlapping H2D / kernel / D2H, and the call returns
 * when out (and *steps_out) are complete.  Mixing host and device for starts
 * and out is EINVAL.
 * Errors: EINVAL (NULL g, NULL starts/out with num_walks > 0, L = 0,
 * num_walks * L overflow, wrong current device); ENOMEM (staging); ECUDA
 * (launch).  With num_walks = 0 the buffers may be NULL.
 */
grape_status grape_walks_first_order(const grape_graph* g, const uint32_t* starts,
                                     uint64_t num_walks, uint64_t walk_id_base,
                                     uint32_t walk_length, uint64_t seed, uint32_t* out,
                                     uint64_t* steps_out, cudaStream_t stream);

/*
 * grape_walks_node2vec — second-order node2vec walks (Eq.1-3) by
 * rejection sampling with integer thresholds (rules above).
 *   p  return parameter, q  in-out parameter: finite, > 0, and
 *      max(p,1,q) / min(p,1,q) <= 2^24 (keeps every T_c >= 2^8 so the
 *      attempt loop ends; §8(c) c10) — else GRAPE_EINVAL.
 * All other arguments, ownership and errors as grape_walks_first_order.
 * Specialisation (the paper's 8 dispatch paths over p = 1?, q = 1?,
 * weighted?) is internal and never changes a result.
 */
grape_status grape_walks_node2vec(const grape_graph* g, const uint32_t* starts,
                                  uint64_t num_walks, uint64_t walk_id_base,
                                  uint32_t walk_length, double p, double q, uint64_t seed,
                                  uint32_t* out, uint64_t* steps_out, cudaStream_t stream);

/*
 * grape_walks_approx — approximated walks (§4.3.3
 * "Approximated random walks", and Fig. 3): at a node v
 * with deg(v) > degree_threshold = k the step considers only a Sorted Unique
 * Sub-Sample of k neighbours — bucket b = [floor(b deg/k), floor((b+1) deg/k))
 * of v's sorted row contributes the index floor(b deg/k) + BOUNDED(h_b, width),
 * h_b being half of the Philox block with counter (wid lo, wid hi, s,
 * 2^31 + floor(b/2)) (words o1:o0 for even b, o3:o2 for odd b) — and then
 * applies the exact rules above to those candidates (proposal by their weights,
 * node2vec class of x relative to the full N(t)).  Nodes with deg <= k take the
 * exact step (bit-identical to grape_walks_*), so k >= the maximum degree, or
 * k = 0, gives the exact walks.
 *   node2vec  0: first-order (p, q ignored); 1: node2vec with p, q.
 * Everything else as grape_walks_node2vec.  Errors: as grape_walks_node2vec;
 * EINVAL if sub-sampling would apply to a graph without sampling tables
 * (GRAPE_NO_TABLES); ENOMEM / ECUDA if the per-lane candidate scratch
 * (weighted graphs: 8 k bytes per resident thread, stream-ordered) cannot be
 * allocated.
 */
grape_status grape_walks_approx(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                uint64_t walk_id_base, uint32_t walk_length, int node2vec, double p,
                                double q, uint32_t degree_threshold, uint64_t seed, uint32_t* out,
                                uint64_t* steps_out, cudaStream_t stream);

/*
 * grape_walks_node2vec_cdf — node2vec walks with the paper's own sampler
 * (§4.3.2, P:507-511 steps 1-4): at each step
 * after the first, the un-normalised probabilities pi_x = w_vx * T_class(x)
 * of every neighbour of v (classes and integer thresholds as above), their
 * exact running sum S_i (128-bit), ONE draw x64 = DRAW(seed, wid, s, 0) mapped
 * to r = floor(x64 * S / 2^64), and the neighbour at the smallest i with
 * S_i > r.  The first step is the first-order step; with p = q = 1 every walk
 * equals grape_walks_first_order's.  Same law as grape_walks_node2vec (Eq.1),
 * different draws, so different walks; O(deg v) work per step.
 * Arguments, ownership and errors as grape_walks_node2vec; EINVAL if the graph
 * has no sampling tables (GRAPE_NO_TABLES).
 */
grape_status grape_walks_node2vec_cdf(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                      uint64_t walk_id_base, uint32_t walk_length, double p, double q,
                                      uint64_t seed, uint32_t* out, uint64_t* steps_out,
                                      cudaStream_t stream);

/*
 * grape_walks_node2vec_folded — node2vec walks with outlier-folded rejection
 * ("outlier-folded proposals"): the same
 * law as grape_walks_node2vec (Eq.1), fewer attempts when the
 * return class dominates (p < min(1, q)).  At v coming from t, with
 * E = max(T_1, T_q), X = T_p - E (> 0), w_t = w_vt (0 if no arc v -> t),
 * N = w_t X and M = W_v E + N: attempt a draws o = DRAW(seed, wid, s, a); if
 * o3 * M < N * 2^32 the walk returns to t; else x = the proposal of o1:o0 and
 * it is accepted iff o2 < A_class(x), A_c = ceil(min(T_c, E) * 2^32 / E).
 * When p >= min(1, q) (T_p <= E) every walk equals grape_walks_node2vec's.
 * Arguments, ownership and errors as grape_walks_node2vec; EINVAL on graphs
 * without sampling tables, and on weighted graphs with asymmetric weights
 * stored in 16-B records (the return arc's weight is not kept there).
 */
grape_status grape_walks_node2vec_folded(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                         uint64_t walk_id_base, uint32_t walk_length, double p, double q,
                                         uint64_t seed, uint32_t* out, uint64_t* steps_out,
                                         cudaStream_t stream);

/*
 * grape_graph_partition — the §8(f) f4 table layout: split every
 * sampling table of a built graph into chunks of 2^k bytes (at most 64 per table),
 * owner j of `parts` holding a contiguous range of chunks (owners differ by at most one
 * chunk) on device devices[j] (peer access from the graph's device is enabled;
 * devices may repeat, e.g. all equal to the graph's device).  Walks then read each
 * table entry from its part (over NVLink for a peer's part) and stay bit-identical
 * to the unpartitioned graph.  Only the default rules run on a partitioned graph
 * (grape_walks_first_order / _node2vec / _stats, grape_skipgram_pairs,
 * grape_walks_skipgram); the approximated, CDF and folded modes return EINVAL.
 * Synchronous.
 *   parts     2 .. 8;   devices  host int[parts]
 * Errors: EINVAL on a NULL graph / device list, parts out of range, a graph without
 * tables or already partitioned, a device that does not exist or that the graph's
 * device cannot access; ECUDA on allocation / copy failure (the graph is then
 * unchanged).  This form partitions a graph built on one GPU; it does not build a
 * graph larger than one GPU's memory.
 */
grape_status grape_graph_partition(grape_graph* g, uint32_t parts, const int* devices);

/*
 * Distributed table build — the §8(f) f4 row for graphs whose sampling tables
 * exceed one GPU (the paper's ClueWeb09 / sk-2005 scale, P:80,
 * P:288).  One process per GPU ("rank" j of `parts`), each holding the whole CSR
 * (8 bytes per arc) and owning part j of every table (records, guide, edge hash:
 * owner j's contiguous range of 2^k-byte chunks, as grape_graph_partition lays them
 * out; each owner's range allocated in whole 2 MB pages).  The ranks
 * exchange CUDA IPC handles of their parts and build in four stages; every rank
 * then walks over all parts (peer parts over NVLink, or the same GPU's memory
 * when ranks share a device), bit-identical to the single-GPU tables.  The ABI
 * runs no collective: the caller moves the exports between ranks and puts a
 * barrier where marked (paper_2110_06196_b200.graph_from_csr_dist does both over
 * torch.distributed).  Sequence, on every rank:
 *   grape_graph_dist_create(..., part = rank, parts = world)
 *   grape_graph_dist_export -> all-gather -> grape_graph_dist_import(all exports)
 *   for stage in 0..3: grape_graph_dist_build(stage), barrier
 *   grape_graph_dist_finish(OR over ranks of the build's flags_out)
 * and before any rank calls grape_graph_free: a barrier (peers read its parts).
 * Only the default walk rules run on the result (as after grape_graph_partition).
 */
typedef struct { unsigned char bytes[64]; } grape_ipc_handle;   /* a cudaIpcMemHandle_t */

typedef struct {
    uint32_t part;            /* the exporting rank's part index */
    int device;               /* its CUDA device */
    uint64_t bytes[4];        /* bytes of its part of: 0 records, 1 guide, 2 edge hash, 3 build flags */
    grape_ipc_handle handle[4];   /* IPC handles of those parts (valid where bytes > 0) */
} grape_part_export;

/* Rank `part` of `parts` (2..8): copy and validate the CSR (as grape_graph_from_csr_opts;
 * same arguments on every rank), choose the table layout for parts x
 * opts->table_budget_bytes bytes (required, equal on every rank, so every rank
 * chooses the same layout; forced fields as in grape_table_options) and allocate
 * this rank's parts.  Synchronous.  EINVAL: bad arguments, table_budget_bytes = 0,
 * GRAPE_NO_TABLES, a graph outside the tables' index ranges; ENOMEM: no layout fits
 * (or allocation failed); ECUDA. */
grape_status grape_graph_dist_create(uint32_t num_nodes, uint64_t num_arcs, const uint64_t* row_offsets,
                                     const uint32_t* col_indices, const uint32_t* weights, int device,
                                     uint32_t flags, const grape_table_options* opts, uint32_t part,
                                     uint32_t parts, grape_graph** out);
/* IPC handles of this rank's parts into *out (host memory). */
grape_status grape_graph_dist_export(const grape_graph* g, grape_part_export* out);
/* Open every other rank's parts: exports[j] = rank j's export, j = 0 .. parts-1.
 * EINVAL when an export's sizes differ from this rank's layout (different graphs). */
grape_status grape_graph_dist_import(grape_graph* g, const grape_part_export* exports);
/* Build stage 0 (edge hash), 1 (no-common-neighbour flags), 2 (records) or 3 (guide)
 * of this rank's parts; synchronous; every rank must finish stage k before any
 * starts stage k+1 (barrier).  *flags_out (may be NULL): bit 0 = a reverse arc of
 * different weight was seen, bit 1 = an arc has no reverse although GRAPE_SYMMETRIC
 * was asserted (stage 2). */
grape_status grape_graph_dist_build(grape_graph* g, uint32_t stage, uint32_t* flags_out);
/* flags_all = OR over ranks of stage 2's flags_out.  Releases the CSR copy; the
 * graph then walks.  EINVAL when called twice or before import, or when a rank saw
 * an arc without its reverse under GRAPE_SYMMETRIC (bit 1). */
grape_status grape_graph_dist_finish(grape_graph* g, uint32_t flags_all);

/*
 * grape_skipgram_pairs — the SkipGram consumer of a walk matrix (SURVEY §8(f)
 * row f3): the (center, context) pairs of the sliding window
 * ("given a window size, these models learn ... the co-occurrence of two nodes
 * in each window"; SkipGram "predicts the contextual nodes of a sequence
 * given its central node") and, per pair, num_negatives negatives from
 * the out-degree "scale-free" distribution — the node whose row holds a uniform
 * arc index, the rank the paper implements on Elias-Fano.
 *   walks          device u32[num_walks][walk_length], rows of walk ids
 *                  walk_id_base + r (as written by grape_walks_*; PAD suffixes)
 *   window         w >= 1: offsets j = -w .. -1, 1 .. w
 *   centers, contexts  device u32[S], S = num_walks * walk_length * 2w; slot
 *                  p = (r * walk_length + i) * 2w + o, o = 0 .. 2w-1 for
 *                  j = -w .. -1, 1 .. w: (row[i], row[i+j]) when 0 <= i+j < L
 *                  and both entries are not PAD, else (PAD, PAD)
 *   negatives      device u32[S][num_negatives] (may be NULL if 0): for a valid
 *                  slot, negative k = rank(floor(x64 * m / 2^64)), x64 = words
 *                  o1:o0 (k even) or o3:o2 (k odd) of Philox4x32-10 with counter
 *                  (P lo, P hi, 0xFFFFFFFF, floor(k/2)), key = seed,
 *                  P = ((walk_id_base + r) * L + i) * 2w + o the
 *                  global slot id (so shards reproduce slices of one call);
 *                  rank(e) = the v with off[v] <= e < off[v+1]; PAD for an
 *                  invalid slot or a graph without arcs.
 * Device buffers only; asynchronous on `stream` (the first call on a graph
 * builds its node guide, ~4 n bytes, synchronously).  Errors: EINVAL on NULL
 * buffers, host buffers, walk_length = 0, window = 0 or > 1024, num_negatives
 * > 1024, walk_length * 2 * window * num_negatives >= 2^32, slot-count overflow,
 * a device mismatch; ECUDA on launch failure.
 */
grape_status grape_skipgram_pairs(const grape_graph* g, const uint32_t* walks, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, uint32_t window,
                                  uint32_t num_negatives, uint64_t seed, uint32_t* centers, uint32_t* contexts,
                                  uint32_t* negatives, cudaStream_t stream);

/*
 * grape_walks_skipgram — walks streamed straight into the SkipGram consumer
 * (DESIGN.md §7e): exactly grape_walks_first_order /
 * grape_walks_node2vec (walk_seed) followed by grape_skipgram_pairs (pair_seed) on
 * the same walk ids, bit for bit, without materialising the walk matrix: walks are
 * generated chunk_walks rows at a time (0 = automatic: 4 rounds of the walker's
 * resident lanes, at most half the walks) into one of two internal device buffers,
 * and the pair kernel consumes each chunk while the walker fills the next (two
 * internal streams): the walker's time overlaps the pair kernel's, and only two
 * chunks of rows exist at a time.  The walks exist to feed this; the paper
 * generates them lazily for the same reason ("static generation ... tens of
 * terabytes").
 *   starts        device u32[num_walks]; walk ids walk_id_base + i
 *   node2vec      0: first order (p, q ignored), else node2vec(p, q)
 *   centers, contexts, negatives, window, num_negatives: as grape_skipgram_pairs
 *   steps_out     device u64 or NULL: realised transitions are added to it
 * Asynchronous on `stream` (the internal streams are ordered after the work already
 * on it, and `stream` is ordered after them).  Device buffers only (EINVAL
 * otherwise); the other errors as grape_walks_node2vec and grape_skipgram_pairs.
 */
grape_status grape_walks_skipgram(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, int node2vec, double p, double q,
                                  uint64_t walk_seed, uint32_t window, uint32_t num_negatives, uint64_t pair_seed,
                                  uint32_t* centers, uint32_t* contexts, uint32_t* negatives, uint64_t* steps_out,
                                  uint64_t chunk_walks, cudaStream_t stream);

/*
 * grape_walks_stats — diagnostics: run the same walks as grape_walks_first_order
 * (node2vec = 0) or grape_walks_node2vec (node2vec = 1) with event counters
 * compiled into the kernel, and return the counts.  `out` receives exactly the
 * walk matrix the plain call writes (a parity check of the counting build).
 * starts / out must be device buffers; the call is synchronous on `stream`.
 * Used by bench.py to turn measured time into the roofline of DESIGN.md §7.
 * Errors as grape_walks_node2vec; EINVAL if starts or out is host memory or
 * stats is NULL.
 */
typedef struct {
    uint64_t sector_loads;      /* 32-B sector loads issued, all kinds */
    uint64_t node_loads;        /* node-record loads of the current node v (+ u64 W_v loads) */
    uint64_t xnode_loads;       /* node-record loads of a proposal x (symmetric membership) */
    uint64_t cw_probes;         /* sector probes of weight-prefix searches (proposals) */
    uint64_t col_probes;        /* sector probes of membership searches */
    uint64_t col_loads;         /* proposal loads: col[i] (v3) or arc records (tables; incl. guide-split scans) */
    uint64_t attempts;          /* proposals drawn (Philox draws) */
    uint64_t membership_tests;  /* "x in N(t)" searches performed */
    uint64_t start_loads;       /* walks started */
    uint64_t steps;             /* realised transitions */
    /* table walker only (zero on the v3 walker): */
    uint64_t guide_loads;       /* guide-table entries read (weighted proposals) */
    uint64_t hash_probes;       /* edge-hash sectors read by membership tests */
    uint64_t alu_decisions;     /* attempts decided without reading the graph */
    uint64_t iterations;        /* lane-iterations of the state machine (one load at most each) */
    uint64_t draw_iterations;   /* ... of them spent drawing only (no load) */
    uint64_t back_iterations;   /* ... of them emitting a register-decided return (no load) */
} grape_walk_stats;

grape_status grape_walks_stats(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                               uint64_t walk_id_base, uint32_t walk_length, int node2vec,
                               double p, double q, uint64_t seed, uint32_t* out,
                               grape_walk_stats* stats, cudaStream_t stream);

/* grape_walks_stats for the other modes: degree_threshold as grape_walks_approx
 * (0: exact), sampler 0 = the default rejection rules, 2 = outlier-folded
 * (grape_walks_node2vec_folded).  EINVAL for the CDF sampler (no counting build)
 * and for combinations the walk calls reject. */
grape_status grape_walks_stats_ex(const grape_graph* g, const uint32_t* starts, uint64_t num_walks,
                                  uint64_t walk_id_base, uint32_t walk_length, int node2vec,
                                  double p, double q, uint32_t degree_threshold, int sampler,
                                  uint64_t seed, uint32_t* out, grape_walk_stats* stats,
                                  cudaStream_t stream);

/* Static string for a status code. */
const char* grape_status_string(grape_status s);

/* Detail of the last error on the calling thread ("" if none). */
const char* grape_last_error(void);

/* Library version string, e.g. "grape-b200 0.1.0 (sm_100a)". */
const char* grape_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GRAPE_WALK_H */
