/*
 * grape_oracle.c — the CPU ORACLE for the GRAPE walk hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or execute this
 * code.  The product path (paper_2110_06196_b200/) never links, imports or
 * calls it, and this file includes no header of the product path.
 *
 * Plain, slow, obviously-correct, single-threaded C.  Every function follows
 * the rule it cites, step by step, in the order SURVEY.md §8(c) writes it:
 *
 *   P:NNN  = /root/reference/PAPER.md line NNN (section / equation named)
 *   S:NNN  = /root/reference/SPEC.md line NNN
 *   §8(c)  = /root/repo/SURVEY.md §8(c), the readings this build adopts
 *            (restated, each with its justification).
 *
 * What the paper fixes (and what the tests pin this file against):
 *   - the node2vec transition law  pi_vx = alpha_pq(t,x) * w_vx   (§4.3.1 Eq.1)
 *     with alpha = 1/p if x == t, 1 if x in N(t), 1/q otherwise   (Eq.2-3 reformulated)
 *   - the weighted first-order law P(x|v) = w_vx / sum_y w_vy       (§4.3.2 steps 1-4)
 *   - the unweighted first-order law: uniform over N(v)
 * What the paper leaves open and §8(c) fixes (parity conventions; pinned
 * against the CUDA toolkit's independent Philox and by exact arithmetic):
 *   - Philox4x32-10 counter = (wid lo, wid hi, step, attempt), key = seed  (§8(c) c7)
 *   - bounded integer = (x64 * W) >> 64                                    (§8(c) c8)
 *   - integer acceptance thresholds from 1/p, 1, 1/q                       (§8(c) c9)
 *   - dead ends pad with 0xFFFFFFFF; bad start ids give all-PAD rows       (§8(c) c3, c14)
 *   - the first node2vec step is a first-order step (attempt 0)            (§8(c) c2)
 *
 * Parity status: every function here is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py (see DESIGN.md §4 for the pin of each one).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define ORACLE_PAD 0xFFFFFFFFu
#define ORACLE_NONE 0xFFFFFFFFu

/* ---------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), the counter-based RNG
 * §8(c) c7 adopts in place of the paper's unspecified assembly PRNG.
 * Constants of the construction: multipliers M0, M1 and Weyl key bumps W0, W1.
 * One round:  (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2   (32x32 -> 64)
 *             c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
 * Ten rounds, the key bumped by (W0, W1) between consecutive rounds.
 * ------------------------------------------------------------------------- */
static const uint32_t PHILOX_M0 = 0xD2511F53u;
static const uint32_t PHILOX_M1 = 0xCD9E8D57u;
static const uint32_t PHILOX_W0 = 0x9E3779B9u;
static const uint32_t PHILOX_W1 = 0xBB67AE85u;

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    int round;
    for (round = 0; round < 10; round++) {
        uint64_t prod0, prod1;
        uint32_t hi0, lo0, hi1, lo1;
        if (round > 0) {
            k0 = k0 + PHILOX_W0;
            k1 = k1 + PHILOX_W1;
        }
        prod0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        prod1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        hi0 = (uint32_t)(prod0 >> 32);
        lo0 = (uint32_t)prod0;
        hi1 = (uint32_t)(prod1 >> 32);
        lo1 = (uint32_t)prod1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* DRAW(seed, wid, s, a)  (§8(c) c7): the four output words of one attempt. */
void oracle_draw(uint64_t seed, uint64_t wid, uint32_t s, uint32_t a, uint32_t out[4])
{
    uint32_t ctr[4];
    uint32_t key[2];
    ctr[0] = (uint32_t)(wid & 0xFFFFFFFFu);
    ctr[1] = (uint32_t)(wid >> 32);
    ctr[2] = s;
    ctr[3] = a;
    key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
    key[1] = (uint32_t)(seed >> 32);
    oracle_philox4x32_10(ctr, key, out);
}

/* BOUNDED(x64, W) = floor(x64 * W / 2^64), a uniform-ish integer in [0, W)
 * (§8(c) c8).  W >= 1. */
uint64_t oracle_bounded(uint64_t x64, uint64_t W)
{
    unsigned __int128 prod = (unsigned __int128)x64 * (unsigned __int128)W;
    return (uint64_t)(prod >> 64);
}

/* THRESHOLDS(p, q) (§8(c) c9): the acceptance thresholds of the three
 * node2vec classes, proportional to alpha = 1/p, 1, 1/q (Eq.1),
 * scaled so that the largest class is accepted with certainty:
 *     mn = min(p, 1, q);  T_c = floor(2^32 * mn / c)  for c in (p, 1, q).
 * Returns 0 on success, 1 if p or q is not finite and > 0, or if
 * max(p,1,q)/min(p,1,q) > 2^24 (§8(c) c10: keeps every T_c >= 2^8). */
int oracle_thresholds(double p, double q, uint64_t T[3])
{
    double mn, mx;
    if (!(p > 0.0) || !(q > 0.0) || isinf(p) || isinf(q) || isnan(p) || isnan(q))
        return 1;
    mn = 1.0;
    if (p < mn) mn = p;
    if (q < mn) mn = q;
    mx = 1.0;
    if (p > mx) mx = p;
    if (q > mx) mx = q;
    if (mx / mn > 16777216.0)
        return 1;
    T[0] = (uint64_t)floor(ldexp(mn / p, 32));
    T[1] = (uint64_t)floor(ldexp(mn, 32));
    T[2] = (uint64_t)floor(ldexp(mn / q, 32));
    return 0;
}

/* Per-row inclusive prefix sums of the integer weights (the paper's
 * "un-normalized cumulative distribution", step 2), built once:
 *     cw[off[v] + i] = w[off[v]] + ... + w[off[v] + i].
 * weights may be NULL (unweighted): then cw[off[v]+i] = i + 1. */
void oracle_prefix(uint32_t n, const uint64_t* off, const uint32_t* w, uint64_t* cw)
{
    uint32_t v;
    for (v = 0; v < n; v++) {
        uint64_t acc = 0;
        uint64_t e;
        for (e = off[v]; e < off[v + 1]; e++) {
            acc += (w != NULL) ? (uint64_t)w[e] : 1u;
            cw[e] = acc;
        }
    }
}

/* Smallest i in [0, d) with row[i] > r, for a non-decreasing row with
 * row[d-1] > r ("a binary search"; §8(c) c11: any search returning
 * this index is valid).  Plain bisection on [lo, hi). */
uint64_t oracle_upper_bound(const uint64_t* row, uint64_t d, uint64_t r)
{
    uint64_t lo = 0, hi = d;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (row[mid] > r)
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

/* INMEMBER(t, x): does x occur in the sorted row col[off[t] .. off[t+1])?
 * (beta_q uses "x in N(t)"; rows are sorted index vectors.) */
int oracle_in_row(const uint64_t* off, const uint32_t* col, uint32_t t, uint32_t x)
{
    uint64_t lo = off[t], hi = off[t + 1];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (col[mid] == x)
            return 1;
        if (col[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return 0;
}

/* PROPOSE(v, x64) (§8(c)): a neighbour of v drawn with probability w_vx / W_v
 * (uniform draw in [0, W_v), then search of the cumulative sum).
 * cw == NULL means unweighted: the index is BOUNDED(x64, deg(v)).
 * Requires deg(v) >= 1. */
uint32_t oracle_propose(const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                        uint32_t v, uint64_t x64)
{
    uint64_t lo = off[v];
    uint64_t d = off[v + 1] - lo;
    uint64_t i;
    if (cw != NULL) {
        uint64_t W = cw[lo + d - 1];
        uint64_t r = oracle_bounded(x64, W);
        i = oracle_upper_bound(cw + lo, d, r);
    } else {
        i = oracle_bounded(x64, d);
    }
    return col[lo + i];
}

static uint64_t x64_of(const uint32_t o[4])
{
    return ((uint64_t)o[1] << 32) | (uint64_t)o[0];
}

/* One node2vec step from v, coming from t (t != ORACLE_NONE), at step index s
 * of walk wid (the attempt loop of §8(c) WALK):  for a = 0, 1, 2, ...:
 *   (x64, u) = DRAW(seed, wid, s, a);  x = PROPOSE(v, x64);
 *   T = T_p if x == t  (gamma_p: d(t,x) = 0)
 *       T_1 if x in N(t) (beta_q: d(t,x) = 1)
 *       T_q otherwise    (d(t,x) = 2)
 *   accept iff u < T.
 * Accepting x with probability T_class(x)/2^32 after proposing it with
 * probability w_vx/W_v samples x with probability proportional to
 * w_vx * T_class(x), i.e. to alpha_pq(t,x) * w_vx (Eq.1) because the T_c are
 * proportional to 1/p, 1, 1/q.  Returns x; *attempts = number of draws used. */
uint32_t oracle_node2vec_step(const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                              const uint64_t T[3], uint64_t seed, uint64_t wid, uint32_t s,
                              uint32_t t, uint32_t v, uint32_t* attempts)
{
    uint32_t a = 0;
    for (;;) {
        uint32_t o[4];
        uint32_t x;
        uint64_t thr;
        oracle_draw(seed, wid, s, a, o);
        x = oracle_propose(off, col, cw, v, x64_of(o));
        if (x == t)
            thr = T[0];
        else if (oracle_in_row(off, col, t, x))
            thr = T[1];
        else
            thr = T[2];
        a++;
        if ((uint64_t)o[2] < thr) {
            *attempts = a;
            return x;
        }
    }
}

/* WALK (§8(c)) for num_walks start nodes.  Row i of out (length L) is the walk
 * with id base + i.  mode 0 = first-order, mode 1 = node2vec
 * (P:415-497).  L = nodes per row including the start (§8(c) c1).  A start id
 * >= n gives an all-PAD row (c14); a node with out-degree 0 ends the walk and
 * the rest of the row stays PAD (c3).  The first node2vec step, having no t,
 * is a first-order step with attempt 0 (c2).
 * Returns 0, or 1 if (mode == 1 and) the thresholds are invalid.
 * If steps_out != NULL, *steps_out += realised transitions;
 * if attempts_out != NULL, *attempts_out += draws used by node2vec steps s >= 2. */
int oracle_walks(uint32_t n, const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                 const uint32_t* starts, uint64_t num_walks, uint64_t base, uint32_t L,
                 int mode, double p, double q, uint64_t seed, uint32_t* out,
                 uint64_t* steps_out, uint64_t* attempts_out)
{
    uint64_t T[3] = {0, 0, 0};
    uint64_t i;
    uint64_t steps = 0, attempts = 0;
    if (mode == 1 && oracle_thresholds(p, q, T) != 0)
        return 1;
    for (i = 0; i < num_walks; i++) {
        uint32_t* row = out + i * (uint64_t)L;
        uint64_t wid = base + i;
        uint32_t start = starts[i];
        uint32_t t, v, s, j;
        for (j = 0; j < L; j++)
            row[j] = ORACLE_PAD;
        if (start >= n || L == 0)
            continue;
        row[0] = start;
        t = ORACLE_NONE;
        v = start;
        for (s = 1; s < L; s++) {
            uint32_t x;
            if (off[v + 1] == off[v])
                break;
            if (mode == 0 || t == ORACLE_NONE) {
                uint32_t o[4];
                oracle_draw(seed, wid, s, 0, o);
                x = oracle_propose(off, col, cw, v, x64_of(o));
            } else {
                uint32_t a = 0;
                x = oracle_node2vec_step(off, col, cw, T, seed, wid, s, t, v, &a);
                attempts += a;
            }
            row[s] = x;
            steps++;
            t = v;
            v = x;
        }
    }
    if (steps_out != NULL)
        *steps_out += steps;
    if (attempts_out != NULL)
        *attempts_out += attempts;
    return 0;
}

/* Batched single steps for the statistical pins (tests only).
 * First-order: x_out[k] = the step-s proposal from v for walk id wid0 + k.
 * Node2vec:    x_out[k], att_out[k] = the step-s node2vec step from v coming
 *              from t for walk id wid0 + k.  Returns 1 on invalid thresholds. */
void oracle_first_order_steps(const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                              uint64_t seed, uint32_t v, uint32_t s, uint64_t wid0,
                              uint64_t count, uint32_t* x_out)
{
    uint64_t k;
    for (k = 0; k < count; k++) {
        uint32_t o[4];
        oracle_draw(seed, wid0 + k, s, 0, o);
        x_out[k] = oracle_propose(off, col, cw, v, x64_of(o));
    }
}

int oracle_node2vec_steps(const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                          double p, double q, uint64_t seed, uint32_t t, uint32_t v,
                          uint32_t s, uint64_t wid0, uint64_t count, uint32_t* x_out,
                          uint32_t* att_out)
{
    uint64_t T[3];
    uint64_t k;
    if (oracle_thresholds(p, q, T) != 0)
        return 1;
    for (k = 0; k < count; k++)
        x_out[k] = oracle_node2vec_step(off, col, cw, T, seed, wid0 + k, s, t, v, &att_out[k]);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Approximated walks with Sorted Unique Sub-Sampling (SUSS) — SURVEY.md §8(f)
 * row f1; §4.3.3 "Approximated random walks" and Fig. 3
 * (P:110-116).  Readings (f1-*):
 *   - degree threshold k = d_T >= 1.  At a node v with deg(v) = n <= k the step
 *     is exactly the exact step ("if degree(v) <= d_T the step is exactly
 *     the exact-walk step").
 *   - n > k: SUSS "divides the range into k uniformly spaced buckets and
 *     then randomly samples a value in each bucket": bucket b = [lo_b, lo_{b+1}),
 *     lo_b = floor(b n / k) (the index range is [0, n): §8(c) c15 garble "[0,n]"),
 *     candidate index c_b = lo_b + BOUNDED(h_b, lo_{b+1} - lo_b); the k candidates
 *     are sorted and distinct by construction.
 *   - the subsample is drawn once per step ("the sub-sampling is repeated
 *     at each step"): h_b comes from the Philox block with counter
 *     (wid lo, wid hi, s, 0x80000000 | floor(b/2)) — words (o1:o0) for even b,
 *     (o3:o2) for odd b — a counter range the attempt counter (< 2^31) never uses.
 *   - the step then runs the exact rules on the candidates only (P:509-511 steps
 *     1-4 on the sub-sampled neighbourhood, Fig. 3b): proposal by BOUNDED(x64,
 *     W_C) and the first candidate whose running weight sum exceeds it; node2vec
 *     acceptance with the class of x relative to t on the full N(t) (the
 *     sub-sampling restricts v's candidates, not the graph).
 * ------------------------------------------------------------------------- */
#define ORACLE_SUSS_CTR 0x80000000u

/* The k SUSS candidate indices (row-local, strictly increasing) of step s of
 * walk wid at a node of degree n > k. */
void oracle_suss(uint64_t seed, uint64_t wid, uint32_t s, uint64_t n, uint32_t k, uint64_t* idx)
{
    uint32_t b;
    for (b = 0; b < k; b++) {
        uint64_t lo = ((uint64_t)b * n) / k;
        uint64_t hi = ((uint64_t)(b + 1) * n) / k;
        uint32_t o[4];
        uint64_t h;
        oracle_draw(seed, wid, s, ORACLE_SUSS_CTR | (b / 2), o);
        h = (b % 2 == 0) ? (((uint64_t)o[1] << 32) | o[0]) : (((uint64_t)o[3] << 32) | o[2]);
        idx[b] = lo + oracle_bounded(h, hi - lo);
    }
}

/* PROPOSE on the candidate set: cand[b] = row-local indices, weights from cw
 * (NULL: unweighted, each candidate weight 1).  ccum = caller scratch of k u64. */
static uint32_t oracle_propose_cand(const uint64_t* off, const uint32_t* col, const uint64_t* cw, uint32_t v,
                                    const uint64_t* cand, uint32_t k, uint64_t* ccum, uint64_t x64)
{
    uint64_t lo = off[v];
    uint64_t acc = 0, r, b;
    uint32_t j;
    for (j = 0; j < k; j++) {
        uint64_t e = lo + cand[j];
        uint64_t w = 1;
        if (cw != NULL)
            w = cw[e] - (cand[j] > 0 ? cw[e - 1] : 0);
        acc += w;
        ccum[j] = acc;
    }
    r = oracle_bounded(x64, acc);
    b = oracle_upper_bound(ccum, k, r);
    return col[lo + cand[b]];
}

/* WALK with degree threshold k (k = 0: no threshold, the exact WALK).
 * cand / ccum: caller scratch of k u64 each.  Same conventions and return
 * value as oracle_walks. */
int oracle_walks_approx(uint32_t n, const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                        const uint32_t* starts, uint64_t num_walks, uint64_t base, uint32_t L,
                        int mode, double p, double q, uint64_t seed, uint32_t k,
                        uint64_t* cand, uint64_t* ccum, uint32_t* out, uint64_t* steps_out)
{
    uint64_t T[3] = {0, 0, 0};
    uint64_t i;
    uint64_t steps = 0;
    if (mode == 1 && oracle_thresholds(p, q, T) != 0)
        return 1;
    for (i = 0; i < num_walks; i++) {
        uint32_t* row = out + i * (uint64_t)L;
        uint64_t wid = base + i;
        uint32_t start = starts[i];
        uint32_t t, v, s, j;
        for (j = 0; j < L; j++)
            row[j] = ORACLE_PAD;
        if (start >= n || L == 0)
            continue;
        row[0] = start;
        t = ORACLE_NONE;
        v = start;
        for (s = 1; s < L; s++) {
            uint64_t deg = off[v + 1] - off[v];
            int sub = k > 0 && deg > k;
            uint32_t x;
            if (deg == 0)
                break;
            if (sub)
                oracle_suss(seed, wid, s, deg, k, cand);
            if (mode == 0 || t == ORACLE_NONE) {
                uint32_t o[4];
                oracle_draw(seed, wid, s, 0, o);
                x = sub ? oracle_propose_cand(off, col, cw, v, cand, k, ccum, x64_of(o))
                        : oracle_propose(off, col, cw, v, x64_of(o));
            } else {
                uint32_t a = 0;
                for (;;) {
                    uint32_t o[4];
                    uint64_t thr;
                    oracle_draw(seed, wid, s, a, o);
                    x = sub ? oracle_propose_cand(off, col, cw, v, cand, k, ccum, x64_of(o))
                            : oracle_propose(off, col, cw, v, x64_of(o));
                    if (x == t)
                        thr = T[0];
                    else if (oracle_in_row(off, col, t, x))
                        thr = T[1];
                    else
                        thr = T[2];
                    a++;
                    if ((uint64_t)o[2] < thr)
                        break;
                }
            }
            row[s] = x;
            steps++;
            t = v;
            v = x;
        }
    }
    if (steps_out != NULL)
        *steps_out += steps;
    return 0;
}

/* ---------------------------------------------------------------------------
 * The paper's own node2vec sampler, step by step — SURVEY.md §8(f) row f2;
 * PAPER.md §4.3.2 "Efficient sampling for Node2Vec random walks":
 *   "1) computation of the un-normalized transition probabilities to each
 *    neighbour of v according to the provided in-out and return biases;
 *    2) computation of the un-normalized cumulative distribution, which is
 *    equivalent to a cumulative sum; 3) uniform sampling of a random value
 *    between 0 and the maximum value in the un-normalized cumulative
 *    distribution; 4) identification of the corresponding index".
 * Readings (f2-*):
 *   - the biases alpha = 1/p, 1, 1/q (Eq.1) enter as the integer
 *     thresholds T_p, T_1, T_q of §8(c) c9 (proportional to them; exact for
 *     every BASELINE config): pi_x = w_vx * T_class(x), a u64;
 *   - the running sum is exact (u128: deg < 2^28 terms below 2^64);
 *   - step 3 draws ONE x64 per step, DRAW(seed, wid, s, 0) words o1:o0, and
 *     maps it by BOUNDED on the total (128-bit): r = floor(x64 * S / 2^64);
 *   - step 4 takes the smallest i with cum_i > r;
 *   - the first step of a walk (no t) is the first-order step (§8(c) c2), and
 *     so is every step when p = q = 1 (then pi = w * T with one T, which
 *     selects exactly the first-order index — see the proof in DESIGN.md §7c).
 * ------------------------------------------------------------------------- */
typedef unsigned __int128 oracle_u128;

/* floor(x64 * S / 2^64) for S < 2^128 with the result < 2^128 (S < 2^92 here). */
static oracle_u128 oracle_bounded128(uint64_t x64, oracle_u128 S)
{
    uint64_t s_lo = (uint64_t)S, s_hi = (uint64_t)(S >> 64);
    oracle_u128 lo = ((oracle_u128)x64 * s_lo) >> 64;
    return (oracle_u128)x64 * s_hi + lo;
}

/* One CDF node2vec step from v coming from t (t != NONE). */
uint32_t oracle_cdf_step(const uint64_t* off, const uint32_t* col, const uint64_t* cw, const uint64_t T[3],
                         uint64_t seed, uint64_t wid, uint32_t s, uint32_t t, uint32_t v)
{
    uint64_t lo = off[v], d = off[v + 1] - lo, i;
    oracle_u128 total = 0, cum = 0, r;
    uint32_t o[4];
    for (i = 0; i < d; i++) {                    /* step 1-2 (first pass: the total) */
        uint32_t x = col[lo + i];
        uint64_t w = cw == NULL ? 1 : cw[lo + i] - (i > 0 ? cw[lo + i - 1] : 0);
        uint64_t Tc = x == t ? T[0] : (oracle_in_row(off, col, t, x) ? T[1] : T[2]);
        total += (oracle_u128)w * Tc;
    }
    oracle_draw(seed, wid, s, 0, o);             /* step 3 */
    r = oracle_bounded128(x64_of(o), total);
    for (i = 0; i < d; i++) {                    /* step 4 (second pass: the running sum) */
        uint32_t x = col[lo + i];
        uint64_t w = cw == NULL ? 1 : cw[lo + i] - (i > 0 ? cw[lo + i - 1] : 0);
        uint64_t Tc = x == t ? T[0] : (oracle_in_row(off, col, t, x) ? T[1] : T[2]);
        cum += (oracle_u128)w * Tc;
        if (cum > r)
            return x;
    }
    return ORACLE_NONE;   /* unreachable: cum reaches total > r */
}

/* WALK with the CDF sampler (node2vec only; conventions as oracle_walks). */
int oracle_walks_cdf(uint32_t n, const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                     const uint32_t* starts, uint64_t num_walks, uint64_t base, uint32_t L,
                     double p, double q, uint64_t seed, uint32_t* out, uint64_t* steps_out)
{
    uint64_t T[3];
    uint64_t i, steps = 0;
    if (oracle_thresholds(p, q, T) != 0)
        return 1;
    for (i = 0; i < num_walks; i++) {
        uint32_t* row = out + i * (uint64_t)L;
        uint64_t wid = base + i;
        uint32_t start = starts[i];
        uint32_t t, v, s, j;
        for (j = 0; j < L; j++)
            row[j] = ORACLE_PAD;
        if (start >= n || L == 0)
            continue;
        row[0] = start;
        t = ORACLE_NONE;
        v = start;
        for (s = 1; s < L; s++) {
            uint32_t x;
            if (off[v + 1] == off[v])
                break;
            if (t == ORACLE_NONE) {
                uint32_t o[4];
                oracle_draw(seed, wid, s, 0, o);
                x = oracle_propose(off, col, cw, v, x64_of(o));
            } else {
                x = oracle_cdf_step(off, col, cw, T, seed, wid, s, t, v);
            }
            row[s] = x;
            steps++;
            t = v;
            v = x;
        }
    }
    if (steps_out != NULL)
        *steps_out += steps;
    return 0;
}

/* Batched single CDF steps for the statistical pins (tests only). */
int oracle_cdf_steps(const uint64_t* off, const uint32_t* col, const uint64_t* cw, double p, double q,
                     uint64_t seed, uint32_t t, uint32_t v, uint32_t s, uint64_t wid0, uint64_t count,
                     uint32_t* x_out)
{
    uint64_t T[3];
    uint64_t k;
    if (oracle_thresholds(p, q, T) != 0)
        return 1;
    for (k = 0; k < count; k++)
        x_out[k] = oracle_cdf_step(off, col, cw, T, seed, wid0 + k, s, t, v);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Outlier-folded rejection ("outlier-folded
 * proposals").  Same law as the default rule — Eq.1
 * — with fewer attempts when the return class dominates (p < min(1, q)):
 *   E = max(T_1, T_q)            envelope of the non-return classes
 *   X = T_p - E if T_p > E else 0  the return's excess over the envelope
 *   w_t = w_vt (0 if no arc v -> t),  N = w_t * X,  M = W_v * E + N  (< 2^64:
 *         M <= W_v * T_p since w_t <= W_v)
 *   A_c = ceil(min(T_c, E) * 2^32 / E)  acceptance thresholds scaled to E
 * attempt a: o = DRAW(seed, wid, s, a);
 *   if N > 0 and o3 * M < N * 2^32 (exact 96-bit compare): x = t, accepted
 *     (the return's excess mass, probability N / M up to 2^-32);
 *   else x = PROPOSE(v, o1:o0) and accept iff o2 < A_class(x).
 * P(x) is proportional to w_vx * min(T_c, E) + [x == t] * N = w_vx * T_c(x),
 * i.e. Eq.1.  When T_p <= E (then E = 2^32 and N = 0, A = T) this is the
 * default rule draw for draw; the first step stays first-order (c2).
 * ------------------------------------------------------------------------- */
static void oracle_fold_consts(const uint64_t T[3], uint64_t* E, uint64_t* X, uint64_t A[3])
{
    int c;
    *E = T[1] > T[2] ? T[1] : T[2];
    *X = T[0] > *E ? T[0] - *E : 0;
    for (c = 0; c < 3; c++) {
        uint64_t tc = T[c] < *E ? T[c] : *E;
        oracle_u128 num = ((oracle_u128)tc << 32) + *E - 1;
        A[c] = (uint64_t)(num / *E);
    }
}

uint32_t oracle_folded_step(const uint64_t* off, const uint32_t* col, const uint64_t* cw, const uint64_t T[3],
                            uint64_t seed, uint64_t wid, uint32_t s, uint32_t t, uint32_t v, uint32_t* attempts)
{
    uint64_t E, X, A[3];
    uint64_t lo = off[v], d = off[v + 1] - lo, W, wt = 0, N, M, i;
    uint32_t a = 0;
    oracle_fold_consts(T, &E, &X, A);
    W = cw != NULL ? cw[lo + d - 1] : d;
    for (i = 0; i < d; i++)   /* w_vt: the weight of the arc v -> t, if any */
        if (col[lo + i] == t)
            wt = cw != NULL ? cw[lo + i] - (i > 0 ? cw[lo + i - 1] : 0) : 1;
    N = wt * X;
    M = W * E + N;
    for (;;) {
        uint32_t o[4];
        uint32_t x;
        uint64_t thr;
        oracle_draw(seed, wid, s, a, o);
        a++;
        if (N > 0 && (oracle_u128)o[3] * M < ((oracle_u128)N << 32)) {
            *attempts = a;
            return t;
        }
        x = oracle_propose(off, col, cw, v, x64_of(o));
        if (x == t)
            thr = A[0];
        else if (oracle_in_row(off, col, t, x))
            thr = A[1];
        else
            thr = A[2];
        if ((uint64_t)o[2] < thr) {
            *attempts = a;
            return x;
        }
    }
}

int oracle_walks_folded(uint32_t n, const uint64_t* off, const uint32_t* col, const uint64_t* cw,
                        const uint32_t* starts, uint64_t num_walks, uint64_t base, uint32_t L,
                        double p, double q, uint64_t seed, uint32_t* out, uint64_t* steps_out,
                        uint64_t* attempts_out)
{
    uint64_t T[3];
    uint64_t i, steps = 0, attempts = 0;
    if (oracle_thresholds(p, q, T) != 0)
        return 1;
    for (i = 0; i < num_walks; i++) {
        uint32_t* row = out + i * (uint64_t)L;
        uint64_t wid = base + i;
        uint32_t start = starts[i];
        uint32_t t, v, s, j;
        for (j = 0; j < L; j++)
            row[j] = ORACLE_PAD;
        if (start >= n || L == 0)
            continue;
        row[0] = start;
        t = ORACLE_NONE;
        v = start;
        for (s = 1; s < L; s++) {
            uint32_t x;
            if (off[v + 1] == off[v])
                break;
            if (t == ORACLE_NONE) {
                uint32_t o[4];
                oracle_draw(seed, wid, s, 0, o);
                x = oracle_propose(off, col, cw, v, x64_of(o));
            } else {
                uint32_t a = 0;
                x = oracle_folded_step(off, col, cw, T, seed, wid, s, t, v, &a);
                attempts += a;
            }
            row[s] = x;
            steps++;
            t = v;
            v = x;
        }
    }
    if (steps_out != NULL)
        *steps_out += steps;
    if (attempts_out != NULL)
        *attempts_out += attempts;
    return 0;
}

int oracle_folded_steps(const uint64_t* off, const uint32_t* col, const uint64_t* cw, double p, double q,
                        uint64_t seed, uint32_t t, uint32_t v, uint32_t s, uint64_t wid0, uint64_t count,
                        uint32_t* x_out, uint32_t* att_out)
{
    uint64_t T[3];
    uint64_t k;
    if (oracle_thresholds(p, q, T) != 0)
        return 1;
    for (k = 0; k < count; k++)
        x_out[k] = oracle_folded_step(off, col, cw, T, seed, wid0 + k, s, t, v, &att_out[k]);
    return 0;
}

/* ---------------------------------------------------------------------------
 * SkipGram consumer (readings f3-a..d): the
 * training pairs of the shallow models the walks feed ("given a window
 * size, these models learn ... the co-occurrence of two nodes in each window";
 * P:399 SkipGram "predicts the contextual nodes of a sequence given its central
 * node") and their negatives, "scale-free negative sampling, which is
 * efficiently implemented using the Elias-Fano data structure rank method"
 * (P:405), over the "outbound ... node degrees scale-free distribution"
 * (P:319): a uniform arc index e in [0, m) and the node whose row holds it.
 * ------------------------------------------------------------------------- */

/* rank(e): the node v whose row holds arc index e, off[v] <= e < off[v+1]
 * (the largest v with off[v] <= e; rows of degree 0 hold no index).  e < m. */
uint32_t oracle_rank(uint32_t n, const uint64_t* off, uint64_t e)
{
    uint32_t lo = 0, hi = n - 1;   /* off[lo] <= e < off[hi + 1] throughout */
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo + 1) / 2;
        if (off[mid] <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

/* Pairs and negatives of walks [0, num_walks) (walk ids base + r), window w,
 * K negatives per pair.  Slot p = ((wid * L + i) * 2w + o) - base * L * 2w,
 * offset o = 0 .. 2w-1 standing for j = -w .. -1, 1 .. w (f3-a):
 *   centers[p] = row[i], contexts[p] = row[i + j] if 0 <= i + j < L and both
 *   are not PAD; otherwise both PAD (f3-b);
 *   negs[p * K + k] = rank(BOUNDED(x, m)) for a valid slot, x = words o1:o0
 *   (k even) or o3:o2 (k odd) of DRAW(seed, P, 0xFFFFFFFF, floor(k / 2)),
 *   P = its global slot index (wid * L + i) * 2w + o (f3-c);
 *   PAD for an invalid slot, or when m = 0.
 * Returns 0. */
int oracle_skipgram(uint32_t n, const uint64_t* off, const uint32_t* walks, uint64_t num_walks,
                    uint64_t base, uint32_t L, uint32_t w, uint32_t K, uint64_t seed,
                    uint32_t* centers, uint32_t* contexts, uint32_t* negs)
{
    const uint64_t m = n ? off[n] : 0;
    uint64_t r, p = 0;
    for (r = 0; r < num_walks; r++) {
        const uint32_t* row = walks + r * L;
        uint32_t i, o, k;
        for (i = 0; i < L; i++) {
            for (o = 0; o < 2 * w; o++, p++) {
                const int64_t j = o < w ? (int64_t)o - (int64_t)w : (int64_t)o - (int64_t)w + 1;
                const int64_t c = (int64_t)i + j;
                const int valid = c >= 0 && c < (int64_t)L && row[i] != ORACLE_PAD && row[c] != ORACLE_PAD;
                const uint64_t P = ((base + r) * L + i) * (uint64_t)(2 * w) + o;
                centers[p] = valid ? row[i] : ORACLE_PAD;
                contexts[p] = valid ? row[c] : ORACLE_PAD;
                for (k = 0; k < K; k++) {
                    uint32_t d[4];
                    if (!valid || m == 0) {
                        negs[p * K + k] = ORACLE_PAD;
                        continue;
                    }
                    /* one Philox block per two negatives (f3-c): words o1:o0 for even k,
                     * o3:o2 for odd k */
                    oracle_draw(seed, P, 0xFFFFFFFFu, k / 2, d);
                    {
                        const uint64_t x64 = (k & 1) ? ((uint64_t)d[3] << 32 | d[2]) : x64_of(d);
                        negs[p * K + k] = oracle_rank(n, off, oracle_bounded(x64, m));
                    }
                }
            }
        }
    }
    return 0;
}
