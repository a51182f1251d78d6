/*
 * PCF Learned Sort -- CPU ORACLE.   *** TEST INFRASTRUCTURE, NOT PRODUCT CODE ***
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load this library.  The product path
 * (paper_2405_07122_b200/, libpcfsort.so) never links, imports or executes it,
 * and the two share no code: no headers, helpers, tables or constants.  The
 * written specs both sides implement independently are in DESIGN.md §3.
 *
 * Plain, slow, obviously-correct, single-threaded C.  Every function cites the
 * passage of /root/reference/PAPER.md it follows (line numbers + section) and
 * the DESIGN.md reading (R1..R16) it takes where the paper is silent.
 *
 *   Algorithm 1 "Learned-Sort"          PAPER.md:132-171  (§3, Alg. 1)
 *   base case n < tau -> Standard-Sort
 *   model-based bucketing               PAPER.md:152-158, 197-209 (§3.1)
 *   fallback |c_j| >= delta
 *   PCF i(x), b, F~(x)                  PAPER.md:288-308 (§3.2)
 *   alpha=beta=gamma=delta=floor(n^3/4) PAPER.md:345, 357 (Thms 1-2), 423
 *
 * Floating point: compiled with -O2 -ffp-contract=off, no -ffast-math, so
 * every double operation below is one IEEE-754 binary64 round-to-nearest-even
 * operation in source order (reading R6).
 *
 * Parity pins: see tests/test_oracle_pins.py.  Function without an external
 * pin: orc_sample_positions (the paper leaves the sampler unspecified, R3) --
 * "parity unpinned" beyond its statistical checks and the published
 * SplitMix64 output vector that pins orc_mix64.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORC_OK 0
#define ORC_ERR_INVALID_ARG 1
#define ORC_ERR_NAN 2
#define ORC_ERR_OOM 4
#define ORC_ERR_INVARIANT 8

#define ORC_KEY_F64 0
#define ORC_KEY_U64 1

#define ORC_FLAG_SAMPLE_ALL 2u /* reading R14: a_k = seg[k], alpha = m (test mode) */

typedef struct orc_node {
    uint32_t level, alpha;
    uint64_t offset, m;
    uint64_t xmin_bits, xmax_bits;
    uint64_t digest_b, digest_h;
    uint32_t n_fallback, n_small, n_recurse, reserved;
} orc_node; /* 72 bytes */

typedef struct orc_ctx {
    uint32_t tau;
    uint32_t flags;
    uint64_t seed;
    int check;          /* run the per-node invariant checks */
    int violation;      /* bitmask of failed invariants (0 = none)            */
    /* pass log (optional; NULL = off) */
    orc_node *nodes;
    uint64_t nodes_cap, nodes_count;
    uint32_t *l1_b;     /* level-1 b[1..beta+1]   */
    uint32_t *l1_h;     /* level-1 H[1..gamma+1]  */
    uint64_t l1_cap, l1_b_len, l1_h_len;
    /* report (SPEC.md:233-237 SortReport fields) */
    uint32_t max_depth;
    uint64_t base_case_calls, fallback_buckets, fallback_keys, degenerate_calls, bucketing_calls;
} orc_ctx;

/* ------------------------------------------------------------------------ */
/* IEEE-754 totalOrder on binary64 (reading R11): a finite/inf/-0 aware total
 * order.  Positive values order like their bit patterns; negative values order
 * reversed; every negative (incl. -0.0) precedes every positive (incl. +0.0). */
static int total_order_less_f64(uint64_t a, uint64_t b)
{
    int sa = (int)(a >> 63), sb = (int)(b >> 63);
    if (sa != sb) return sa > sb;      /* negative < positive             */
    if (sa == 0) return a < b;         /* both positive: larger bits = larger */
    return a > b;                      /* both negative: larger bits = smaller */
}

static int cmp_f64_total(const void *pa, const void *pb)
{
    uint64_t a = *(const uint64_t *)pa, b = *(const uint64_t *)pb;
    if (total_order_less_f64(a, b)) return -1;
    if (total_order_less_f64(b, a)) return 1;
    return 0;
}

static int cmp_u64(const void *pa, const void *pb)
{
    uint64_t a = *(const uint64_t *)pa, b = *(const uint64_t *)pb;
    return (a > b) - (a < b);
}

static int key_less(int kt, uint64_t a, uint64_t b)
{
    return kt == ORC_KEY_F64 ? total_order_less_f64(a, b) : (a < b);
}

static double as_f64(uint64_t bits) { double d; memcpy(&d, &bits, 8); return d; }

static int is_nan_bits(uint64_t bits)
{
    return (bits & 0x7fffffffffffffffULL) > 0x7ff0000000000000ULL;
}

/* "Standard-Sort": any O(n log n) sort (reading R2).
 * libc qsort with the totalOrder comparator; keys are bit patterns. */
void orc_standard_sort(uint64_t *x, uint64_t m, int kt)
{
    if (m > 1) qsort(x, (size_t)m, 8, kt == ORC_KEY_F64 ? cmp_f64_total : cmp_u64);
}

/* ------------------------------------------------------------------------ */
/* SURVEY.md 8(f) F1, key-value / argsort variant.  The paper sorts keys only
 * (Alg. 1 input/output); carrying a payload needs a rule for
 * equal keys, and the one permutation every stable sort produces is the plain
 * definition: perm[k] = the index of the k-th smallest key, equal keys in
 * increasing index order (reading R18 in DESIGN.md).  Plain top-down stable merge
 * sort of the indices (ties keep the left run first). */
static void argsort_rec(int kt, const uint64_t *x, uint64_t *p, uint64_t *tmp, uint64_t lo, uint64_t hi)
{
    if (hi - lo < 2) return;
    uint64_t mid = lo + (hi - lo) / 2, i = lo, j = mid, k = lo;
    argsort_rec(kt, x, p, tmp, lo, mid);
    argsort_rec(kt, x, p, tmp, mid, hi);
    while (i < mid && j < hi) {
        if (key_less(kt, x[p[j]], x[p[i]])) tmp[k++] = p[j++];   /* strictly smaller right key first */
        else tmp[k++] = p[i++];
    }
    while (i < mid) tmp[k++] = p[i++];
    while (j < hi) tmp[k++] = p[j++];
    for (k = lo; k < hi; ++k) p[k] = tmp[k];
}

int orc_stable_argsort(int kt, const uint64_t *x, uint64_t n, uint64_t *perm)
{
    for (uint64_t i = 0; i < n; ++i) {
        if (kt == ORC_KEY_F64 && is_nan_bits(x[i])) return ORC_ERR_NAN;
        perm[i] = i;
    }
    uint64_t *tmp = (uint64_t *)malloc((size_t)(n ? n : 1) * 8);
    if (!tmp) return ORC_ERR_OOM;
    argsort_rec(kt, x, perm, tmp, 0, n);
    free(tmp);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* alpha = beta = gamma = delta = floor(m^{3/4})  (
 * reading R5): the largest c with c^4 <= m^3, in exact 128-bit integers. */
uint64_t orc_iroot34(uint64_t m)   /* defined for m < 2^42 */
{
    if (m == 0) return 0;
    unsigned __int128 m3 = (unsigned __int128)m * m * m;
    /* plain bisection on [0, m]: c^4 <= m^3 is monotone in c */
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo + 1) / 2;
        unsigned __int128 c2 = (unsigned __int128)mid * mid;
        /* c^4 may exceed 128 bits only if c2 >= 2^64; then c^4 > m^3 surely
         * because m^3 < 2^128 needs m < 2^42.67 and c <= m. */
        int gt;
        if (c2 >> 64) gt = 1;
        else gt = (c2 * c2) > m3;
        if (gt) hi = mid - 1; else lo = mid;
    }
    return lo;
}

/* i(x) = floor((x - x_min)/(x_max - x_min) * beta) + 1.
 * Reading R6: d = x - xmin, q = d / r, t = q * beta, each binary64 RN; floor of
 * the non-negative t. */
uint64_t orc_interval_index_f64(double x, double xmin, double xmax, uint64_t beta)
{
    double r = xmax - xmin;
    double d = x - xmin;
    double q = d / r;
    double t = q * (double)beta;
    return (uint64_t)floor(t) + 1;
}

/* Reading R15: u64 keys -- exact integer differences, then one RN conversion. */
uint64_t orc_interval_index_u64(uint64_t x, uint64_t xmin, uint64_t xmax, uint64_t beta)
{
    double r = (double)(xmax - xmin);
    double d = (double)(x - xmin);
    double q = d / r;
    double t = q * (double)beta;
    return (uint64_t)floor(t) + 1;
}

static uint64_t interval_index(int kt, uint64_t xbits, uint64_t minbits, uint64_t maxbits, uint64_t beta)
{
    if (kt == ORC_KEY_F64)
        return orc_interval_index_f64(as_f64(xbits), as_f64(minbits), as_f64(maxbits), beta);
    return orc_interval_index_u64(xbits, minbits, maxbits, beta);
}

/* ------------------------------------------------------------------------ */
/* Counter-based sampler (reading R3/R4).  SplitMix64's output
 * finaliser (Steele, Lea, Flood 2014), used as a hash. */
uint64_t orc_mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Position of the k-th (0-based) of the alpha samples of the bucketing node at
 * recursion level L whose segment starts at global offset o and has m keys:
 *   key_node = mix64(seed ^ mix64(o + L * 0x9E3779B97F4A7C15))
 *   h_k      = mix64(key_node + (k + 1) * 0x9E3779B97F4A7C15)
 *   p_k      = floor(h_k * m / 2^64)                       (with replacement) */
uint64_t orc_sample_position(uint64_t seed, uint32_t level, uint64_t o, uint64_t m, uint64_t k)
{
    uint64_t key = orc_mix64(seed ^ orc_mix64(o + (uint64_t)level * 0x9E3779B97F4A7C15ULL));
    uint64_t h = orc_mix64(key + (k + 1) * 0x9E3779B97F4A7C15ULL);
    return (uint64_t)(((unsigned __int128)h * m) >> 64);
}

void orc_sample_positions(uint64_t seed, uint32_t level, uint64_t o, uint64_t m, uint64_t alpha, uint64_t *out)
{
    for (uint64_t k = 0; k < alpha; k++) out[k] = orc_sample_position(seed, level, o, m, k);
}

/* digest(v[1..K]) = sum_{i=1..K} mix64((i << 32) ^ v_i)  mod 2^64 */
uint64_t orc_digest(const uint32_t *v1, uint64_t K)
{
    uint64_t s = 0;
    for (uint64_t i = 1; i <= K; i++) s += orc_mix64((i << 32) ^ (uint64_t)v1[i - 1]);
    return s;
}

/* PCF training: b_i = |{ j : i(a_j) <= i }|, i = 1..beta+1,
 * by counting per interval then an inclusive prefix sum (the O(alpha+beta)
 * construction of the Thm 1 proof).  b1 is b[1..beta+1]
 * stored 0-based.  Returns 0, or ORC_ERR_INVARIANT if b_{beta+1} != alpha. */
int orc_train_pcf(int kt, const uint64_t *a, uint64_t alpha, uint64_t minbits, uint64_t maxbits,
                  uint64_t beta, uint32_t *b1)
{
    for (uint64_t i = 0; i <= beta; i++) b1[i] = 0;
    for (uint64_t k = 0; k < alpha; k++) {
        uint64_t i = interval_index(kt, a[k], minbits, maxbits, beta);
        b1[i - 1] += 1;
    }
    for (uint64_t i = 1; i <= beta; i++) b1[i] += b1[i - 1];
    return b1[beta] == alpha ? 0 : ORC_ERR_INVARIANT;
}

/* Bucket index j = floor(F~(x) * gamma) + 1 with F~(x) = b_{i(x)} / alpha
 * (PAPER.md:156, 305).  Reading R7: evaluated exactly in integers,
 * j = floor(b_i * gamma / alpha) + 1. */
uint64_t orc_bucket_of(uint64_t b_i, uint64_t alpha, uint64_t gamma)
{
    return (uint64_t)(((unsigned __int128)b_i * gamma) / alpha) + 1;
}

/* F~(x) itself, as a double, for the SPEC.md:136-138 pins. */
double orc_infer_cdf(int kt, const uint32_t *b1, uint64_t alpha, uint64_t xbits, uint64_t minbits,
                     uint64_t maxbits, uint64_t beta)
{
    uint64_t i = interval_index(kt, xbits, minbits, maxbits, beta);
    return (double)b1[i - 1] / (double)alpha;
}

/* ------------------------------------------------------------------------ */
/* One model-based bucketing step M_PCF on
 * seg[0..m) with explicit (alpha, beta, gamma) and the sample a[0..alpha):
 * bucket[k] receives j(seg[k]) in 1..gamma+1, H[1..gamma+1] the counts, and
 * the keys are appended to their buckets in index order (stable; R16) into
 * out.  b1 receives b[1..beta+1].  minbits/maxbits are the segment min/max.
 * Returns 0 or ORC_ERR_INVARIANT. */
int orc_bucketing(int kt, const uint64_t *seg, uint64_t m, const uint64_t *a, uint64_t alpha,
                  uint64_t beta, uint64_t gamma, uint64_t minbits, uint64_t maxbits,
                  uint32_t *b1, uint32_t *H1, uint32_t *bucket, uint64_t *out)
{
    int rc = orc_train_pcf(kt, a, alpha, minbits, maxbits, beta, b1);
    for (uint64_t j = 0; j <= gamma; j++) H1[j] = 0;
    for (uint64_t k = 0; k < m; k++) {
        uint64_t i = interval_index(kt, seg[k], minbits, maxbits, beta);
        uint64_t j = orc_bucket_of(b1[i - 1], alpha, gamma);
        bucket[k] = (uint32_t)j;
        H1[j - 1] += 1;
    }
    /* c_j.Append(x_i) for i = 1..n: two-pass counting
     * placement, identical to appending in index order. */
    uint64_t *start = (uint64_t *)malloc((size_t)(gamma + 1) * 8);
    if (!start) return ORC_ERR_OOM;
    uint64_t run = 0;
    for (uint64_t j = 0; j <= gamma; j++) { start[j] = run; run += H1[j]; }
    for (uint64_t k = 0; k < m; k++) out[start[bucket[k] - 1]++] = seg[k];
    free(start);
    return rc;
}

/* ------------------------------------------------------------------------ */
typedef struct ls_state {
    int kt;
    orc_ctx *ctx;
    uint64_t *tmp; /* scratch, same length as the array */
} ls_state;

static void log_node(orc_ctx *c, const orc_node *nd)
{
    if (c->nodes && c->nodes_count < c->nodes_cap) c->nodes[c->nodes_count] = *nd;
    c->nodes_count++;
}

/* Learned-Sort(x) (Alg. 1) on y[o, o+m) at recursion level L
 * (level 1 = the whole array).  Order of checks per reading R13. */
static int learned_sort_rec(ls_state *st, uint64_t *y, uint64_t o, uint64_t m, uint32_t L)
{
    orc_ctx *c = st->ctx;
    int kt = st->kt;
    uint64_t *seg = y + o;
    if (L > c->max_depth) c->max_depth = L;

    /* if n < tau: return Standard-Sort(x) */
    if (m < c->tau) {
        orc_standard_sort(seg, m, kt);
        c->base_case_calls++;
        return 0;
    }

    /* x_min, x_max over the whole segment, totalOrder (R11) */
    uint64_t mn = seg[0], mx = seg[0];
    for (uint64_t k = 1; k < m; k++) {
        if (key_less(kt, seg[k], mn)) mn = seg[k];
        if (key_less(kt, mx, seg[k])) mx = seg[k];
    }
    /* Readings R9/R10: i(x) is undefined unless 0 < x_max - x_min < inf. */
    int degenerate;
    if (kt == ORC_KEY_F64) {
        double r = as_f64(mx) - as_f64(mn);
        degenerate = !(r > 0.0) || isinf(r);
    } else {
        degenerate = !(mx > mn);
    }
    if (degenerate) {
        orc_standard_sort(seg, m, kt);
        c->degenerate_calls++;
        return 0;
    }

    /* alpha = beta = gamma = delta = floor(m^{3/4})  (Thms 1-2; R5, R14) */
    uint64_t p = orc_iroot34(m);
    uint64_t beta = p, gamma = p, delta = p;
    uint64_t alpha = (c->flags & ORC_FLAG_SAMPLE_ALL) ? m : p;

    uint64_t *a = (uint64_t *)malloc((size_t)alpha * 8);
    uint32_t *b1 = (uint32_t *)malloc((size_t)(beta + 1) * 4);
    uint32_t *H1 = (uint32_t *)malloc((size_t)(gamma + 1) * 4);
    uint32_t *bucket = (uint32_t *)malloc((size_t)m * 4);
    if (!a || !b1 || !H1 || !bucket) { free(a); free(b1); free(H1); free(bucket); return ORC_ERR_OOM; }

    /* "alpha samples are taken at random from x" (R3, R4) */
    if (c->flags & ORC_FLAG_SAMPLE_ALL) {
        for (uint64_t k = 0; k < alpha; k++) a[k] = seg[k];
    } else {
        for (uint64_t k = 0; k < alpha; k++) a[k] = seg[orc_sample_position(c->seed, L, o, m, k)];
    }

    int rc = orc_bucketing(kt, seg, m, a, alpha, beta, gamma, mn, mx, b1, H1, bucket, st->tmp);
    if (rc == ORC_ERR_OOM) { free(a); free(b1); free(H1); free(bucket); return rc; }
    if (rc) c->violation |= 1;
    memcpy(seg, st->tmp, (size_t)m * 8);
    c->bucketing_calls++;

    orc_node nd;
    memset(&nd, 0, sizeof nd);
    nd.level = L; nd.alpha = (uint32_t)alpha; nd.offset = o; nd.m = m;
    nd.xmin_bits = mn; nd.xmax_bits = mx;
    nd.digest_b = orc_digest(b1, beta + 1);
    nd.digest_h = orc_digest(H1, gamma + 1);
    for (uint64_t j = 0; j <= gamma; j++) {
        if (H1[j] == 0) continue;
        if (H1[j] >= delta) nd.n_fallback++;
        else if (H1[j] < c->tau) nd.n_small++;
        else nd.n_recurse++;
    }
    if (L == 1 && c->l1_b) {
        uint64_t nb = beta + 1 < c->l1_cap ? beta + 1 : c->l1_cap;
        memcpy(c->l1_b, b1, (size_t)nb * 4);
        c->l1_b_len = beta + 1;
    }
    if (L == 1 && c->l1_h) {
        uint64_t nh = gamma + 1 < c->l1_cap ? gamma + 1 : c->l1_cap;
        memcpy(c->l1_h, H1, (size_t)nh * 4);
        c->l1_h_len = gamma + 1;
    }
    log_node(c, &nd);

    /* Per-node invariant checks */
    if (c->check) {
        uint64_t sum = 0;
        for (uint64_t j = 0; j <= gamma; j++) sum += H1[j];
        if (sum != m) c->violation |= 2;
        for (uint64_t i = 1; i <= beta; i++) if (b1[i] < b1[i - 1]) c->violation |= 4;
        if (b1[beta] != alpha) c->violation |= 4;
        if (orc_bucket_of(b1[beta], alpha, gamma) != gamma + 1) c->violation |= 8;
        if (H1[gamma] < 1) c->violation |= 8;
        /* order property: p in c_j, q in c_k, j < k => p < q */
        uint64_t pos = 0, prev_max = 0;
        int have_prev = 0;
        for (uint64_t j = 0; j <= gamma; j++) {
            if (H1[j] == 0) continue;
            uint64_t bmin = seg[pos], bmax = seg[pos];
            for (uint64_t k = pos; k < pos + H1[j]; k++) {
                if (key_less(kt, seg[k], bmin)) bmin = seg[k];
                if (key_less(kt, bmax, seg[k])) bmax = seg[k];
            }
            if (have_prev && !key_less(kt, prev_max, bmin)) c->violation |= 16;
            prev_max = bmax; have_prev = 1;
            pos += H1[j];
        }
    }

    /* Recursively sort and concatenate: c_j in place. */
    uint64_t pos = 0;
    for (uint64_t j = 0; j <= gamma && rc != ORC_ERR_OOM; j++) {
        uint64_t h = H1[j];
        if (h == 0) continue;
        if (h >= delta) {                 /* |c_j| >= delta: Standard-Sort (R12) */
            orc_standard_sort(seg + pos, h, kt);
            c->fallback_buckets++;
            c->fallback_keys += h;
        } else {                          /* else Learned-Sort(c_j) */
            int r2 = learned_sort_rec(st, y, o + pos, h, L + 1);
            if (r2 == ORC_ERR_OOM) rc = r2;
        }
        pos += h;
    }
    free(a); free(b1); free(H1); free(bucket);
    return rc == ORC_ERR_OOM ? rc : 0;
}

/* Entry point: sorts x[0..n) (bit patterns of kt keys) in place.
 * NaN keys are an input-domain error raised before any work. */
int orc_learned_sort(int kt, uint64_t *x, uint64_t n, orc_ctx *ctx)
{
    /* n <= 2^40 keeps m^3 inside 128 bits for the exact floor(m^{3/4}) (R5) */
    if (!ctx || (n && !x) || ctx->tau < 2 || (kt != ORC_KEY_F64 && kt != ORC_KEY_U64) ||
        n > (1ULL << 40))
        return ORC_ERR_INVALID_ARG;
    if (kt == ORC_KEY_F64)
        for (uint64_t k = 0; k < n; k++)
            if (is_nan_bits(x[k])) return ORC_ERR_NAN;
    if (n == 0) return ORC_OK;
    ls_state st;
    st.kt = kt; st.ctx = ctx;
    st.tmp = (uint64_t *)malloc((size_t)n * 8);
    if (!st.tmp) return ORC_ERR_OOM;
    int rc = learned_sort_rec(&st, x, 0, n, 1);
    free(st.tmp);
    if (rc) return rc;
    return ctx->violation ? ORC_ERR_INVARIANT : ORC_OK;
}

/* Deterministic recursion-depth bound (Eqs. 1-3; Lemma 1
 * sketch PAPER.md:239): Learned-Sort recurses only on buckets of size
 * < delta = floor(m^{3/4}), so level sizes obey m_{k+1} <= floor(m_k^{3/4}) - 1;
 * the bound is the number of levels whose size can still be >= tau, plus the
 * final base-case level. */
uint32_t orc_depth_bound(uint64_t n, uint32_t tau)
{
    uint32_t d = 1;
    uint64_t m = n;
    while (m >= tau) {
        uint64_t p = orc_iroot34(m);
        if (p == 0) break;
        m = p - 1;
        d++;
    }
    return d;
}
