/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference's CPU oracle for the fused
 * AllGather-GEMM / GEMM-ReduceScatter path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * Pinned against the reference's golden vectors (proj/tests/golden/*.csv via
 * tests/golden/) and, in this container, bitwise against the reference itself
 * compiled from /root/reference (oracle/_ref, see oracle/Makefile).
 *
 * Every function cites the reference code it restates
 * (paths relative to /root/reference/proj).
 *
 * Build with -ffp-contract=off: the reference's k-ascending fp64 sums must not
 * be contracted into FMAs for the outputs to be bit-identical.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

/* ---- Rng: splitmix64 + uniform[-1,1) (core/include/overlap/matrix.hpp:56-77) ---- */
typedef struct {
    uint64_t state;
} orc_rng;

static void rng_init(orc_rng* r, uint64_t seed) { r->state = seed ? seed : 0x9e3779b97f4a7c15ull; }

static uint64_t rng_next_u64(orc_rng* r) {
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static double rng_uniform(orc_rng* r) {
    return (double)(rng_next_u64(r) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

/* Round a double to the nearest bfloat16 (round-to-nearest-even), returned as
 * a double. Inputs are in [-1, 1), so no overflow/NaN handling is needed beyond
 * the generic path. This is the rounding the B200 harness applies to the
 * reference Rng stream before upload. */
double orc_round_bf16(double x) {
    float f = (float)x; /* double -> float is RNE; then float -> bf16 RNE */
    /* Double rounding d->f->bf16 can differ from direct d->bf16 only when the
     * float lands exactly on a bf16 tie; resolve ties against the double. */
    uint32_t u;
    memcpy(&u, &f, 4);
    uint32_t lower = u & 0xFFFFu;
    uint32_t base = u & 0xFFFF0000u;
    float lo, hi;
    memcpy(&lo, &base, 4);
    uint32_t up = base + 0x10000u;
    memcpy(&hi, &up, 4);
    uint32_t out;
    if (lower > 0x8000u) {
        out = up;
    } else if (lower < 0x8000u) {
        out = base;
    } else {
        /* float is exactly halfway between lo and hi: decide with the double */
        double dlo = (double)lo, dhi = (double)hi;
        double mid = 0.5 * (dlo + dhi);
        if (fabs(x) > fabs(mid)) out = up;
        else if (fabs(x) < fabs(mid)) out = base;
        else out = ((base >> 16) & 1u) ? up : base; /* true tie: even */
    }
    float r;
    memcpy(&r, &out, 4);
    return (double)r;
}

uint16_t orc_bf16_bits(double x) {
    float f = (float)orc_round_bf16(x);
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)(u >> 16);
}

/* ---- workspace fill (core/src/workspace.cpp:5-29) ----
 * Rank r draws from Rng(seed * 0x100000001b3 + r + 1): A shard row-major, then
 * B shard row-major (reference layout: AG A [m/tp, k], B [k, n/tp];
 * RS A [m, k/tp], B [k/tp, n]). round_bf16 != 0 rounds every value. */
void orc_fill_rank(int pattern, int m, int n, int k, int tp, uint64_t seed, int rank, int round_bf16, double* a,
                   double* b) {
    orc_rng rng;
    rng_init(&rng, seed * 0x100000001b3ull + (uint64_t)rank + 1);
    const int rpr = m / tp;
    size_t na, nb;
    if (pattern == 0) {
        na = (size_t)rpr * k;
        nb = (size_t)k * (n / tp);
    } else {
        na = (size_t)m * (k / tp);
        nb = (size_t)(k / tp) * n;
    }
    for (size_t i = 0; i < na; ++i) {
        double v = rng_uniform(&rng);
        a[i] = round_bf16 ? orc_round_bf16(v) : v;
    }
    for (size_t i = 0; i < nb; ++i) {
        double v = rng_uniform(&rng);
        b[i] = round_bf16 ? orc_round_bf16(v) : v;
    }
}

/* C[rows, cols] = A[rows, kk] * B[kk, cols] with every element summed from 0.0
 * in ascending k (oracle.cpp:10-19). The i-k-j loop performs exactly the same
 * sequence of (acc + a*b) roundings per element as the reference's i-j-k loop. */
static void matmul_rows(const double* a, int lda, const double* b, int ldb, double* c, int ldc, int rows, int kk,
                        int cols) {
    for (int i = 0; i < rows; ++i) {
        double* ci = c + (size_t)i * ldc;
        for (int j = 0; j < cols; ++j) ci[j] = 0.0;
        const double* ai = a + (size_t)i * lda;
        for (int x = 0; x < kk; ++x) {
            const double av = ai[x];
            const double* bx = b + (size_t)x * ldb;
            for (int j = 0; j < cols; ++j) ci[j] += av * bx[j];
        }
    }
}

/* AllGather-GEMM oracle for one rank (oracle.cpp:44-48): out [m, n/tp] =
 * gathered A [m, k] (shards stacked in rank order) * B_rank [k, n/tp].
 * a_shards[r] is rank r's [m/tp, k] shard. Only rows [row0, row0+rows). */
void orc_ag_rank(int m, int n, int k, int tp, const double* const* a_shards, const double* b_rank, double* out,
                 int row0, int rows) {
    const int rpr = m / tp, nl = n / tp;
    for (int i = row0; i < row0 + rows; ++i) {
        const int src = i / rpr;
        matmul_rows(a_shards[src] + (size_t)(i - src * rpr) * k, k, b_rank, nl, out + (size_t)(i - row0) * nl, nl, 1,
                    k, nl);
    }
}

/* GEMM-ReduceScatter oracle for one owner (oracle.cpp:49-60): out [rows, n] =
 * rows [owner*m/tp + lrow0, +rows) of sum_{r=0..tp-1} A_r [m, k/tp] * B_r [k/tp, n],
 * the sum taken in rank order starting from 0.0. scratch: n doubles. */
void orc_rs_rows(int m, int n, int k, int tp, const double* const* a_shards, const double* const* b_shards, int owner,
                 int lrow0, int rows, double* out, double* scratch) {
    const int rpr = m / tp, kl = k / tp;
    for (int i = 0; i < rows; ++i) {
        const int row = owner * rpr + lrow0 + i;
        double* o = out + (size_t)i * n;
        for (int j = 0; j < n; ++j) o[j] = 0.0;
        for (int r = 0; r < tp; ++r) {
            matmul_rows(a_shards[r] + (size_t)row * kl, kl, b_shards[r], n, scratch, n, 1, kl, n);
            for (int j = 0; j < n; ++j) o[j] += scratch[j];
        }
    }
}

/* max |a-b| / max(1, |a|, |b|) (matrix.cpp:11-25). */
double orc_max_rel_error(const double* a, const double* b, size_t count) {
    double worst = 0.0;
    for (size_t i = 0; i < count; ++i) {
        double fa = fabs(a[i]), fb = fabs(b[i]);
        double denom = fa > fb ? fa : fb;
        if (denom < 1.0) denom = 1.0;
        double e = fabs(a[i] - b[i]) / denom;
        if (e > worst) worst = e;
    }
    return worst;
}

/* ||a-b||_F / ||b||_F (normwise variant for bf16-exchange modes). */
double orc_normwise_error(const double* a, const double* b, size_t count) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < count; ++i) {
        double d = a[i] - b[i];
        num += d * d;
        den += b[i] * b[i];
    }
    return den > 0 ? sqrt(num / den) : sqrt(num);
}

/* Fill one rank directly as bf16 bit patterns in the B200 device layout:
 * A row-major as the reference (AG [m/tp, k], RS [m, k/tp]); B transposed to
 * K-major [cols, kk] (AG cols = n/tp, kk = k; RS cols = n, kk = k/tp), i.e.
 * bT[j*kk + x] = round_bf16(reference b_shard(x, j)). Same Rng stream as
 * orc_fill_rank (workspace.cpp:11,22-23). */
void orc_fill_rank_bits(int pattern, int m, int n, int k, int tp, uint64_t seed, int rank, uint16_t* a_bits,
                        uint16_t* bt_bits) {
    orc_rng rng;
    rng_init(&rng, seed * 0x100000001b3ull + (uint64_t)rank + 1);
    const int rpr = m / tp;
    int arows, acols, kk, cols;
    if (pattern == 0) {
        arows = rpr; acols = k; kk = k; cols = n / tp;
    } else {
        arows = m; acols = k / tp; kk = k / tp; cols = n;
    }
    for (size_t i = 0; i < (size_t)arows * acols; ++i) a_bits[i] = orc_bf16_bits(rng_uniform(&rng));
    for (int x = 0; x < kk; ++x)
        for (int j = 0; j < cols; ++j) bt_bits[(size_t)j * kk + x] = orc_bf16_bits(rng_uniform(&rng));
}

/* bf16 bits -> double (exact). */
void orc_bits_to_double(const uint16_t* bits, double* out, size_t count) {
    for (size_t i = 0; i < count; ++i) {
        uint32_t u = (uint32_t)bits[i] << 16;
        float f;
        memcpy(&f, &u, 4);
        out[i] = (double)f;
    }
}
