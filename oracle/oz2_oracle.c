/*
 * oz2_oracle.c — CPU restatement of the reference's Ozaki-II accurate-mode
 * emulation (`oz2::os_ii<T>`), used ONLY as test infrastructure:
 *   - tests/ compare the CUDA product path against it bit for bit;
 *   - bench.py's cpu_baseline leg / `--impl reference` time it;
 *   - __graft_entry__.smoke() checks one small product call against it.
 * Nothing in the product package (paper_2602_02549_b200/) links, imports or
 * calls this file.
 *
 * Every function cites the reference line it restates (paths relative to
 * /root/reference/proj/include/oz2/).  Compile with -ffp-contract=off and no
 * -march flags, like the reference build (CMakeLists.txt:3-10), so that every
 * `a*b+c` below is two roundings and every fma() is libm's single rounding.
 *
 * The per-(N, mode) constants (moduli, s1/s2, P1/P2, P_inv, P') are computed
 * in exact arithmetic by oracle/moduli.py (restating moduli.hpp:93-142 and
 * mp.hpp:59-93) and passed in through `ora_table`.
 *
 * Error codes mirror the reference's exception classes:
 *   0 ok, 1 std::invalid_argument, 2 std::domain_error, 3 std::range_error,
 *   4 std::logic_error.
 */
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_INVALID 1
#define ORA_DOMAIN 2
#define ORA_RANGE 3
#define ORA_LOGIC 4

#define ORA_MAX_MODULI 49
#define ORA_MAX_INNER (1LL << 17) /* int8gemm.hpp:12 kMaxInnerDim */

typedef struct {
    int n;                     /* number of moduli N */
    int mode;                  /* 0 = fp32 (Prec::F32), 1 = fp64 (Prec::F64) */
    int p[ORA_MAX_MODULI];     /* moduli.hpp:31-36 first N entries */
    double s1[ORA_MAX_MODULI]; /* moduli.hpp:120-138 */
    double s2[ORA_MAX_MODULI];
    double P1, P2, P_inv;      /* moduli.hpp:112-117 */
    float P_prime;             /* moduli.hpp:140, mp.hpp:67-85 */
    float coeff;               /* mp.hpp:89-93 scaling_coeff_fp32() */
} ora_table;

/* Optional outputs; any NULL pointer is skipped (emulate.hpp:17-24 fields). */
typedef struct {
    int16_t *mu, *nu, *mu_prime, *nu_prime; /* scaling.hpp:20-28 */
    float *e, *f;
    double *Aprime, *Bprime;                /* m*k, k*n */
    int32_t *Cbar;                          /* m*n */
    float *Dbar;                            /* m*n */
    int8_t *W;                              /* N*m*n, crt.hpp:81-87 */
    double *C1, *C2, *Q, *Cpp64;            /* m*n */
    float *Cpp32;                           /* m*n (fp32 mode) */
    int8_t *Ares, *Bres;                    /* N*m*k, N*k*n residue planes (crt.hpp:160-161) */
    int32_t *Cprod;                         /* N*m*n wrapped INT32 products (crt.hpp:70) */
    int32_t *cmax_row, *cmax_col;           /* out: row/col maxima of Cbar (scaling.hpp:175-192) */
    const int32_t *ext_cmax_row;            /* in: if set, maxima already reduced across ranks */
    const int32_t *ext_cmax_col;            /*     (multi-rank 2-D partition) */
    int subnormal;                          /* emulate.hpp:23 */
    char msg[256];                          /* exception what() */
} ora_out;

static int set_err(ora_out *o, int code, const char *what) {
    if (o) {
        strncpy(o->msg, what, sizeof(o->msg) - 1);
        o->msg[sizeof(o->msg) - 1] = 0;
    }
    return code;
}

/* ---------------------------------------------------------------------------
 * parallel.hpp:22-40 — contiguous-block fork/join over threads; results are
 * independent of the thread count because workers never share outputs.
 * ------------------------------------------------------------------------- */
typedef void (*ora_body)(int64_t i, void *ctx);
typedef struct { int64_t lo, hi; ora_body fn; void *ctx; } ora_chunk;

static void *ora_chunk_run(void *arg) {
    ora_chunk *c = (ora_chunk *)arg;
    for (int64_t i = c->lo; i < c->hi; ++i) c->fn(i, c->ctx);
    return NULL;
}

static int g_threads = 1;

void ora_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

static void parallel_for(int64_t count, ora_body fn, void *ctx) {
    int threads = g_threads;
    if (threads > count) threads = (int)count;
    if (threads <= 1) {
        for (int64_t i = 0; i < count; ++i) fn(i, ctx);
        return;
    }
    const int64_t block = (count + threads - 1) / threads;
    pthread_t tid[256];
    ora_chunk ch[256];
    int used = 0;
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = t * block;
        int64_t hi = lo + block;
        if (hi > count) hi = count;
        if (lo >= hi) break;
        ch[used].lo = lo; ch[used].hi = hi; ch[used].fn = fn; ch[used].ctx = ctx;
        pthread_create(&tid[used], NULL, ora_chunk_run, &ch[used]);
        ++used;
    }
    for (int t = 0; t < used; ++t) pthread_join(tid[t], NULL);
}

/* ---------------------------------------------------------------------------
 * prng.hpp:48-82 and gen.hpp:15-31 — the reference's synthetic generator.
 * ------------------------------------------------------------------------- */
static uint64_t splitmix64(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s[4]; } xoshiro;

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static void xo_seed(xoshiro *r, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&sm);
}

static uint64_t xo_next(xoshiro *r) {
    uint64_t *s = r->s;
    const uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

static double xo_uniform(xoshiro *r) { return (double)((xo_next(r) >> 11) + 1) * 0x1p-53; }

static double xo_normal(xoshiro *r) {
    const double u1 = xo_uniform(r);
    const double u2 = xo_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

uint64_t ora_xoshiro_next(uint64_t seed, int64_t count, uint64_t *out) {
    xoshiro r;
    xo_seed(&r, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = xo_next(&r);
    return 0;
}

int ora_gen_matrix_f64(int64_t rows, int64_t cols, double phi, uint64_t seed, double *out) {
    if (phi < 0) return ORA_DOMAIN;
    xoshiro r;
    xo_seed(&r, seed);
    for (int64_t i = 0; i < rows * cols; ++i) {
        double v;
        do {
            const double u = xo_uniform(&r);
            const double g = xo_normal(&r);
            v = (u - 0.5) * exp(g * phi);
        } while (v == 0.0 || !isfinite(v));
        out[i] = v;
    }
    return ORA_OK;
}

int ora_gen_matrix_f32(int64_t rows, int64_t cols, double phi, uint64_t seed, float *out) {
    if (phi < 0) return ORA_DOMAIN;
    xoshiro r;
    xo_seed(&r, seed);
    for (int64_t i = 0; i < rows * cols; ++i) {
        float v;
        do {
            const double u = xo_uniform(&r);
            const double g = xo_normal(&r);
            v = (float)((u - 0.5) * exp(g * phi));
        } while (v == 0.0f || !isfinite((double)v));
        out[i] = v;
    }
    return ORA_OK;
}

/* experiment.hpp:83-88 */
uint64_t ora_derive_seed(uint64_t seed, uint64_t trial, uint64_t role) {
    uint64_t s = seed;
    (void)splitmix64(&s);
    s ^= 0x5851f42d4c957f2dull * (trial + 1) + 0x14057b7ef767814full * (role + 1);
    return splitmix64(&s);
}

/* ---------------------------------------------------------------------------
 * softfp.hpp scalar primitives.
 * ------------------------------------------------------------------------- */

/* softfp.hpp:94-102 round_nearest_even */
static double round_nearest_even(double x) {
    if (fabs(x) >= 0x1p52) return x;
    const double fl = floor(x);
    const double frac = x - fl;
    if (frac > 0.5) return fl + 1.0;
    if (frac < 0.5) return fl;
    return fmod(fl, 2.0) == 0.0 ? fl : fl + 1.0;
}

/* softfp.hpp:117-125 signed_mod (int64 variant) */
static long long signed_mod_ll(long long x, long long p) {
    long long r0 = x % p;
    if (r0 < 0) r0 += p;
    if (2 * r0 < p) return r0;
    if (2 * r0 > p) return r0 - p;
    const long long q0 = (x - r0) / p;
    return (q0 % 2 == 0) ? r0 : r0 - p;
}

/* softfp.hpp:147-150 log2_fp32: extended log2 then one fp32 rounding */
float ora_log2_fp32(float x) { return (float)log2((double)x); }

/* softfp.hpp:153-159 fp32_round_up */
float ora_fp32_round_up(int64_t v) {
    float f = (float)v;
    if ((double)f < (double)v) f = nextafterf(f, INFINITY);
    return f;
}

/*
 * softfp.hpp:89-91 fma_fp32(a, b, c, Rnd::Down): single downward rounding of
 * the exact a*b + c.  For fp32 a, b the product is exact in fp64 (48 bits);
 * TwoSum gives the exact sum as hi + lo; the largest float <= hi + lo is then
 * found from RN(hi) with one correction step.
 */
float ora_fma_fp32_down(float a, float b, float c) {
    const double prod = (double)a * (double)b; /* exact */
    const double cd = (double)c;
    const double hi = prod + cd;
    const double bb = hi - prod;
    const double lo = (prod - (hi - bb)) + (cd - bb); /* TwoSum: hi + lo == prod + cd */
    float f = (float)hi;
    if ((double)f > hi || ((double)f == hi && lo < 0.0)) f = nextafterf(f, -INFINITY);
    return f;
}

/* scaling.hpp:159-194 shift_from: floor(fma_fp32(coeff, e, P', Down)) */
long ora_shift_from(float coeff, float e, float p_prime) {
    const float inner = ora_fma_fp32_down(coeff, e, p_prime);
    return (long)floor((double)inner);
}

/* The full scaling-exponent step for one clearance max c (integer, exact):
 * D = RU32(c) (softfp.hpp:153-159), mx = max(1, D) (scaling.hpp:176-177),
 * e = log2f(mx) (:178), shift = floor(fma_down(coeff, e, P')) (:171-172). */
long ora_shift_of_cmax(int64_t c, float coeff, float p_prime, float *e_out) {
    float d = ora_fp32_round_up(c);
    float mx = 1.0f;
    if (d > mx) mx = d;
    const float e = ora_log2_fp32(mx);
    if (e_out) *e_out = e;
    return ora_shift_from(coeff, e, p_prime);
}

/* ---------------------------------------------------------------------------
 * scaling.hpp — Algorithm 2.  Inputs are fp64 arrays; the fp32 mode passes
 * the exactly widened float values, matching the reference, which converts
 * every float entry to double before each scaling operation (scaling.hpp:36,
 * :46, :116, :127, :205, :219).
 * ------------------------------------------------------------------------- */

/* scaling.hpp:61-79 ceil_abs_scaled */
static int ceil_abs_scaled(double a, int sft, int8_t *out) {
    if (a == 0.0) { *out = 0; return ORA_OK; }
    int e;
    const double f = frexp(fabs(a), &e);
    const uint64_t mant = (uint64_t)ldexp(f, 53);
    const long exp2 = (long)e - 53 + sft;
    if (exp2 >= 0) return ORA_LOGIC;
    const long s = -exp2;
    uint64_t v;
    if (s >= 53) {
        v = 1;
    } else {
        const uint64_t q = mant >> s;
        const uint64_t rem = mant & ((1ull << s) - 1);
        v = q + (rem != 0 ? 1 : 0);
    }
    if (v > 64) return ORA_LOGIC;
    *out = (int8_t)v;
    return ORA_OK;
}

/* int8gemm.hpp:17-34 gemm_i8_wrap: i-j-h loops, uint32 wraparound. */
typedef struct { const int8_t *a, *b; int32_t *c; int64_t m, k, n; } gemm_ctx;

static void gemm_row(int64_t i, void *vctx) {
    const gemm_ctx *g = (const gemm_ctx *)vctx;
    for (int64_t j = 0; j < g->n; ++j) {
        uint32_t acc = 0;
        for (int64_t h = 0; h < g->k; ++h) {
            const int32_t prod = (int32_t)g->a[i * g->k + h] * (int32_t)g->b[h * g->n + j];
            acc += (uint32_t)prod;
        }
        g->c[i * g->n + j] = (int32_t)acc;
    }
}

int ora_gemm_i8_wrap(int64_t m, int64_t k, int64_t n, const int8_t *a, const int8_t *b, int32_t *c) {
    if (k > ORA_MAX_INNER) return ORA_DOMAIN;
    gemm_ctx g = {a, b, c, m, k, n};
    parallel_for(m, gemm_row, &g);
    return ORA_OK;
}

/* crt.hpp:20-28 pow2_mod */
static long pow2_mod(long e, long p) {
    long base = 2 % p, acc = 1 % p;
    while (e > 0) {
        if (e & 1) acc = (acc * base) % p;
        base = (base * base) % p;
        e >>= 1;
    }
    return acc;
}

/* crt.hpp:32-53 residue_of */
int ora_residue_of(double x, int p, int8_t *out) {
    if (x == 0.0) { *out = 0; return ORA_OK; }
    if (!isfinite(x)) return ORA_DOMAIN;
    int e;
    const double f = frexp(fabs(x), &e);
    uint64_t mant = (uint64_t)ldexp(f, 53);
    long ex = (long)e - 53;
    if (ex < 0) {
        const uint64_t low = (-ex >= 64) ? mant : (mant & ((1ull << -ex) - 1));
        if (low != 0) return ORA_DOMAIN;
        mant = (-ex >= 64) ? 0 : (mant >> -ex);
        ex = 0;
    }
    long r0 = (long)(mant % (uint64_t)p);
    r0 = (r0 * pow2_mod(ex, p)) % p;
    if (x < 0.0) r0 = (p - r0) % p;
    if (2 * r0 > p) { *out = (int8_t)(r0 - p); return ORA_OK; }
    if (2 * r0 == p) { *out = (int8_t)(-p / 2); return ORA_OK; }
    *out = (int8_t)r0;
    return ORA_OK;
}

/* Exported scalar primitives for the KAT suite. */
int ora_ceil_abs_scaled(double a, int sft, int8_t *out) { return ceil_abs_scaled(a, sft, out); }
long long ora_signed_mod(long long x, long long p) { return signed_mod_ll(x, p); }
double ora_round_nearest_even(double x) { return round_nearest_even(x); }

/* ---------------------------------------------------------------------------
 * Work contexts for the row-parallel loops.
 * ------------------------------------------------------------------------- */
typedef struct {
    const double *x; int64_t rows, cols;
    const int16_t *sft; int by_col; /* sft indexed by row (0) or column (1) */
    int8_t *out; double *outd; int p; volatile int err;
} map_ctx;

static void ceil_row(int64_t i, void *v) {
    map_ctx *c = (map_ctx *)v;
    for (int64_t h = 0; h < c->cols; ++h) {
        const int sft = c->by_col ? c->sft[h] : c->sft[i];
        int8_t r;
        if (ceil_abs_scaled(c->x[i * c->cols + h], sft, &r) != ORA_OK) { c->err = ORA_LOGIC; return; }
        c->out[i * c->cols + h] = r;
    }
}

/* scaling.hpp:199-225 truncate_scaled_rows/cols */
static void trunc_row(int64_t i, void *v) {
    map_ctx *c = (map_ctx *)v;
    for (int64_t h = 0; h < c->cols; ++h) {
        const int sft = c->by_col ? c->sft[h] : c->sft[i];
        const double scaled = ldexp(c->x[i * c->cols + h], sft);
        if (!isfinite(scaled)) { c->err = ORA_RANGE; return; }
        c->outd[i * c->cols + h] = trunc(scaled);
    }
}

/* crt.hpp:58-65 residue_matrix */
static void resid_row(int64_t i, void *v) {
    map_ctx *c = (map_ctx *)v;
    for (int64_t h = 0; h < c->cols; ++h) {
        int8_t r;
        if (ora_residue_of(c->x[i * c->cols + h], c->p, &r) != ORA_OK) { c->err = ORA_DOMAIN; return; }
        c->out[i * c->cols + h] = r;
    }
}

typedef struct {
    const int8_t *const *w; int64_t n; const ora_table *t; double *c1, *c2;
} acc_ctx;

/* crt.hpp:91-110 accumulate: ordered fma chain starting at +0.0 */
static void acc_row(int64_t i, void *v) {
    acc_ctx *c = (acc_ctx *)v;
    const int dd = c->t->mode == 1;
    for (int64_t j = 0; j < c->n; ++j) {
        double acc1 = 0.0, acc2 = 0.0;
        for (int l = 0; l < c->t->n; ++l) {
            const double wv = (double)c->w[l][i * c->n + j];
            acc1 = fma(c->t->s1[l], wv, acc1);
            if (dd) acc2 = fma(c->t->s2[l], wv, acc2);
        }
        c->c1[i * c->n + j] = acc1;
        c->c2[i * c->n + j] = acc2;
    }
}

/* ---------------------------------------------------------------------------
 * emulate.hpp:54-88 os_ii<T> — the whole pipeline.
 *   prec: 0 = float (A, B, C are float*), 1 = double.
 * ------------------------------------------------------------------------- */
static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) { fprintf(stderr, "oz2_oracle: out of memory (%zu bytes)\n", n); abort(); }
    return p;
}

int ora_os_ii(int prec, int64_t m, int64_t k, int64_t n, const void *Ain, const void *Bin,
              void *Cout, const ora_table *t, ora_out *o) {
    if (o) { o->subnormal = 0; o->msg[0] = 0; }
    if (k > ORA_MAX_INNER) return set_err(o, ORA_DOMAIN, "os_ii: k exceeds 2^17");
    if (t->n < 2 || t->n > ORA_MAX_MODULI) return set_err(o, ORA_DOMAIN, "build_table: N out of [2, 49]");
    const int N = t->n;
    int rc = ORA_OK;

    /* widen inputs exactly (fp32 mode converts per element in the reference) */
    double *A = (double *)xmalloc(sizeof(double) * (size_t)(m * k));
    double *B = (double *)xmalloc(sizeof(double) * (size_t)(k * n));
    for (int64_t i = 0; i < m * k; ++i) A[i] = prec ? ((const double *)Ain)[i] : (double)((const float *)Ain)[i];
    for (int64_t i = 0; i < k * n; ++i) B[i] = prec ? ((const double *)Bin)[i] : (double)((const float *)Bin)[i];

    int16_t *mup = (int16_t *)xmalloc(sizeof(int16_t) * (size_t)m);
    int16_t *nup = (int16_t *)xmalloc(sizeof(int16_t) * (size_t)n);
    int16_t *mu = (int16_t *)xmalloc(sizeof(int16_t) * (size_t)m);
    int16_t *nu = (int16_t *)xmalloc(sizeof(int16_t) * (size_t)n);
    float *ev = (float *)xmalloc(sizeof(float) * (size_t)m);
    float *fv = (float *)xmalloc(sizeof(float) * (size_t)n);
    int8_t *abar = NULL, *bbar = NULL, **W = NULL, *al = NULL, *bl = NULL;
    int32_t *cbar = NULL, *cl = NULL;
    double *Ap = NULL, *Bp = NULL, *c1 = NULL, *c2 = NULL;
    char buf[128];

    /* scaling.hpp:86-96 row_pre_exponents (row_abs_max :33-42) */
    for (int64_t i = 0; i < m; ++i) {
        double mx = 0;
        for (int64_t h = 0; h < k; ++h) {
            const double v = fabs(A[i * k + h]);
            if (!isfinite(v)) { rc = set_err(o, ORA_DOMAIN, "matrix entry is not finite"); goto done; }
            mx = v > mx ? v : mx;
        }
        if (mx == 0.0) {
            snprintf(buf, sizeof buf, "row_pre_exponents: zero row %lld", (long long)i);
            rc = set_err(o, ORA_DOMAIN, buf); goto done;
        }
        mup[i] = (int16_t)(5l - ilogb(mx));
    }
    /* scaling.hpp:98-107 col_pre_exponents (col_abs_max :44-52) */
    for (int64_t j = 0; j < n; ++j) {
        double mx = 0;
        for (int64_t h = 0; h < k; ++h) {
            const double v = fabs(B[h * n + j]);
            if (!isfinite(v)) { rc = set_err(o, ORA_DOMAIN, "matrix entry is not finite"); goto done; }
            mx = v > mx ? v : mx;
        }
        if (mx == 0.0) {
            snprintf(buf, sizeof buf, "col_pre_exponents: zero column %lld", (long long)j);
            rc = set_err(o, ORA_DOMAIN, buf); goto done;
        }
        nup[j] = (int16_t)(5l - ilogb(mx));
    }

    /* scaling.hpp:111-131 ceil_abs_scale_rows/cols */
    abar = (int8_t *)xmalloc((size_t)(m * k));
    bbar = (int8_t *)xmalloc((size_t)(k * n));
    {
        map_ctx ca = {A, m, k, mup, 0, abar, NULL, 0, 0};
        parallel_for(m, ceil_row, &ca);
        map_ctx cb = {B, k, n, nup, 1, bbar, NULL, 0, 0};
        parallel_for(k, ceil_row, &cb);
        if (ca.err || cb.err) { rc = set_err(o, ORA_LOGIC, "ceil_abs_scaled: entry above row/column max"); goto done; }
    }

    /* scaling.hpp:140-148 clearance_product */
    cbar = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(m * n));
    ora_gemm_i8_wrap(m, k, n, abar, bbar, cbar);
    if (o && o->Cbar) memcpy(o->Cbar, cbar, sizeof(int32_t) * (size_t)(m * n));
    if (o && o->Dbar)
        for (int64_t i = 0; i < m * n; ++i) o->Dbar[i] = ora_fp32_round_up(cbar[i]);

    /* scaling.hpp:159-194 scaling_exponents */
    for (int64_t i = 0; i < m; ++i) {
        float mx = 1.0f;
        int32_t cm = 0;
        for (int64_t j = 0; j < n; ++j) {
            const float d = ora_fp32_round_up(cbar[i * n + j]);
            mx = d > mx ? d : mx;
            cm = cbar[i * n + j] > cm ? cbar[i * n + j] : cm;
        }
        if (o && o->cmax_row) o->cmax_row[i] = cm;
        if (o && o->ext_cmax_row) {  /* RU32 is monotone: max of RU32 == RU32 of max */
            const float d = ora_fp32_round_up(o->ext_cmax_row[i]);
            mx = d > 1.0f ? d : 1.0f;
        }
        const float ei = ora_log2_fp32(mx);
        if (!(ei < 31.0f)) { rc = set_err(o, ORA_LOGIC, "scaling_exponents: e_i >= 31"); goto done; }
        ev[i] = ei;
        const long v = (long)mup[i] + ora_shift_from(t->coeff, ei, t->P_prime);
        if (v < -32768 || v > 32767) { rc = set_err(o, ORA_RANGE, "mu: exceeds 16-bit range"); goto done; }
        mu[i] = (int16_t)v;
    }
    for (int64_t j = 0; j < n; ++j) {
        float mx = 1.0f;
        int32_t cm = 0;
        for (int64_t i = 0; i < m; ++i) {
            const float d = ora_fp32_round_up(cbar[i * n + j]);
            mx = d > mx ? d : mx;
            cm = cbar[i * n + j] > cm ? cbar[i * n + j] : cm;
        }
        if (o && o->cmax_col) o->cmax_col[j] = cm;
        if (o && o->ext_cmax_col) {
            const float d = ora_fp32_round_up(o->ext_cmax_col[j]);
            mx = d > 1.0f ? d : 1.0f;
        }
        const float fj = ora_log2_fp32(mx);
        if (!(fj < 31.0f)) { rc = set_err(o, ORA_LOGIC, "scaling_exponents: f_j >= 31"); goto done; }
        fv[j] = fj;
        const long v = (long)nup[j] + ora_shift_from(t->coeff, fj, t->P_prime);
        if (v < -32768 || v > 32767) { rc = set_err(o, ORA_RANGE, "nu: exceeds 16-bit range"); goto done; }
        nu[j] = (int16_t)v;
    }

    /* scaling.hpp:199-225 truncate_scaled_rows/cols */
    Ap = (double *)xmalloc(sizeof(double) * (size_t)(m * k));
    Bp = (double *)xmalloc(sizeof(double) * (size_t)(k * n));
    {
        map_ctx ta = {A, m, k, mu, 0, NULL, Ap, 0, 0};
        parallel_for(m, trunc_row, &ta);
        if (ta.err) { rc = set_err(o, ORA_RANGE, "truncate_scaled: 2^mu*a overflow"); goto done; }
        map_ctx tb = {B, k, n, nu, 1, NULL, Bp, 0, 0};
        parallel_for(k, trunc_row, &tb);
        if (tb.err) { rc = set_err(o, ORA_RANGE, "truncate_scaled: b*2^nu overflow"); goto done; }
    }

    /* crt.hpp:154-173 run_crt: per-modulus residues, GEMM, reduction */
    W = (int8_t **)xmalloc(sizeof(int8_t *) * (size_t)N);
    for (int l = 0; l < N; ++l) W[l] = (int8_t *)xmalloc((size_t)(m * n));
    al = (int8_t *)xmalloc((size_t)(m * k));
    bl = (int8_t *)xmalloc((size_t)(k * n));
    cl = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(m * n));
    for (int l = 0; l < N; ++l) {
        const int p = t->p[l];
        map_ctx ra = {Ap, m, k, NULL, 0, al, NULL, p, 0};
        parallel_for(m, resid_row, &ra);
        map_ctx rb = {Bp, k, n, NULL, 0, bl, NULL, p, 0};
        parallel_for(k, resid_row, &rb);
        if (ra.err || rb.err) { rc = set_err(o, ORA_DOMAIN, "residue_of: entry is not an integer"); goto done; }
        if (o && o->Ares) memcpy(o->Ares + (size_t)l * (size_t)(m * k), al, (size_t)(m * k));
        if (o && o->Bres) memcpy(o->Bres + (size_t)l * (size_t)(k * n), bl, (size_t)(k * n));
        /* crt.hpp:69-79 residue_gemm_and_reduce */
        ora_gemm_i8_wrap(m, k, n, al, bl, cl);
        if (o && o->Cprod) memcpy(o->Cprod + (size_t)l * (size_t)(m * n), cl, sizeof(int32_t) * (size_t)(m * n));
        for (int64_t i = 0; i < m * n; ++i) {
            long long v = signed_mod_ll((long long)cl[i], p);
            if (2 * v == p) v = -v;
            W[l][i] = (int8_t)v;
        }
        if (o && o->W) memcpy(o->W + (size_t)l * (size_t)(m * n), W[l], (size_t)(m * n));
    }

    c1 = (double *)xmalloc(sizeof(double) * (size_t)(m * n));
    c2 = (double *)xmalloc(sizeof(double) * (size_t)(m * n));
    {
        acc_ctx ac = {(const int8_t *const *)W, n, t, c1, c2};
        parallel_for(m, acc_row, &ac);
    }
    if (o && o->C1) memcpy(o->C1, c1, sizeof(double) * (size_t)(m * n));
    if (o && o->C2) memcpy(o->C2, c2, sizeof(double) * (size_t)(m * n));

    /* crt.hpp:113-119 compute_q and crt.hpp:129-150 final_reduce, then
     * emulate.hpp:30-46 inverse_scale<T>.  The reference completes the whole
     * final_reduce (including its fp32 range check) before inverse_scale. */
    {
        int any_range_fr = 0, any_range_inv = 0, sub = 0;
        double *cpp = (double *)xmalloc(sizeof(double) * (size_t)(m * n));
        for (int64_t i = 0; i < m * n; ++i) {
            const double q = round_nearest_even(t->P_inv * c1[i]);
            if (o && o->Q) o->Q[i] = q;
            const double t1 = fma(-q, t->P1, c1[i]);
            const double t2 = t1 + c2[i];
            cpp[i] = fma(-q, t->P2, t2);
            if (o && o->Cpp64) o->Cpp64[i] = cpp[i];
            if (t->mode == 0 && fabs(cpp[i]) >= 0x1.ffffffp+127) any_range_fr = 1;
        }
        if (any_range_fr) {
            free(cpp);
            rc = set_err(o, ORA_RANGE, "final_reduce: single(C'') overflows fp32 (N too large for fp32 mode)");
            goto done;
        }
        for (int64_t i = 0; i < m && !any_range_inv; ++i)
            for (int64_t j = 0; j < n; ++j) {
                const int64_t idx = i * n + j;
                if (prec == 0) {
                    const float cp32 = (float)cpp[idx];
                    if (o && o->Cpp32) o->Cpp32[idx] = cp32;
                    const float x = ldexpf(cp32, -mu[i]);
                    const float y = ldexpf(x, -nu[j]);
                    if (!isfinite(y) || !isfinite(x)) { any_range_inv = 1; break; }
                    if ((x != 0 && fabsf(x) < FLT_MIN) || (y != 0 && fabsf(y) < FLT_MIN)) sub = 1;
                    ((float *)Cout)[idx] = y;
                } else {
                    const double x = ldexp(cpp[idx], -mu[i]);
                    const double y = ldexp(x, -nu[j]);
                    if (!isfinite(y) || !isfinite(x)) { any_range_inv = 1; break; }
                    if ((x != 0 && fabs(x) < DBL_MIN) || (y != 0 && fabs(y) < DBL_MIN)) sub = 1;
                    ((double *)Cout)[idx] = y;
                }
            }
        free(cpp);
        if (any_range_inv) { rc = set_err(o, ORA_RANGE, "os_ii: inverse scaling overflow"); goto done; }
        if (o) o->subnormal = sub;
    }

    if (o) {
        if (o->mu) memcpy(o->mu, mu, sizeof(int16_t) * (size_t)m);
        if (o->nu) memcpy(o->nu, nu, sizeof(int16_t) * (size_t)n);
        if (o->mu_prime) memcpy(o->mu_prime, mup, sizeof(int16_t) * (size_t)m);
        if (o->nu_prime) memcpy(o->nu_prime, nup, sizeof(int16_t) * (size_t)n);
        if (o->e) memcpy(o->e, ev, sizeof(float) * (size_t)m);
        if (o->f) memcpy(o->f, fv, sizeof(float) * (size_t)n);
        if (o->Aprime) memcpy(o->Aprime, Ap, sizeof(double) * (size_t)(m * k));
        if (o->Bprime) memcpy(o->Bprime, Bp, sizeof(double) * (size_t)(k * n));
    }

done:
    free(A); free(B); free(mup); free(nup); free(mu); free(nu); free(ev); free(fv);
    free(abar); free(bbar); free(cbar); free(Ap); free(Bp); free(al); free(bl); free(cl);
    free(c1); free(c2);
    if (W) { for (int l = 0; l < N; ++l) free(W[l]); free(W); }
    return rc;
}

/* Exhaustive monotonicity check of the log2f model over every value D̄ can
 * take (RU32 of integers in [1, 2^29]): returns the number of adjacent float
 * pairs x < y with log2f(x) > log2f(y).  Used by the oracle tests to justify
 * the product's threshold-table evaluation of mu/nu. */
int64_t ora_log2f_monotone_violations(void) {
    int64_t bad = 0;
    float prev_x = 1.0f, prev_e = ora_log2_fp32(1.0f);
    for (float x = nextafterf(1.0f, INFINITY); x <= 0x1p29f; x = nextafterf(x, INFINITY)) {
        const float e = ora_log2_fp32(x);
        if (e < prev_e) ++bad;
        prev_x = x; prev_e = e;
    }
    (void)prev_x;
    return bad;
}

/* Element-wise log2f over a float array (used to check device log2 parity). */
void ora_log2f_array(const float *x, int64_t count, float *out) {
    for (int64_t i = 0; i < count; ++i) out[i] = ora_log2_fp32(x[i]);
}

/* ---------------------------------------------------------------------------
 * Sampled full-size checks (test infrastructure): pieces of os_ii evaluated
 * exactly as above for selected rows / columns / entries, so that a device
 * result at BASELINE sizes (16384^3) can be verified without the O(N m n k)
 * CPU emulation.
 * ------------------------------------------------------------------------- */

/* scaling.hpp:86-107 for every row of A (m x k) / column of B (k x n);
 * returns ORA_DOMAIN on a zero row / column or non-finite entry. */
int ora_pre_exponents(const double *X, int64_t rows, int64_t cols, int by_col, int16_t *out) {
    const int64_t cnt = by_col ? cols : rows, len = by_col ? rows : cols;
    for (int64_t t = 0; t < cnt; ++t) {
        double mx = 0;
        for (int64_t h = 0; h < len; ++h) {
            const double v = fabs(by_col ? X[h * cols + t] : X[t * cols + h]);
            if (!isfinite(v)) return ORA_DOMAIN;
            mx = v > mx ? v : mx;
        }
        if (mx == 0.0) return ORA_DOMAIN;
        out[t] = (int16_t)(5l - ilogb(mx));
    }
    return ORA_OK;
}

/* Abar / Bbar (scaling.hpp:111-131) as int8 matrices in the reference layout. */
typedef struct { const double *x; int64_t rows, cols; const int16_t *sft; int by_col; int8_t *out; volatile int err; } cs_ctx;
static void cs_row(int64_t i, void *v) {
    cs_ctx *c = (cs_ctx *)v;
    for (int64_t h = 0; h < c->cols; ++h)
        if (ceil_abs_scaled(c->x[i * c->cols + h], c->by_col ? c->sft[h] : c->sft[i], &c->out[i * c->cols + h]) != ORA_OK)
            c->err = 1;
}
int ora_ceil_scale(const double *X, int64_t rows, int64_t cols, const int16_t *sft, int by_col, int8_t *out) {
    cs_ctx c = {X, rows, cols, sft, by_col, out, 0};
    parallel_for(rows, cs_row, &c);
    return c.err ? ORA_LOGIC : ORA_OK;
}

/* Row maxima of Cbar = Abar * Bbar for selected rows (scaling.hpp:175-183);
 * one selected row per parallel_for index. */
typedef struct { const int8_t *abar, *bbar; int64_t m, k, n; const int64_t *idx; int32_t *out; } cm_ctx;
static void cm_row(int64_t q, void *v) {
    const cm_ctx *c = (const cm_ctx *)v;
    int32_t *acc = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)c->n);
    memset(acc, 0, sizeof(int32_t) * (size_t)c->n);
    const int8_t *a = c->abar + c->idx[q] * c->k;
    for (int64_t h = 0; h < c->k; ++h) {
        const int32_t av = a[h];
        if (!av) continue;
        const int8_t *b = c->bbar + h * c->n;
        for (int64_t j = 0; j < c->n; ++j) acc[j] += av * (int32_t)b[j];
    }
    int32_t mx = 0;
    for (int64_t j = 0; j < c->n; ++j) mx = acc[j] > mx ? acc[j] : mx;
    c->out[q] = mx;
    free(acc);
}
int ora_cbar_row_max(const int8_t *abar, const int8_t *bbar, int64_t k, int64_t n, const int64_t *rows,
                     int64_t count, int32_t *out) {
    cm_ctx c = {abar, bbar, 0, k, n, rows, out};
    parallel_for(count, cm_row, &c);
    return ORA_OK;
}

/* Column maxima of Cbar for selected columns (scaling.hpp:184-192). */
static void cm_col(int64_t q, void *v) {
    const cm_ctx *c = (const cm_ctx *)v;
    int8_t *bc = (int8_t *)xmalloc((size_t)c->k);
    for (int64_t h = 0; h < c->k; ++h) bc[h] = c->bbar[h * c->n + c->idx[q]];
    int32_t mx = 0;
    for (int64_t i = 0; i < c->m; ++i) {
        const int8_t *a = c->abar + i * c->k;
        int32_t s = 0;
        for (int64_t h = 0; h < c->k; ++h) s += (int32_t)a[h] * (int32_t)bc[h];
        mx = s > mx ? s : mx;
    }
    c->out[q] = mx;
    free(bc);
}
int ora_cbar_col_max(const int8_t *abar, const int8_t *bbar, int64_t m, int64_t k, int64_t n, const int64_t *cols,
                     int64_t count, int32_t *out) {
    cm_ctx c = {abar, bbar, m, k, n, cols, out};
    parallel_for(count, cm_col, &c);
    return ORA_OK;
}

/* C entries (i, j) by the reference pipeline given the scaling exponents
 * mu_i, nu_j: trunc (scaling.hpp:199-225), residues (crt.hpp:32-53), the N
 * wrapped dot products and signed mod (crt.hpp:69-79), accumulate / Q /
 * final_reduce (crt.hpp:91-150), inverse_scale (emulate.hpp:30-46).
 * prec: 0 fp32 (C out as float), 1 fp64. */
typedef struct {
    int prec; const double *A, *B; int64_t k, n; const int16_t *mu, *nu; const int64_t *ri, *cj;
    const ora_table *t; void *out; volatile int err;
} en_ctx;
static void en_one(int64_t q, void *v) {
    en_ctx *c = (en_ctx *)v;
    const ora_table *t = c->t;
    const int N = t->n;
    const int64_t k = c->k, n = c->n, i = c->ri[q], j = c->cj[q];
    int8_t *ar = (int8_t *)xmalloc((size_t)k), *bc = (int8_t *)xmalloc((size_t)k);
    double c1 = 0.0, c2 = 0.0;
    for (int l = 0; l < N; ++l) {
        const int p = t->p[l];
        for (int64_t h = 0; h < k; ++h) {
            const double a = trunc(ldexp(c->A[i * k + h], c->mu[i]));
            const double b = trunc(ldexp(c->B[h * n + j], c->nu[j]));
            if (!isfinite(a) || !isfinite(b)) { c->err = ORA_RANGE; free(ar); free(bc); return; }
            ora_residue_of(a, p, &ar[h]);
            ora_residue_of(b, p, &bc[h]);
        }
        uint32_t acc = 0;
        for (int64_t h = 0; h < k; ++h) acc += (uint32_t)((int32_t)ar[h] * (int32_t)bc[h]);
        long long w = signed_mod_ll((long long)(int32_t)acc, p);
        if (2 * w == p) w = -w;
        const double wv = (double)(int8_t)w;
        c1 = fma(t->s1[l], wv, c1);
        if (t->mode == 1) c2 = fma(t->s2[l], wv, c2);
    }
    const double qv = round_nearest_even(t->P_inv * c1);
    const double t1 = fma(-qv, t->P1, c1);
    const double t2 = t1 + c2;
    const double cpp = fma(-qv, t->P2, t2);
    if (c->prec == 0) {
        const float x = ldexpf((float)cpp, -c->mu[i]);
        ((float *)c->out)[q] = ldexpf(x, -c->nu[j]);
    } else {
        const double x = ldexp(cpp, -c->mu[i]);
        ((double *)c->out)[q] = ldexp(x, -c->nu[j]);
    }
    free(ar); free(bc);
}
int ora_entries(int prec, const double *A, const double *B, int64_t k, int64_t n, const int16_t *mu,
                const int16_t *nu, const int64_t *ri, const int64_t *cj, int64_t count, const ora_table *t,
                void *out) {
    en_ctx c = {prec, A, B, k, n, mu, nu, ri, cj, t, out, 0};
    parallel_for(count, en_one, &c);
    return c.err ? c.err : ORA_OK;
}
