/*
 * oz2g.h — C ABI of the B200-native Ozaki-II (accurate mode) GEMM emulation.
 *
 * This is the drop-in boundary for the reference's hot path
 *   template<class T> EmulationResult<T> oz2::os_ii(const Matrix<T>& a,
 *        const Matrix<T>& b, int n, bool keep_intermediates = false)
 *   (/root/reference/proj/include/oz2/emulate.hpp:54-88)
 * and for the constant registry it reads
 *   const ModuliTable& table_for(int n, Prec mode)   (moduli.hpp:145-153).
 * The reference has no FFI of its own; include/oz2g/emulate.hpp re-presents
 * `oz2::os_ii<T>` / `EmulationResult<T>` unchanged on top of this ABI, and
 * INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Plain pointers and sizes only.  Matrices are row-major (matrix.hpp:25-26)
 * with explicit leading dimensions.  Results are bit-identical to the
 * reference for any launch configuration (integer GEMMs are exact and the
 * fp64 accumulation order over moduli is fixed, crt.hpp:99-104).
 *
 * Status codes map 1:1 onto the reference's exception classes.
 */
#ifndef OZ2G_H
#define OZ2G_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZ2G_API_VERSION 4

/* Status codes (return value of every entry point). */
#define OZ2G_OK 0
#define OZ2G_INVALID_ARGUMENT 1 /* std::invalid_argument (matrix.hpp:47-49) */
#define OZ2G_DOMAIN_ERROR 2     /* std::domain_error (emulate.hpp:59, scaling.hpp:90/102, moduli.hpp:94) */
#define OZ2G_RANGE_ERROR 3      /* std::range_error (scaling.hpp:145/206/220, crt.hpp:144, emulate.hpp:39) */
#define OZ2G_LOGIC_ERROR 4      /* std::logic_error (scaling.hpp:67/77/179/189) */
#define OZ2G_CUDA_ERROR 5       /* device / driver failure (no reference counterpart) */

/* Precision of A, B, C (moduli.hpp:23 enum class Prec). */
#define OZ2G_FP32 0
#define OZ2G_FP64 1

/* Flags for oz2g_gemm. */
#define OZ2G_HOST_PTRS 0u    /* A, B, C are host pointers (copies are done inside) */
#define OZ2G_DEVICE_PTRS 1u  /* A, B, C are device pointers on the current device */
#define OZ2G_TIMING 2u       /* fill oz2g_diag::stage_ms with per-stage CUDA-event times */
#define OZ2G_ASYNC 4u        /* enqueue and return (see oz2g_synchronize); C only, no timing */

/* Limits (int8gemm.hpp:12, moduli.hpp:38). */
#define OZ2G_MAX_INNER_DIM (1LL << 17)
#define OZ2G_MAX_MODULI 49

/*
 * Optional intermediates (EmulationResult::scaling / ::crt, emulate.hpp:17-24,
 * scaling.hpp:20-28, crt.hpp:81-87).  Every non-NULL pointer is a HOST buffer
 * that is filled; NULL members are skipped.  Shapes (row-major, dense):
 *   mu, mu_prime, e : m        nu, nu_prime, f : n
 *   Aprime : m*k (fp64)        Bprime : k*n (fp64)
 *   Cbar : m*n (int32)         Dbar : m*n (fp32)
 *   W : N*m*n (int8)           C1, C2, Q, Cpp64 : m*n (fp64)   Cpp32 : m*n
 * Extra evidence beyond the reference's struct (for bit-parity checks of the
 * device stages):
 *   Ares : N*m*k int8 residues of A' (crt.hpp:160)
 *   Bres : N*k*n int8 residues of B' (crt.hpp:161), row-major k x n
 *   Cprod: N*m*n int32 wrapped INT8 products (crt.hpp:70)
 *   cmax_row : m, cmax_col : n int32 clearance-product maxima (scaling.hpp:175-192)
 *   bounds : when non-NULL, the deterministic error bounds of the paper
 *            (bounds.hpp:182-206) are evaluated in the same pass (below).
 */
/*
 * Error bounds on |A B - C| per entry (bounds.hpp:143-206), every operation
 * rounded upward so each value is a certificate:
 *   cheap: bound_cheap (bounds.hpp:198-206), r_b scalar;
 *   tight: bound_tight (bounds.hpp:182-195) with the exact |A'B'| replaced by
 *          the sound device bound (|C''| + r_const) / (1 - u_coef).
 * `cheap` / `tight` are optional m*n outputs (host buffers, or device buffers
 * when `device` != 0); the maxima are always returned.  With `relative` != 0
 * also max_ij tight_ij / (|A||B|)_ij, against a lower bound of (|A||B|)_ij
 * (floor(|A| 2^(mu'+1)) floor(|B| 2^(nu'+1)), one extra int8 GEMM), so it
 * is >= the exact ratio.
 */
typedef struct oz2g_bounds {
    double *cheap, *tight;
    int device;
    double cheap_max, tight_max;
    int relative;           /* in: also evaluate tight_rel_max */
    double tight_rel_max;   /* out */
} oz2g_bounds;

typedef struct oz2g_intermediates {
    int16_t *mu, *nu, *mu_prime, *nu_prime;
    float *e, *f;
    double *Aprime, *Bprime;
    int32_t *Cbar;
    float *Dbar;
    int8_t *W;
    double *C1, *C2, *Q, *Cpp64;
    float *Cpp32;
    int8_t *Ares, *Bres;
    int32_t *Cprod;
    int32_t *cmax_row, *cmax_col;
    oz2g_bounds *bounds;
} oz2g_intermediates;

/* Per-call diagnostics. */
typedef struct oz2g_diag {
    int subnormal;          /* EmulationResult::subnormal (emulate.hpp:23) */
    int kernels_launched;   /* device kernels launched by this call */
    double stage_ms[8];     /* with OZ2G_TIMING: 0 H2D, 1 scale (K1), 2 clearance GEMM, 3 exponents,
                               4 residues, 5 residue GEMMs, 6 CRT + unscale, 7 D2H (ms) */
    int speculation;        /* pipelined host-pointer calls (speculated column exponents): 0 not used,
                               1 confirmed, 2 some column tiles recomputed, 3 every stage after the
                               upload redone; C is the same in every case */
} oz2g_diag;

/*
 * Multi-GPU hook.  After the clearance product, the per-row and per-column
 * maxima of C̄ (int32, device memory, lengths m and n) must be max-reduced
 * across every rank that shares the same rows (resp. columns) of C before the
 * scaling exponents are formed.  When non-NULL, the callback is
 * invoked on the calling thread with device pointers, to be reduced IN PLACE
 * (e.g. ncclAllReduce(..., ncclInt32, ncclMax, row_comm/col_comm, stream)).
 * Return 0 on success.
 */
typedef int (*oz2g_reduce_maxima_fn)(int32_t *cmax_row, int64_t m, int32_t *cmax_col, int64_t n,
                                     void *stream, void *user);

/*
 * C = os_ii(A, B, nmod) for A (m x k) and B (k x n), row-major with leading
 * dimensions lda >= k, ldb >= n, ldc >= n; `prec` is OZ2G_FP32 (float*) or
 * OZ2G_FP64 (double*).  `stream` is a cudaStream_t (NULL = legacy default).
 * `inter`, `diag`, `reduce_fn` may be NULL.
 */
int oz2g_gemm(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B,
              int64_t ldb, void *C, int64_t ldc, int nmod, unsigned flags, void *stream,
              oz2g_intermediates *inter, oz2g_diag *diag, oz2g_reduce_maxima_fn reduce_fn, void *reduce_user);

/*
 * One emulated GEMM tiled over several devices of this process:
 * C is split into an R x Cg grid of tiles (count 1 -> 1x1, 2 -> 2x1, 4 -> 2x2,
 * 8 -> 2x4, otherwise count x 1; oz2g_grid_shape), tile t = (t / Cg, t % Cg)
 * runs on devices[t], and the clearance maxima are max-reduced across tiles
 * before the scaling exponents, so C equals the single-device result bit for
 * bit.  Host pointers only (each device uploads its own blocks); a device may
 * be listed more than once.  Errors: the one the single-device call reports.
 * Replaces os_ii<T> (emulate.hpp:54-88) for callers that own several GPUs.
 */
int oz2g_gemm_multi(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B,
                    int64_t ldb, void *C, int64_t ldc, int nmod, unsigned flags, const int *devices, int count,
                    oz2g_diag *diag);

/*
 * The same A, B emulated for several moduli counts (the N sweep of the
 * paper's experiments): the scaling scans and the clearance product do not
 * depend on N and are computed once.  C[i] (leading dimension ldc) receives
 * the result for nmods[i], bit-identical to oz2g_gemm with nmods[i].  Host or
 * device pointers (flags); no OZ2G_ASYNC / OZ2G_TIMING.
 */
int oz2g_gemm_sweep(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B,
                    int64_t ldb, void *const *C, int64_t ldc, const int *nmods, int count, unsigned flags,
                    void *stream, oz2g_diag *diag);

/* The tile grid oz2g_gemm_multi uses for `count` devices. */
int oz2g_grid_shape(int count, int *rows, int *cols);

/*
 * Optional warm-up: create the workspaces and streams of the listed devices
 * and upload the residue constants of every table (N = 2..49, fp32 and fp64),
 * the work the first call on a device would otherwise do (moduli.hpp:145-153
 * builds tables lazily the same way).
 */
int oz2g_init(const int *devices, int count);

/* Convenience wrappers mirroring os_ii<double>/os_ii<float>. */
int oz2g_dgemm(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *B, int64_t ldb,
               double *C, int64_t ldc, int nmod, unsigned flags, void *stream, oz2g_diag *diag);
int oz2g_sgemm(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, const float *B, int64_t ldb,
               float *C, int64_t ldc, int nmod, unsigned flags, void *stream, oz2g_diag *diag);

/* Message of the last failing call on this thread (exception::what()). */
const char *oz2g_last_error(void);

/*
 * table_for(n, mode) (moduli.hpp:78-91, :145-153) without the mpz members;
 * P is returned as a decimal string.  Callable without a GPU.
 */
typedef struct oz2g_table {
    int n, mode;
    int p[OZ2G_MAX_MODULI], q[OZ2G_MAX_MODULI], beta[OZ2G_MAX_MODULI];
    double s1[OZ2G_MAX_MODULI], s2[OZ2G_MAX_MODULI];
    long rho;
    double P1, P2, P_inv;
    float P_prime;
    char P_dec[160];
    /* Scaling-exponent step table (scaling.hpp:159-194 as a step function of
     * the integer clearance maximum c):  shift(c) = shift0 - #{t : c >= thr[t]}. */
    int shift0, nthr;
    int32_t thr[64];
} oz2g_table;

int oz2g_table_for(int n, int mode, oz2g_table *out);

/* fp32_safe_moduli_max() (moduli.hpp:157-170).  Callable without a GPU. */
int oz2g_fp32_safe_moduli_max(void);

/* The scaling-exponent shift for one clearance maximum c, evaluated directly
 * (fp32_round_up, log2f, fma_fp32(.., Down), floor — scaling.hpp:171-180).
 * Callable without a GPU; used to validate the step table. */
int oz2g_shift_of_cmax(int n, int64_t c);

/* Device-side log2f evaluation used for the e/f diagnostics, exposed so tests
 * can compare it exhaustively with the host libm (log2_fp32, softfp.hpp:147). */
int oz2g_device_log2f(const float *x_dev, float *out_dev, int64_t count, void *stream);

/* suggest_n (bounds.hpp:217-243): the smallest N in [2, 49] (fp32: [2, 16])
 * whose cheap-bound maximum (bounds.hpp:198-206) is <= `target` (absolute).
 * *n_out = 0 when no N achieves it; *bound_max = the cheap-bound maximum at
 * the returned N (or at the cap).  One clearance pass; A, B as in oz2g_gemm. */
int oz2g_suggest_n(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B, int64_t ldb,
                   double target, unsigned flags, void *stream, int *n_out, double *bound_max);

/* suggest_n with the tight bound (bounds.hpp:182-195; the paper's choice of N
 * for a target accuracy): the smallest N in [2, 49] (fp32: [2, 16])
 * whose device tight-bound maximum is <= `target` — absolute, or with
 * `relative` != 0 relative to (|A||B|)_ij (oz2g_bounds.tight_rel_max).  Every
 * smaller N is shown to fail: by a lower estimate of the tight bound
 * (N < excluded_below) or by its own emulation.  n = 0: not achievable. */
typedef struct oz2g_suggest {
    int n;                  /* chosen N (0: none in range meets the target) */
    int cheap_n;            /* oz2g_suggest_n's answer for the same target (absolute, cheap bound) */
    int excluded_below;     /* every N < this was excluded by the lower estimate */
    int emulations;         /* full emulations run (N = excluded_below .. n) */
    double bound_max;       /* the criterion's maximum at n (or at the last N tried) */
    double tight_max, tight_rel_max;
} oz2g_suggest;
int oz2g_suggest_n_tight(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B,
                         int64_t ldb, double target, int relative, unsigned flags, void *stream, oz2g_suggest *out);

/* Double-double reference product C = A B (hi + lo) for DEVICE fp64
 * matrices: every product exact (TwoProd), the k-term sum in double-double
 * (error <= ~k 2^-104 sum|a||b|).  Used to measure the emulation error
 * against the paper's bounds (the role of error_matrix, oracle.hpp:164-172). */
int oz2g_dd_gemm(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *B, int64_t ldb,
                 double *Chi, double *Clo, int64_t ldc, void *stream);

/* Experiment-harness pieces:
 *  oz2g_gen_matrix   the reference's synthetic stream (gen.hpp:15-31, prng.hpp),
 *                    host memory, bit-identical to the reference for a seed;
 *  oz2g_derive_seed  experiment.hpp:83-88;
 *  oz2g_native_gemm  the "native" working-precision GEMM of the error report
 *                    (experiment.hpp:55-68: sequential loop, separate RN mul
 *                    and add), DEVICE pointers. */
int oz2g_gen_matrix(int prec, int64_t rows, int64_t cols, double phi, uint64_t seed, void *out);
uint64_t oz2g_derive_seed(uint64_t seed, uint64_t trial, uint64_t role);
int oz2g_native_gemm(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B,
                     int64_t ldb, void *C, int64_t ldc, void *stream);

/* Dense INT8 tensor-core peak (the roofline denominator of the residue GEMM):
 * `launches` back-to-back launches of a kernel in which every SM issues
 * `iters` x 4 tcgen05.mma.kind::i8 128x256x32 from shared memory (no loads,
 * no epilogue), on a low-toggle operand pattern (random = 0: the clock-limited
 * peak) or pseudo-random bytes (random = 1: the power draw of real residue
 * planes).  *ms_out = device time of all launches (CUDA events), *ops_out =
 * int8 operations (2 per multiply-add) they performed. */
int oz2g_i8_peak(long long iters, int launches, int random, double *ms_out, double *ops_out);

/* Tuning options for this process (every default is
 * the measured best).  Names: "gemm" (0 single-CTA tiles, 1 CTA pair, 2
 * multicast cluster), "fused", "fused_mc", "fused_fence", "spec" (-1 by size,
 * 0, 1, 2), "graph", "pdl" (0, 1 small calls, 2), "group_m", "group_n",
 * "l2hint", "crt_overlap", "crt_cv" (4 | 8), "wblock_min_mb", "gemm_fence",
 * "epi_warps" (0 | 4 | 8), "pair_stages" (4..6), "rowscan_threads" (0 | 256 |
 * 512 | 1024), "resid_stream", "spec_tail" (1..3), "dist_pipeline",
 * "debug_sync", "resid_fast" (1 balanced-digit residue split, 0 exponent
 * buckets only).  Unset options take OZ2G_<NAME> from the environment at first
 * use.  A set applies from the next call (captured graphs are re-captured).
 * Unknown names and out-of-range values: OZ2G_INVALID_ARGUMENT.
 * oz2g_option_name(i) lists the names (NULL past the last). */
int oz2g_set_option(const char *name, long long value);
int oz2g_get_option(const char *name, long long *value);
const char *oz2g_option_name(int index);

/*
 * One emulated GEMM across P processes (one GPU each) with NCCL driven by the
 * library.  C is tiled R x C (oz2g_grid_shape), rank q = r*C + c
 * owns tile (r, c): rows [r*ceil(m/R), ...) and columns [c*ceil(n/C), ...).
 *
 *   oz2g_comm_unique_id   rank 0 creates the id (128 bytes) and shares it
 *                         (e.g. torch.distributed broadcast);
 *   oz2g_comm_init        every rank, with its CUDA device current: the world
 *                         comm plus the row / column comms (ncclCommSplit);
 *   oz2g_gemm_dist        the rank's C tile.  Device pointers.  Inputs:
 *     default (OZ2G_DIST_SHARDS): 1-D shards — A rows [q m/P, (q+1) m/P)
 *       (lda >= k) and the B columns of shard s = c*R + r, width n/P
 *       (ldb >= n/P); m, n multiples of P.  The row / column blocks are
 *       all-gathered over NVLink inside the call.
 *     OZ2G_DIST_TILES: A is the row block r (all of k), B the column block c.
 *   The clearance maxima are max-reduced (ncclAllReduce, int32, MAX) over the
 *   row / column comms between the clearance product and the scaling
 *   exponents, so every tile equals the corresponding part of the
 *   single-device C bit for bit.  Errors are the tile's own.
 * Failures of the comm functions: oz2g_comm_last_error().
 */
#define OZ2G_DIST_SHARDS 0u
#define OZ2G_DIST_TILES 8u
typedef struct oz2g_comm oz2g_comm;
typedef struct oz2g_dist_tile {
    int R, C, r, c;
    int64_t row0, rows, col0, cols;                 /* this rank's C tile */
    int64_t a_shard_row0, a_shard_rows;             /* its A shard (OZ2G_DIST_SHARDS) */
    int64_t b_shard_col0, b_shard_cols;             /* its B shard */
} oz2g_dist_tile;
int oz2g_comm_available(void);
int oz2g_comm_unique_id(unsigned char *id_out);
int oz2g_comm_init(const unsigned char *id, int nranks, int rank, oz2g_comm **out);
int oz2g_comm_grid(const oz2g_comm *comm, int *R, int *C, int *r, int *c);
int oz2g_comm_destroy(oz2g_comm *comm);
const char *oz2g_comm_last_error(void);
/* Tile and shard ranges of `rank` (host-only; callable without a GPU). */
int oz2g_dist_layout(int nranks, int rank, int64_t m, int64_t n, oz2g_dist_tile *out);
int oz2g_gemm_dist(int prec, int64_t m, int64_t n, int64_t k, const void *A, int64_t lda, const void *B,
                   int64_t ldb, void *C, int64_t ldc, int nmod, unsigned flags, void *stream, oz2g_comm *comm,
                   oz2g_diag *diag);

/* Library information (compiled arch, number of SMs used, version). */
int oz2g_version(void);

/*
 * Complete every OZ2G_ASYNC call enqueued on the current device: wait for
 * them, then report the first failure in call order (the status the blocking
 * call would have returned; later calls' C are still written).  With
 * OZ2G_ASYNC, host buffers (A, B, C) must stay valid and C must not be read
 * until this returns; the next call's uploads overlap the previous call's
 * residue GEMMs, so a stream of calls is bounded by PCIe rather than by
 * upload + compute.
 */
int oz2g_synchronize(void);

/* Release cached device workspaces of this thread's current device. */
void oz2g_release_workspace(void);

#ifdef __cplusplus
}
#endif
#endif /* OZ2G_H */
