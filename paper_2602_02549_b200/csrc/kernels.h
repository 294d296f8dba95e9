// kernels.h — host-visible launchers of the oz2g device stages.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace oz2g {

struct DevStatus;

// Speculated exponents (api.cu run_gemm): the exponents kernel compares each
// value it writes with the one in place and marks the row / column group that
// moved: flags[0] = any, flags[1 + i / row_div] for row i (row_div > 0),
// flags[1 + col_slot0 + j / col_div] for column j (col_div > 0).
struct ChangeFlags {
    int32_t* flags;
    int64_t row_div, col_div, col_slot0;
};

enum GemmEpilogue { EPI_MAX = 0, EPI_RESID = 1, EPI_I32 = 2 };

struct GemmParams {
    int m, n;                 // valid output rows / columns
    int kblocks;              // kp / 128
    int planes;               // number of (A_l, B_l) pairs
    int tiles_m, tiles_n;
    int group_m;              // tile-rows per raster group (L2 reuse of the B operand)
    uint64_t hintA, hintB;    // TMA L2 cache policies for the A / B operand loads
    // EPI_MAX
    int32_t* rowmax;
    int32_t* colmax;
    // EPI_RESID: W[l*wplane + i*ldw + j]
    int8_t* W;
    int64_t ldw, wplane;
    // EPI_I32: C32[l*cplane + i*ldc32 + j]
    int32_t* C32;
    int64_t ldc32, cplane;
    uint32_t p[49], magic[49], off[49];
    // unit fence (experiment, OZ2G_GEMM_FENCE): a zeroed counter; before its
    // j-th unit a CTA waits until every CTA issued the loads of j units
    unsigned long long* fence;
};

int gemm_smem_bytes();
cudaError_t launch_i8_peak(long long iters, int random, int num_sms, int* sink, cudaStream_t stream, double* ops);
int gemm_tile_m();
int gemm_tile_n();
int gemm_tile_k();
cudaError_t launch_gemm_i8(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                           int num_sms, cudaStream_t stream);
// cluster of 2 CTAs, 128 x 256 tiles each, B tile multicast (tmB box: 128 rows)
cudaError_t launch_gemm_i8_mc(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                              int num_sms, cudaStream_t stream);
int gemm_pair_tile_m();
int gemm_pair_tile_n();
int gemm_pair_box_rows();
cudaError_t launch_gemm_i8_pair(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                                int num_sms, cudaStream_t stream);

// Residue constants for the residue kernels (uploaded once per table): a
// header followed by the weight table w[l][G][s] (G in [0, kResidE8), s = sign)
// of two packed words whose signed bytes are the symmetric representatives of
// (-1)^s 2^(8 (t + G)) mod p_l, t = 0..7 (resid.cu explains the arithmetic).
// Per-modulus constants of the balanced-digit path (resid.cu), one 16-byte
// load: the weights of G = 0, s = 0, RN32(1 / p) and -p (mod 2^32).
struct alignas(16) FastMod {
    int32_t w0, w1;
    float inv_p;
    uint32_t negp;
};
struct alignas(16) ResidHeader {  // size a multiple of 16: the table that follows is read as int2/uint4
    int n, pad;
    uint32_t p[49];
    float inv_p[49];  // RN32(1 / p)
    FastMod fm[49];
};
constexpr int kResidE8 = 16;  // E' / 8 <= 15: |A'| < 2^(6 + P') and P' < 171 for N <= 49
constexpr int kResidRow = kResidE8 * 2 * 8;  // bytes per modulus: [G][sign][8 bytes]
__host__ __device__ inline size_t resid_consts_bytes(int n) { return sizeof(ResidHeader) + (size_t)kResidRow * n; }
typedef ResidHeader ResidConsts;

// Stage launchers (scale.cu).  T = float or double inputs; prec selects.
cudaError_t launch_row_scan_A(int prec, const void* A, int64_t lda, int64_t m, int64_t k, int64_t kp,
                              int32_t* mu_prime, int8_t* abar, DevStatus* st, cudaStream_t s, int64_t row0);
cudaError_t launch_col_max_B(int prec, const void* B, int64_t ldb, int64_t k, int64_t n,
                             unsigned long long* bmax, DevStatus* st, cudaStream_t s);
// col0: global index of column 0 (zero-column messages of a column chunk)
cudaError_t launch_col_exp_B(const unsigned long long* bmax, int64_t n, int32_t* nu_prime, DevStatus* st,
                             cudaStream_t s, int64_t col0 = 0);
// Bbar = ceil(|B| 2^nu') in B's layout [kp][ldn] (rows k..kp and columns n..ldn zero)
cudaError_t launch_bbar_rows(int prec, const void* B, int64_t ldb, int64_t k, int64_t n, int64_t kp, int64_t ldn,
                             const int32_t* nu_prime, int8_t* bbar, DevStatus* st, cudaStream_t s,
                             int64_t cols_out = -1);
cudaError_t launch_exponents(const int32_t* cmax_row, int64_t m, const int32_t* cmax_col, int64_t n,
                             const int32_t* mu_prime, const int32_t* nu_prime, int shift0, int nthr,
                             const int32_t* thr, int32_t* mu, int32_t* nu, float* e, float* f, DevStatus* st,
                             cudaStream_t s, const ChangeFlags* changed = nullptr);
// plane_stride: bytes between residue planes (0 = m * kp); a row block of the
// planes is written by passing the block's A / mu / planes offsets.
cudaError_t launch_resid_A(int prec, const void* A, int64_t lda, int64_t m, int64_t k, int64_t kp,
                           const int32_t* mu, const ResidConsts* rc_dev, int nmod, int8_t* planes,
                           int64_t plane_stride, DevStatus* st, cudaStream_t s);
// residue planes of trunc(B 2^nu) in B's layout, [l][kp][ldn]
cudaError_t launch_resid_B_rows(int prec, const void* B, int64_t ldb, int64_t k, int64_t n, int64_t kp, int64_t ldn,
                                const int32_t* nu, const ResidConsts* rc_dev, int nmod, int8_t* planes,
                                DevStatus* st, cudaStream_t s, int64_t cols_out = -1);
cudaError_t launch_trunc_scaled(int prec, const void* X, int64_t ldx, int64_t rows, int64_t cols,
                                const int32_t* shift, int by_col, double* out, cudaStream_t s);
cudaError_t launch_log2f(const float* x, float* out, int64_t count, cudaStream_t s);
cudaError_t launch_init_call(DevStatus* st, unsigned long long* bmax, int64_t nb, int32_t* rmax, int64_t nr,
                             int32_t* cmax, int64_t nc, cudaStream_t s);
cudaError_t launch_merge_status(DevStatus* dst, const DevStatus* src, int64_t count, cudaStream_t s);

// Error-bound factors (bounds.cu): RA_i = t (|A|v)_i, PA_i = sqrt(max(1, rowmax_i)),
// ea_i = alpha_i; CB_j, PB_j, eb_j likewise for the columns of B (all rounded up).
struct BoundVecs {
    double *RA, *PA, *CB, *PB;
    int32_t *ea, *eb;
};
cudaError_t launch_bound_vectors(int prec, const void* A, int64_t lda, int64_t m, const void* B, int64_t ldb,
                                 int64_t k, int64_t n, const int32_t* cmax_row, const int32_t* cmax_col,
                                 const int32_t* mu_prime, const int32_t* nu_prime, double t_up, double* scratch,
                                 const BoundVecs& v, cudaStream_t s);
size_t bound_scratch_doubles(int64_t m, int64_t n, int64_t k);
cudaError_t launch_cheap_bound_max(const BoundVecs& v, int64_t m, int64_t n, double t_up, double kt2_up,
                                   unsigned long long* out_bits, int num_sms, cudaStream_t s);
cudaError_t launch_tight_lower_max(const BoundVecs& v, int64_t m, int64_t n, int64_t k, double t_up, double kt2_up,
                                   const int32_t* lo, const int32_t* rsum, const int32_t* csum,
                                   unsigned long long* out_bits, int num_sms, cudaStream_t s);
cudaError_t launch_ab_lower(int prec, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t m, int64_t n,
                            int64_t k, const int32_t* lo, const int32_t* mup, const int32_t* nup, const int32_t* rsum,
                            const int32_t* csum, double* out, unsigned long long* budget, unsigned long long cap,
                            cudaStream_t s);
cudaError_t launch_floor_operands(int prec, const void* A, int64_t lda, int64_t m, const void* B, int64_t ldb,
                                  int64_t k, int64_t n, int64_t kp, int64_t ldn, const int32_t* mu_prime,
                                  const int32_t* nu_prime, int8_t* a_out, int8_t* b_out, int32_t* rsum,
                                  int32_t* csum, cudaStream_t s);
cudaError_t launch_dd_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t m, int64_t n,
                           int64_t k, double* Chi, double* Clo, int64_t ldc, cudaStream_t s);
cudaError_t launch_native_gemm(int prec, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t m,
                               int64_t n, int64_t k, void* C, int64_t ldc, cudaStream_t s);

// Residue GEMMs with the CRT + inverse scaling in the epilogue (fused.cu):
// one launch over every 128 x 128 tile of C, all N planes per tile.
struct FusedParams {
    GemmParams g;                // m, n, kblocks, planes = N, tiles, group_m, hints, p / magic / off
    double s1[49], s2[49];
    double P1, P2, P_inv;
    int mode;                    // 1: fp64 table (C2 chain), 0: fp32 table
    int probe;                   // experiments (OZ2G_FUSED=2: skip the CRT epilogue); 0 normally
    unsigned long long* plane_sync;  // zeroed counter of the plane fence (fused.cu), or nullptr
    const int32_t* mu;           // [m]
    const int32_t* nu;           // [n]
    void* C;                     // T [m][ldc]
    int64_t ldc;
    DevStatus* st;
    int dbg;                     // diagnostics (option debug_sync): bounded barrier waits that report a stall
};
int fused_tile_m();
int fused_tile_n();
int fused_b_box_rows(bool mc);  // K-rows of the B TMA box (half a stage with multicast)
cudaError_t launch_gemm_crt_fused(int prec, const CUtensorMap& tmA, const CUtensorMap& tmB, const FusedParams& P,
                                  int num_sms, bool mc, cudaStream_t stream);

// CRT + inverse scaling (crt.cu).
struct CrtConsts {
    int n, mode;
    double s1[49], s2[49];
    double P1, P2, P_inv;
};
struct BoundCtx {  // evaluated in the CRT pass when `on`
    int on;
    BoundVecs v;
    double t2_up, rconst_up, ucoef, kpr_cheap_up, k_rconst_up;
    double *cheap, *tight;             // optional m x n outputs (device)
    unsigned long long* max_bits;      // [0] cheap max, [1] tight max, [2] tight / |A||B| max (bits)
    // relative criterion: (|A||B|)_ij >= ab_lo[i * n + j] (launch_ab_lower); nullptr: no relative maximum
    const double* ab_lo;
};
// Status flags per (row group, column group) of C instead of the launch's
// single status (speculated exponents, api.cu): entry (i, j) of the launch
// flags base[((row0 + i) / row_div) * slots + (col0 + j) / col_div]; col_div
// and col0 are multiples of 8 (one CRT thread's columns share an entry).
struct StatusGrid {
    DevStatus* base;  // nullptr: the launch's status
    int64_t row0, col0, row_div, col_div, slots;
};
struct CrtExtra {  // optional device outputs (nullptr = skip)
    double *C1, *C2, *Q, *Cpp64;
    float* Cpp32;
    BoundCtx bnd;
    StatusGrid sg;
};
cudaError_t launch_crt(int prec, const int8_t* W, int64_t ldw, int64_t wplane, int64_t m, int64_t n,
                       const CrtConsts& cc, const int32_t* mu, const int32_t* nu, void* C, int64_t ldc,
                       const CrtExtra& extra, DevStatus* st, cudaStream_t s);

}  // namespace oz2g
