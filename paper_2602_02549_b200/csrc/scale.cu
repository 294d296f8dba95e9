// scale.cu — the HBM-bound stages of Algorithm 2 (scaling) and the residue
// split of Algorithm 3, one coalesced pass each over A / B.
//
//   row_scan_A   row_abs_max + row_pre_exponents + ceil_abs_scale_rows
//                (scaling.hpp:33-42, :86-96, :61-79, :111-120): mu'_i and
//                Abar = ceil(2^mu'|A|) written K-major (row-major, padded to kp)
//   col_max_B /  col_abs_max + col_pre_exponents (scaling.hpp:44-52, :98-107)
//   col_exp_B
//   exponents    scaling_exponents (scaling.hpp:159-194) from the clearance
//                maxima with the host-built step table (tables.cpp)
//   (the residue planes and Bbar^T are written by resid.cu)
#include <cfloat>
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace oz2g {

namespace {

template <class T>
__device__ __forceinline__ double ld_d(const T* p) { return (double)__ldg(p); }

__device__ __forceinline__ void flag(DevStatus* st, uint32_t bits) { atomicOr(&st->err, bits); }

__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

// ---------------------------------------------------------------------------
// A: one CTA per row (two passes; the second re-reads the row from L2).
// blockDim is 256, 512 or 1024 (launcher); the reductions handle each.  Each
// thread takes 8 consecutive elements per step (16-byte loads, one 8-byte
// store of Abar); the max runs on the fp64 pipe (fmax of |x|, non-finite
// detected by |x| <= DBL_MAX) and Abar = ceil(2^mu' |a|) too (ceil_scaled_p2),
// with the integer routine for the rows whose 2^mu' is not a normal double.
// ---------------------------------------------------------------------------
constexpr int kRowE = 8;

template <class T>
__device__ __forceinline__ void load8(const T* __restrict__ p, int64_t h0, int64_t k, bool vec, double (&x)[kRowE]) {
    if (vec && h0 + kRowE <= k) {
        if constexpr (sizeof(T) == 8) {
#pragma unroll
            for (int j = 0; j < kRowE; j += 2) {
                const double2 t = __ldg(reinterpret_cast<const double2*>(p + h0 + j));
                x[j] = t.x;
                x[j + 1] = t.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kRowE; j += 4) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(p + h0 + j));
                x[j] = t.x; x[j + 1] = t.y; x[j + 2] = t.z; x[j + 3] = t.w;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < kRowE; ++j) x[j] = h0 + j < k ? (double)__ldg(p + h0 + j) : 0.0;
    }
}

// Abar of 8 elements packed in two words; logic |= an entry above 64
__device__ __forceinline__ uint2 abar8(const double (&x)[kRowE], int sft, bool fast, double p2, bool& logic) {
    uint32_t w[2] = {0u, 0u};
#pragma unroll
    for (int j = 0; j < kRowE; ++j) {
        const int c = fast ? ceil_scaled_p2(x[j], p2) : ceil_abs_scaled(x[j], sft);
        logic |= c < 0;
        w[j >> 2] |= (uint32_t)(c & 0xff) << (8 * (j & 3));
    }
    return make_uint2(w[0], w[1]);
}

// block-wide max of the (non-negative) row maxima; thread 0 sets mu' (or the
// zero-row error) and every thread gets it back
__device__ __forceinline__ int row_mu_prime(double mxd, int32_t* __restrict__ mu_prime, DevStatus* st, int64_t i,
                                            int64_t row0) {
    unsigned long long mx = (unsigned long long)__double_as_longlong(mxd);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = t > mx ? t : mx;
    }
    __shared__ unsigned long long red[32];
    __shared__ int s_mup;
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m2 = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m2 = red[w] > m2 ? red[w] : m2;
        int mup = 0;
        if (m2 == 0) {
            flag(st, ERR_A_ZERO_ROW);
            atomicMin((unsigned long long*)&st->first_row, status_key(row0 + i, false));
        } else {
            mup = 5 - ilogb_exact(__longlong_as_double((long long)m2));
        }
        mu_prime[i] = mup;
        s_mup = mup;
    }
    __syncthreads();
    return s_mup;
}

// U: first-pass steps unrolled (loads in flight per thread); 1 at two rows per
// SM (32 registers), 4 for the long rows held to one row per SM (launcher)
template <class T, int U>
__global__ void __launch_bounds__(1024) row_scan_A_kernel(const T* __restrict__ A, int64_t lda, int64_t k,
                                                         int64_t kp, int32_t* __restrict__ mu_prime,
                                                         int8_t* __restrict__ abar, DevStatus* st,
                                                         int64_t row0) {
    pdl_enter();
    const int64_t i = blockIdx.x;  // row within this launch; row0 + i in the whole matrix
    const T* row = A + i * lda;
    const bool vec = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
    double mxd = 0.0;
    bool bad = false;
#pragma unroll U
    for (int64_t h0 = (int64_t)threadIdx.x * kRowE; h0 < k; h0 += (int64_t)blockDim.x * kRowE) {
        double x[kRowE];
        load8(row, h0, k, vec, x);
#pragma unroll
        for (int j = 0; j < kRowE; ++j) {
            bad |= !(fabs(x[j]) <= DBL_MAX);
            mxd = fmax(mxd, fabs(x[j]));
        }
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) {
            flag(st, ERR_A_NONFINITE);
            atomicMin((unsigned long long*)&st->first_row, status_key(row0 + i, true));
        }
        return;
    }
    const int sft = row_mu_prime(mxd, mu_prime, st, i, row0);
    const bool fast = pow2_normal(sft);
    const double p2 = fast ? pow2d(sft) : 0.0;
    int8_t* out = abar + i * kp;
    bool logic = false;
    // second pass (row re-read from L2); kp is a multiple of 128, columns k.. are zero
#pragma unroll (U > 1 ? 2 : 1)
    for (int64_t h0 = (int64_t)threadIdx.x * kRowE; h0 < kp; h0 += (int64_t)blockDim.x * kRowE) {
        double x[kRowE];
        load8(row, h0, k, vec, x);
        *reinterpret_cast<uint2*>(out + h0) = abar8(x, sft, fast, p2, logic);
    }
    if (logic) flag(st, ERR_CEIL_LOGIC);
}

// Single-pass variant for k <= 16 * blockDim.x (launched up to k = 8192): each
// thread keeps 16 consecutive elements of the row in registers, so the row is
// read from HBM once and the ceil pass needs no second load.
constexpr int kRowVPT = 16;

template <class T>
__global__ void __launch_bounds__(512) row_scan_A_reg_kernel(const T* __restrict__ A, int64_t lda, int64_t k,
                                                             int64_t kp, int32_t* __restrict__ mu_prime,
                                                             int8_t* __restrict__ abar, DevStatus* st,
                                                             int64_t row0) {
    pdl_enter();
    const int64_t i = blockIdx.x;
    const T* row = A + i * lda;
    const bool vec = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
    const int64_t h0 = (int64_t)threadIdx.x * kRowVPT;
    double x0[kRowE], x1[kRowE];
    load8(row, h0, k, vec, x0);
    load8(row, h0 + kRowE, k, vec, x1);
    double mxd = 0.0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kRowE; ++j) {
        bad |= !(fabs(x0[j]) <= DBL_MAX) || !(fabs(x1[j]) <= DBL_MAX);
        mxd = fmax(mxd, fmax(fabs(x0[j]), fabs(x1[j])));
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) {
            flag(st, ERR_A_NONFINITE);
            atomicMin((unsigned long long*)&st->first_row, status_key(row0 + i, true));
        }
        return;
    }
    const int sft = row_mu_prime(mxd, mu_prime, st, i, row0);
    const bool fast = pow2_normal(sft);
    const double p2 = fast ? pow2d(sft) : 0.0;
    int8_t* out = abar + i * kp;
    bool logic = false;
    // columns k .. kp are zero; a thread past kp (blockDim * 16 > kp) writes nothing
    if (h0 < kp) *reinterpret_cast<uint2*>(out + h0) = abar8(x0, sft, fast, p2, logic);
    if (h0 + kRowE < kp) *reinterpret_cast<uint2*>(out + h0 + kRowE) = abar8(x1, sft, fast, p2, logic);
    if (logic) flag(st, ERR_CEIL_LOGIC);
}

// ---------------------------------------------------------------------------
// B column maxima: 256 columns x `rows` rows per CTA, atomicMax on |x| bits
// (monotone for non-negative doubles).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) col_max_B_kernel(const T* __restrict__ B, int64_t ldb, int64_t k,
                                                        int64_t n, int rows, unsigned long long* __restrict__ bmax,
                                                        DevStatus* st) {
    pdl_enter();
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j >= n) return;
    const int64_t h0 = (int64_t)blockIdx.y * rows;
    const int64_t h1 = h0 + rows < k ? h0 + rows : k;
    unsigned long long mx = 0;
    bool bad = false;
    for (int64_t h = h0; h < h1; ++h) {
        const unsigned long long b = abs_bits(ld_d(B + h * ldb + j));
        bad |= b >= 0x7ff0000000000000ull;
        mx = b > mx ? b : mx;
    }
    // a non-finite entry leaves bits >= 0x7ff0... in bmax[j]: col_exp_B reports
    // it with the column index, so the first failing column decides the message
    (void)bad;
    if (mx) atomicMax(&bmax[j], mx);
}

__global__ void col_exp_B_kernel(const unsigned long long* __restrict__ bmax, int64_t n,
                                 int32_t* __restrict__ nu_prime, DevStatus* st, int64_t col0) {
    pdl_enter();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const unsigned long long b = bmax[j];
    if (b >= 0x7ff0000000000000ull) {  // col_abs_max: non-finite entry (scaling.hpp:43-51)
        flag(st, ERR_B_NONFINITE);
        atomicMin((unsigned long long*)&st->first_col, status_key(col0 + j, true));
        nu_prime[j] = 0;
        return;
    }
    if (b == 0) {
        flag(st, ERR_B_ZERO_COL);
        atomicMin((unsigned long long*)&st->first_col, status_key(col0 + j, false));
        nu_prime[j] = 0;
        return;
    }
    nu_prime[j] = 5 - ilogb_exact(__longlong_as_double((long long)b));
}

// ---------------------------------------------------------------------------
// scaling_exponents from the clearance maxima (scaling.hpp:159-194).
// ---------------------------------------------------------------------------
struct ThrTable {
    int shift0, nthr;
    int32_t thr[64];
};

__global__ void exponents_kernel(const int32_t* __restrict__ cmax_row, int64_t m,
                                 const int32_t* __restrict__ cmax_col, int64_t n,
                                 const int32_t* __restrict__ mu_prime, const int32_t* __restrict__ nu_prime,
                                 const ThrTable tt, int32_t* __restrict__ mu, int32_t* __restrict__ nu,
                                 float* __restrict__ e, float* __restrict__ f, DevStatus* st,
                                 const ChangeFlags cf) {
    pdl_enter();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m + n) return;
    const bool is_row = t < m;
    const int64_t idx = is_row ? t : t - m;
    const int32_t c = is_row ? cmax_row[idx] : cmax_col[idx];
    int cnt = 0;
    for (int q = 0; q < tt.nthr; ++q) cnt += c >= tt.thr[q];
    const int shift = tt.shift0 - cnt;
    // diagnostics e_i / f_j = log2f(max(1, RU32(c))) (softfp.hpp:147-159)
    float d = __int2float_ru(c);
    d = d > 1.0f ? d : 1.0f;
    const float ev = (float)log2((double)d);
    if (!(ev < 31.0f)) flag(st, ERR_E_LOGIC);
    const int base = is_row ? mu_prime[idx] : nu_prime[idx];
    const int v = base + shift;
    if (v < -32768 || v > 32767) flag(st, is_row ? ERR_MU_RANGE : ERR_NU_RANGE);
    // cf.flags: mu / nu hold exponents speculated from partial maxima; mark
    // every row / column group in which one of them moves
    if (is_row) {
        if (cf.flags && cf.row_div && mu[idx] != v) {
            cf.flags[0] = 1;
            cf.flags[1 + idx / cf.row_div] = 1;
        }
        mu[idx] = v;
        if (e) e[idx] = ev;
    } else {
        if (cf.flags && cf.col_div && nu[idx] != v) {
            cf.flags[0] = 1;
            cf.flags[1 + cf.col_slot0 + idx / cf.col_div] = 1;
        }
        nu[idx] = v;
        if (f) f[idx] = ev;
    }
}

template <class T>
__global__ void trunc_scaled_kernel(const T* __restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                    const int32_t* __restrict__ shift, int by_col, double* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * cols) return;
    const int64_t i = t / cols, j = t - i * cols;
    const double x = ld_d(X + i * ldx + j);
    const int s = by_col ? shift[j] : shift[i];
    out[t] = trunc(ldexp_rn(x, s));
}

__global__ void log2f_kernel(const float* __restrict__ x, float* __restrict__ out, int64_t count) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) out[t] = (float)log2((double)x[t]);
}

// OR the error bits and subnormal flags of src[0 .. count) into dst (the
// per-chunk / per-tile statuses of the speculated path, api.cu).
__global__ void merge_status_kernel(DevStatus* __restrict__ dst, const DevStatus* __restrict__ src, int64_t count) {
    uint32_t err = 0, sub = 0;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
        err |= src[i].err;
        sub |= src[i].subnormal;
    }
    err = __reduce_or_sync(0xffffffffu, err);
    sub = __reduce_or_sync(0xffffffffu, sub);
    if ((threadIdx.x & 31) == 0 && (err | sub)) {
        if (err) atomicOr(&dst->err, err);
        if (sub) atomicOr(&dst->subnormal, 1u);
    }
}


// ---------------------------------------------------------------------------
// Lower-bound operands for the relative error criterion of suggest_n (f1):
// Acheck_ih = floor(|a_ih| 2^(mu'_i + 1)), Bcheck_hj = floor(|b_hj| 2^(nu'_j + 1)),
// both in [0, 127] because |a| 2^mu' < 64 (scaling.hpp:86-107).  Then
//   2^-(mu'_i + nu'_j + 2) (Acheck Bcheck)_ij <= (|A||B|)_ij
//     < 2^-(mu'_i + nu'_j + 2) ((Acheck Bcheck)_ij + SA_i + SB_j + k),
// with SA / SB the row / column sums of Acheck / Bcheck.  Layouts as Abar /
// Bbar: [m][kp] and [kp][ldn], zero padded.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) floor_rows_A_kernel(const T* __restrict__ A, int64_t lda, int64_t k,
                                                           int64_t kp, const int32_t* __restrict__ mu_prime,
                                                           int8_t* __restrict__ out, int32_t* __restrict__ rsum) {
    const int64_t i = blockIdx.x;
    const int s = mu_prime[i] + 1;
    int acc = 0;
    for (int64_t h = threadIdx.x; h < kp; h += blockDim.x) {
        int v = 0;
        if (h < k) v = (int)floor(ldexp_rn(fabs((double)A[i * lda + h]), s));
        out[i * kp + h] = (int8_t)v;
        acc += v;
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(&rsum[i], acc);
}

template <class T>
__global__ void __launch_bounds__(256) floor_rows_B_kernel(const T* __restrict__ B, int64_t ldb, int64_t k,
                                                           int64_t n, int64_t kp, int64_t ldn,
                                                           const int32_t* __restrict__ nu_prime,
                                                           int8_t* __restrict__ out, int32_t* __restrict__ csum) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j >= ldn) return;
    const int64_t h0 = (int64_t)blockIdx.y * 64;
    const int s = j < n ? nu_prime[j] + 1 : 0;
    int acc = 0;
    for (int64_t h = h0; h < h0 + 64 && h < kp; ++h) {
        int v = 0;
        if (h < k && j < n) v = (int)floor(ldexp_rn(fabs((double)B[h * ldb + j]), s));
        out[h * ldn + j] = (int8_t)v;
        acc += v;
    }
    if (j < n && acc) atomicAdd(&csum[j], acc);
}


// Start of a call: clear the status word (first-failure keys to their maximum)
// and zero the maxima the scans and the clearance GEMM accumulate into.
__global__ void init_call_kernel(DevStatus* st, unsigned long long* bmax, int64_t nb, int32_t* rmax, int64_t nr,
                                 int32_t* cmax, int64_t nc) {
    pdl_enter();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) {
        st->err = 0;
        st->subnormal = 0;
        st->first_row = 0x7f7f7f7f7f7f7f7fll;
        st->first_col = 0x7f7f7f7f7f7f7f7fll;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t; i < nb; i += stride) bmax[i] = 0;
    for (int64_t i = t; i < nr; i += stride) rmax[i] = 0;
    for (int64_t i = t; i < nc; i += stride) cmax[i] = 0;
}

inline unsigned blocks_for(int64_t work, int per) { return (unsigned)((work + per - 1) / per); }

}  // namespace

cudaError_t launch_row_scan_A(int prec, const void* A, int64_t lda, int64_t m, int64_t k, int64_t kp,
                              int32_t* mu_prime, int8_t* abar, DevStatus* st, cudaStream_t s, int64_t row0) {
    if (m == 0) return cudaSuccess;
    // ~16 elements per thread, 32..512 threads per row: up to k = 8192 the row
    // stays in registers (one HBM pass, several rows per SM); longer rows use
    // two passes (the second hits L2) — measured faster at k = 16384 than one
    // 1024-thread register-resident row per SM (0.86 vs 0.90-0.98 ms at 16384^2)
    const int64_t want = (k + kRowVPT - 1) / kRowVPT;
    if (want <= 512) {
        const unsigned threads = (unsigned)(want <= 32 ? 32 : (want + 31) / 32 * 32);
        if (prec)
            return launch_pdl(row_scan_A_reg_kernel<double>, dim3((unsigned)m), dim3(threads), 0, s, (const double*)A, lda,
                              k, kp, mu_prime, abar, st, row0);
        return launch_pdl(row_scan_A_reg_kernel<float>, dim3((unsigned)m), dim3(threads), 0, s, (const float*)A, lda, k,
                          kp, mu_prime, abar, st, row0);
    } else {
        // rows over 256 KB (k = 65536 fp64): two rows per SM in flight would
        // outgrow L2 and the second pass would re-read HBM, so an unused
        // dynamic shared-memory request holds it to one row per SM (cfg5:
        // DRAM read 2.11 -> 1.11 GB per launch, 0.337 -> 0.324-0.331 ms; the
        // kernel is bound by the max -> second-pass turnaround, not by HBM)
        const size_t row_bytes = (size_t)k * (prec ? 8 : 4);
        const bool long_row = row_bytes > (256u << 10);
        cudaError_t err;
        if (long_row) {
            const size_t pin = 120u << 10;
            if (prec) {
                if ((err = cudaFuncSetAttribute(row_scan_A_kernel<double, 4>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pin)) != cudaSuccess)
                    return err;
                return launch_pdl(row_scan_A_kernel<double, 4>, dim3((unsigned)m), dim3(1024), pin, s, (const double*)A,
                                  lda, k, kp, mu_prime, abar, st, row0);
            } else {
                if ((err = cudaFuncSetAttribute(row_scan_A_kernel<float, 4>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pin)) != cudaSuccess)
                    return err;
                return launch_pdl(row_scan_A_kernel<float, 4>, dim3((unsigned)m), dim3(1024), pin, s, (const float*)A,
                                  lda, k, kp, mu_prime, abar, st, row0);
            }
        } else {
            // 512 threads (4 rows per SM in flight) up to 128 KB rows, 1024 (2
            // per SM) above, so the rows in flight stay within L2: at 16384^2
            // 0.51 vs 0.62 ms per launch (256 threads: 0.65, 4.2 GB read);
            // option "rowscan_threads" 256/512/1024 overrides (experiments)
            const int thr_env = (int)opt(OPT_ROWSCAN_THREADS);
            const unsigned thr = thr_env ? (unsigned)thr_env : row_bytes <= (128u << 10) ? 512u : 1024u;
            if (prec)
                return launch_pdl(row_scan_A_kernel<double, 1>, dim3((unsigned)m), dim3(thr), 0, s, (const double*)A,
                                  lda, k, kp, mu_prime, abar, st, row0);
            return launch_pdl(row_scan_A_kernel<float, 1>, dim3((unsigned)m), dim3(thr), 0, s, (const float*)A, lda,
                              k, kp, mu_prime, abar, st, row0);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_col_max_B(int prec, const void* B, int64_t ldb, int64_t k, int64_t n,
                             unsigned long long* bmax, DevStatus* st, cudaStream_t s) {
    if (n == 0 || k == 0) return cudaSuccess;
    // 64 rows per CTA, fewer when that leaves under ~16 CTAs per SM
    const int64_t cols = blocks_for(n, 256);
    int rows = 64;
    while (rows > 8 && cols * blocks_for(k, rows) < 16 * current_sm_count()) rows /= 2;
    dim3 grid((unsigned)cols, blocks_for(k, rows));
    if (prec) return launch_pdl(col_max_B_kernel<double>, grid, dim3(256), 0, s, (const double*)B, ldb, k, n, rows, bmax, st);
    return launch_pdl(col_max_B_kernel<float>, grid, dim3(256), 0, s, (const float*)B, ldb, k, n, rows, bmax, st);
}

cudaError_t launch_col_exp_B(const unsigned long long* bmax, int64_t n, int32_t* nu_prime, DevStatus* st,
                             cudaStream_t s, int64_t col0) {
    if (n == 0) return cudaSuccess;
    return launch_pdl(col_exp_B_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, s, bmax, n, nu_prime, st, col0);
}

cudaError_t launch_exponents(const int32_t* cmax_row, int64_t m, const int32_t* cmax_col, int64_t n,
                             const int32_t* mu_prime, const int32_t* nu_prime, int shift0, int nthr,
                             const int32_t* thr, int32_t* mu, int32_t* nu, float* e, float* f, DevStatus* st,
                             cudaStream_t s, const ChangeFlags* changed) {
    if (m + n == 0) return cudaSuccess;
    ThrTable tt;
    tt.shift0 = shift0;
    tt.nthr = nthr;
    for (int q = 0; q < 64; ++q) tt.thr[q] = q < nthr ? thr[q] : 0;
    return launch_pdl(exponents_kernel, dim3(blocks_for(m + n, 256)), dim3(256), 0, s, cmax_row, m, cmax_col, n,
                      mu_prime, nu_prime, tt, mu, nu, e, f, st, changed ? *changed : ChangeFlags{nullptr, 0, 0, 0});
}

cudaError_t launch_trunc_scaled(int prec, const void* X, int64_t ldx, int64_t rows, int64_t cols,
                                const int32_t* shift, int by_col, double* out, cudaStream_t s) {
    if (rows * cols == 0) return cudaSuccess;
    if (prec) trunc_scaled_kernel<double><<<blocks_for(rows * cols, 256), 256, 0, s>>>((const double*)X, ldx, rows, cols, shift, by_col, out);
    else trunc_scaled_kernel<float><<<blocks_for(rows * cols, 256), 256, 0, s>>>((const float*)X, ldx, rows, cols, shift, by_col, out);
    return cudaGetLastError();
}

cudaError_t launch_log2f(const float* x, float* out, int64_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    log2f_kernel<<<blocks_for(count, 256), 256, 0, s>>>(x, out, count);
    return cudaGetLastError();
}

cudaError_t launch_merge_status(DevStatus* dst, const DevStatus* src, int64_t count, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    merge_status_kernel<<<1, 256, 0, s>>>(dst, src, count);
    return cudaGetLastError();
}


cudaError_t launch_floor_operands(int prec, const void* A, int64_t lda, int64_t m, const void* B, int64_t ldb,
                                  int64_t k, int64_t n, int64_t kp, int64_t ldn, const int32_t* mu_prime,
                                  const int32_t* nu_prime, int8_t* a_out, int8_t* b_out, int32_t* rsum,
                                  int32_t* csum, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(rsum, 0, 4 * (size_t)(m > 0 ? m : 1), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(csum, 0, 4 * (size_t)(n > 0 ? n : 1), s);
    if (e != cudaSuccess) return e;
    if (m && kp) {
        if (prec) floor_rows_A_kernel<double><<<(unsigned)m, 256, 0, s>>>((const double*)A, lda, k, kp, mu_prime, a_out, rsum);
        else floor_rows_A_kernel<float><<<(unsigned)m, 256, 0, s>>>((const float*)A, lda, k, kp, mu_prime, a_out, rsum);
    }
    if (ldn && kp) {
        dim3 grid(blocks_for(ldn, 256), blocks_for(kp, 64));
        if (prec) floor_rows_B_kernel<double><<<grid, 256, 0, s>>>((const double*)B, ldb, k, n, kp, ldn, nu_prime, b_out, csum);
        else floor_rows_B_kernel<float><<<grid, 256, 0, s>>>((const float*)B, ldb, k, n, kp, ldn, nu_prime, b_out, csum);
    }
    return cudaGetLastError();
}


cudaError_t launch_init_call(DevStatus* st, unsigned long long* bmax, int64_t nb, int32_t* rmax, int64_t nr,
                             int32_t* cmax, int64_t nc, cudaStream_t s) {
    const int64_t most = nb > nr ? (nb > nc ? nb : nc) : (nr > nc ? nr : nc);
    const int64_t blocks = (most + 255) / 256;
    return launch_pdl(init_call_kernel, dim3((unsigned)(blocks < 1 ? 1 : (blocks > 1184 ? 1184 : blocks))), dim3(256), 0,
                      s, st, bmax, nb, rmax, nr, cmax, nc);
}

}  // namespace oz2g
