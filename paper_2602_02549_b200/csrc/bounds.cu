// bounds.cu — the paper's deterministic error bounds evaluated on the device
// (SURVEY §8 row f1), and a double-double reference GEMM for measuring the
// actual error (row f2).
//
// Restates bounds.hpp:143-206 (eval_bound):
//   bound_ij = t (|A|v)_i 2^beta'_j + t 2^alpha'_i (v^T|B|)_j
//              + kpR_ij t^2 2^(alpha'_i + beta'_j)
// with 2^alpha'_i = 2^alpha_i sqrt(max(1, rowmax_i Cbar)), alpha_i =
// ilogb(max_h |a_ih|) = 5 - mu'_i (same for beta / nu'), t = 1/sqrt(2^5 (P-1)).
//   cheap: kpR = k + r_const + u_coef P/2                   (bounds.hpp:198-206)
//   tight: kpR = k + r_const + u_coef |A'B'|_ij              (bounds.hpp:182-195)
// The reference evaluates in 128-bit MPFR with upward rounding; here every
// operation is an fp64 upward rounding (_ru intrinsics), so each reported
// value is >= the exact formula (a certificate) and within a few ulps of it.
// For the tight form the exact |A'B'| is replaced by the sound device bound
// |A'B'| <= (|C''| + r_const) / (1 - u_coef), from |A'B' - C''| <= R_b
// (the property test_crt.cpp:158-164 checks), so it is >= the reference's.
#include "device_common.cuh"
#include "kernels.h"

namespace oz2g {

namespace {

template <class T>
__device__ __forceinline__ double ld_d(const T* p) { return (double)__ldg(p); }

// Sum of |a_ih| over a row, rounded upward (any order of RU additions gives
// an upper bound of the exact sum).
template <class T>
__global__ void __launch_bounds__(256) abs_sum_rows_kernel(const T* __restrict__ A, int64_t lda, int64_t k,
                                                           double* __restrict__ rs) {
    const T* row = A + (int64_t)blockIdx.x * lda;
    double s = 0.0;
#pragma unroll 4
    for (int64_t h = threadIdx.x; h < k; h += blockDim.x) s = __dadd_ru(s, fabs(ld_d(row + h)));
#pragma unroll
    for (int o = 16; o; o >>= 1) s = __dadd_ru(s, __shfl_xor_sync(0xffffffffu, s, o));
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = __dadd_ru(t, red[w]);
        rs[blockIdx.x] = t;
    }
}

// Column sums of |b_hj|: partial sums over 256-row chunks, then a final pass.
template <class T>
__global__ void __launch_bounds__(256) abs_sum_cols_part_kernel(const T* __restrict__ B, int64_t ldb, int64_t k,
                                                                int64_t n, double* __restrict__ part) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j >= n) return;
    const int64_t h0 = (int64_t)blockIdx.y * 256;
    const int64_t h1 = h0 + 256 < k ? h0 + 256 : k;
    double s = 0.0;
#pragma unroll 4
    for (int64_t h = h0; h < h1; ++h) s = __dadd_ru(s, fabs(ld_d(B + h * ldb + j)));
    part[(int64_t)blockIdx.y * n + j] = s;
}

__global__ void abs_sum_cols_final_kernel(const double* __restrict__ part, int64_t chunks, int64_t n,
                                          double* __restrict__ cs) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t c = 0; c < chunks; ++c) s = __dadd_ru(s, part[c * n + j]);
    cs[j] = s;
}

// Per-row / per-column factors of the bound (bounds.hpp:115-125).
__global__ void bound_vectors_kernel(const double* __restrict__ rs, const int32_t* __restrict__ cmax_row,
                                     const int32_t* __restrict__ mu_prime, int64_t m, const double* __restrict__ cs,
                                     const int32_t* __restrict__ cmax_col, const int32_t* __restrict__ nu_prime,
                                     int64_t n, double t_up, BoundVecs v) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) {
        v.RA[t] = __dmul_ru(t_up, rs[t]);
        v.PA[t] = __dsqrt_ru((double)max(1, cmax_row[t]));
        v.ea[t] = 5 - mu_prime[t];
    } else if (t < m + n) {
        const int64_t j = t - m;
        v.CB[j] = __dmul_ru(t_up, cs[j]);
        v.PB[j] = __dsqrt_ru((double)max(1, cmax_col[j]));
        v.eb[j] = 5 - nu_prime[j];
    }
}

// ---------------------------------------------------------------------------
// Double-double reference GEMM (device pointers, fp64 inputs): C = A B with
// every product exact (TwoProd by FMA) and the k-term sum carried in
// double-double (Dekker/Knuth TwoSum), error <= ~k 2^-104 sum |a||b|.
// 64 x 64 output tile per 256-thread block, 4 x 4 outputs per thread.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dd_add(double& hi, double& lo, double p, double e) {
    const double s = __dadd_rn(hi, p);
    const double bb = __dadd_rn(s, -hi);
    const double err = __dadd_rn(__dadd_rn(hi, -__dadd_rn(s, -bb)), __dadd_rn(p, -bb));
    const double t = __dadd_rn(__dadd_rn(lo, e), err);
    hi = __dadd_rn(s, t);
    lo = __dadd_rn(t, -__dadd_rn(hi, -s));
}

__global__ void __launch_bounds__(256) dd_gemm_kernel(const double* __restrict__ A, int64_t lda,
                                                      const double* __restrict__ B, int64_t ldb, int64_t m,
                                                      int64_t n, int64_t k, double* __restrict__ Chi,
                                                      double* __restrict__ Clo, int64_t ldc) {
    __shared__ double sA[16][64 + 1];
    __shared__ double sB[16][64 + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.y * 64, j0 = (int64_t)blockIdx.x * 64;
    double hi[4][4], lo[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) hi[a][b] = lo[a][b] = 0.0;
    for (int64_t h0 = 0; h0 < k; h0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int r = e >> 4, c = e & 15;       // A tile: 64 rows x 16 cols
            const int64_t gi = i0 + r, gh = h0 + c;
            sA[c][r] = (gi < m && gh < k) ? A[gi * lda + gh] : 0.0;
            const int rb = e >> 6, cb = e & 63;     // B tile: 16 rows x 64 cols
            const int64_t gh2 = h0 + rb, gj = j0 + cb;
            sB[rb][cb] = (gh2 < k && gj < n) ? B[gh2 * ldb + gj] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int c = 0; c < 16; ++c) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = sA[c][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = sB[c][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const double p = __dmul_rn(av[a], bv[b]);
                    const double e = __fma_rn(av[a], bv[b], -p);
                    dd_add(hi[a][b], lo[a][b], p, e);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gi = i0 + ty + 16 * a, gj = j0 + tx + 16 * b;
            if (gi < m && gj < n) {
                Chi[gi * ldc + gj] = hi[a][b];
                Clo[gi * ldc + gj] = lo[a][b];
            }
        }
}

// max_ij of the cheap bound for one N (bounds.hpp:198-206), every operation
// rounded up; used by suggest_n (bounds.hpp:217-243).
__global__ void __launch_bounds__(256) cheap_bound_max_kernel(BoundVecs v, int64_t m, int64_t n, double t_up,
                                                              double kt2_up, unsigned long long* out_bits) {
    unsigned long long best = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        // RA/CB hold t_ref*(|A|v), t_ref*(v^T|B|) for t_ref = 1; scale by this N's t
        const double b1 = ldexp_ru(__dmul_ru(__dmul_ru(t_up, v.RA[i]), v.PB[j]), v.eb[j]);
        const double b2 = ldexp_ru(__dmul_ru(__dmul_ru(t_up, v.CB[j]), v.PA[i]), v.ea[i]);
        const double b3 = ldexp_ru(__dmul_ru(kt2_up, __dmul_ru(v.PA[i], v.PB[j])), v.ea[i] + v.eb[j]);
        const double bnd = __dadd_ru(__dadd_ru(b1, b2), b3);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(bnd);
        best = bits > best ? bits : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
        best = t > best ? t : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, best);
}


// Pruning for the tight-bound search of suggest_n (api.cu run_suggest_tight):
// max_ij of a LOWER estimate of the tight bound for one N — the tight formula
// (bounds.hpp:182-195) without its u_coef |A'B'| term (>= 0), evaluated with
// upward roundings and then scaled by (1 - 2^-30), which is below the exact
// formula because the upward roundings overshoot by < 2^-34 relative — divided
// (rounded down) by an UPPER bound of (|A||B|)_ij when `lo` is set (relative
// criterion), see launch_floor_operands.  A maximum above the target proves
// that N cannot meet it.
__global__ void __launch_bounds__(256) tight_lower_max_kernel(BoundVecs v, int64_t m, int64_t n, int64_t k,
                                                              double t_up, double kt2_up, const int32_t* lo,
                                                              const int32_t* rsum, const int32_t* csum,
                                                              unsigned long long* out_bits) {
    unsigned long long best = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        const double b1 = ldexp_ru(__dmul_ru(__dmul_ru(t_up, v.RA[i]), v.PB[j]), v.eb[j]);
        const double b2 = ldexp_ru(__dmul_ru(__dmul_ru(t_up, v.CB[j]), v.PA[i]), v.ea[i]);
        const double b3 = ldexp_ru(__dmul_ru(kt2_up, __dmul_ru(v.PA[i], v.PB[j])), v.ea[i] + v.eb[j]);
        double r = __dmul_rd(__dadd_ru(__dadd_ru(b1, b2), b3), 1.0 - 0x1p-30);
        if (lo) {
            const long long hi = (long long)lo[e] + rsum[i] + csum[j] + k;  // exact, < 2^33
            const double up = ldexp_ru(__ll2double_ru(hi), v.ea[i] + v.eb[j] - 12);
            r = up > 0.0 ? __ddiv_rd(r, up) : 0.0;
        }
        const unsigned long long bits = (unsigned long long)__double_as_longlong(r);
        best = bits > best ? bits : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
        best = t > best ? t : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, best);
}


// Lower bound of (|A||B|)_ij for the relative criterion, m x n fp64:
// lo_ij 2^-(mu'_i + nu'_j + 2) from the floor-operand product, or — where
// that is loose (its upper counterpart exceeds it by more than 1/16, e.g.
// entries whose large terms do not meet: wide exponent spreads) — the dot
// product sum_h |a_ih||b_hj| with every operation rounded down (each term is
// exact for fp32 inputs, and rounding down keeps a lower bound), within a
// global budget of refined multiply-adds (the rest keep the floor bound).
template <class T>
__global__ void __launch_bounds__(256) ab_lower_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                                       int64_t ldb, int64_t m, int64_t n, int64_t k,
                                                       const int32_t* __restrict__ lo, const int32_t* __restrict__ mup,
                                                       const int32_t* __restrict__ nup,
                                                       const int32_t* __restrict__ rsum,
                                                       const int32_t* __restrict__ csum, double* __restrict__ out,
                                                       unsigned long long* budget, unsigned long long cap) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e / n, j = e - i * n;
    const long long l = lo[e];
    const long long slack = (long long)rsum[i] + csum[j] + k;
    const int sc = -(mup[i] + nup[j] + 2);
    double v = l > 0 ? ldexp_rd(__ll2double_rd(l), sc) : 0.0;
    if (16 * slack > l && atomicAdd(budget, (unsigned long long)k) + (unsigned long long)k <= cap) {
        double acc = 0.0;
        for (int64_t h = 0; h < k; ++h)
            acc = __fma_rd(fabs((double)A[i * lda + h]), fabs((double)B[h * ldb + j]), acc);
        v = acc > v ? acc : v;
    }
    out[e] = v;
}

// The experiment harness's "native" GEMM (experiment.hpp:55-68): per entry a
// sequential loop h = 0..k-1 with a separate RN multiply and RN add in the
// working precision T (no FMA), exactly the reference's err_native reference.
template <class T>
__global__ void native_gemm_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ B, int64_t ldb,
                                   int64_t m, int64_t n, int64_t k, T* __restrict__ C, int64_t ldc) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m * n) return;
    const int64_t i = t / n, j = t - i * n;
    T acc = 0;
    for (int64_t h = 0; h < k; ++h) {
        if constexpr (sizeof(T) == 8) acc = __dadd_rn(acc, __dmul_rn(A[i * lda + h], B[h * ldb + j]));
        else acc = __fadd_rn(acc, __fmul_rn(A[i * lda + h], B[h * ldb + j]));
    }
    C[i * ldc + j] = acc;
}

inline unsigned blocks_for(int64_t work, int per) { return (unsigned)((work + per - 1) / per); }

}  // namespace

cudaError_t launch_native_gemm(int prec, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t m,
                               int64_t n, int64_t k, void* C, int64_t ldc, cudaStream_t s) {
    if (m * n == 0) return cudaSuccess;
    if (prec)
        native_gemm_kernel<double><<<blocks_for(m * n, 128), 128, 0, s>>>((const double*)A, lda, (const double*)B, ldb,
                                                                         m, n, k, (double*)C, ldc);
    else
        native_gemm_kernel<float><<<blocks_for(m * n, 128), 128, 0, s>>>((const float*)A, lda, (const float*)B, ldb, m,
                                                                        n, k, (float*)C, ldc);
    return cudaGetLastError();
}

cudaError_t launch_cheap_bound_max(const BoundVecs& v, int64_t m, int64_t n, double t_up, double kt2_up,
                                   unsigned long long* out_bits, int num_sms, cudaStream_t s) {
    if (m * n == 0) return cudaSuccess;
    const int64_t want = (m * n + 255) / 256;
    const unsigned grid = (unsigned)(want < (int64_t)num_sms * 8 ? want : (int64_t)num_sms * 8);
    cheap_bound_max_kernel<<<grid, 256, 0, s>>>(v, m, n, t_up, kt2_up, out_bits);
    return cudaGetLastError();
}

cudaError_t launch_bound_vectors(int prec, const void* A, int64_t lda, int64_t m, const void* B, int64_t ldb,
                                 int64_t k, int64_t n, const int32_t* cmax_row, const int32_t* cmax_col,
                                 const int32_t* mu_prime, const int32_t* nu_prime, double t_up, double* scratch,
                                 const BoundVecs& v, cudaStream_t s) {
    // scratch: rs[m] | cs[n] | part[ceil(k/256) * n]
    double* rs = scratch;
    double* cs = scratch + m;
    double* part = cs + n;
    const int64_t chunks = (k + 255) / 256;
    if (m) {
        if (prec) abs_sum_rows_kernel<double><<<(unsigned)m, 256, 0, s>>>((const double*)A, lda, k, rs);
        else abs_sum_rows_kernel<float><<<(unsigned)m, 256, 0, s>>>((const float*)A, lda, k, rs);
    }
    if (n) {
        dim3 grid(blocks_for(n, 256), (unsigned)chunks);
        if (prec) abs_sum_cols_part_kernel<double><<<grid, 256, 0, s>>>((const double*)B, ldb, k, n, part);
        else abs_sum_cols_part_kernel<float><<<grid, 256, 0, s>>>((const float*)B, ldb, k, n, part);
        abs_sum_cols_final_kernel<<<blocks_for(n, 256), 256, 0, s>>>(part, chunks, n, cs);
    }
    if (m + n) bound_vectors_kernel<<<blocks_for(m + n, 256), 256, 0, s>>>(rs, cmax_row, mu_prime, m, cs, cmax_col,
                                                                           nu_prime, n, t_up, v);
    return cudaGetLastError();
}

size_t bound_scratch_doubles(int64_t m, int64_t n, int64_t k) { return (size_t)(m + n + ((k + 255) / 256) * n); }

cudaError_t launch_dd_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t m, int64_t n,
                           int64_t k, double* Chi, double* Clo, int64_t ldc, cudaStream_t s) {
    if (m * n == 0) return cudaSuccess;
    dim3 grid(blocks_for(n, 64), blocks_for(m, 64));
    dd_gemm_kernel<<<grid, 256, 0, s>>>(A, lda, B, ldb, m, n, k, Chi, Clo, ldc);
    return cudaGetLastError();
}


cudaError_t launch_tight_lower_max(const BoundVecs& v, int64_t m, int64_t n, int64_t k, double t_up, double kt2_up,
                                   const int32_t* lo, const int32_t* rsum, const int32_t* csum,
                                   unsigned long long* out_bits, int num_sms, cudaStream_t s) {
    if (m * n == 0) return cudaSuccess;
    const int64_t want = (m * n + 255) / 256;
    const unsigned grid = (unsigned)(want < (int64_t)num_sms * 8 ? want : (int64_t)num_sms * 8);
    tight_lower_max_kernel<<<grid, 256, 0, s>>>(v, m, n, k, t_up, kt2_up, lo, rsum, csum, out_bits);
    return cudaGetLastError();
}


cudaError_t launch_ab_lower(int prec, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t m, int64_t n,
                            int64_t k, const int32_t* lo, const int32_t* mup, const int32_t* nup, const int32_t* rsum,
                            const int32_t* csum, double* out, unsigned long long* budget, unsigned long long cap,
                            cudaStream_t s) {
    if (m * n == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(budget, 0, 8, s);
    if (e != cudaSuccess) return e;
    if (prec)
        ab_lower_kernel<double><<<blocks_for(m * n, 256), 256, 0, s>>>((const double*)A, lda, (const double*)B, ldb, m,
                                                                      n, k, lo, mup, nup, rsum, csum, out, budget, cap);
    else
        ab_lower_kernel<float><<<blocks_for(m * n, 256), 256, 0, s>>>((const float*)A, lda, (const float*)B, ldb, m, n,
                                                                     k, lo, mup, nup, rsum, csum, out, budget, cap);
    return cudaGetLastError();
}

}  // namespace oz2g
