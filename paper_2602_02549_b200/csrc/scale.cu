// scale.cu — the HBM-bound stages of Algorithm 2 (scaling) and the residue
// split of Algorithm 3, one coalesced pass each over A / B.
//
//   row_scan_A   row_abs_max + row_pre_exponents + ceil_abs_scale_rows
//                (scaling.hpp:33-42, :86-96, :61-79, :111-120): mu'_i and
//                Abar = ceil(2^mu'|A|) written K-major (row-major, padded to kp)
//   col_max_B /  col_abs_max + col_pre_exponents (scaling.hpp:44-52, :98-107)
//   col_exp_B
//   bbar_T       ceil_abs_scale_cols (scaling.hpp:122-131), written transposed
//                (K-major Bbar^T [n][kp]) through shared memory
//   exponents    scaling_exponents (scaling.hpp:159-194) from the clearance
//                maxima with the host-built step table (tables.cpp)
//   resid_A /    truncate_scaled_rows/cols (scaling.hpp:199-225) fused with
//   resid_BT     residue_matrix (crt.hpp:20-65): A' = trunc(2^mu A) is never
//                materialised; every element is decomposed once and all N
//                int8 residue planes are emitted in the same pass.
#include <cfloat>

#include "device_common.cuh"
#include "kernels.h"

namespace oz2g {

namespace {

template <class T>
__device__ __forceinline__ double ld_d(const T* p) { return (double)__ldg(p); }

// ceil(2^sft |a|) exactly (scaling.hpp:61-79); returns -1 on the logic_error paths.
__device__ __forceinline__ int ceil_abs_scaled(double a, int sft) {
    if (a == 0.0) return 0;
    uint64_t mant; int e2;
    decompose(a, mant, e2);
    const int exp2 = e2 + sft;  // == e - 53 + sft with frexp's e = e2 + 53
    if (exp2 >= 0) return -1;
    const int s = -exp2;
    uint64_t v;
    if (s >= 53) {
        v = 1;
    } else {
        const uint64_t q = mant >> s;
        const uint64_t rem = mant & ((1ull << s) - 1);
        v = q + (rem != 0 ? 1 : 0);
    }
    return v > 64 ? -1 : (int)v;
}

__device__ __forceinline__ void flag(DevStatus* st, uint32_t bits) { atomicOr(&st->err, bits); }

__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

// ---------------------------------------------------------------------------
// A: one CTA per row (two passes; the second re-reads the row from L2).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) row_scan_A_kernel(const T* __restrict__ A, int64_t lda, int64_t k,
                                                         int64_t kp, int32_t* __restrict__ mu_prime,
                                                         int8_t* __restrict__ abar, DevStatus* st) {
    const int64_t i = blockIdx.x;
    const T* row = A + i * lda;
    unsigned long long mx = 0;
    bool bad = false;
    for (int64_t h = threadIdx.x; h < k; h += blockDim.x) {
        const double v = ld_d(row + h);
        const unsigned long long b = abs_bits(v);
        bad |= b >= 0x7ff0000000000000ull;
        mx = b > mx ? b : mx;
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) { flag(st, ERR_A_NONFINITE); atomicMin((unsigned long long*)&st->first_row, i); }
        return;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = t > mx ? t : mx;
    }
    __shared__ unsigned long long red[8];
    __shared__ int s_mup;
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m2 = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m2 = red[w] > m2 ? red[w] : m2;
        int mup = 0;
        if (m2 == 0) {
            flag(st, ERR_A_ZERO_ROW);
            atomicMin((unsigned long long*)&st->first_row, i);
        } else {
            mup = 5 - ilogb_exact(__longlong_as_double((long long)m2));
        }
        mu_prime[i] = mup;
        s_mup = mup;
    }
    __syncthreads();
    const int sft = s_mup;
    int8_t* out = abar + i * kp;
    bool logic = false;
    // 16 consecutive bytes per thread, one 16-byte store
    for (int64_t h0 = (int64_t)threadIdx.x * 16; h0 < kp; h0 += (int64_t)blockDim.x * 16) {
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int64_t h = h0 + j;
            int v = 0;
            if (h < k) v = ceil_abs_scaled(ld_d(row + h), sft);
            logic |= v < 0;
            w[j >> 2] |= (uint32_t)(v & 0xff) << (8 * (j & 3));
        }
        *reinterpret_cast<uint4*>(out + h0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (logic) flag(st, ERR_CEIL_LOGIC);
}

// ---------------------------------------------------------------------------
// B column maxima: 256 columns x 64 rows per CTA, atomicMax on |x| bits
// (monotone for non-negative doubles).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) col_max_B_kernel(const T* __restrict__ B, int64_t ldb, int64_t k,
                                                        int64_t n, unsigned long long* __restrict__ bmax,
                                                        DevStatus* st) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j >= n) return;
    const int64_t h0 = (int64_t)blockIdx.y * 64;
    const int64_t h1 = h0 + 64 < k ? h0 + 64 : k;
    unsigned long long mx = 0;
    bool bad = false;
    for (int64_t h = h0; h < h1; ++h) {
        const unsigned long long b = abs_bits(ld_d(B + h * ldb + j));
        bad |= b >= 0x7ff0000000000000ull;
        mx = b > mx ? b : mx;
    }
    if (bad) { flag(st, ERR_B_NONFINITE); return; }
    if (mx) atomicMax(&bmax[j], mx);
}

__global__ void col_exp_B_kernel(const unsigned long long* __restrict__ bmax, int64_t n,
                                 int32_t* __restrict__ nu_prime, DevStatus* st) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const unsigned long long b = bmax[j];
    if (b == 0) {
        flag(st, ERR_B_ZERO_COL);
        atomicMin((unsigned long long*)&st->first_col, j);
        nu_prime[j] = 0;
        return;
    }
    nu_prime[j] = 5 - ilogb_exact(__longlong_as_double((long long)b));
}

// ---------------------------------------------------------------------------
// Residues of A' = trunc(2^shift x) for one element, all moduli.
// ---------------------------------------------------------------------------
struct ElemDec {
    uint64_t mant;  // 53-bit significand (0 for x == 0)
    int E;          // |A'| = floor(mant * 2^E)
    bool neg;
};

__device__ __forceinline__ ElemDec elem_dec(double x, int shift, bool& overflow) {
    ElemDec d{0, 0, false};
    if (x == 0.0) return d;
    int e2;
    decompose(x, d.mant, e2);
    d.E = e2 + shift;
    d.neg = x < 0.0;
    // ldexp(x, shift) overflows iff |x| 2^shift >= 2^1024 (scaling.hpp:206/220)
    overflow |= d.E + 53 > 1024;
    return d;
}

// signed residue in the reference's representative range (crt.hpp:48-52)
__device__ __forceinline__ uint32_t resid_byte(const ElemDec& d, int l, const ResidConsts& rc) {
    if (d.mant == 0) return 0;
    const uint32_t p = rc.p[l];
    uint32_t r;
    if (p == 256u) {
        if (d.E >= 0) r = d.E >= 8 ? 0u : (uint32_t)((d.mant << d.E) & 0xffu);
        else r = (-d.E >= 64) ? 0u : (uint32_t)((d.mant >> (-d.E)) & 0xffu);
        if (d.neg) r = (256u - r) & 0xffu;
        return r;  // int8 wrap of [0,255]: 128 -> -128 as the reference stores it
    }
    const ModP mp{p, rc.magic[l]};
    uint64_t X = d.mant;
    if (d.E < 0) X = (-d.E >= 64) ? 0ull : (X >> (-d.E));
    const uint32_t hi = (uint32_t)(X >> 32), lo = (uint32_t)X;
    r = mod_u32(hi * rc.c32[l] + mod_u32(lo, mp), mp);
    if (d.E > 0) r = mod_u32(r * (uint32_t)rc.pow2[l][d.E < 255 ? d.E : 255], mp);
    if (d.neg && r) r = p - r;
    const int32_t s = (2u * r > p) ? (int32_t)r - (int32_t)p : (int32_t)r;
    return (uint32_t)s & 0xffu;
}

template <class T>
__global__ void __launch_bounds__(256) resid_A_kernel(const T* __restrict__ A, int64_t lda, int64_t m,
                                                      int64_t k, int64_t kp, const int32_t* __restrict__ mu,
                                                      const ResidConsts* __restrict__ rc_g, int nmod,
                                                      int8_t* __restrict__ planes, DevStatus* st) {
    extern __shared__ uint8_t sh[];
    ResidConsts& rc = *reinterpret_cast<ResidConsts*>(sh);
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(rc_g);
        uint32_t* dst = reinterpret_cast<uint32_t*>(sh);
        for (int t = threadIdx.x; t < (int)(sizeof(ResidConsts) / 4); t += blockDim.x) dst[t] = src[t];
    }
    __syncthreads();
    const int64_t chunks = kp / 16;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= m * chunks) return;
    const int64_t i = gid / chunks;
    const int64_t h0 = (gid - i * chunks) * 16;
    const int sft = mu[i];
    const T* row = A + i * lda;
    ElemDec d[16];
    bool ovf = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int64_t h = h0 + j;
        const double x = h < k ? ld_d(row + h) : 0.0;
        d[j] = elem_dec(x, sft, ovf);
    }
    if (ovf) flag(st, ERR_TRUNC_A_RANGE);
    const int64_t plane = m * kp;
    int8_t* out = planes + i * kp + h0;
    for (int l = 0; l < nmod; ++l) {
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j >> 2] |= resid_byte(d[j], l, rc) << (8 * (j & 3));
        *reinterpret_cast<uint4*>(out + (int64_t)l * plane) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---------------------------------------------------------------------------
// B transposed writers: tile 64 (h) x 64 (j), output [plane][j][kp].
//   OP 0: Bbar^T = ceil(|B| 2^nu')   OP 1: residue planes of trunc(B 2^nu)
// ---------------------------------------------------------------------------
constexpr int TB = 64;
constexpr int TROW = TB + 16;  // padded smem row (bytes) to spread banks

template <class T, int OP>
__global__ void __launch_bounds__(256) transpose_B_kernel(const T* __restrict__ B, int64_t ldb, int64_t k,
                                                          int64_t n, int64_t kp, const int32_t* __restrict__ shift,
                                                          const ResidConsts* __restrict__ rc_g, int nmod,
                                                          int8_t* __restrict__ out, DevStatus* st) {
    extern __shared__ uint8_t sh[];
    constexpr int CH = 8;  // moduli per smem round
    uint8_t* tile = sh;    // [CH][TB][TROW]
    ResidConsts* rcp = reinterpret_cast<ResidConsts*>(sh + CH * TB * TROW);
    if (OP == 1) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(rc_g);
        uint32_t* dst = reinterpret_cast<uint32_t*>(rcp);
        for (int t = threadIdx.x; t < (int)(sizeof(ResidConsts) / 4); t += blockDim.x) dst[t] = src[t];
    }
    const int tx = threadIdx.x & 63;  // column within tile
    const int ty = threadIdx.x >> 6;  // 4 groups of 16 rows
    const int64_t j = (int64_t)blockIdx.x * TB + tx;
    const int64_t hbase = (int64_t)blockIdx.y * TB + ty * 16;
    const bool jok = j < n;
    const int sft = jok ? shift[j] : 0;
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int64_t h = hbase + r;
        x[r] = (jok && h < k) ? ld_d(B + h * ldb + j) : 0.0;
    }
    __syncthreads();
    const int nplanes = OP == 0 ? 1 : nmod;
    const int64_t plane = n * kp;
    ElemDec d[16];
    bool flagbit = false;
    if (OP == 1) {
#pragma unroll
        for (int r = 0; r < 16; ++r) d[r] = elem_dec(x[r], sft, flagbit);
    }
    for (int l0 = 0; l0 < nplanes; l0 += CH) {
        const int lc = nplanes - l0 < CH ? nplanes - l0 : CH;
        for (int c = 0; c < lc; ++c) {
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                uint32_t b;
                if (OP == 0) {
                    const int v = ceil_abs_scaled(x[r], sft);
                    flagbit |= v < 0;
                    b = (uint32_t)(v & 0xff);
                } else {
                    b = resid_byte(d[r], l0 + c, *rcp);
                }
                w[r >> 2] |= b << (8 * (r & 3));
            }
            *reinterpret_cast<uint4*>(tile + (c * TB + tx) * TROW + ty * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        __syncthreads();
        // write out: per (c, row jj) 64 contiguous bytes = 4 x 16 B
        for (int idx = threadIdx.x; idx < lc * TB * 4; idx += blockDim.x) {
            const int q = idx & 3;
            const int jj = (idx >> 2) % TB;
            const int c = (idx >> 2) / TB;
            const int64_t jg = (int64_t)blockIdx.x * TB + jj;
            if (jg >= n) continue;
            const int64_t hg = (int64_t)blockIdx.y * TB + q * 16;
            const uint4 val = *reinterpret_cast<const uint4*>(tile + (c * TB + jj) * TROW + q * 16);
            *reinterpret_cast<uint4*>(out + (int64_t)(l0 + c) * plane + jg * kp + hg) = val;
        }
        __syncthreads();
    }
    if (flagbit) flag(st, OP == 0 ? ERR_CEIL_LOGIC : ERR_TRUNC_B_RANGE);
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
                                 float* __restrict__ e, float* __restrict__ f, DevStatus* st) {
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
    if (is_row) { mu[idx] = v; if (e) e[idx] = ev; }
    else { nu[idx] = v; if (f) f[idx] = ev; }
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

inline unsigned blocks_for(int64_t work, int per) { return (unsigned)((work + per - 1) / per); }

}  // namespace

cudaError_t launch_row_scan_A(int prec, const void* A, int64_t lda, int64_t m, int64_t k, int64_t kp,
                              int32_t* mu_prime, int8_t* abar, DevStatus* st, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    if (prec) row_scan_A_kernel<double><<<(unsigned)m, 256, 0, s>>>((const double*)A, lda, k, kp, mu_prime, abar, st);
    else row_scan_A_kernel<float><<<(unsigned)m, 256, 0, s>>>((const float*)A, lda, k, kp, mu_prime, abar, st);
    return cudaGetLastError();
}

cudaError_t launch_col_max_B(int prec, const void* B, int64_t ldb, int64_t k, int64_t n,
                             unsigned long long* bmax, DevStatus* st, cudaStream_t s) {
    if (n == 0 || k == 0) return cudaSuccess;
    dim3 grid(blocks_for(n, 256), blocks_for(k, 64));
    if (prec) col_max_B_kernel<double><<<grid, 256, 0, s>>>((const double*)B, ldb, k, n, bmax, st);
    else col_max_B_kernel<float><<<grid, 256, 0, s>>>((const float*)B, ldb, k, n, bmax, st);
    return cudaGetLastError();
}

cudaError_t launch_col_exp_B(const unsigned long long* bmax, int64_t n, int32_t* nu_prime, DevStatus* st,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    col_exp_B_kernel<<<blocks_for(n, 256), 256, 0, s>>>(bmax, n, nu_prime, st);
    return cudaGetLastError();
}

static size_t transpose_smem(int op) {
    return (size_t)8 * TB * TROW + (op == 1 ? sizeof(ResidConsts) : 0);
}

cudaError_t launch_bbar_T(int prec, const void* B, int64_t ldb, int64_t k, int64_t n, int64_t kp,
                          const int32_t* nu_prime, int8_t* bbar_t, DevStatus* st, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    dim3 grid(blocks_for(n, TB), (unsigned)(kp / TB));
    const size_t sm = transpose_smem(0);
    if (prec)
        transpose_B_kernel<double, 0><<<grid, 256, sm, s>>>((const double*)B, ldb, k, n, kp, nu_prime, nullptr, 1, bbar_t, st);
    else
        transpose_B_kernel<float, 0><<<grid, 256, sm, s>>>((const float*)B, ldb, k, n, kp, nu_prime, nullptr, 1, bbar_t, st);
    return cudaGetLastError();
}

cudaError_t launch_resid_BT(int prec, const void* B, int64_t ldb, int64_t k, int64_t n, int64_t kp,
                            const int32_t* nu, const ResidConsts* rc_dev, int nmod, int8_t* planes,
                            DevStatus* st, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    dim3 grid(blocks_for(n, TB), (unsigned)(kp / TB));
    const size_t sm = transpose_smem(1);
    cudaError_t err;
    if (prec) {
        err = cudaFuncSetAttribute(transpose_B_kernel<double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (err != cudaSuccess) return err;
        transpose_B_kernel<double, 1><<<grid, 256, sm, s>>>((const double*)B, ldb, k, n, kp, nu, rc_dev, nmod, planes, st);
    } else {
        err = cudaFuncSetAttribute(transpose_B_kernel<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (err != cudaSuccess) return err;
        transpose_B_kernel<float, 1><<<grid, 256, sm, s>>>((const float*)B, ldb, k, n, kp, nu, rc_dev, nmod, planes, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_resid_A(int prec, const void* A, int64_t lda, int64_t m, int64_t k, int64_t kp,
                           const int32_t* mu, const ResidConsts* rc_dev, int nmod, int8_t* planes,
                           DevStatus* st, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    const int64_t work = m * (kp / 16);
    const size_t sm = sizeof(ResidConsts);
    cudaError_t err;
    if (prec) {
        err = cudaFuncSetAttribute(resid_A_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (err != cudaSuccess) return err;
        resid_A_kernel<double><<<blocks_for(work, 256), 256, sm, s>>>((const double*)A, lda, m, k, kp, mu, rc_dev, nmod, planes, st);
    } else {
        err = cudaFuncSetAttribute(resid_A_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (err != cudaSuccess) return err;
        resid_A_kernel<float><<<blocks_for(work, 256), 256, sm, s>>>((const float*)A, lda, m, k, kp, mu, rc_dev, nmod, planes, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_exponents(const int32_t* cmax_row, int64_t m, const int32_t* cmax_col, int64_t n,
                             const int32_t* mu_prime, const int32_t* nu_prime, int shift0, int nthr,
                             const int32_t* thr, int32_t* mu, int32_t* nu, float* e, float* f, DevStatus* st,
                             cudaStream_t s) {
    if (m + n == 0) return cudaSuccess;
    ThrTable tt;
    tt.shift0 = shift0;
    tt.nthr = nthr;
    for (int q = 0; q < 64; ++q) tt.thr[q] = q < nthr ? thr[q] : 0;
    exponents_kernel<<<blocks_for(m + n, 256), 256, 0, s>>>(cmax_row, m, cmax_col, n, mu_prime, nu_prime, tt, mu,
                                                            nu, e, f, st);
    return cudaGetLastError();
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

}  // namespace oz2g
