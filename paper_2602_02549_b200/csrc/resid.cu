// resid.cu — the residue split of Algorithm 3 fused with the truncation of
// Algorithm 2, and the transposed writer of Bbar:
//
//   resid_A      truncate_scaled_rows (scaling.hpp:199-211) + residue_matrix
//                (crt.hpp:20-65) for every modulus: A' = trunc(2^mu A) is never
//                materialised; each element is decomposed once and all N int8
//                planes [l][m][kp] (K-major) are written in the same pass.
//   resid_B      the same for B (truncate_scaled_cols, scaling.hpp:213-225)
//                in B's own layout, planes [l][kp][ldn] (MN-major for the GEMM).
//   bbar         ceil_abs_scale_cols (scaling.hpp:122-131) -> Bbar [kp][ldn].
//
// Two decompositions of A' feed the same exact reduction: balanced base-256
// digits with one weight set per modulus (the fast path below, every chunk of
// 8 elements with |A'| < 2^62 — practically all of them), and the exponent
// buckets described here (the rest, or option resid_fast = 0).
//
// Residue arithmetic.  |A'| = m' * 2^E' with m' < 2^53 (m' = mant >> -E if
// E < 0, E' = max(E, 0)); write it as g * 2^(8 G) with g = m' << (E' mod 8)
// < 2^60 and G = E' / 8.  With the signed byte weights
//   w[l][G][s][t] = symmetric representative of (-1)^s 2^(8 (t + G)) mod p_l
//   S = sum_t byte_t(g) * w[l][G][sgn(x)][t]     (two dp4a.u32.s32, |S| < 2^18)
// is congruent to A' mod p_l.  The dp4a accumulator starts at the bit pattern
// of M = 1.5 * 2^23, so the integer result is the bit pattern of the float
// M + S (exact: the float has ulp 1 on [2^23, 2^24)).  Then, in fp32,
//   q = round(S / p) = RN(S * RN(1/p) + M) - M      (|error| < 2^-13.5, while
//       S / p is >= 1/(2p) > 2^-9 away from a half-integer for odd p;
//       for p = 256 the product is exact)
// and r = S - p q is read off the integer bit patterns: bits(M + S) -
// p * bits(M + q) = r + 0x4B400000 (1 - p), whose low byte is r as int8
// because 0x4B400000 is a multiple of 256.  r is the reference's
// representative of A' mod p_l (crt.hpp:48-52), symmetric for odd p; for
// p = 256, r = +-128 both give the byte 0x80, which is how the reference
// stores the class 128 (-128).  Per (element, modulus): one LDS.64, two IDP,
// one FADD, one FFMA, one IMAD, and 3/4 of a PRMT to pack.  Bucketing E' by 8
// keeps the table small (256 B per modulus) and the lanes of a warp on one or
// two entries, so the weight loads are broadcasts.
#include "device_common.cuh"
#include "kernels.h"
#include "options.h"

namespace oz2g {

namespace {

__device__ __forceinline__ void flag(DevStatus* st, uint32_t bits) { atomicOr(&st->err, bits); }

template <class T>
__device__ __forceinline__ double ld_d(const T* p) { return (double)__ldg(p); }

struct ElemDec {
    uint32_t lo, hi;  // bytes 0-3 / 4-7 of m' << (E' mod 8)  (< 2^60)
    uint32_t off;     // byte offset of the weights: 16 * (E' / 8) (+ 8 for x < 0)
};

// Branch-free: x = mant * 2^(max(ef, 1) - 1075) holds for normals, subnormals
// (ef = 0, no hidden bit) and zero (mant = 0, which gives S = 0 for any table
// row), so no case needs separate code.
__device__ __forceinline__ ElemDec elem_dec(double x, int shift, bool& overflow) {
    const uint64_t bits = (uint64_t)__double_as_longlong(x);
    const int ef = (int)((bits >> 52) & 0x7ff);
    const uint64_t mant = (bits & 0x000fffffffffffffull) | ((uint64_t)(ef != 0) << 52);
    const int E = max(ef, 1) - 1075 + shift;
    // ldexp(x, shift) overflows iff |x| 2^shift >= 2^1024 (scaling.hpp:206/220);
    // |A'| < 2^(6 + P') < 2^177 for every valid input, so E' <= 124 < 8 * kResidE8
    const int Ep = max(E, 0);
    overflow |= mant != 0 && (E > 1024 - 53 || Ep > 8 * kResidE8 - 1);
    const int Ec = min(Ep, 8 * kResidE8 - 1);
    const uint64_t g = (mant >> min(max(-E, 0), 63)) << (Ec & 7);  // trunc for E < 0, then E' mod 8
    ElemDec d;
    d.lo = (uint32_t)g;
    d.hi = (uint32_t)(g >> 32);
    d.off = (uint32_t)(Ec >> 3) * 16u + (uint32_t)(bits >> 63) * 8u;
    return d;
}

__device__ __forceinline__ int dp4a_us(uint32_t a, int32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

struct ModC {
    float inv_p;
    uint32_t p;
};

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23 (bits 0x4B400000): ulp 1 on [2^23, 2^24)

// Word whose low byte is the reference's representative of sgn * m' * 2^E' mod p
// (see the file header).  bits = bits(M + S) = 0x4B400000 + S and
// bits(t) = 0x4B400000 + q with q = round(S / p) (the only inexact fp32 step
// rounds to that integer), so bits - p * bits(t) = S - p q + 0x4B400000 (1 - p),
// whose low byte is r = S - p q: 0x4B400000 is a multiple of 256.
__device__ __forceinline__ uint32_t resid_w(const ElemDec& d, const uint8_t* __restrict__ row_l, const ModC& c) {
    const int2 w = *reinterpret_cast<const int2*>(row_l + d.off);
    const int bits = dp4a_us(d.hi, w.y, dp4a_us(d.lo, w.x, 0x4B400000));  // bits of the float M + S
    const float u = __fsub_rn(__int_as_float(bits), kMagic);              // S
    const float t = __fmaf_rn(u, c.inv_p, kMagic);                         // M + round(S / p)
    return (uint32_t)bits - (uint32_t)__float_as_int(t) * c.p;
}

__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
    const uint32_t lo = __byte_perm(b0, b1, 0x0040);
    const uint32_t hi = __byte_perm(b2, b3, 0x0040);
    return __byte_perm(lo, hi, 0x5410);
}

// ---------------------------------------------------------------------------
// Fast path (every element of a thread's chunk with |A'| < 2^62, i.e. E <= 9:
// the common case — |A'| < 2^(6 + mu_i - mu'_i) and the shift exceeds 56 only
// for rows whose clearance maximum is tiny).  A' is formed as a 64-bit two's
// complement integer x (one fp64 multiply by 2^shift and a truncating
// conversion) and written in balanced base-256 digits
//   x = sum_t d_t 256^t,  d_t in [-128, 127]:  the bytes of
//   z = (x + 0x80..80) ^ 0x80..80  (adding 128 per byte, then flipping bit 7)
// so one set of constant weights per modulus serves every element — the
// weights of G = 0, s = 0 of the table, read once per modulus and chunk (a
// broadcast), not once per element.  S = sum_t d_t w_t (two dp4a.s32.s32,
// |S| <= 2^17; one when d_4..d_7 = 0 for the whole chunk) then goes through the
// same exact fp32 reduction.  The p = 256 plane is d_0 itself (x mod 256 in
// [-128, 127]), no arithmetic.
// ---------------------------------------------------------------------------
struct FastDec {
    uint32_t lo, hi;  // the balanced digits d_0..d_3 / d_4..d_7 as signed bytes
};

__device__ __forceinline__ FastDec fast_dec(double x, int shift, bool& ok) {
    // A' = trunc(x 2^shift): the product is exact unless it is subnormal, and
    // then |A'| < 1 truncates to 0 either way (one DMUL, one F2I.S64.TRUNC)
    ok &= pow2_normal(shift);
    const double y = __dmul_rn(x, pow2d(shift));
    ok &= (uint32_t)(__double2hiint(y) & 0x7fffffff) < 0x43D00000u;  // |y| < 2^62 (also rejects inf / nan)
    constexpr uint64_t C = 0x8080808080808080ull;
    const uint64_t z = ((uint64_t)__double2ll_rz(y) + C) ^ C;  // balanced digits
    FastDec d;
    d.lo = (uint32_t)z;
    d.hi = (uint32_t)(z >> 32);
    return d;
}

__device__ __forceinline__ int dp4a_ss(uint32_t a, int32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// a * b + c (mod 2^32), opaque to the compiler (which would otherwise negate
// each product instead of using the negated modulus once)
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t resid_fast(const FastDec& d, const FastMod& f) {
    const int bits = dp4a_ss(d.hi, f.w1, dp4a_ss(d.lo, f.w0, 0x4B400000));  // bits of the float M + S
    const float u = __fsub_rn(__int_as_float(bits), kMagic);
    const float t = __fmaf_rn(u, f.inv_p, kMagic);
    return mad_u32(__float_as_uint(t), f.negp, (uint32_t)bits);
}

// All N planes of one 8-element chunk from its balanced digits.
// Four digits: every element of the chunk has d_4 = .. = d_7 = 0 (|A'| within
// [-0x80808080, 0x7F7F7F7F]), so one dp4a per element and modulus.
__device__ __forceinline__ uint32_t resid_fast4(uint32_t lo, const FastMod& f) {
    const int bits = dp4a_ss(lo, f.w0, 0x4B400000);
    const float u = __fsub_rn(__int_as_float(bits), kMagic);
    const float t = __fmaf_rn(u, f.inv_p, kMagic);
    return mad_u32(__float_as_uint(t), f.negp, (uint32_t)bits);
}

// All N planes of one 8-element chunk from its balanced digits.
__device__ __forceinline__ void write_fast(const FastDec (&f)[8], const ResidHeader& hd, int nmod, int8_t* out,
                                           int64_t plane) {
    int l0 = 0;
    if (hd.p[0] == 256u) {  // the table's first modulus: the plane is d_0
        *reinterpret_cast<uint2*>(out) =
            make_uint2(pack4(f[0].lo, f[1].lo, f[2].lo, f[3].lo), pack4(f[4].lo, f[5].lo, f[6].lo, f[7].lo));
        l0 = 1;
    }
    const uint32_t hi = f[0].hi | f[1].hi | f[2].hi | f[3].hi | f[4].hi | f[5].hi | f[6].hi | f[7].hi;
    if (hi == 0u) {  // small |A'| (fp32 inputs, few moduli): four digits
#pragma unroll 2
        for (int l = l0; l < nmod; ++l) {
            const FastMod fm = hd.fm[l];
            const uint32_t w0 = pack4(resid_fast4(f[0].lo, fm), resid_fast4(f[1].lo, fm), resid_fast4(f[2].lo, fm),
                                      resid_fast4(f[3].lo, fm));
            const uint32_t w1 = pack4(resid_fast4(f[4].lo, fm), resid_fast4(f[5].lo, fm), resid_fast4(f[6].lo, fm),
                                      resid_fast4(f[7].lo, fm));
            *reinterpret_cast<uint2*>(out + (int64_t)l * plane) = make_uint2(w0, w1);
        }
        return;
    }
#pragma unroll 2
    for (int l = l0; l < nmod; ++l) {
        const FastMod fm = hd.fm[l];  // one 16-byte broadcast load per modulus
        const uint32_t w0 = pack4(resid_fast(f[0], fm), resid_fast(f[1], fm), resid_fast(f[2], fm), resid_fast(f[3], fm));
        const uint32_t w1 = pack4(resid_fast(f[4], fm), resid_fast(f[5], fm), resid_fast(f[6], fm), resid_fast(f[7], fm));
        *reinterpret_cast<uint2*>(out + (int64_t)l * plane) = make_uint2(w0, w1);
    }
}

__device__ __forceinline__ void load_resid_consts(const ResidHeader* __restrict__ g, int n, uint8_t* sh) {
    const uint4* src = reinterpret_cast<const uint4*>(g);
    uint4* dst = reinterpret_cast<uint4*>(sh);
    const int words = (int)(resid_consts_bytes(n) / 16);
    for (int t = threadIdx.x; t < words; t += blockDim.x) dst[t] = src[t];
}

__device__ __forceinline__ ModC modc(const ResidHeader& hd, int l) { return ModC{hd.inv_p[l], hd.p[l]}; }

// ---------------------------------------------------------------------------
// Row-major writers (A and B alike): each thread owns 8 consecutive columns of
// one row (16-byte vector loads, one 8-byte store per output plane); grid.x
// covers the 2048-column chunks of a row and a CTA walks rows blockIdx.y,
// blockIdx.y + gridDim.y, ... so the weight table is loaded once per CTA.
//   A residues: rows m, shift mu per row, planes [l][m][kp] (K-major for the GEMM)
//   B residues: rows kp (k real, the rest zero), shift nu per column, planes
//               [l][kp][ldn] (B's own layout, read MN-major by the GEMM)
//   Bbar (OP 0): ceil(|b| 2^nu'_j) into [kp][ldn] (scaling.hpp:122-131)
// Columns past the valid ones (up to the padded width) are written as zeros.
// ---------------------------------------------------------------------------
constexpr int RA_E = 8;

// A: the row-shift case of the writer below, kept as its own kernel (per-row
// shift; 64 registers, 4 CTAs per SM — 65 would leave 3).
template <class T>
__global__ void __launch_bounds__(256, 4) resid_A_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t k,
                                                      int64_t kp, const int32_t* __restrict__ mu,
                                                      const ResidHeader* __restrict__ rc_g, int nmod,
                                                      int8_t* __restrict__ planes, int64_t plane, DevStatus* st,
                                                      int fast_on) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t sh[];
    load_resid_consts(rc_g, nmod, sh);
    __syncthreads();
    const ResidHeader& hd = *reinterpret_cast<const ResidHeader*>(sh);
    const uint8_t* tab = sh + sizeof(ResidHeader);
    const int64_t h0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * RA_E;
    bool ovf = false;
    if (h0 >= kp) return;
    for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
        const int sft = mu[i];
        const T* row = A + i * lda + h0;
        int8_t* out = planes + i * kp + h0;
        const bool vec = h0 + RA_E <= k && ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
        if (fast_on && vec) {
            FastDec f[RA_E];
            bool ok = true;
            if (sizeof(T) == 8) {
#pragma unroll
                for (int j = 0; j < RA_E; j += 2) {
                    const double2 v = __ldg(reinterpret_cast<const double2*>(row + j));
                    f[j] = fast_dec(v.x, sft, ok);
                    f[j + 1] = fast_dec(v.y, sft, ok);
                }
            } else {
#pragma unroll
                for (int j = 0; j < RA_E; j += 4) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(row + j));
                    f[j] = fast_dec((double)v.x, sft, ok);
                    f[j + 1] = fast_dec((double)v.y, sft, ok);
                    f[j + 2] = fast_dec((double)v.z, sft, ok);
                    f[j + 3] = fast_dec((double)v.w, sft, ok);
                }
            }
            if (ok) {
                write_fast(f, hd, nmod, out, plane);
                continue;
            }
        }
        ElemDec d[RA_E];
        if (sizeof(T) == 8 && h0 + RA_E <= k && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < RA_E; j += 2) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(row + j));
                d[j] = elem_dec(v.x, sft, ovf);
                d[j + 1] = elem_dec(v.y, sft, ovf);
            }
        } else if (sizeof(T) == 4 && h0 + RA_E <= k && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < RA_E; j += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(row + j));
                d[j] = elem_dec((double)v.x, sft, ovf);
                d[j + 1] = elem_dec((double)v.y, sft, ovf);
                d[j + 2] = elem_dec((double)v.z, sft, ovf);
                d[j + 3] = elem_dec((double)v.w, sft, ovf);
            }
        } else {
#pragma unroll
            for (int j = 0; j < RA_E; ++j) d[j] = elem_dec(h0 + j < k ? ld_d(row + j) : 0.0, sft, ovf);
        }
#pragma unroll 2
        for (int l = 0; l < nmod; ++l) {
            const ModC c = modc(hd, l);
            const uint8_t* rl = tab + (size_t)l * kResidRow;
            const uint32_t w0 = pack4(resid_w(d[0], rl, c), resid_w(d[1], rl, c), resid_w(d[2], rl, c),
                                      resid_w(d[3], rl, c));
            const uint32_t w1 = pack4(resid_w(d[4], rl, c), resid_w(d[5], rl, c), resid_w(d[6], rl, c),
                                      resid_w(d[7], rl, c));
            *reinterpret_cast<uint2*>(out + (int64_t)l * plane) = make_uint2(w0, w1);
        }
    }
    if (ovf) flag(st, ERR_TRUNC_A_RANGE);
}

template <class T, bool COLSHIFT, int OP>
__global__ void __launch_bounds__(256, 4) resid_rows_kernel(const T* __restrict__ X, int64_t ldx, int64_t rows_valid,
                                                         int64_t rows_total, int64_t cols_valid, int64_t cols_out,
                                                         int64_t ld_out, const int32_t* __restrict__ shift,
                                                         const ResidHeader* __restrict__ rc_g, int nmod,
                                                         int8_t* __restrict__ planes, int64_t plane, uint32_t err_bit,
                                                         DevStatus* st, int fast_on) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t sh[];
    if (OP == 1) {
        load_resid_consts(rc_g, nmod, sh);
        __syncthreads();
    }
    const ResidHeader& hd = *reinterpret_cast<const ResidHeader*>(sh);
    const uint8_t* tab = sh + sizeof(ResidHeader);
    const int64_t h0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * RA_E;
    if (h0 >= cols_out) return;
    bool bad = false;
    int csft[RA_E];  // per-column shifts (B): the same for every row
    if (COLSHIFT) {
#pragma unroll
        for (int j = 0; j < RA_E; ++j) csft[j] = h0 + j < cols_valid ? __ldg(shift + h0 + j) : 0;
    }
    const bool full = h0 + RA_E <= cols_valid;
    const int nplanes = OP == 0 ? 1 : nmod;
    // Bbar: 2^nu'_j as doubles for the fp64-pipe ceil (ceil_scaled_p2) when all are normal
    double p2c[RA_E] = {};
    bool fastc = OP == 0 && COLSHIFT;
    if (OP == 0 && COLSHIFT) {
#pragma unroll
        for (int j = 0; j < RA_E; ++j) {
            fastc &= pow2_normal(csft[j]);
            p2c[j] = pow2_normal(csft[j]) ? pow2d(csft[j]) : 0.0;
        }
    }
    for (int64_t i = blockIdx.y; i < rows_total; i += gridDim.y) {
        int8_t* out = planes + i * ld_out + h0;
        if (i >= rows_valid) {  // zero padding rows (B: k .. kp)
            for (int l = 0; l < nplanes; ++l) *reinterpret_cast<uint2*>(out + (int64_t)l * plane) = make_uint2(0u, 0u);
            continue;
        }
        const T* row = X + i * ldx + h0;
        const int rsft = COLSHIFT ? 0 : __ldg(shift + i);
        const bool vec = full && ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
        if (OP == 0) {
            double x[RA_E];
            if (vec && sizeof(T) == 8) {
#pragma unroll
                for (int j = 0; j < RA_E; j += 2) {
                    const double2 t = __ldg(reinterpret_cast<const double2*>(row + j));
                    x[j] = t.x;
                    x[j + 1] = t.y;
                }
            } else if (vec && sizeof(T) == 4) {
#pragma unroll
                for (int j = 0; j < RA_E; j += 4) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(row + j));
                    x[j] = t.x; x[j + 1] = t.y; x[j + 2] = t.z; x[j + 3] = t.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < RA_E; ++j) x[j] = h0 + j < cols_valid ? (double)__ldg(row + j) : 0.0;
            }
            uint32_t w[2] = {0u, 0u};
#pragma unroll
            for (int j = 0; j < RA_E; ++j) {
                const int c = fastc ? ceil_scaled_p2(x[j], p2c[j]) : ceil_abs_scaled(x[j], COLSHIFT ? csft[j] : rsft);
                bad |= c < 0;
                w[j >> 2] |= (uint32_t)(c & 0xff) << (8 * (j & 3));
            }
            *reinterpret_cast<uint2*>(out) = make_uint2(w[0], w[1]);
            continue;
        }
        if (fast_on && vec) {
            FastDec f[RA_E];
            bool ok = true;
            if (sizeof(T) == 8) {
#pragma unroll
                for (int j = 0; j < RA_E; j += 2) {
                    const double2 t = __ldg(reinterpret_cast<const double2*>(row + j));
                    f[j] = fast_dec(t.x, COLSHIFT ? csft[j] : rsft, ok);
                    f[j + 1] = fast_dec(t.y, COLSHIFT ? csft[j + 1] : rsft, ok);
                }
            } else {
#pragma unroll
                for (int j = 0; j < RA_E; j += 4) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(row + j));
                    f[j] = fast_dec((double)t.x, COLSHIFT ? csft[j] : rsft, ok);
                    f[j + 1] = fast_dec((double)t.y, COLSHIFT ? csft[j + 1] : rsft, ok);
                    f[j + 2] = fast_dec((double)t.z, COLSHIFT ? csft[j + 2] : rsft, ok);
                    f[j + 3] = fast_dec((double)t.w, COLSHIFT ? csft[j + 3] : rsft, ok);
                }
            }
            if (ok) {
                write_fast(f, hd, nmod, out, plane);
                continue;
            }
        }
        // decode straight from the loads (no staging array: fewer live registers)
        ElemDec d[RA_E];
        if (vec && sizeof(T) == 8) {
#pragma unroll
            for (int j = 0; j < RA_E; j += 2) {
                const double2 t = __ldg(reinterpret_cast<const double2*>(row + j));
                d[j] = elem_dec(t.x, COLSHIFT ? csft[j] : rsft, bad);
                d[j + 1] = elem_dec(t.y, COLSHIFT ? csft[j + 1] : rsft, bad);
            }
        } else if (vec && sizeof(T) == 4) {
#pragma unroll
            for (int j = 0; j < RA_E; j += 4) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(row + j));
                d[j] = elem_dec((double)t.x, COLSHIFT ? csft[j] : rsft, bad);
                d[j + 1] = elem_dec((double)t.y, COLSHIFT ? csft[j + 1] : rsft, bad);
                d[j + 2] = elem_dec((double)t.z, COLSHIFT ? csft[j + 2] : rsft, bad);
                d[j + 3] = elem_dec((double)t.w, COLSHIFT ? csft[j + 3] : rsft, bad);
            }
        } else {
#pragma unroll
            for (int j = 0; j < RA_E; ++j)
                d[j] = elem_dec(h0 + j < cols_valid ? (double)__ldg(row + j) : 0.0, COLSHIFT ? csft[j] : rsft, bad);
        }
#pragma unroll 2
        for (int l = 0; l < nmod; ++l) {
            const ModC c = modc(hd, l);
            const uint8_t* rl = tab + (size_t)l * kResidRow;
            const uint32_t w0 = pack4(resid_w(d[0], rl, c), resid_w(d[1], rl, c), resid_w(d[2], rl, c),
                                      resid_w(d[3], rl, c));
            const uint32_t w1 = pack4(resid_w(d[4], rl, c), resid_w(d[5], rl, c), resid_w(d[6], rl, c),
                                      resid_w(d[7], rl, c));
            *reinterpret_cast<uint2*>(out + (int64_t)l * plane) = make_uint2(w0, w1);
        }
    }
    if (bad) flag(st, err_bit);
}

inline unsigned blocks_for(int64_t work, int per) { return (unsigned)((work + per - 1) / per); }

template <class K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// grid: x = column chunks, y = enough row strides for kResidWaves waves of
// resident CTAs (each CTA then loads the weight table once for rows / y rows).
constexpr int kResidWaves = 4;

template <class K>
cudaError_t rows_grid(K kernel, size_t smem, int64_t rows, unsigned chunks, dim3& grid) {
    cudaError_t err = set_smem(kernel, smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem)) != cudaSuccess) return err;
    const int64_t ctas = (int64_t)current_sm_count() * (per_sm > 0 ? per_sm : 1) * kResidWaves;
    int64_t r = (ctas + chunks - 1) / chunks;
    r = r < rows ? r : rows;
    grid = dim3(chunks, (unsigned)(r < 65535 ? (r > 0 ? r : 1) : 65535));
    return cudaSuccess;
}

template <class T, bool COLSHIFT, int OP>
cudaError_t launch_rows(const void* X, int64_t ldx, int64_t rows_valid, int64_t rows_total, int64_t cols_valid,
                        int64_t cols_out, int64_t ld_out, const int32_t* shift, const ResidConsts* rc, int nmod,
                        int8_t* planes, int64_t plane, uint32_t err_bit, DevStatus* st, cudaStream_t s) {
    if (rows_total == 0 || cols_out == 0) return cudaSuccess;
    const unsigned chunks = blocks_for(cols_out, 256 * RA_E);
    const size_t sm = OP == 1 ? resid_consts_bytes(nmod) : 0;
    dim3 grid;
    cudaError_t err = rows_grid(resid_rows_kernel<T, COLSHIFT, OP>, sm, rows_total, chunks, grid);
    if (err != cudaSuccess) return err;
    return launch_pdl(resid_rows_kernel<T, COLSHIFT, OP>, grid, dim3(256), sm, s, (const T*)X, ldx, rows_valid,
                      rows_total, cols_valid, cols_out, ld_out, shift, rc, nmod, planes, plane, err_bit, st,
                      (int)opt(OPT_RESID_FAST));
}

}  // namespace

cudaError_t launch_bbar_rows(int prec, const void* B, int64_t ldb, int64_t k, int64_t n, int64_t kp, int64_t ldn,
                             const int32_t* nu_prime, int8_t* bbar, DevStatus* st, cudaStream_t s, int64_t cols_out) {
    if (n == 0) return cudaSuccess;
    if (cols_out < 0) cols_out = ldn;
    return prec ? launch_rows<double, true, 0>(B, ldb, k, kp, n, cols_out, ldn, nu_prime, nullptr, 1, bbar, 0,
                                               ERR_CEIL_LOGIC, st, s)
                : launch_rows<float, true, 0>(B, ldb, k, kp, n, cols_out, ldn, nu_prime, nullptr, 1, bbar, 0,
                                              ERR_CEIL_LOGIC, st, s);
}

cudaError_t launch_resid_B_rows(int prec, const void* B, int64_t ldb, int64_t k, int64_t n, int64_t kp, int64_t ldn,
                                const int32_t* nu, const ResidConsts* rc_dev, int nmod, int8_t* planes,
                                DevStatus* st, cudaStream_t s, int64_t cols_out) {
    if (n == 0) return cudaSuccess;
    if (cols_out < 0) cols_out = ldn;
    const int64_t plane = kp * ldn;
    return prec ? launch_rows<double, true, 1>(B, ldb, k, kp, n, cols_out, ldn, nu, rc_dev, nmod, planes, plane,
                                               ERR_TRUNC_B_RANGE, st, s)
                : launch_rows<float, true, 1>(B, ldb, k, kp, n, cols_out, ldn, nu, rc_dev, nmod, planes, plane,
                                              ERR_TRUNC_B_RANGE, st, s);
}

cudaError_t launch_resid_A(int prec, const void* A, int64_t lda, int64_t m, int64_t k, int64_t kp,
                           const int32_t* mu, const ResidConsts* rc_dev, int nmod, int8_t* planes,
                           int64_t plane_stride, DevStatus* st, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    const int64_t plane = plane_stride ? plane_stride : m * kp;
    const unsigned chunks = blocks_for(kp, 256 * RA_E);
    const size_t sm = resid_consts_bytes(nmod);
    dim3 grid;
    cudaError_t err;
    if (prec) {
        if ((err = rows_grid(resid_A_kernel<double>, sm, m, chunks, grid)) != cudaSuccess) return err;
        return launch_pdl(resid_A_kernel<double>, grid, dim3(256), sm, s, (const double*)A, lda, m, k, kp, mu, rc_dev,
                          nmod, planes, plane, st, (int)opt(OPT_RESID_FAST));
    }
    if ((err = rows_grid(resid_A_kernel<float>, sm, m, chunks, grid)) != cudaSuccess) return err;
    return launch_pdl(resid_A_kernel<float>, grid, dim3(256), sm, s, (const float*)A, lda, m, k, kp, mu, rc_dev, nmod,
                      planes, plane, st, (int)opt(OPT_RESID_FAST));
}

}  // namespace oz2g
