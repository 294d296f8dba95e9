// crt.cu — Chinese-Remainder reconstruction and inverse scaling, fused into
// one HBM-bound pass over the N int8 residue products W_l.
//
// Restates, element by element and in the reference's exact operation order:
//   accumulate    crt.hpp:91-110  C1 = fma chain of s1_l * W_l over l = 0..N-1
//                                 from +0.0; C2 likewise with s2 (fp64 mode)
//   compute_q     crt.hpp:113-119 Q = round_half_even(RN(P_inv * C1))
//   final_reduce  crt.hpp:129-150 C'' = fma(-Q, P2, fma(-Q, P1, C1) + C2);
//                                 fp32 mode: |C''| >= 0x1.ffffffp+127 is a
//                                 range error, else C''32 = RN32(C'')
//   inverse_scale emulate.hpp:30-46 x = ldexp(C'', -mu_i), y = ldexp(x, -nu_j)
//                                 (two RN scalings), subnormal / overflow flags
// Every operation is an explicit _rn intrinsic so nvcc cannot contract or
// reorder; the result is bit-identical to the reference.
//
// Optionally (BND) the same pass evaluates the cheap and tight error bounds
// of bounds.hpp:143-206 for every entry (see bounds.cu for the derivation).
#include <cfloat>
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace oz2g {

namespace {

// CV consecutive columns per thread: one 8-byte (CV = 8) or 4-byte (CV = 4)
// load per modulus plane
template <int CV> struct WordOf;
template <> struct WordOf<8> {
    using T = uint2;
    static __device__ __forceinline__ uint32_t lo(uint2 w) { return w.x; }
    static __device__ __forceinline__ uint32_t hi(uint2 w) { return w.y; }
};
template <> struct WordOf<4> {
    using T = uint32_t;
    static __device__ __forceinline__ uint32_t lo(uint32_t w) { return w; }
    static __device__ __forceinline__ uint32_t hi(uint32_t) { return 0u; }
};

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// Exact int8 -> fp64 on the fp64 pipe instead of the conversion (XU) pipe: the
// double with bits 0x43300000:(w ^ 0x80) is 2^52 + w + 128, and subtracting
// 2^52 + 128 is exact.  wx = the packed word with every byte XORed by 0x80.
__device__ __forceinline__ double i8_to_f64_fp(uint32_t wx, int b) {
    const uint32_t lo = __byte_perm(wx, 0u, 0x4440u | (uint32_t)b);
    return __dsub_rn(__hiloint2double(0x43300000, (int)lo), 4503599627370624.0);
}

// Byte t of w as a signed int8 -> fp64 with one I2F.F64.S8 (XU) reading the
// byte in place (a plain C cast of byte 0 compiled to two PRMTs and an S16
// conversion here).
__device__ __forceinline__ double i8_to_f64_xu(uint32_t w, int t) {
    if (t != 0) return (double)(int8_t)((w >> (8 * t)) & 0xffu);  // folds into I2F.F64.S8 R.Bt
    double r;
    asm("{.reg .s8 b; cvt.s8.u32 b, %1; cvt.rn.f64.s8 %0, b;}" : "=d"(r) : "r"(w));
    return r;
}

// NFP of the CV columns convert through i8_to_f64_fp, the rest with I2F (XU):
// XU converts 16 values/clk/SM, the fp64 pipe 64, so splitting balances them.
// 8 columns per thread: capped at 64 registers (4 CTAs per SM; the kernel is
// latency-bound and was at 3 CTAs with 70 registers): 0.238 -> 0.206 ms per
// 2048-row block at 16384^2 with one group of 8 plane loads in flight per
// thread (double-buffering the groups spilled at 64 registers: 0.216 ms);
// 5 CTAs spill and lose (0.32 ms).
template <class T, bool DD, bool BND, int NFP, bool INTER, int CV>
__global__ void __launch_bounds__(256, CV == 8 ? 4 : 1) crt_kernel(const int8_t* __restrict__ W, int64_t ldw, int64_t wplane,
                                                  int64_t m, int64_t n, const CrtConsts cc,
                                                  const int32_t* __restrict__ mu, const int32_t* __restrict__ nu,
                                                  T* __restrict__ C, int64_t ldc, const CrtExtra ex,
                                                  DevStatus* st) {
    pdl_enter();
    const int64_t qn = (n + CV - 1) / CV;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = t < m * qn;
    unsigned long long bmax_cheap = 0, bmax_tight = 0, bmax_rel = 0;
    if (active) {
        const int64_t i = t / qn;
        const int64_t j0 = (t - i * qn) * CV;
        const int jn = (int)(n - j0 < CV ? n - j0 : CV);
        double c1[CV], c2[CV];
#pragma unroll
        for (int b = 0; b < CV; ++b) { c1[b] = 0.0; c2[b] = 0.0; }
        const int8_t* wp = W + i * ldw + j0;
        // crt.hpp:99-104: acc = fma(s_l, W_l, acc) in the fixed order l = 0..N-1.
        // Loads are issued 4 planes ahead of their use to keep HBM busy.
        using Wt = typename WordOf<CV>::T;
        auto fold = [&](const Wt word, int l) {
            const double s1 = cc.s1[l];
            const double s2 = cc.s2[l];
            const uint32_t wlo = WordOf<CV>::lo(word), whi = WordOf<CV>::hi(word);
            const uint32_t xx = wlo ^ 0x80808080u, xy = whi ^ 0x80808080u;
#pragma unroll
            for (int b = 0; b < CV; ++b) {
                const uint32_t w32 = b < 4 ? wlo : whi;
                const double wv = b >= CV - NFP ? i8_to_f64_fp(b < 4 ? xx : xy, b & 3) : i8_to_f64_xu(w32, b & 3);
                c1[b] = __fma_rn(s1, wv, c1[b]);
                if (DD) c2[b] = __fma_rn(s2, wv, c2[b]);
            }
        };
        // planes in groups of 8 loads in flight per thread
        int l = 0;
        const int nfull = cc.n & ~7;
        for (; l < nfull; l += 8) {  // 8 loads in flight per thread; occupancy hides the rest
            Wt cur[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) cur[u] = __ldcs(reinterpret_cast<const Wt*>(wp + (int64_t)(l + u) * wplane));
#pragma unroll
            for (int u = 0; u < 8; ++u) fold(cur[u], l + u);
        }
        for (; l + 4 <= cc.n; l += 4) {
            Wt wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) wv[u] = __ldcs(reinterpret_cast<const Wt*>(wp + (int64_t)(l + u) * wplane));
#pragma unroll
            for (int u = 0; u < 4; ++u) fold(wv[u], l + u);
        }
        for (; l < cc.n; ++l) fold(__ldg(reinterpret_cast<const Wt*>(wp + (int64_t)l * wplane)), l);

        const int mui = mu[i];
        double RAi = 0, PAi = 0;
        int eai = 0;
        if (BND) { RAi = ex.bnd.v.RA[i]; PAi = ex.bnd.v.PA[i]; eai = ex.bnd.v.ea[i]; }
        bool fr_range = false, inv_range = false, sub = false;
        // the column shifts of this thread (two 16-byte loads when whole and aligned)
        int nuv[CV];
        if (jn == CV && (reinterpret_cast<uintptr_t>(nu + j0) & 15) == 0) {
#pragma unroll
            for (int b = 0; b < CV; b += 4) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(nu + j0 + b));
                nuv[b] = v.x; nuv[b + 1] = v.y; nuv[b + 2] = v.z; nuv[b + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int b = 0; b < CV; ++b) nuv[b] = b < jn ? __ldg(nu + j0 + b) : 0;
        }
        // 2^-mu_i and every 2^-nu_j normal (in T): each ldexp is one
        // multiplication (ldexp_rn's / ldexpf_rn's own fast path)
        auto p2ok = [](int e) { return sizeof(T) == 4 ? (e >= -126 && e <= 127) : pow2_normal(e); };
        bool fastsc = p2ok(-mui);
#pragma unroll
        for (int b = 0; b < CV; ++b) fastsc &= p2ok(-nuv[b]);
        const double pmu = fastsc && sizeof(T) == 8 ? pow2d(-mui) : 0.0;
        const float pmuf = fastsc && sizeof(T) == 4 ? pow2f(-mui) : 0.0f;
        T yv[CV];  // this thread's C entries, stored together below
#pragma unroll
        for (int b = 0; b < CV; ++b) {
            yv[b] = T(0);
            if (b >= jn) break;
            const int64_t j = j0 + b;
            // crt.hpp:113-119, round_nearest_even (softfp.hpp:94-102): rint,
            // except that the reference's floor(x) + 1 returns +0.0 for x in
            // [-0.5, -0.0) where rint gives -0.0; adding +0.0 maps exactly that
            // -0.0 to +0.0 (qx itself is never -0.0: C1 is an fma chain from
            // +0.0 with s1_l > 0, so an exact zero sum is +0.0)
            const double qx = __dmul_rn(cc.P_inv, c1[b]);
            const double q = __dadd_rn(rint(qx), 0.0);
            const double t1 = __fma_rn(-q, cc.P1, c1[b]);         // crt.hpp:136-138
            const double t2 = __dadd_rn(t1, c2[b]);
            const double cpp = __fma_rn(-q, cc.P2, t2);
            const int64_t o = i * n + j;
            if (INTER) {
                if (ex.C1) ex.C1[o] = c1[b];
                if (ex.C2) ex.C2[o] = c2[b];
                if (ex.Q) ex.Q[o] = q;
                if (ex.Cpp64) ex.Cpp64[o] = cpp;
            }
            const int nuj = nuv[b];
            if (BND) {
                const BoundCtx& bc = ex.bnd;
                const double PBj = bc.v.PB[j], CBj = bc.v.CB[j];
                const int ebj = bc.v.eb[j];
                const double base = __dadd_ru(ldexp_ru(__dmul_ru(RAi, PBj), ebj), ldexp_ru(__dmul_ru(PAi, CBj), eai));
                const double pp = __dmul_ru(PAi, PBj);
                const double cheap =
                    __dadd_ru(base, ldexp_ru(__dmul_ru(__dmul_ru(bc.kpr_cheap_up, bc.t2_up), pp), eai + ebj));
                const double ab_up = __ddiv_ru(__dadd_ru(fabs(cpp), bc.rconst_up), 1.0 - bc.ucoef);
                const double kpr_t = __dadd_ru(bc.k_rconst_up, __dmul_ru(bc.ucoef, ab_up));
                const double tight = __dadd_ru(base, ldexp_ru(__dmul_ru(__dmul_ru(kpr_t, bc.t2_up), pp), eai + ebj));
                if (bc.cheap) bc.cheap[o] = cheap;
                if (bc.tight) bc.tight[o] = tight;
                const unsigned long long cb = (unsigned long long)__double_as_longlong(cheap);
                const unsigned long long tb = (unsigned long long)__double_as_longlong(tight);
                bmax_cheap = cb > bmax_cheap ? cb : bmax_cheap;
                bmax_tight = tb > bmax_tight ? tb : bmax_tight;
                if (bc.ab_lo) {  // tight / (|A||B|)_ij, rounded up against a lower bound of |A||B|
                    const double lv = bc.ab_lo[o];
                    const double rel = lv > 0.0 ? __ddiv_ru(tight, lv) : __longlong_as_double(0x7ff0000000000000ll);
                    const unsigned long long rb = (unsigned long long)__double_as_longlong(rel);
                    bmax_rel = rb > bmax_rel ? rb : bmax_rel;
                }
            }
            if constexpr (sizeof(T) == 4) {
                if (fabs(cpp) >= 0x1.ffffffp+127) { fr_range = true; continue; }  // crt.hpp:144-145
                const float c32 = __double2float_rn(cpp);
                if (INTER && ex.Cpp32) ex.Cpp32[o] = c32;
                const float x = fastsc ? __fmul_rn(c32, pmuf) : ldexpf_rn(c32, -mui);  // emulate.hpp:37-38
                const float y = fastsc ? __fmul_rn(x, pow2f(-nuj)) : ldexpf_rn(x, -nuj);
                const uint32_t ux = (__float_as_uint(x) >> 23) & 0xffu, uy = (__float_as_uint(y) >> 23) & 0xffu;
                if (((ux + 1u) & 0xfeu) == 0u || ((uy + 1u) & 0xfeu) == 0u) {  // zero / subnormal / inf / nan
                    inv_range |= !isfinite(x) || !isfinite(y);
                    sub |= (x != 0.0f && fabsf(x) < FLT_MIN) || (y != 0.0f && fabsf(y) < FLT_MIN);
                }
                yv[b] = y;
            } else {
                const double x = fastsc ? __dmul_rn(cpp, pmu) : ldexp_rn(cpp, -mui);
                const double y = fastsc ? __dmul_rn(x, pow2d(-nuj)) : ldexp_rn(x, -nuj);
                // exponent field 0 (zero, subnormal) or 0x7ff (inf, nan) in either: check
                // precisely (integer test on the high words; rarely taken)
                const uint32_t ux = ((uint32_t)__double2hiint(x) >> 20) & 0x7ffu;
                const uint32_t uy = ((uint32_t)__double2hiint(y) >> 20) & 0x7ffu;
                if (((ux + 1u) & 0x7feu) == 0u || ((uy + 1u) & 0x7feu) == 0u) {
                    inv_range |= !isfinite(x) || !isfinite(y);
                    sub |= (x != 0.0 && fabs(x) < DBL_MIN) || (y != 0.0 && fabs(y) < DBL_MIN);
                }
                yv[b] = y;
            }
        }
        // C: 32-byte stores when the thread's CV entries are whole and aligned
        // (a warp's stores then cover its 2 KB of C exactly once), else scalar
        T* crow = C + i * ldc + j0;
        if (jn == CV && (reinterpret_cast<uintptr_t>(crow) & 31) == 0) {
            if constexpr (sizeof(T) == 8) {
#pragma unroll
                for (int b = 0; b < CV; b += 4)
                    st_global_v4f64(reinterpret_cast<double*>(crow) + b, yv[b], yv[b + 1], yv[b + 2], yv[b + 3]);
            } else {
#pragma unroll
                for (int b = 0; b < CV; b += 4)
                    *reinterpret_cast<float4*>(crow + b) = make_float4(yv[b], yv[b + 1], yv[b + 2], yv[b + 3]);
            }
        } else {
#pragma unroll
            for (int b = 0; b < CV; ++b)
                if (b < jn) crow[b] = yv[b];
        }
        if (fr_range | inv_range | sub) {
            DevStatus* s = ex.sg.base ? ex.sg.base + ((ex.sg.row0 + i) / ex.sg.row_div) * ex.sg.slots +
                                            (ex.sg.col0 + j0) / ex.sg.col_div
                                      : st;
            if (fr_range) atomicOr(&s->err, (uint32_t)ERR_FR_RANGE);
            if (inv_range) atomicOr(&s->err, (uint32_t)ERR_INV_RANGE);
            if (sub) atomicOr(&s->subnormal, 1u);
        }
    }
    if (BND) {
        bmax_cheap = warp_max_u64(bmax_cheap);
        bmax_tight = warp_max_u64(bmax_tight);
        bmax_rel = warp_max_u64(bmax_rel);
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&ex.bnd.max_bits[0], bmax_cheap);
            atomicMax(&ex.bnd.max_bits[1], bmax_tight);
            if (ex.bnd.ab_lo) atomicMax(&ex.bnd.max_bits[2], bmax_rel);
        }
    }
}

template <class T, bool DD, int NFP, bool INTER, int CV>
cudaError_t launch_n(cudaStream_t s, const int8_t* W, int64_t ldw, int64_t wplane, int64_t m, int64_t n,
                     const CrtConsts& cc, const int32_t* mu, const int32_t* nu, T* C, int64_t ldc, const CrtExtra& ex,
                     DevStatus* st) {
    const int64_t work = m * ((n + CV - 1) / CV);
    const unsigned grid = (unsigned)((work + 255) / 256);
    if (ex.bnd.on)
        return launch_pdl(crt_kernel<T, DD, true, NFP, INTER, CV>, dim3(grid), dim3(256), 0, s, W, ldw, wplane, m, n,
                          cc, mu, nu, C, ldc, ex, st);
    return launch_pdl(crt_kernel<T, DD, false, NFP, INTER, CV>, dim3(grid), dim3(256), 0, s, W, ldw, wplane, m, n, cc,
                      mu, nu, C, ldc, ex, st);
}

int crt_cv() { return opt(OPT_CRT_CV) == 4 ? 4 : 8; }

// Conversions on the fp64 pipe: 3 of 8 with the double-double chain (two DFMA
// per byte; measured best of {0, 3, 5, 8} at 16384^2, N = 16), 6 of 8 with the
// single chain of fp32 mode (one DFMA per byte); half of that with 4 columns.
template <class T, bool DD>
cudaError_t launch_t(cudaStream_t s, const int8_t* W, int64_t ldw, int64_t wplane, int64_t m, int64_t n,
                     const CrtConsts& cc, const int32_t* mu, const int32_t* nu, T* C, int64_t ldc, const CrtExtra& ex,
                     DevStatus* st) {
    const bool inter = ex.C1 || ex.C2 || ex.Q || ex.Cpp64 || ex.Cpp32;
    if (crt_cv() == 4) {
        constexpr int NFP = DD ? 2 : 3;
        if (inter) return launch_n<T, DD, NFP, true, 4>(s, W, ldw, wplane, m, n, cc, mu, nu, C, ldc, ex, st);
        return launch_n<T, DD, NFP, false, 4>(s, W, ldw, wplane, m, n, cc, mu, nu, C, ldc, ex, st);
    }
    constexpr int NFP = DD ? 3 : 6;
    if (inter) return launch_n<T, DD, NFP, true, 8>(s, W, ldw, wplane, m, n, cc, mu, nu, C, ldc, ex, st);
    return launch_n<T, DD, NFP, false, 8>(s, W, ldw, wplane, m, n, cc, mu, nu, C, ldc, ex, st);
}

}  // namespace

cudaError_t launch_crt(int prec, const int8_t* W, int64_t ldw, int64_t wplane, int64_t m, int64_t n,
                       const CrtConsts& cc, const int32_t* mu, const int32_t* nu, void* C, int64_t ldc,
                       const CrtExtra& extra, DevStatus* st, cudaStream_t s) {
    if (m * n == 0) return cudaSuccess;
    if (prec) {
        if (cc.mode == 1) return launch_t<double, true>(s, W, ldw, wplane, m, n, cc, mu, nu, (double*)C, ldc, extra, st);
        return launch_t<double, false>(s, W, ldw, wplane, m, n, cc, mu, nu, (double*)C, ldc, extra, st);
    }
    return launch_t<float, false>(s, W, ldw, wplane, m, n, cc, mu, nu, (float*)C, ldc, extra, st);
}

}  // namespace oz2g
