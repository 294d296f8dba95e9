// fused.cu — the N residue GEMMs with the Chinese-Remainder reconstruction
// and the inverse scaling in their epilogue (the north star's stage 3: no
// residue product ever reaches HBM).
//
// Replaces, for one C tile at a time, the chain
//   residue_gemm_and_reduce  crt.hpp:69-79     (W_l = signed_mod(A'_l B'_l, p_l))
//   accumulate               crt.hpp:91-110    (C1, C2 ordered fma chains over l)
//   compute_q / final_reduce crt.hpp:113-150
//   inverse_scale            emulate.hpp:30-46
// that the two-pass path (gemm_tc.cu EPI_RESID writing int8 W per plane, then
// crt.cu) runs as two kernels.
//
// A CTA owns a 128 x 128 tile of C and walks the planes l = 0 .. N-1 in order:
//   warp 0        TMA producer: A_l tile 128 x 128 B (K-major), B_l tile 128
//                 columns x 128 K-rows (MN-major), 6-stage ring;
//   warp 1        TMEM allocator + MMA issuer: 4 x tcgen05.mma kind::i8
//                 128x128x32 per stage into accumulator l & 1 (two 128-column
//                 TMEM buffers, so plane l+1 multiplies while plane l is folded);
//   warps 2..9    epilogue, 8 warps: warp w reads TMEM lanes 32 (w % 4) ..
//                 (the tcgen05.ld lane restriction) and columns 64 ((w-2) / 4)
//                 .. +63, so each thread owns 64 entries of one row.
// Per entry the state across planes is C1 (fp64, in the thread's registers
// for 32 of its entries, in shared memory for the other 32) and C2 (fp64, in
// TMEM columns 256..511 — 2 columns per entry), both updated
// by the reference's fma in plane order l = 0, 1, ..., so C1 and C2 are the
// reference's ordered chains bit for bit (in fp64 mode C1 is even exact,
// Lemma 2; in fp32 mode it is not, and the order is what makes it match).
// After plane N-1 the thread finishes its 64 entries: Q, C'', the fp32 guard,
// the two ldexp of the inverse scaling, the subnormal / range flags, and
// writes C.  Accumulators 2 x 128 + C2 256 = all 512 TMEM columns.
#include <cfloat>
#include <cstdlib>

#include <cstdio>

#include "device_common.cuh"
#include "kernels.h"

namespace oz2g {

namespace {

constexpr int FBM = 128, FBN = 128, FBK = 128, FSTAGES = 5;
constexpr int FA_BYTES = FBM * FBK;  // 16 KB
constexpr int FB_BYTES = FBN * FBK;  // 16 KB (one MN-major box: 128 columns x 128 K-rows)
constexpr int F_EPI_WARPS = 8;
constexpr int F_COLS = FBN / (F_EPI_WARPS / 4);  // columns of the tile per epilogue thread
constexpr int F_THREADS = 64 + 32 * F_EPI_WARPS;
constexpr uint32_t FIDESC = idesc_i8(FBM, FBN, true);
// C1 of the upper half of each thread's columns lives in shared memory
// ([column][row] doubles: a warp's lanes hit consecutive words), the lower half
// in registers: 10 warps are 3 per SM sub-partition, whose 16K registers
// allow 168 per thread, too few for 64 fp64 accumulators plus the work.
constexpr int F_COLS_REG = 32;
constexpr int F_C1S_BYTES = (FBN / 2) * FBM * 8;  // 64 KB: 2 column groups x 32 columns x 128 rows
constexpr int F_SMEM = FSTAGES * (FA_BYTES + FB_BYTES) + F_C1S_BYTES + 1024 + 256;
constexpr uint32_t F_C2_COL = 256;  // first TMEM column of the C2 state

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Grouped raster over the C tiles (B tiles reused across group_m tile-rows).
__device__ __forceinline__ void decode_tile(int u, int tiles_m, int tiles_n, int group_m, int& tm, int& tn) {
    const int group = group_m * tiles_n;
    const int g = u / group;
    const int first_m = g * group_m;
    const int gm = min(tiles_m - first_m, group_m);
    const int r = u - g * group;
    tm = first_m + r % gm;
    tn = r / gm;
}

// W = signed_mod(C', p) (softfp.hpp:117-125 with the p/2 tie to -p/2),
// branch-free for every modulus: r = (C' + off) mod p with off a multiple of
// p >= 2^31; the representative is r - p when 2r >= p (for odd p the same as
// 2r > p; for p = 256, magic = 2^24 makes q exact and maps 128 to -128 as the
// two-pass epilogue's byte cast does).  Returned as the exact double
// W = (2^52 + 128 + W) - (2^52 + 128), built on the fp64 pipe (the I2F
// conversion would run on the XU pipe, the epilogue's bottleneck).
__device__ __forceinline__ double residue_wd(uint32_t v, uint32_t p, uint32_t magic, uint32_t off) {
    const uint32_t x = v + off;
    const uint32_t q = __umulhi(x, magic);
    uint32_t r = x - q * p;
    r = r >= p ? r - p : r;
    const uint32_t biased = (2u * r >= p ? r - p : r) + 128u;  // W + 128 in [0, 255]
    return __dsub_rn(__hiloint2double(0x43300000, (int)biased), 4503599627370624.0);
}

// Diagnostics (FusedParams.dbg): a barrier wait bounded to ~2^32 clocks that
// reports the stalled barrier and gives up instead of hanging.
__device__ __noinline__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int tag, int a, int b) {
    const long long t0 = clock64();
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680) : "memory");
        if (ok) return;
        if (clock64() - t0 > (1ll << 32)) {
            unsigned long long raw;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(raw) : "r"(smem_u32(bar)));
            if ((threadIdx.x & 31) == 0)
                printf("oz2g fused stall: block %d warp %d barrier %d (parity %u) at %d / %d raw %016llx\n",
                       (int)blockIdx.x, (int)(threadIdx.x >> 5), tag, parity, a, b, raw);
            return;
        }
    }
}

// MC: CTAs run in clusters of 2 on vertically adjacent tiles that share the
// B tile; each CTA loads half of the B stage's K-rows with .multicast::cluster
// into both CTAs (B crosses L2 -> SM once per pair), and a stage is refilled
// only when both CTAs' MMAs have read it (commits multicast to both).
template <class T, bool DD, bool MC>
__global__ void __launch_bounds__(F_THREADS, 1)
    gemm_crt_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ FusedParams P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + FSTAGES * FA_BYTES;
    double* c1s = reinterpret_cast<double*>(sB + FSTAGES * FB_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + FSTAGES * FB_BYTES + F_C1S_BYTES);
    uint64_t* empty = full + FSTAGES;
    uint64_t* tfull = empty + FSTAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const GemmParams& G = P.g;

    const uint32_t rank = MC ? cluster_ctarank() : 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < FSTAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MC ? 2 : 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], F_EPI_WARPS); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
    if (warp == 1) { tmem_alloc(tmem_slot, 512); tmem_relinquish(); }
    tc_fence_before();
    if (MC) cluster_sync_all();  // the peer's barriers exist before any multicast reaches them
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // work units: tiles (or vertically adjacent tile pairs for MC) in raster order
    const int units_m = MC ? (G.tiles_m + 1) >> 1 : G.tiles_m;
    const int ugroup = MC ? max(1, G.group_m >> 1) : G.group_m;
    const int total = units_m * G.tiles_n;
    const int first = MC ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int stride = MC ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int N = G.planes;

    if (warp == 0) {
        // ===== TMA producer: for each tile, planes in order, all of K =====
        // Plane fence: before the loads of its g-th plane step a CTA waits until
        // every CTA has issued all loads of its first g steps, so the CTAs of a
        // wave stay within one plane of each other and the wave's operand blocks
        // (~50 MB per plane at k = 16384) stay in L2 — unsynchronised, the CTAs
        // drift over several planes and re-read the planes from HBM (381 GB per
        // 16384^3 call, measured).  Bounded wait: a CTA that is not resident
        // (another kernel holds its SM) only costs the time-out, not a hang.
        int stage = 0;
        uint32_t phase = 0;
        uint32_t g = 0;
        const uint32_t steps_total = (uint32_t)((total + stride - 1) / stride) * (uint32_t)N;
        for (int u = first; u < total; u += stride) {
            int tm, tn;
            decode_tile(u, units_m, G.tiles_n, ugroup, tm, tn);
            if (MC) tm = 2 * tm + (int)rank;  // rows past m are TMA zero fill
            for (int l = 0; l < N; ++l, ++g) {
                if (P.plane_sync && lane == 0) {
                    const unsigned long long need = (unsigned long long)g * gridDim.x;
                    const long long t0 = clock64();
                    while (ld_acquire_u64(P.plane_sync) < need && clock64() - t0 < (1ll << 26)) __nanosleep(64);
                }
                __syncwarp();
                for (int kb = 0; kb < G.kblocks; ++kb) {
                    if (P.dbg) mbar_wait_dbg(&empty[stage], phase ^ 1u, 1, u, l);
                    else mbar_wait(&empty[stage], phase ^ 1u);
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&full[stage], FA_BYTES + FB_BYTES);
                        tma_load_3d(sA + stage * FA_BYTES, &tmA, &full[stage], kb * FBK, tm * FBM, l, G.hintA);
                        if (MC)  // this CTA's half of the K-rows, into both CTAs of the pair
                            tma_load_3d_mc(sB + stage * FB_BYTES + (int)rank * (FB_BYTES / 2), &tmB, &full[stage],
                                           tn * FBN, kb * FBK + (int)rank * (FBK / 2), l, (uint16_t)0x3, G.hintB);
                        else
                            tma_load_3d(sB + stage * FB_BYTES, &tmB, &full[stage], tn * FBN, kb * FBK, l, G.hintB);
                    }
                    __syncwarp();
                    if (++stage == FSTAGES) { stage = 0; phase ^= 1u; }
                }
                if (P.plane_sync && lane == 0) atomicAdd(P.plane_sync, 1ull);
            }
        }
        // CTAs with fewer tiles release the steps they do not have
        if (P.plane_sync && lane == 0 && g < steps_total) atomicAdd(P.plane_sync, (unsigned long long)(steps_total - g));
        if (MC) {  // every stage released by both CTAs before the pair may exit (the peer's commits target us)
            for (int s2 = 0; s2 < FSTAGES; ++s2) {
                if (P.dbg) mbar_wait_dbg(&empty[stage], phase ^ 1u, 2, s2, stage);
                else mbar_wait(&empty[stage], phase ^ 1u);
                if (++stage == FSTAGES) { stage = 0; phase ^= 1u; }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: plane l of a tile into accumulator (running plane count) & 1 =====
        const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA));
        const uint64_t bdesc0 = umma_desc_sw128_mn(smem_u32(sB), FB_BYTES);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int u = first; u < total; u += stride) {
            for (int l = 0; l < N; ++l, ++it) {
                const int acc = it & 1;
                if (P.dbg) mbar_wait_dbg(&tempty[acc], (uint32_t)((it >> 1) & 1) ^ 1u, 3, u, l);
                else mbar_wait(&tempty[acc], (uint32_t)((it >> 1) & 1) ^ 1u);
                tc_fence_after();
                const uint32_t dtmem = tmem_base + (uint32_t)(acc * FBN);
                for (int kb = 0; kb < G.kblocks; ++kb) {
                    if (P.dbg) mbar_wait_dbg(&full[stage], phase, 4, u, l);
                    else mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        // descriptors = the stage-0 descriptor + the byte offset / 16 in the
                        // 14-bit address field (shared addresses < 2^18: no carry out)
                        const uint64_t ad = adesc0 + (uint64_t)((stage * FA_BYTES) >> 4);
                        const uint64_t bd = bdesc0 + (uint64_t)((stage * FB_BYTES) >> 4);
#pragma unroll
                        for (int k = 0; k < FBK / 32; ++k)
                            mma_i8(dtmem, ad + (uint64_t)(k * 32 >> 4), bd + (uint64_t)(k * 32 * 128 >> 4), FIDESC,
                                   (kb | k) != 0 ? 1u : 0u);
                        if (MC) mma_commit_mc(&empty[stage], (uint16_t)0x3);
                        else mma_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == FSTAGES) { stage = 0; phase ^= 1u; }
                }
                if (lane == 0) mma_commit(&tfull[acc]);
                __syncwarp();
            }
        }
    } else {
        // ===== Epilogue: 32 entries of one row per thread, state over the planes =====
        const int quad = warp & 3;            // TMEM lanes 32 quad .. 32 quad + 31
        const int cgrp = (warp - 2) >> 2;     // columns F_COLS cgrp .. F_COLS (cgrp + 1) - 1 of the tile
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        int it = 0;
        uint32_t err_bits = 0, sub = 0;
        for (int u = first; u < total; u += stride) {
            int tm, tn;
            decode_tile(u, units_m, G.tiles_n, ugroup, tm, tn);
            if (MC) tm = 2 * tm + (int)rank;
            const int64_t row = (int64_t)tm * FBM + quad * 32 + lane;
            const int64_t col0 = (int64_t)tn * FBN + cgrp * F_COLS;
            double c1[F_COLS_REG];                           // columns 0 .. 31 of the thread's 64
#pragma unroll
            for (int j = 0; j < F_COLS_REG; ++j) c1[j] = 0.0;   // crt.hpp:99: both chains start at +0.0
            // columns 32 .. 63: c1s[(cgrp * 32 + j) * 128 + row in tile]
            double* c1x = c1s + (size_t)cgrp * 32 * FBM + quad * 32 + lane;
            for (int l = 0; l < N; ++l, ++it) {
                const int acc = it & 1;
                if (P.dbg) mbar_wait_dbg(&tfull[acc], (uint32_t)((it >> 1) & 1), 5, u, l);
                else mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
                tc_fence_after();
                if (P.probe == 1) {  // experiment: MMA + operand feed alone (no CRT; C not written)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    continue;
                }
                const uint32_t p = G.p[l], magic = G.magic[l], off = G.off[l];
                const double s1 = P.s1[l], s2 = P.s2[l];
                const bool last = l == N - 1;
                const bool live = row < G.m;
                const int mui = (last && live) ? P.mu[row] : 0;
#pragma unroll
                for (int ch = 0; ch < F_COLS / 8; ++ch) {
                    __syncwarp();  // the tcgen05.ld / .st below are warp-collective
                    uint32_t v[8];
                    tmem_ld8(lane_base + (uint32_t)(acc * FBN + cgrp * F_COLS + ch * 8), v);
                    uint32_t c2w[16];
                    if (DD && l > 0) tmem_ld16(lane_base + F_C2_COL + (uint32_t)(cgrp * 2 * F_COLS + ch * 16), c2w);
                    tmem_ld_wait();
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const double wv = residue_wd(v[b], p, magic, off);
                        const int jj = ch * 8 + b;
                        if (jj < F_COLS_REG) {
                            c1[jj] = __fma_rn(s1, wv, c1[jj]);                          // crt.hpp:99-104
                        } else {
                            double* cp = c1x + (size_t)(jj - F_COLS_REG) * FBM;
                            *cp = __fma_rn(s1, wv, l > 0 ? *cp : 0.0);
                        }
                        if (DD) {
                            const double prev = l > 0 ? __hiloint2double((int)c2w[2 * b + 1], (int)c2w[2 * b]) : 0.0;
                            const double c2 = __fma_rn(s2, wv, prev);
                            c2w[2 * b] = (uint32_t)__double2loint(c2);
                            c2w[2 * b + 1] = (uint32_t)__double2hiint(c2);
                        }
                    }
                    if (!last) {
                        if (DD) tmem_st16(lane_base + F_C2_COL + (uint32_t)(cgrp * 2 * F_COLS + ch * 16), c2w);
                    } else if (live) {
                    // ---- plane N-1 folded: finish these 8 entries (crt.hpp:113-150, emulate.hpp:30-46) ----
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const int64_t j = col0 + ch * 8 + b;
                        if (j >= G.n) break;
                        const int jj = ch * 8 + b;
                        const double c1v = jj < F_COLS_REG ? c1[jj] : c1x[(size_t)(jj - F_COLS_REG) * FBM];
                        const double c2v = DD ? __hiloint2double((int)c2w[2 * b + 1], (int)c2w[2 * b]) : 0.0;
                        const double qx = __dmul_rn(P.P_inv, c1v);
                        double q = rint(qx);
                        if (q == 0.0 && qx != 0.0) q = 0.0;  // round_nearest_even's +0.0 (crt.cu)
                        const double t1 = __fma_rn(-q, P.P1, c1v);
                        const double t2 = __dadd_rn(t1, c2v);
                        const double cpp = __fma_rn(-q, P.P2, t2);
                        const int nuj = __ldg(P.nu + j);
                        if constexpr (sizeof(T) == 4) {
                            if (fabs(cpp) >= 0x1.ffffffp+127) { err_bits |= ERR_FR_RANGE; continue; }
                            const float c32 = __double2float_rn(cpp);
                            const float x = ldexpf_rn(c32, -mui);
                            const float y = ldexpf_rn(x, -nuj);
                            if (!isfinite(x) || !isfinite(y)) err_bits |= ERR_INV_RANGE;
                            sub |= (x != 0.0f && fabsf(x) < FLT_MIN) || (y != 0.0f && fabsf(y) < FLT_MIN);
                            reinterpret_cast<float*>(P.C)[row * P.ldc + j] = y;
                        } else {
                            const double x = ldexp_rn(cpp, -mui);
                            const double y = ldexp_rn(x, -nuj);
                            if (!isfinite(x) || !isfinite(y)) err_bits |= ERR_INV_RANGE;
                            sub |= (x != 0.0 && fabs(x) < DBL_MIN) || (y != 0.0 && fabs(y) < DBL_MIN);
                            reinterpret_cast<double*>(P.C)[row * P.ldc + j] = y;
                        }
                    }
                    }
                }
                if (DD && !last) tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
            }
        }
        if (err_bits) atomicOr(&P.st->err, err_bits);
        if (sub) atomicOr(&P.st->subnormal, 1u);
    }

    tc_fence_before();
    if (MC) cluster_sync_all();
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

template <class T, bool DD, bool MC>
cudaError_t launch_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const FusedParams& P, int grid,
                     cudaStream_t stream) {
    static int configured[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        const cudaError_t err = cudaFuncSetAttribute(gemm_crt_fused_kernel<T, DD, MC>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
        if (err != cudaSuccess) return err;
        configured[dev] = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(F_THREADS);
    cfg.dynamicSmemBytes = F_SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = MC ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_crt_fused_kernel<T, DD, MC>, tmA, tmB, P);
}

template <class T, bool DD>
cudaError_t launch_mc(bool mc, const CUtensorMap& tmA, const CUtensorMap& tmB, const FusedParams& P, int grid,
                      cudaStream_t stream) {
    return mc ? launch_t<T, DD, true>(tmA, tmB, P, grid, stream) : launch_t<T, DD, false>(tmA, tmB, P, grid, stream);
}

}  // namespace

int fused_tile_m() { return FBM; }
int fused_tile_n() { return FBN; }

int fused_b_box_rows(bool mc) { return mc ? FBK / 2 : FBK; }

cudaError_t launch_gemm_crt_fused(int prec, const CUtensorMap& tmA, const CUtensorMap& tmB, const FusedParams& P,
                                  int num_sms, bool mc, cudaStream_t stream) {
    const int units = (mc ? (P.g.tiles_m + 1) / 2 : P.g.tiles_m) * P.g.tiles_n;
    if (units == 0) return cudaSuccess;
    const int per = mc ? 2 : 1;
    const int slots = num_sms / per;
    const int grid = (units < slots ? units : slots) * per;
    const bool dd = P.mode != 0;
    if (prec) return dd ? launch_mc<double, true>(mc, tmA, tmB, P, grid, stream)
                        : launch_mc<double, false>(mc, tmA, tmB, P, grid, stream);
    return dd ? launch_mc<float, true>(mc, tmA, tmB, P, grid, stream) : launch_mc<float, false>(mc, tmA, tmB, P, grid, stream);
}

}  // namespace oz2g
