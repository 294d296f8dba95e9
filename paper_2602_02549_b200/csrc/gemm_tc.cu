// gemm_tc.cu — INT8 x INT8 -> INT32 GEMMs of the Ozaki-II scheme on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, sm_100a).
//
// Replaces the reference's software INT8 engine
//   gemm_i8_wrap       /root/reference/proj/include/oz2/int8gemm.hpp:17-34
// at its two call sites, each with a fused epilogue so that the INT32 product
// is never written to HBM:
//   EPI_MAX   clearance_product (scaling.hpp:140-148) + the row/column maxima
//             of scaling_exponents (scaling.hpp:175-192): per-tile max, then
//             one atomicMax per row / column.  (fp32_round_up and log2f are
//             monotone, so max commutes with them; they run later on m+n
//             scalars.)
//   EPI_RESID residue_gemm_and_reduce (crt.hpp:69-79): W = signed_mod(C', p)
//             with the p/2 tie mapped to -p/2, stored as int8.
//   EPI_I32   debug/evidence: store the wrapped INT32 product itself.
//
// Exactness: |a|,|b| <= 128 and k <= 2^17 give |sum| <= 2^31; the tensor core
// accumulates in 32-bit two's complement, which is exactly the reference's
// uint32 wraparound (int8gemm.hpp:24-30) — and for p = 256 the residue
// survives the wrap because 256 | 2^32.
//
// Kernel shape: persistent, one CTA per SM, 256 threads —
//   warp 0      TMA producer (one elected lane): A tile 128x128 B and
//               B tile 128 rows x 256 columns per stage (two 128-column
//               boxes), 128-byte swizzle, 4 stages;
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma 128x256x32 per stage
//               into a TMEM accumulator (2 x 256 columns, double-buffered);
//   warp 2      TMEM allocator;
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns, fused reduction.
// A is K-major (planes [l][m][kp]); B is MN-major in its own row-major layout
// (planes [l][kp][ldn], ldn = n rounded to 16), which tcgen05 accepts for INT8
// (instruction-descriptor bit 16), so B's planes are written without a
// transpose.
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace oz2g {

namespace {

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_BYTES = BM * BK;  // 16 KB
constexpr int B_BYTES = BN * BK;  // 32 KB
// B is MN-major ([plane][k][n] in HBM, B's own layout): a B tile is two TMA
// boxes of 128 columns x BK rows, B_CHUNK bytes apart in shared memory
constexpr int B_CHUNK = 128 * BK;  // 16 KB
constexpr uint32_t IDESC = idesc_i8(BM, BN, true);
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 1024 /*align*/ + 256 /*barriers*/;

struct TileCoord { int l, tm, tn; };

// Grouped raster: group_m > 0 walks groups of group_m tile-rows column by
// column (B tiles reused across the group); group_m < 0 walks groups of
// -group_m tile-columns row by row (A tiles reused).
__device__ __forceinline__ TileCoord decode_unit(int u, int tiles_m, int tiles_n, int group_m) {
    const int per_plane = tiles_m * tiles_n;
    TileCoord c;
    c.l = u / per_plane;
    const int t = u - c.l * per_plane;
    if (group_m > 0) {
        const int group = group_m * tiles_n;
        const int g = t / group;
        const int first_m = g * group_m;
        const int gm = min(tiles_m - first_m, group_m);
        const int r = t - g * group;
        c.tm = first_m + r % gm;
        c.tn = r / gm;
    } else {
        const int group_n = -group_m;
        const int group = group_n * tiles_m;
        const int g = t / group;
        const int first_n = g * group_n;
        const int gn = min(tiles_n - first_n, group_n);
        const int r = t - g * group;
        c.tn = first_n + r % gn;
        c.tm = r / gn;
    }
    return c;
}

template <int MODE>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&v)[32], int row, int col0, int l,
                                               const GemmParams& P) {
    const int lane = threadIdx.x & 31;
    if constexpr (MODE == EPI_MAX) {
        // row max over this chunk (values are exact non-negative integers)
        int32_t rmax = 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) rmax = max(rmax, (int32_t)v[c]);
        // column max across the 32 rows of this warp: lane c keeps column c
        int32_t mine = 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            const int32_t cm = (int32_t)__reduce_max_sync(0xffffffffu, v[c]);
            if (lane == c) mine = cm;
        }
        // columns beyond n and rows beyond m hold TMA zero-fill (harmless for max)
        if (col0 + lane < P.n) atomicMax(&P.colmax[col0 + lane], mine);
        if (row < P.m) {
            // accumulate the row max in a register across chunks: done by caller
            (void)rmax;
        }
    } else if constexpr (MODE == EPI_RESID) {
        if (row >= P.m) return;
        const uint32_t p = P.p[l];
        uint32_t packed[8];
        if (p == 256u) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                packed[c] = (v[4 * c] & 0xffu) | ((v[4 * c + 1] & 0xffu) << 8) | ((v[4 * c + 2] & 0xffu) << 16) |
                            ((v[4 * c + 3] & 0xffu) << 24);
        } else {
            const ModP mp{p, P.magic[l]};
            const uint32_t off = P.off[l];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint32_t word = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t r = mod_u32(v[4 * c + b] + off, mp);  // (C' mod p) in [0, p)
                    const int32_t w = (2u * r > p) ? (int32_t)r - (int32_t)p : (int32_t)r;
                    word |= ((uint32_t)w & 0xffu) << (8 * b);
                }
                packed[c] = word;
            }
        }
        int8_t* dst = P.W + (int64_t)l * P.wplane + (int64_t)row * P.ldw + col0;
        if (col0 + 32 <= P.n) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
            d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        } else {
            for (int c = 0; c < 32 && col0 + c < P.n; ++c) dst[c] = (int8_t)((packed[c >> 2] >> (8 * (c & 3))) & 0xff);
        }
    } else {  // EPI_I32
        if (row >= P.m) return;
        int32_t* dst = P.C32 + (int64_t)l * P.cplane + (int64_t)row * P.ldc32 + col0;
        for (int c = 0; c < 32 && col0 + c < P.n; ++c) dst[c] = (int32_t)v[c];
    }
}

// 8 epilogue warps (warps 4..11): warp w reads TMEM lanes 32 (w % 4) .. and
// the column half (w - 4) / 4 of the 256-column accumulator, so the epilogue
// of a tile takes half as long — it bounds the GEMM when k is small (each
// tile's MMAs then take little longer than its epilogue).
constexpr int tc_threads(int epi_warps) { return 128 + 32 * epi_warps; }

template <int MODE, int EPI_WARPS>
__global__ void __launch_bounds__(tc_threads(EPI_WARPS), 1)
    gemm_i8_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], EPI_WARPS); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
    if (warp == 2) { tmem_alloc(tmem_slot, 512); tmem_relinquish(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // the set-up above overlaps the previous kernel's tail

    const int total = P.planes * P.tiles_m * P.tiles_n;

    if (warp == 0) {
        // ===== TMA producer =====
        int stage = 0;
        uint32_t phase = 0;
        unsigned long long j = 0;
        for (int u = blockIdx.x; u < total; u += gridDim.x, ++j) {
            const TileCoord tc = decode_unit(u, P.tiles_m, P.tiles_n, P.group_m);
            if (P.fence && lane == 0) step_fence_wait(P.fence, j * gridDim.x);
            __syncwarp();
            for (int kb = 0; kb < P.kblocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1u);
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[stage], A_BYTES + B_BYTES);
                    // A row groups are reused by every wave of a raster group: keep them in L2;
                    // B tiles stream through
                    tma_load_3d(sA + stage * A_BYTES, &tmA, &full[stage], kb * BK, tc.tm * BM, tc.l, P.hintA);
                    tma_load_3d(sB + stage * B_BYTES, &tmB, &full[stage], tc.tn * BN, kb * BK, tc.l, P.hintB);
                    tma_load_3d(sB + stage * B_BYTES + B_CHUNK, &tmB, &full[stage], tc.tn * BN + 128, kb * BK, tc.l,
                                P.hintB);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
            if (P.fence && lane == 0) atomicAdd(P.fence, 1ull);
        }
        if (P.fence && lane == 0) {  // release the units this CTA does not have
            const unsigned long long steps = (unsigned long long)((total + (int)gridDim.x - 1) / (int)gridDim.x);
            if (j < steps) atomicAdd(P.fence, steps - j);
        }
        // the next kernel may be scheduled once every CTA has issued its last
        // loads (earlier, its waiting CTAs would sit beside the whole GEMM)
        if (lane == 0) pdl_trigger();
    } else if (warp == 1) {
        // ===== MMA issuer =====
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t aph = (uint32_t)((it >> 1) & 1);
            mbar_wait(&tempty[acc], aph ^ 1u);
            tc_fence_after();
            const uint32_t dtmem = tmem_base + (uint32_t)(acc * BN);
            for (int kb = 0; kb < P.kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k)
                        mma_i8(dtmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128_mn(b0 + k * 32 * 128, B_CHUNK), IDESC,
                               (kb | k) != 0 ? 1u : 0u);
                    mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
            if (lane == 0) mma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== Epilogue =====
        const int wq = warp & 3;                                  // TMEM lane quadrant
        const int c_lo = ((warp - 4) / 4) * (BN / 32 / (EPI_WARPS / 4));  // first 32-column chunk
        const int c_hi = c_lo + BN / 32 / (EPI_WARPS / 4);
        int it = 0;
        for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
            const TileCoord tc = decode_unit(u, P.tiles_m, P.tiles_n, P.group_m);
            const int acc = it & 1;
            const uint32_t aph = (uint32_t)((it >> 1) & 1);
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = tc.tm * BM + wq * 32 + lane;
            int32_t rowmax = 0;
#pragma unroll 1
            for (int c = c_lo; c < c_hi; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
                tmem_ld_wait();
                const int col0 = tc.tn * BN + c * 32;
                if constexpr (MODE == EPI_MAX) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) rowmax = max(rowmax, (int32_t)v[j]);
                }
                epilogue_chunk<MODE>(v, row, col0, tc.l, P);
            }
            if constexpr (MODE == EPI_MAX) {
                if (row < P.m) atomicMax(&P.rowmax[row], rowmax);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }

    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------------------
// Multicast variant: a cluster of 2 CTAs computes two vertically adjacent
// 128 x 256 tiles that share one B tile.  Each CTA loads its own A tile and
// HALF of the B tile with .multicast::cluster into both CTAs' shared memory,
// so B crosses L2 -> SM once per pair; MMAs stay cta_group::1 (each CTA owns
// its accumulator).  A stage may be refilled only when both CTAs' MMAs have
// read it: every MMA commit arrives on the empty barrier of both CTAs.
// ---------------------------------------------------------------------------
constexpr int MC_HALF_B = B_CHUNK;  // 128 columns of B x BK rows

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_i8_tc_mc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
    if (warp == 2) { tmem_alloc(tmem_slot, 512); tmem_relinquish(); }
    tc_fence_before();
    cluster_sync_all();  // the peer's barriers exist before any multicast reaches them
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int clusters = gridDim.x >> 1;
    const int cid = blockIdx.x >> 1;
    const int tiles_m2 = (P.tiles_m + 1) >> 1;  // tile-row pairs
    const int total = P.planes * tiles_m2 * P.tiles_n;
    const int group2 = P.group_m > 1 ? P.group_m >> 1 : 1;

    if (warp == 0) {
        // ===== TMA producer (both CTAs) =====
        int stage = 0;
        uint32_t phase = 0;
        for (int u = cid; u < total; u += clusters) {
            const TileCoord tc = decode_unit(u, tiles_m2, P.tiles_n, group2);
            const int arow = (2 * tc.tm + (int)rank) * BM;  // rows past m are TMA zero fill
            const int bcol = tc.tn * BN + (int)rank * (BN / 2);
            for (int kb = 0; kb < P.kblocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1u);
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[stage], A_BYTES + B_BYTES);
                    tma_load_3d(sA + stage * A_BYTES, &tmA, &full[stage], kb * BK, arow, tc.l, P.hintA);
                    tma_load_3d_mc(sB + stage * B_BYTES + (int)rank * MC_HALF_B, &tmB, &full[stage], bcol, kb * BK,
                                   tc.l, (uint16_t)0x3, P.hintB);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
        }
        // producer tail: every stage released by both CTAs before the cluster
        // may exit (the peer's last commits target our barriers)
        for (int s = 0; s < STAGES; ++s) {
            mbar_wait(&empty[stage], phase ^ 1u);
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (each CTA, its own accumulator) =====
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int u = cid; u < total; u += clusters, ++it) {
            const int acc = it & 1;
            const uint32_t aph = (uint32_t)((it >> 1) & 1);
            mbar_wait(&tempty[acc], aph ^ 1u);
            tc_fence_after();
            const uint32_t dtmem = tmem_base + (uint32_t)(acc * BN);
            for (int kb = 0; kb < P.kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k)
                        mma_i8(dtmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128_mn(b0 + k * 32 * 128, B_CHUNK), IDESC,
                               (kb | k) != 0 ? 1u : 0u);
                    mma_commit_mc(&empty[stage], (uint16_t)0x3);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
            if (lane == 0) mma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== Epilogue =====
        const int wq = warp - 4;
        int it = 0;
        for (int u = cid; u < total; u += clusters, ++it) {
            const TileCoord tc = decode_unit(u, tiles_m2, P.tiles_n, group2);
            const int acc = it & 1;
            const uint32_t aph = (uint32_t)((it >> 1) & 1);
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = (2 * tc.tm + (int)rank) * BM + wq * 32 + lane;
            int32_t rowmax = 0;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
                tmem_ld_wait();
                const int col0 = tc.tn * BN + c * 32;
                if constexpr (MODE == EPI_MAX) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) rowmax = max(rowmax, (int32_t)v[j]);
                }
                epilogue_chunk<MODE>(v, row, col0, tc.l, P);
            }
            if constexpr (MODE == EPI_MAX) {
                if (row < P.m) atomicMax(&P.rowmax[row], rowmax);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant: a cluster of 2 CTAs computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 256).  Each CTA loads its 128-row half
// of A and its 128-row half of B^T per stage (32 KB instead of 48 KB for the
// same MACs per SM) and keeps its 128 x 256 half of the accumulator in its own
// TMEM.  The even CTA ("leader") issues the MMAs; its full barrier receives the
// transaction bytes of both CTAs' TMA loads; MMA completion is committed with
// multicast to the barriers of both CTAs; both CTAs' epilogue warps release an
// accumulator stage on the leader's tmem-empty barrier.
// ---------------------------------------------------------------------------
constexpr int P_BM = 256, P_BN = 256;     // pair tile
constexpr int P_HALF = 128;               // rows of A and columns of B per CTA
constexpr int P_STAGE_BYTES = 2 * P_HALF * BK;  // 32 KB per CTA per stage
constexpr uint32_t P_IDESC = idesc_i8(P_BM, P_BN, true);
constexpr int p_smem_bytes(int stages) { return stages * P_STAGE_BYTES + 1024 + 256; }

template <int MODE, int P_STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_i8_tc_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;                                   // [stage][128][128]
    uint8_t* sB = smem + P_STAGES * P_HALF * BK;          // [stage][128][128]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE_BYTES);
    uint64_t* empty = full + P_STAGES;
    uint64_t* tfull = empty + P_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < P_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
    if (warp == 2) { tmem_alloc_pair(tmem_slot, 512); tmem_relinquish_pair(); }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int clusters = gridDim.x >> 1;
    const int cid = blockIdx.x >> 1;
    const int total = P.planes * P.tiles_m * P.tiles_n;

    if (warp == 0) {
        // ===== TMA producer (both CTAs) =====
        int stage = 0;
        uint32_t phase = 0;
        unsigned long long j = 0;
        for (int u = cid; u < total; u += clusters, ++j) {
            const TileCoord tc = decode_unit(u, P.tiles_m, P.tiles_n, P.group_m);
            const int arow = tc.tm * P_BM + (int)rank * P_HALF;
            const int bcol = tc.tn * P_BN + (int)rank * P_HALF;  // this CTA's 128 columns of B
            if (P.fence && lane == 0) step_fence_wait(P.fence, j * gridDim.x);
            __syncwarp();
            for (int kb = 0; kb < P.kblocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1u);
                if (lane == 0) {
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
                    tma_load_3d_pair(sA + stage * P_HALF * BK, &tmA, &full[stage], kb * BK, arow, tc.l, P.hintA);
                    tma_load_3d_pair(sB + stage * P_HALF * BK, &tmB, &full[stage], bcol, kb * BK, tc.l, P.hintB);
                }
                __syncwarp();
                if (++stage == P_STAGES) { stage = 0; phase ^= 1u; }
            }
            if (P.fence && lane == 0) atomicAdd(P.fence, 1ull);
        }
        if (P.fence && lane == 0) {
            const unsigned long long steps = (unsigned long long)((total + clusters - 1) / clusters);
            if (j < steps) atomicAdd(P.fence, steps - j);
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader CTA only) =====
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int u = cid; u < total; u += clusters, ++it) {
                const int acc = it & 1;
                const uint32_t aph = (uint32_t)((it >> 1) & 1);
                mbar_wait(&tempty[acc], aph ^ 1u);
                tc_fence_after();
                const uint32_t dtmem = tmem_base + (uint32_t)(acc * P_BN);
                for (int kb = 0; kb < P.kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * P_HALF * BK);
                        const uint32_t b0 = smem_u32(sB + stage * P_HALF * BK);
#pragma unroll
                        for (int k = 0; k < BK / 32; ++k)
                            mma_i8_pair(dtmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128_mn(b0 + k * 32 * 128, P_HALF * BK), P_IDESC,
                                        (kb | k) != 0 ? 1u : 0u);
                        mma_commit_pair(&empty[stage], (uint16_t)0x3);
                    }
                    __syncwarp();
                    if (++stage == P_STAGES) { stage = 0; phase ^= 1u; }
                }
                if (lane == 0) mma_commit_pair(&tfull[acc], (uint16_t)0x3);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ===== Epilogue (both CTAs): rows tm*256 + rank*128 + [0, 128) =====
        const int wq = warp - 4;
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
        int it = 0;
        for (int u = cid; u < total; u += clusters, ++it) {
            const TileCoord tc = decode_unit(u, P.tiles_m, P.tiles_n, P.group_m);
            const int acc = it & 1;
            const uint32_t aph = (uint32_t)((it >> 1) & 1);
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = tc.tm * P_BM + (int)rank * P_HALF + wq * 32 + lane;
            int32_t rowmax = 0;
#pragma unroll 1
            for (int c = 0; c < P_BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * P_BN + c * 32), v);
                tmem_ld_wait();
                const int col0 = tc.tn * P_BN + c * 32;
                if constexpr (MODE == EPI_MAX) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) rowmax = max(rowmax, (int32_t)v[j]);
                }
                epilogue_chunk<MODE>(v, row, col0, tc.l, P);
            }
            if constexpr (MODE == EPI_MAX) {
                if (row < P.m) atomicMax(&P.rowmax[row], rowmax);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * sizeof(uint64_t)));
        }
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, 512);
    }
}


// ---------------------------------------------------------------------------
// Dense INT8 tensor-core peak (the roofline denominator of the residue GEMM,
// SURVEY §6): one CTA per SM issues `iters` x 4 tcgen05.mma kind::i8
// 128x256x32 from one shared-memory stage (the residue GEMM's own operand
// layouts and instruction descriptor) into one TMEM accumulator — no TMA, no
// epilogue — so the launch time is the tensor pipe's alone.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(long long iters, int random, int* sink) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + A_BYTES;
    uint64_t* done = reinterpret_cast<uint64_t*>(sB + B_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // operand bytes: a low-toggle pattern (the tensor pipe's clock-limited peak) or
    // pseudo-random bytes (its power draw on data like the residue planes)
    for (int i = threadIdx.x; i < (A_BYTES + B_BYTES) / 4; i += blockDim.x) {
        uint32_t x = (uint32_t)i * 0x9E3779B1u + blockIdx.x * 0x85EBCA77u;
        x ^= x >> 15; x *= 0x2C1B3C6Du; x ^= x >> 12; x *= 0x297A2D39u; x ^= x >> 15;
        reinterpret_cast<uint32_t*>(smem)[i] = random ? x : 0x01010101u * (uint32_t)(i & 3);
    }
    if (threadIdx.x == 0) { mbar_init(done, 1); fence_mbar_init(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 1) { tmem_alloc(tmem_slot, 256); tmem_relinquish(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0 && lane == 0) {
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (long long it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < BK / 32; ++k)
                mma_i8(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128_mn(b0 + k * 32 * 128, B_CHUNK), IDESC,
                       (it | k) != 0 ? 1u : 0u);
        }
        mma_commit(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    tc_fence_after();
    if (warp == 0) {  // keep the result live
        uint32_t v[32];
        tmem_ld32(tmem, v);
        tmem_ld_wait();
        if (v[0] == 0x7fffffffu && lane == 0) *sink = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

}  // namespace

int gemm_smem_bytes() { return SMEM_BYTES; }
int gemm_tile_m() { return BM; }
int gemm_tile_n() { return BN; }
int gemm_tile_k() { return BK; }

template <int EW>
cudaError_t launch_tc(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P, int grid,
                      cudaStream_t stream) {
    static int configured[64][3] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int mi = mode == EPI_MAX ? 0 : mode == EPI_RESID ? 1 : 2;
    auto kern = mode == EPI_MAX ? gemm_i8_tc_kernel<EPI_MAX, EW>
              : mode == EPI_RESID ? gemm_i8_tc_kernel<EPI_RESID, EW> : gemm_i8_tc_kernel<EPI_I32, EW>;
    if (dev < 64 && !configured[dev][mi]) {  // once per device and kernel
        const cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        if (err != cudaSuccess) return err;
        configured[dev][mi] = 1;
    }
    return launch_pdl(kern, dim3(grid), dim3(tc_threads(EW)), SMEM_BYTES, stream, tmA, tmB, P);
}

cudaError_t launch_gemm_i8(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                           int num_sms, cudaStream_t stream) {
    const int total = P.planes * P.tiles_m * P.tiles_n;
    if (total == 0) return cudaSuccess;
    const int grid = total < num_sms ? total : num_sms;
    // epilogue warps: 8 when k is small (k <= 2048: a tile's MMAs take little
    // longer than its epilogue; cfg1 1024^3 79 vs 88 us per call), 4 above
    // (equal at 4096^3, 4 within noise ahead at 16384^3); option "epi_warps" 4|8 forces
    const int env = (int)opt(OPT_EPI_WARPS);
    const int ew = env == 4 || env == 8 ? env : (P.kblocks <= 16 ? 8 : 4);
    return ew == 4 ? launch_tc<4>(mode, tmA, tmB, P, grid, stream) : launch_tc<8>(mode, tmA, tmB, P, grid, stream);
}

cudaError_t launch_gemm_i8_mc(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                              int num_sms, cudaStream_t stream) {
    const int total = P.planes * ((P.tiles_m + 1) / 2) * P.tiles_n;  // tile pairs
    if (total == 0) return cudaSuccess;
    const int pairs = num_sms / 2;
    const int grid = 2 * (total < pairs ? total : pairs);
    cudaError_t err = cudaSuccess;
    switch (mode) {
        case EPI_MAX:
            err = cudaFuncSetAttribute(gemm_i8_tc_mc_kernel<EPI_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM_BYTES);
            if (err != cudaSuccess) return err;
            gemm_i8_tc_mc_kernel<EPI_MAX><<<grid, 256, SMEM_BYTES, stream>>>(tmA, tmB, P);
            break;
        case EPI_RESID:
            err = cudaFuncSetAttribute(gemm_i8_tc_mc_kernel<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM_BYTES);
            if (err != cudaSuccess) return err;
            gemm_i8_tc_mc_kernel<EPI_RESID><<<grid, 256, SMEM_BYTES, stream>>>(tmA, tmB, P);
            break;
        default:
            err = cudaFuncSetAttribute(gemm_i8_tc_mc_kernel<EPI_I32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM_BYTES);
            if (err != cudaSuccess) return err;
            gemm_i8_tc_mc_kernel<EPI_I32><<<grid, 256, SMEM_BYTES, stream>>>(tmA, tmB, P);
            break;
    }
    return cudaGetLastError();
}

int gemm_pair_tile_m() { return P_BM; }
int gemm_pair_tile_n() { return P_BN; }
int gemm_pair_box_rows() { return P_HALF; }

template <int MODE, int ST>
cudaError_t launch_pair_t(int grid, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                          cudaStream_t stream) {
    cudaError_t err = cudaFuncSetAttribute(gemm_i8_tc_pair_kernel<MODE, ST>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_bytes(ST));
    if (err != cudaSuccess) return err;
    gemm_i8_tc_pair_kernel<MODE, ST><<<grid, 256, p_smem_bytes(ST), stream>>>(tmA, tmB, P);
    return cudaGetLastError();
}

template <int ST>
cudaError_t launch_pair_s(int mode, int grid, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                          cudaStream_t stream) {
    switch (mode) {
        case EPI_MAX: return launch_pair_t<EPI_MAX, ST>(grid, tmA, tmB, P, stream);
        case EPI_RESID: return launch_pair_t<EPI_RESID, ST>(grid, tmA, tmB, P, stream);
        default: return launch_pair_t<EPI_I32, ST>(grid, tmA, tmB, P, stream);
    }
}

cudaError_t launch_gemm_i8_pair(int mode, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& P,
                                int num_sms, cudaStream_t stream) {
    const int total = P.planes * P.tiles_m * P.tiles_n;  // pair tiles
    if (total == 0) return cudaSuccess;
    const int pairs = num_sms / 2;
    const int grid = 2 * (total < pairs ? total : pairs);
    const int stages = (int)opt(OPT_PAIR_STAGES);
    // deeper pipelines let the clusters drift apart and lose L2 sharing:
    // DRAM reads 82 GB (4 stages), 245 GB (6), 250 GB (7) at 16384^3, N = 16
    if (stages == 6) return launch_pair_s<6>(mode, grid, tmA, tmB, P, stream);
    if (stages == 5) return launch_pair_s<5>(mode, grid, tmA, tmB, P, stream);
    return launch_pair_s<4>(mode, grid, tmA, tmB, P, stream);
}


// Dense INT8 peak microbenchmark: one launch of i8_peak_kernel on every SM,
// `iters` x 4 MMAs (2 x 128 x 256 x 32 int8 ops each) per SM.
cudaError_t launch_i8_peak(long long iters, int random, int num_sms, int* sink, cudaStream_t stream, double* ops) {
    const int smem = A_BYTES + B_BYTES + 1024 + 64;
    cudaError_t err = cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    i8_peak_kernel<<<num_sms, 128, smem, stream>>>(iters, random, sink);
    if (ops) *ops = (double)num_sms * (double)iters * 4.0 * 2.0 * BM * BN * 32.0;
    return cudaGetLastError();
}

}  // namespace oz2g
