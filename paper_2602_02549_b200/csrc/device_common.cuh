// device_common.cuh — sm_100a device helpers shared by the oz2g kernels:
// inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma kind::i8 / commit / ld) and the exact scalar arithmetic the
// Ozaki-II stages need (fp decomposition, modular reduction, RN scaling).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "options.h"

namespace oz2g {

// ----------------------------------------------------------------------------
// Error word bits (first failure in reference pipeline order wins on the host)
// ----------------------------------------------------------------------------
enum ErrBits : uint32_t {
    ERR_A_NONFINITE = 1u << 0,   // scaling.hpp:127 (row_abs_max)
    ERR_A_ZERO_ROW = 1u << 1,    // scaling.hpp:180
    ERR_B_NONFINITE = 1u << 2,   // scaling.hpp:138 (col_abs_max)
    ERR_B_ZERO_COL = 1u << 3,    // scaling.hpp:192
    ERR_CEIL_LOGIC = 1u << 4,    // scaling.hpp:67/77 (cannot happen for valid inputs)
    ERR_E_LOGIC = 1u << 5,       // scaling.hpp:179/189 e_i >= 31
    ERR_MU_RANGE = 1u << 6,      // scaling.hpp:145 mu int16 overflow
    ERR_NU_RANGE = 1u << 7,
    ERR_TRUNC_A_RANGE = 1u << 8, // scaling.hpp:206
    ERR_TRUNC_B_RANGE = 1u << 9, // scaling.hpp:220
    ERR_FR_RANGE = 1u << 10,     // crt.hpp:144 fp32 C'' overflow
    ERR_INV_RANGE = 1u << 11,    // emulate.hpp:39 inverse scaling overflow
};

// Device status block: error bits, first offending index per bit class and
// the subnormal flag.
struct DevStatus {
    uint32_t err;
    uint32_t subnormal;
    int64_t first_row;  // atomicMin targets: status_key of the first failing row of A /
    int64_t first_col;  // column of B (zero or non-finite), as the reference scans in order
};

// 2 * index + kind: the smallest key is the first failing row / column, and
// its low bit says whether it failed as non-finite (1) or all-zero (0)
// (scaling.hpp:33-52 throws at the first bad row, whichever the kind).
__host__ __device__ inline long long status_key(int64_t index, bool nonfinite) {
    return 2 * (long long)index + (nonfinite ? 1 : 0);
}

// ----------------------------------------------------------------------------
// Exact fp helpers
// ----------------------------------------------------------------------------
// |x| = mant * 2^e2 with mant in [2^52, 2^53) for finite nonzero x (normal or
// subnormal) — the reference's frexp/ldexp(f, 53) decomposition (crt.hpp:41-43,
// scaling.hpp:64-66) with e = e2 + 53.
__device__ __forceinline__ void decompose(double x, uint64_t& mant, int& e2) {
    const uint64_t bits = (uint64_t)__double_as_longlong(x);
    const int ef = (int)((bits >> 52) & 0x7ff);
    const uint64_t frac = bits & 0x000fffffffffffffull;
    if (ef) {
        mant = frac | (1ull << 52);
        e2 = ef - 1075;
    } else {
        const int lz = __clzll(frac) - 11;
        mant = frac << lz;
        e2 = -1074 - lz;
    }
}

// ilogb for finite nonzero double (scaling.hpp:182 std::ilogb).
__device__ __forceinline__ int ilogb_exact(double x) {
    uint64_t mant; int e2;
    decompose(x, mant, e2);
    return e2 + 52;
}

// ceil(2^sft |a|) for a shift with 2^sft a normal double (p2 = 2^sft), on the
// fp64 pipe: |a| p2 is exact unless the product is subnormal, and then the
// exact value lies in (0, 2^-1022), whose ceiling is 1 (a product rounded to 0
// is lifted to 1 for a != 0).  Same result as ceil_abs_scaled below; -1 above 64.
__device__ __forceinline__ bool pow2_normal(int sft) { return sft >= -1022 && sft <= 1023; }
__device__ __forceinline__ int ceil_scaled_p2(double a, double p2) {
    double c = ceil(__dmul_rn(fabs(a), p2));
    c = (c == 0.0 && a != 0.0) ? 1.0 : c;
    // c is an integer in [0, 2^53) (or inf): its value from the low word of c + 1.5 * 2^52
    return c > 64.0 ? -1 : (int)(uint32_t)__double_as_longlong(__dadd_rn(c, 6755399441055744.0));
}

// ceil(2^sft |a|) exactly (scaling.hpp:61-79); -1 on the logic_error paths.
__device__ __forceinline__ int ceil_abs_scaled(double a, int sft) {
    if (a == 0.0) return 0;
    uint64_t mant; int e2;
    decompose(a, mant, e2);
    const int exp2 = e2 + sft;  // == e - 53 + sft with frexp's e = e2 + 53
    if (exp2 >= 0) return -1;
    const int s = -exp2;
    uint64_t v;
    if (s >= 53) {
        v = 1;  // 0 < 2^sft |a| < 1
    } else {
        const uint64_t q = mant >> s;
        const uint64_t rem = mant & ((1ull << s) - 1);
        v = q + (rem != 0 ? 1 : 0);
    }
    return v > 64 ? -1 : (int)v;
}

// 2^s as a double for s in [-1022, 1023].
__device__ __forceinline__ double pow2d(int s) { return __longlong_as_double((long long)(s + 1023) << 52); }
__device__ __forceinline__ float pow2f(int s) { return __int_as_float((s + 127) << 23); }

// RN(x * 2^s) with a single rounding: glibc ldexp/scalbn semantics used by
// inverse_scale (emulate.hpp:37-38).
static __device__ __noinline__ double ldexp_rn_slow(double x, int s);
__device__ __forceinline__ double ldexp_rn(double x, int s) {
    // 2^s normal: one multiplication is one RN rounding of the exact x*2^s
    // (exact unless the result is subnormal, inf on overflow) == scalbn.
    if (s >= -1022 && s <= 1023) return __dmul_rn(x, pow2d(s));
    return ldexp_rn_slow(x, s);  // out of line: keeps unrolled epilogues small
}
static __device__ __noinline__ double ldexp_rn_slow(double x, int s) {
    if (x == 0.0 || !isfinite(x)) return x;
    const int ex = ilogb_exact(x);
    const int et = ex + s;
    if (et > 1023) return copysign(__longlong_as_double(0x7ff0000000000000ll), x);
    if (et >= -1022) {
        // exact: intermediates stay between ex and et, both in the normal range
        while (s > 1000) { x = __dmul_rn(x, pow2d(1000)); s -= 1000; }
        while (s < -1000) { x = __dmul_rn(x, pow2d(-1000)); s += 1000; }
        return __dmul_rn(x, pow2d(s));
    }
    if (et < -1075) return copysign(0.0, x);  // |x 2^s| < 2^-1075: RN gives 0
    // subnormal target: m = x * 2^-ex in [1,2) exact; (m * 2^-1022) exact; one rounding
    double m = x;
    int t = -ex;
    while (t > 1000) { m = __dmul_rn(m, pow2d(1000)); t -= 1000; }
    while (t < -1000) { m = __dmul_rn(m, pow2d(-1000)); t += 1000; }
    m = __dmul_rn(m, pow2d(t));
    m = __dmul_rn(m, pow2d(-1022));
    return __dmul_rn(m, pow2d(et + 1022));
}

// x * 2^s rounded upward, x >= 0 (each step rounds up: the result is >= exact).
__device__ __forceinline__ double ldexp_rd(double x, int s) {
    while (s > 1000) { x = __dmul_rd(x, pow2d(1000)); s -= 1000; }
    while (s < -1000) { x = __dmul_rd(x, pow2d(-1000)); s += 1000; }
    return __dmul_rd(x, pow2d(s));
}

__device__ __forceinline__ double ldexp_ru(double x, int s) {
    while (s > 1000) { x = __dmul_ru(x, pow2d(1000)); s -= 1000; }
    while (s < -1000) { x = __dmul_ru(x, pow2d(-1000)); s += 1000; }
    return __dmul_ru(x, pow2d(s));
}

__device__ __forceinline__ int ilogbf_exact(float x) {
    const uint32_t bits = (uint32_t)__float_as_int(x);
    const int ef = (int)((bits >> 23) & 0xff);
    const uint32_t frac = bits & 0x7fffffu;
    if (ef) return ef - 127;
    return -149 + (31 - __clz(frac));
}

// RN(x * 2^s) for float (std::ldexp(float, int) == scalbnf).
static __device__ __noinline__ float ldexpf_rn_slow(float x, int s);
__device__ __forceinline__ float ldexpf_rn(float x, int s) {
    if (s >= -126 && s <= 127) return __fmul_rn(x, pow2f(s));
    return ldexpf_rn_slow(x, s);
}
static __device__ __noinline__ float ldexpf_rn_slow(float x, int s) {
    if (x == 0.0f || !isfinite(x)) return x;
    const int ex = ilogbf_exact(x);
    const int et = ex + s;
    if (et > 127) return copysignf(__int_as_float(0x7f800000), x);
    if (et >= -126) {
        while (s > 120) { x = __fmul_rn(x, pow2f(120)); s -= 120; }
        while (s < -120) { x = __fmul_rn(x, pow2f(-120)); s += 120; }
        return __fmul_rn(x, pow2f(s));
    }
    if (et < -150) return copysignf(0.0f, x);  // |x 2^s| < 2^-150: RN gives 0
    float m = x;
    int t = -ex;
    while (t > 120) { m = __fmul_rn(m, pow2f(120)); t -= 120; }
    while (t < -120) { m = __fmul_rn(m, pow2f(-120)); t += 120; }
    m = __fmul_rn(m, pow2f(t));
    m = __fmul_rn(m, pow2f(-126));
    return __fmul_rn(m, pow2f(et + 126));
}

// ----------------------------------------------------------------------------
// Modular reduction by a small odd modulus p (<= 255) with a precomputed
// magic M = floor(2^32 / p): q = umulhi(x, M) is floor(x/p) or one less.
// ----------------------------------------------------------------------------
struct ModP {
    uint32_t p, magic;
};

__device__ __forceinline__ uint32_t mod_u32(uint32_t x, ModP mp) {
    const uint32_t q = __umulhi(x, mp.magic);
    uint32_t r = x - q * mp.p;
    if (r >= mp.p) r -= mp.p;
    return r;
}

// 32-byte global store (sm_100 STG.256): 4 doubles or 8 floats at a 32-byte
// aligned address.
__device__ __forceinline__ void st_global_v4f64(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// Grid-wide step fence of persistent kernels (one producer lane per CTA):
// wait until `counter` >= need, bounded (~2^26 cycles) so that CTAs that are
// not resident cannot hang the launch.
__device__ __forceinline__ void step_fence_wait(const unsigned long long* counter, unsigned long long need) {
    const long long t0 = clock64();
    for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
        if (v >= need || clock64() - t0 > (1ll << 26)) break;
        __nanosleep(64);
    }
}

// ----------------------------------------------------------------------------
// Programmatic dependent launch.  A kernel launched by launch_pdl may be
// scheduled while its predecessor in the stream is still running: it calls
// pdl_wait() before touching global memory (the predecessor's results become
// visible there — and every earlier kernel's, since the predecessor waited
// too) and pdl_trigger() to let its own successor be scheduled into the SMs
// its tail leaves idle.  Without the launch attribute both are no-ops.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}

// Set by run_gemm for the calls PDL pays on (small problems, where kernel
// ramps are a visible share of the call); option "pdl" 0 never, 2 always.
inline thread_local bool g_pdl_call = false;
inline bool pdl_enabled() {
    const long long mode = opt(OPT_PDL);
    return mode == 2 || (mode == 1 && g_pdl_call);
}

// kernel<<<grid, block, smem, s>>>(args...) with programmatic stream
// serialisation; the kernel must begin with pdl_wait() (pdl_enter()).
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ----------------------------------------------------------------------------
// mbarrier / TMA / tcgen05 PTX wrappers
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t"
        "}" ::"r"(addr),
        "r"(parity), "r"(0x989680)
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* desc) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* desc, uint64_t* bar, int c0,
                                            int c1, int c2, uint64_t cache_hint) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
        : "memory");
}

// L2 cache-policy constants (CUTLASS TMA::CacheHintSm90 values).
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem], int8 x int8 -> int32, one CTA.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
        "}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread
// complete (implicit tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// ---- CTA-pair (cta_group::2) variants ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load by either CTA of a pair; transaction bytes land on the even CTA's barrier.
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* desc, uint64_t* bar, int c0, int c1,
                                                 int c2, uint64_t cache_hint) {
    const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_leader), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
        : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish_pair() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
        "}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on the barrier at the same smem offset in every CTA of `mask` once
// the pair's previously issued MMAs complete.
// ---- cluster multicast with single-CTA MMAs ----
// TMA load whose bytes land at the same smem offset in every CTA of `mask`,
// each signalling its own mbarrier at the offset of `bar`.
__device__ __forceinline__ void tma_load_3d_mc(void* smem_dst, const CUtensorMap* desc, uint64_t* bar, int c0, int c1,
                                               int c2, uint16_t mask, uint64_t cache_hint) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6, %7;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask),
        "l"(cache_hint)
        : "memory");
}
// MMA completion arriving on the mbarrier at the offset of `bar` in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// 32 lanes x 32 columns of 32-bit TMEM -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row core
// groups 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;   // SBO
    d |= (uint64_t)1 << 46;             // descriptor version
    d |= (uint64_t)2 << 61;             // SWIZZLE_128B
    return d;
}

// MN-major operand with 128-byte swizzle (canonical layout, in 16-byte units,
// ((8, n), (8, k)) : ((1, LBO), (8, SBO))): every K-row holds 128 contiguous
// bytes along N, 8 K-rows form a 1 KB swizzle atom (SBO = 1024 B), and the
// next 128 columns of N start `lbo_bytes` further on.  Advancing K by 32 rows
// adds 32 * 128 B to the start address.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;  // LBO: between 128-column chunks of N
    d |= (uint64_t)(1024 >> 4) << 32;                  // SBO: between 8-row groups of K
    d |= (uint64_t)1 << 46;                            // descriptor version
    d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::i8: s8 x s8 -> s32, A K-major, B K-major or
// (b_mn) MN-major (valid for INT8 operands).
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool b_mn = false) {
    return (2u << 4)                       // D format S32
           | (1u << 7) | (1u << 10)        // A, B signed int8
           | ((b_mn ? 1u : 0u) << 16)      // B major: 0 K, 1 MN
           | ((uint32_t)(N >> 3) << 17)    // N / 8
           | ((uint32_t)(M >> 4) << 24);   // M / 16
}

// SM count of the current device (cached per device); launch shapes aim for a
// number of CTAs per SM.
inline int current_sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

}  // namespace oz2g
