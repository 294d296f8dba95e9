// api.cu — host orchestration of the B200 pipeline that replaces
// oz2::os_ii<T> (emulate.hpp:54-88): the single-device pipeline run_gemm and
// the shared helpers (api_internal.h).  The C ABI (include/oz2g.h) and the
// graph / suggest_n / multi-device / sweep runners are in api_ext.cu.
//
//   validation (emulate.hpp:58-61, moduli.hpp:94)
//   K1  row_scan_A / col_max_B / col_exp_B / bbar_T  (scale_matrices part 1)
//   K2  tcgen05 clearance GEMM, fused row/col max    (scaling.hpp:140-148)
//   [optional multi-GPU max-reduction of the maxima]
//   K3  scaling exponents via the step table          (scaling.hpp:159-194)
//   K4  fused trunc + N-plane residues of A and B     (scaling.hpp:199-225, crt.hpp:20-65)
//   K5  N tcgen05 residue GEMMs, fused signed mod p   (crt.hpp:69-79)
//   K6  CRT accumulate / Q / final reduce / unscale   (crt.hpp:91-150, emulate.hpp:30-46)
// Errors are raised through a device status word and mapped, in the
// reference's pipeline order, onto its exception classes.
#include "api_internal.h"

#include <cstdio>
#include <thread>

namespace oz2g {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_alloc_gen{0};
thread_local bool g_capture = false;

std::mutex g_ws_mtx;
std::map<int, Workspace*> g_ws;  // key device * 256 + slot

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Fail{OZ2G_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable"};
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D uint8 tensor [planes][rows][kp] (kp contiguous), box {128, box_rows, 1}, 128-B swizzle.
// plane_stride (bytes) defaults to rows * kp; a larger stride addresses a row
// block of every plane.
CUtensorMap make_plane_map(const void* base, int64_t kp, int64_t rows, int64_t planes, int box_rows,
                           int64_t plane_stride) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(plane_stride ? plane_stride : kp * rows)};
    cuuint32_t box[3] = {128u, (cuuint32_t)box_rows, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Fail{OZ2G_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
    return tm;
}

// 3-D uint8 tensor [planes][rows][cols] read as MN-major B tiles: box {128
// columns, 128 rows, 1}, 128-B swizzle; `pitch` = bytes between rows (16-byte
// multiple), columns past `cols` read as zeros.
CUtensorMap make_plane_map_mn(const void* base, int64_t cols, int64_t pitch, int64_t rows, int64_t planes,
                              int64_t plane_stride, int box_rows) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)plane_stride};
    cuuint32_t box[3] = {128u, (cuuint32_t)box_rows, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Fail{OZ2G_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
    return tm;
}

std::vector<uint8_t> build_resid_consts(const Table& t) {
    std::vector<uint8_t> buf(resid_consts_bytes(t.n), 0);
    ResidHeader* h = reinterpret_cast<ResidHeader*>(buf.data());
    h->n = t.n;
    uint32_t* tab = reinterpret_cast<uint32_t*>(buf.data() + sizeof(ResidHeader));
    for (int l = 0; l < t.n; ++l) {
        const uint32_t p = (uint32_t)t.p[l];
        h->p[l] = p;
        h->inv_p[l] = (float)(1.0 / (double)p);  // any value within 2^-20 relative of 1/p works (resid.cu)
        for (int G = 0; G < kResidE8; ++G) {
            for (int sg = 0; sg < 2; ++sg) {
                uint32_t w[8];
                for (int b = 0; b < 8; ++b) {  // symmetric representative of +-2^(8(b + G)) mod p, as a byte
                    uint32_t v = 1 % p;
                    for (int s = 0; s < 8 * (b + G); ++s) v = (v * 2u) % p;
                    int rep = (2 * v > p) ? (int)v - (int)p : (int)v;  // p = 256: 128 (byte -128)
                    if (sg) rep = -rep;                                  // -128 == 128 (mod 256)
                    w[b] = (uint32_t)rep & 0xffu;
                }
                uint32_t* cell = tab + 2 * (((size_t)l * kResidE8 + G) * 2 + sg);  // [l][G][sign]
                cell[0] = w[0] | (w[1] << 8) | (w[2] << 16) | (w[3] << 24);
                cell[1] = w[4] | (w[5] << 8) | (w[6] << 16) | (w[7] << 24);
            }
        }
        const uint32_t* c0 = tab + 2 * ((size_t)l * kResidE8 * 2);  // G = 0, s = 0
        h->fm[l] = FastMod{(int32_t)c0[0], (int32_t)c0[1], h->inv_p[l], 0u - p};
    }
    return buf;
}

void fill_gemm_moduli(GemmParams& P, const Table& t) {
    for (int l = 0; l < t.n; ++l) {
        const uint32_t p = (uint32_t)t.p[l];
        P.p[l] = p;
        P.magic[l] = (uint32_t)(0x100000000ull / p);
        P.off[l] = (uint32_t)(p * ((0x80000000ull + p - 1) / p));  // multiple of p >= 2^31
    }
}

// One workspace per (device, slot): slot 0 serves oz2g_gemm; oz2g_gemm_multi
// gives tile t slot t, so a device listed twice gets two independent workspaces.
Workspace& workspace(int dev, int slot) {
    std::lock_guard<std::mutex> lk(g_ws_mtx);
    const int key = dev * 256 + slot;
    auto it = g_ws.find(key);
    if (it == g_ws.end()) {
        Workspace* w = new Workspace();
        CUDA_TRY(cudaDeviceGetAttribute(&w->num_sms, cudaDevAttrMultiProcessorCount, dev));
        it = g_ws.emplace(key, w).first;
    }
    return *it->second;
}


// GEMM variant (option "gemm"): 0 single-CTA 128x256 tiles (default), 1
// "pair" CTA-pair cta_group::2 256x256 tiles, 2 "mcast" 2-CTA clusters sharing
// a multicast B tile.
int gemm_variant() { return (int)opt(OPT_GEMM); }

// TMA L2 policies (CUTLASS CacheHintSm90 encodings).  Default EVICT_NORMAL for
// both operands: measured at 16384^3, EVICT_LAST on A / EVICT_FIRST on B doubled
// the residue GEMM's DRAM reads (81 -> 156 GB: B tiles are shared by the CTAs of
// a wave and were evicted before reuse).  OZ2G_L2HINT=1 re-enables for study.
// TMA L2 eviction hints of the GEMM operand loads (option "l2hint"):
//   0 normal/normal (default), 1 A last / B first, 2 A last / B normal,
//   3 A normal / B first
void set_l2_hints(GemmParams& g) {
    const int mode = (int)opt(OPT_L2HINT);
    constexpr uint64_t kNormal = 0x1000000000000000ull, kLast = 0x14F0000000000000ull,
                       kFirst = 0x12F0000000000000ull;
    g.hintA = (mode == 1 || mode == 2) ? kLast : kNormal;
    g.hintB = (mode == 1 || mode == 3) ? kFirst : kNormal;
}

// Option "crt_overlap" = B > 1: the residue GEMMs + CRT of a large call run in
// B row blocks and each block's CRT runs on a side stream while the next
// block's GEMM computes (the CRT CTAs fit beside the persistent GEMM CTAs).
int crt_overlap_blocks() { return (int)opt(OPT_CRT_OVERLAP); }

// Residue GEMMs + CRT fused in one kernel (fused.cu) instead of the int8-W
// GEMM epilogue followed by the CRT pass: option "fused" 1 on, 0 off.
int fused_mode() { return (int)opt(OPT_FUSED); }

// Speculated exponents on the pipelined host path (run_gemm): option "spec"
// 0 off, 1 column exponents only (B uploaded first), 2 row and column
// exponents (A row chunks interleaved with B column chunks).  Default (-1): 2
// for inputs of at least 3 GiB, 1 below (measured: row + column speculation
// wins at 16384^3, 4 GiB, by 4-6%; below that its per-arrival overhead
// outweighs the earlier start, e.g. 3.8 vs 3.0 ms for SGEMM 4096^3, 41.7 vs
// 39.9 ms at 2048 x 65536 x 2048).
int speculation_mode(size_t input_bytes) {
    const long long v = opt(OPT_SPEC);
    if (v >= 0) return (int)v;
    return input_bytes >= (size_t(3) << 30) ? 2 : 1;
}

// Raster group height: one wave of persistent CTAs covers group_m tile-rows,
// so B tiles are streamed from HBM about tiles_m / group_m times per plane.
// Option "group_n" > 0 groups tile-columns instead (returned negated).
int group_m_for(int tiles_m, int tiles_n) {
    const int env = (int)opt(OPT_GROUP_M);
    const int env_n = (int)opt(OPT_GROUP_N);
    if (env_n > 0) return -(env_n < tiles_n ? env_n : (tiles_n > 0 ? tiles_n : 1));
    int g = env > 0 ? env : 16;  // best of {8, 12, 16, 24, 32} at 16384^3 (interleaved A/B)
    return g < tiles_m ? g : (tiles_m > 0 ? tiles_m : 1);
}


// The failure the reference would raise for a device status word, in its
// pipeline order (false when the status is clean).
bool status_failure(const DevStatus& hs, int64_t row_base, int64_t col_base, Fail& out) {
    const uint32_t e = hs.err;
    char buf[160];
    auto fail = [&](int code, std::string what, int order, int64_t index = 0) {
        out = Fail{code, std::move(what)};
        out.order = order;
        out.index = index;
        return true;
    };
    if (e & (ERR_A_NONFINITE | ERR_A_ZERO_ROW)) {  // the first failing row decides (status_key)
        const int64_t row = (hs.first_row >> 1) + row_base;
        if (hs.first_row & 1) return fail(OZ2G_DOMAIN_ERROR, "matrix entry is not finite", 0, row);
        snprintf(buf, sizeof buf, "row_pre_exponents: zero row %lld", (long long)row);
        return fail(OZ2G_DOMAIN_ERROR, buf, 0, row);
    }
    if (e & (ERR_B_NONFINITE | ERR_B_ZERO_COL)) {
        const int64_t col = (hs.first_col >> 1) + col_base;
        if (hs.first_col & 1) return fail(OZ2G_DOMAIN_ERROR, "matrix entry is not finite", 1, col);
        snprintf(buf, sizeof buf, "col_pre_exponents: zero column %lld", (long long)col);
        return fail(OZ2G_DOMAIN_ERROR, buf, 1, col);
    }
    if (e & ERR_CEIL_LOGIC) return fail(OZ2G_LOGIC_ERROR, "ceil_abs_scaled: entry above row/column max", 2);
    if (e & ERR_E_LOGIC) return fail(OZ2G_LOGIC_ERROR, "scaling_exponents: e_i >= 31", 3);
    if (e & ERR_MU_RANGE) return fail(OZ2G_RANGE_ERROR, "mu: exceeds 16-bit range", 4);
    if (e & ERR_NU_RANGE) return fail(OZ2G_RANGE_ERROR, "nu: exceeds 16-bit range", 5);
    if (e & ERR_TRUNC_A_RANGE) return fail(OZ2G_RANGE_ERROR, "truncate_scaled: 2^mu*a overflow", 6);
    if (e & ERR_TRUNC_B_RANGE) return fail(OZ2G_RANGE_ERROR, "truncate_scaled: b*2^nu overflow", 7);
    if (e & ERR_FR_RANGE)
        return fail(OZ2G_RANGE_ERROR, "final_reduce: single(C'') overflows fp32 (N too large for fp32 mode)", 8);
    if (e & ERR_INV_RANGE) return fail(OZ2G_RANGE_ERROR, "os_ii: inverse scaling overflow", 9);
    return false;
}

// Wait for every pending OZ2G_ASYNC call of `ws` and return the first failure
// in call order (caller holds ws.mtx).
bool complete_pending(Workspace& ws, Fail& first) {
    bool failed = false;
    if (ws.pending.empty()) return false;
    for (const auto& p : ws.pending) CUDA_TRY(cudaStreamSynchronize(p.stream));
    std::vector<DevStatus> hs(kStatusRing);
    CUDA_TRY(cudaMemcpy(hs.data(), ws.status_ring.p, sizeof(DevStatus) * kStatusRing, cudaMemcpyDeviceToHost));
    for (const auto& p : ws.pending) {
        Fail f{OZ2G_OK, ""};
        if (!failed && status_failure(hs[(size_t)p.slot], p.row_base, p.col_base, f)) {
            first = f;
            failed = true;
        }
    }
    ws.pending.clear();
    return failed;
}


// Operands of the relative criterion (bounds "relative", suggest_n tight):
// with Acheck = floor(|A| 2^(mu' + 1)), Bcheck = floor(|B| 2^(nu' + 1))
// (launch_floor_operands), lo = Acheck Bcheck (one tcgen05 EPI_I32 launch)
// bounds (|A||B|)_ij from below by lo_ij 2^-(mu'_i + nu'_j + 2) and, with
// the row / column sums, from above.  Needs mu', nu' of these inputs.
void compute_relative_operands(Workspace& ws, int prec, const void* dA, int64_t lda, const void* dB, int64_t ldb,
                               int64_t m, int64_t n, int64_t k, const int32_t* mup, const int32_t* nup,
                               cudaStream_t stream, int& launches) {
    const int64_t kp = round_up(k, 128), ldn = round_up(n > 0 ? n : 1, 16);
    int8_t* la = (int8_t*)ws.lo_a.get((size_t)(m * kp));
    int8_t* lb = (int8_t*)ws.lo_b.get((size_t)(kp * ldn));
    int32_t* sums = (int32_t*)ws.lo_sum.get(4 * (size_t)(m + n));
    int32_t* lab = (int32_t*)ws.lo_ab.get(4 * (size_t)(m * n));
    CUDA_TRY(launch_floor_operands(prec, dA, lda, m, dB, ldb, k, n, kp, ldn, mup, nup, la, lb, sums, sums + m, stream));
    launches += 2;
    GemmParams g;
    std::memset(&g, 0, sizeof g);
    g.m = (int)m;
    g.n = (int)n;
    g.kblocks = (int)(kp / 128);
    g.tiles_m = (int)((m + gemm_tile_m() - 1) / gemm_tile_m());
    g.tiles_n = (int)((n + gemm_tile_n() - 1) / gemm_tile_n());
    g.group_m = group_m_for(g.tiles_m, g.tiles_n);
    set_l2_hints(g);
    g.planes = 1;
    g.C32 = lab;
    g.ldc32 = n;
    g.cplane = m * n;
    CUDA_TRY(launch_gemm_i8(EPI_I32, make_plane_map(la, kp, m, 1, gemm_tile_m()),
                            make_plane_map_mn(lb, n, ldn, kp, 1, kp * ldn), g, ws.num_sms, stream));
    // the fp64 lower bound per entry, refined by rounded-down dot products
    // where the floor product is loose (at most 2^32 multiply-adds)
    double* abl = (double*)ws.ab_lo.get(8 * (size_t)(m * n));
    unsigned long long* budget = (unsigned long long*)ws.x_bmax.get(32) + 3;
    CUDA_TRY(launch_ab_lower(prec, dA, lda, dB, ldb, m, n, k, lab, mup, nup, sums, sums + m, abl, budget,
                             1ull << 32, stream));
    launches += 2;
    ws.lo_ready = true;
}


// row_base / col_base: global index of the first row / column of this call's
// tile (error messages of oz2g_gemm_multi); slot: workspace slot.
int run_gemm(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
             void* C, int64_t ldc, int nmod, unsigned flags, cudaStream_t stream, oz2g_intermediates* inter,
             oz2g_diag* diag, oz2g_reduce_maxima_fn reduce_fn, void* reduce_user, int64_t row_base,
             int64_t col_base, int slot, bool reuse_scaling, const Arrivals* arr) {
    if (prec != OZ2G_FP32 && prec != OZ2G_FP64) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: prec must be OZ2G_FP32 or OZ2G_FP64"};
    if (m < 0 || n < 0 || k < 0) throw Fail{OZ2G_INVALID_ARGUMENT, "Matrix: negative dimension"};
    if (lda < k || ldb < n || ldc < n) throw Fail{OZ2G_INVALID_ARGUMENT, "dimension mismatch: leading dimension"};
    if (k > OZ2G_MAX_INNER_DIM) throw Fail{OZ2G_DOMAIN_ERROR, "os_ii: k exceeds 2^17"};
    const Table& tab = table_for(nmod, prec);  // std::domain_error for N outside [2, 49]
    if (diag) std::memset(diag, 0, sizeof *diag);
    // programmatic dependent launches for small problems only: at 1024^3 they
    // hide kernel ramps (77.7 -> 76.0 us per call); from 3072^3 up the
    // early-scheduled CTAs waiting beside the running kernels cost more than
    // that (8192^3: 8.38 -> 9.6 ms with the GEMM's trigger at its start)
    struct PdlScope {
        bool prev;
        explicit PdlScope(bool on) : prev(g_pdl_call) { g_pdl_call = on; }
        ~PdlScope() { g_pdl_call = prev; }
    } pdl_scope((double)m * (double)n * (double)k <= kPdlMaxWork);
    // k == 0: every row of A (and column of B) is zero (scaling.hpp:180/192)
    if (k == 0) {
        if (m > 0) throw Fail{OZ2G_DOMAIN_ERROR, "row_pre_exponents: zero row 0"};
        if (n > 0) throw Fail{OZ2G_DOMAIN_ERROR, "col_pre_exponents: zero column 0"};
        return OZ2G_OK;
    }
    const bool host = (flags & OZ2G_DEVICE_PTRS) == 0;
    const bool async = (flags & OZ2G_ASYNC) != 0;
    if (async && (inter || reduce_fn || (flags & OZ2G_TIMING)))
        throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: OZ2G_ASYNC computes C only (no intermediates, hook or timing)"};
    const size_t esz = prec ? 8 : 4;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    Workspace& ws = workspace(dev, slot);
    std::lock_guard<std::recursive_mutex> dev_lock(ws.mtx);
    int launches = 0;
    if (!async && !ws.pending.empty()) {  // a blocking call completes earlier async calls first
        Fail f{OZ2G_OK, ""};
        if (complete_pending(ws, f)) throw f;
    }
    if (async && !ws.pending.empty() && ws.last_async_stream != stream)
        CUDA_TRY(cudaStreamWaitEvent(stream, ws.ev_last_async, 0));

    Timer tm;
    tm.on = diag && (flags & OZ2G_TIMING);

    const int64_t kp = round_up(k, 128);
    const int64_t ldw = round_up(n > 0 ? n : 1, 16);
    const int64_t ldn = ldw;  // row pitch of Bbar and of the B residue planes [kp][ldn]
    const void* dA = A;
    const void* dB = B;
    void* dC = C;
    int64_t lda_d = lda, ldb_d = ldb, ldc_d = ldc;
    // pipelined host path: plain calls (no intermediates / multi-GPU hook) on large problems
    // Matrix-sized intermediates need whole-matrix buffers; the O(m + n) scaling
    // vectors (which the reference returns even with keep = false) do not.
    const bool inter_mats = inter && (inter->Aprime || inter->Bprime || inter->Cbar || inter->Dbar || inter->W ||
                                      inter->C1 || inter->C2 || inter->Q || inter->Cpp64 || inter->Cpp32 ||
                                      inter->Ares || inter->Bres || inter->Cprod || inter->bounds);
    // With a multi-rank reduce hook the uploads still overlap the scans and the
    // clearance products, but the exponents (and everything after) wait for
    // the all-reduced maxima: no per-chunk exponents, no speculation.
    // Inputs arriving on other streams (arr, the multi-GPU exchange) take the
    // same chunked path with device pointers: B first, then A row chunks.
    if (arr && (host || inter || async)) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: arrivals need device pointers, C only"};
    const bool pipe = (host && !inter_mats && m >= 2048 && n >= 256) || arr;
    const bool hooked = reduce_fn != nullptr;
    const int64_t chunk_rows =
        arr ? std::max<int64_t>(1, arr->chunk_rows) : pipe ? round_up((m + kPipeChunks - 1) / kPipeChunks, 256) : m;
    const int nchunks = m > 0 ? (int)((m + chunk_rows - 1) / chunk_rows) : 1;
    if (arr && (nchunks > kMaxArrivalChunks || (m > 0 && nchunks != arr->nchunks)))
        throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: arrival chunks do not cover A"};
    const cudaEvent_t ev_b_in = arr ? arr->b : nullptr;
    // speculated exponents (blocking pipelined calls): 2 = rows and columns
    // (A row chunks and B column chunks uploaded alternately), 1 = columns
    // (asynchronous calls: rows + columns only; its statuses are merged on the device)
    const int spec_mode = (pipe && !arr && !hooked && !reuse_scaling && crt_overlap_blocks() <= 1)
                              ? speculation_mode(esz * (size_t)(m * k + k * n)) : 0;
    const bool spec2 = spec_mode == 2 && n >= 2 * 256;
    // spec2 column chunks: units of cu columns (a multiple of 128), chunks of
    // 2^T units (T = option "spec_tail") and a halving tail — the last 2^T
    // units arrive as 2^(T-1), ..., 1, 1 units — so the last arrival, and the
    // work left after the upload, is short; cstart[c] = first column of chunk
    // c, cstart[ncc] = n
    const int tail_t = (int)opt(OPT_SPEC_TAIL);
    const int64_t per_chunk = int64_t(1) << tail_t;
    const int64_t col_chunk = round_up((n + kPipeChunks - 1) / kPipeChunks, 128 * per_chunk);
    const int64_t cu = col_chunk / per_chunk;
    const int64_t nunits = (n + cu - 1) / cu;
    std::vector<int64_t> cstart;
    for (int64_t u = 0; spec2 && u < nunits;) {
        cstart.push_back(u * cu);
        const int64_t rem = nunits - u;
        int64_t step = per_chunk;
        if (rem <= per_chunk) {  // the tail: the largest power of two below rem (1 for rem <= 2)
            step = 1;
            while (2 * step < rem) step *= 2;
        }
        u += step;
    }
    const int ncc = (int)cstart.size();
    if (ncc > kMaxColChunks) throw Fail{OZ2G_LOGIC_ERROR, "oz2g_gemm: too many column chunks"};
    cstart.push_back(n);
    std::vector<std::pair<bool, int>> arrivals;  // spec2 upload order: (is an A row chunk, index)
    for (int j = 0; spec2 && j < std::max(nchunks, ncc); ++j) {
        if (j < nchunks) arrivals.emplace_back(true, j);
        if (j < ncc) arrivals.emplace_back(false, j);
    }
    if (host) {
        dA = ws.A.get(esz * (size_t)(m * k));
        dB = ws.B.get(esz * (size_t)(k * n));
        dC = ws.C.get(esz * (size_t)(m * n));
        lda_d = k; ldb_d = n; ldc_d = n;
        if (pipe) {
            ws.ensure_streams();
            // the device copies of A and B are free once the previous call's last
            // reader ran (its residue GEMMs may still be running: uploads overlap them)
            CUDA_TRY(cudaStreamWaitEvent(ws.s_h2d, ws.ev_inputs_free, 0));
            for (const auto& a : arrivals) {  // spec2: A row chunks and B column chunks alternately
                if (a.first) {
                    const int64_t r0 = a.second * chunk_rows, rc = std::min<int64_t>(chunk_rows, m - r0);
                    tm.span(0, ws.s_h2d, [&] {
                        CUDA_TRY(cudaMemcpy2DAsync((char*)const_cast<void*>(dA) + esz * (size_t)(r0 * k), esz * k,
                                                   (const char*)A + esz * (size_t)(r0 * lda), esz * lda, esz * k, rc,
                                                   cudaMemcpyHostToDevice, ws.s_h2d));
                    });
                    CUDA_TRY(cudaEventRecord(ws.ev_a[a.second], ws.s_h2d));
                } else {
                    const int64_t c0 = cstart[(size_t)a.second], nc = cstart[(size_t)a.second + 1] - c0;
                    tm.span(0, ws.s_h2d, [&] {
                        CUDA_TRY(cudaMemcpy2DAsync((char*)const_cast<void*>(dB) + esz * (size_t)c0, esz * n,
                                                   (const char*)B + esz * (size_t)c0, esz * ldb, esz * nc, k,
                                                   cudaMemcpyHostToDevice, ws.s_h2d));
                    });
                    CUDA_TRY(cudaEventRecord(ws.ev_bc[a.second], ws.s_h2d));
                }
            }
        }
        if (pipe && !spec2) {
            // B first: the column scan needs all of it
            tm.span(0, ws.s_h2d, [&] {
                CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dB), esz * n, B, esz * ldb, esz * n, k,
                                           cudaMemcpyHostToDevice, ws.s_h2d));
            });
            CUDA_TRY(cudaEventRecord(ws.ev_b, ws.s_h2d));
            for (int c = 0; c < nchunks; ++c) {
                const int64_t r0 = c * chunk_rows, rc = std::min<int64_t>(chunk_rows, m - r0);
                tm.span(0, ws.s_h2d, [&] {
                    CUDA_TRY(cudaMemcpy2DAsync((char*)const_cast<void*>(dA) + esz * (size_t)(r0 * k), esz * k,
                                               (const char*)A + esz * (size_t)(r0 * lda), esz * lda, esz * k, rc,
                                               cudaMemcpyHostToDevice, ws.s_h2d));
                });
                CUDA_TRY(cudaEventRecord(ws.ev_a[c], ws.s_h2d));
            }
        } else if (!pipe) {
            tm.span(0, stream, [&] {
                if (m * k) CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dA), esz * k, A, esz * lda, esz * k, m, cudaMemcpyHostToDevice, stream));
                if (k * n) CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dB), esz * n, B, esz * ldb, esz * n, k, cudaMemcpyHostToDevice, stream));
            });
        }
    }

    DevStatus* st;
    int ring_slot = -1;
    if (async) {
        ws.ensure_streams();
        if ((int)ws.pending.size() >= kStatusRing) {  // ring full: complete the oldest calls first
            Fail f{OZ2G_OK, ""};
            if (complete_pending(ws, f)) throw f;
        }
        ring_slot = ws.ring_next;
        ws.ring_next = (ws.ring_next + 1) % kStatusRing;
        st = (DevStatus*)ws.status_ring.get(sizeof(DevStatus) * kStatusRing) + ring_slot;
    } else {
        st = (DevStatus*)ws.status.get(sizeof(DevStatus));
    }
    int32_t* mup = (int32_t*)ws.mup.get(4 * (size_t)m);
    int32_t* nup = (int32_t*)ws.nup.get(4 * (size_t)n);
    int32_t* mu = (int32_t*)ws.mu.get(4 * (size_t)m);
    int32_t* nu = (int32_t*)ws.nu.get(4 * (size_t)n);
    unsigned long long* bmax = (unsigned long long*)ws.bmax.get(8 * (size_t)n);
    int32_t* cmax_row = (int32_t*)ws.cmax_row.get(4 * (size_t)m);
    int32_t* cmax_col = (int32_t*)ws.cmax_col.get(4 * (size_t)n);
    float* ev = (float*)ws.e.get(4 * (size_t)m);
    float* fv = (float*)ws.f.get(4 * (size_t)n);
    int8_t* abar = (int8_t*)ws.abar.get((size_t)(m * kp));
    int8_t* bbar = (int8_t*)ws.bbar.get((size_t)(kp * ldn));
    // reuse_scaling (oz2g_gemm_sweep, device pointers): mu', nu' and the
    // clearance maxima of the previous call on these same inputs are still in
    // the workspace — they do not depend on N — so K1 / K2 are skipped
    const bool scan = !reuse_scaling;
    if (scan) ws.lo_ready = false;  // new inputs: the relative-criterion operands are stale
    // one launch instead of five memsets: the status word (first-failure keys
    // at their maximum) and, for a scan, the column maxima of B and the
    // clearance row / column maxima
    CUDA_TRY(launch_init_call(st, scan ? bmax : nullptr, scan ? n : 0, scan ? cmax_row : nullptr, scan ? m : 0,
                              scan ? cmax_col : nullptr, scan ? n : 0, stream));
    ++launches;

    // Unpipelined calls run the independent A-side and B-side passes (the
    // scans, then the residue splits) on two streams: at small sizes each
    // kernel alone leaves most of the GPU idle.  Joined before each GEMM.
    const bool fork = !pipe && !spec_mode && m > 0 && n > 0;
    size_t evn = 0;  // per-call event index (downloads wait for their CRT; stream forks / joins)
    cudaStream_t sB = stream;
    if (fork) {
        ws.ensure_streams();
        sB = ws.s_aux;
        const cudaEvent_t ef = ws.pool_event(evn++);
        CUDA_TRY(cudaEventRecord(ef, stream));
        CUDA_TRY(cudaStreamWaitEvent(sB, ef, 0));
    }
    // ---- K1 (B): column pre-exponents and Bbar^T ----
    if (pipe && !spec2) CUDA_TRY(cudaStreamWaitEvent(stream, arr ? ev_b_in : ws.ev_b, 0));
    if (scan && !spec2) tm.span(1, sB, [&] {
        CUDA_TRY(launch_col_max_B(prec, dB, ldb_d, k, n, bmax, st, sB)); launches += n > 0;
        CUDA_TRY(launch_col_exp_B(bmax, n, nup, st, sB)); launches += n > 0;
        CUDA_TRY(launch_bbar_rows(prec, dB, ldb_d, k, n, kp, ldn, nup, bbar, st, sB)); launches += n > 0;
    });
    cudaEvent_t ev_bdone = nullptr;
    if (fork) {
        ev_bdone = ws.pool_event(evn++);
        CUDA_TRY(cudaEventRecord(ev_bdone, sB));
    }

    // tile shape: single-CTA 128x256 tiles, CTA-pair 256x256 tiles (cta_group::2),
    // or 128x256 tiles in 2-CTA clusters with a multicast B tile
    const int variant = gemm_variant();
    const bool pair = variant == 1;
    const int BM = pair ? gemm_pair_tile_m() : gemm_tile_m();
    const int BN = pair ? gemm_pair_tile_n() : gemm_tile_n();
    const int boxA = pair ? gemm_pair_box_rows() : BM;
    auto launch_gemm = [&](int mode, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& g) {
        if (variant == 1) return launch_gemm_i8_pair(mode, ta, tb, g, ws.num_sms, stream);
        if (variant == 2) return launch_gemm_i8_mc(mode, ta, tb, g, ws.num_sms, stream);
        return launch_gemm_i8(mode, ta, tb, g, ws.num_sms, stream);
    };
    GemmParams gp;
    std::memset(&gp, 0, sizeof gp);
    gp.n = (int)n;
    gp.kblocks = (int)(kp / 128);
    gp.tiles_n = (int)((n + BN - 1) / BN);
    set_l2_hints(gp);
    auto set_rows = [&](GemmParams& g, int64_t rows) {
        g.m = (int)rows;
        g.tiles_m = (int)((rows + BM - 1) / BM);
        g.group_m = group_m_for(g.tiles_m, g.tiles_n);
    };

    // residue constants (uploaded once per table) and planes
    const int N = tab.n;
    const auto key = std::make_pair(tab.n, tab.mode);
    if (!ws.rc.count(key)) {
        const std::vector<uint8_t> h = build_resid_consts(tab);
        ResidConsts* d = nullptr;
        CUDA_TRY(cudaMalloc(&d, h.size()));
        CUDA_TRY(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
        ws.rc[key] = d;
    }
    const ResidConsts* rc_dev = ws.rc[key];
    int8_t* ares = (int8_t*)ws.ares.get((size_t)N * (size_t)(m * kp));
    int8_t* bres = (int8_t*)ws.bres.get((size_t)N * (size_t)(kp * ldn));

    // ---- CRT constants, W and the row blocks of C (host-side set-up) ----
    CrtConsts cc;
    std::memset(&cc, 0, sizeof cc);
    cc.n = N;
    cc.mode = tab.mode;
    for (int l = 0; l < N; ++l) { cc.s1[l] = tab.s1[l]; cc.s2[l] = tab.s2[l]; }
    cc.P1 = tab.P1; cc.P2 = tab.P2; cc.P_inv = tab.P_inv;
    CrtExtra ex;
    std::memset(&ex, 0, sizeof ex);
    const size_t mn8 = 8 * (size_t)(m * n);
    oz2g_bounds* bo = inter ? inter->bounds : nullptr;
    unsigned long long* bmax_dev = nullptr;
    if (inter) {
        if (inter->C1) ex.C1 = (double*)ws.x_c1.get(mn8);
        if (inter->C2) ex.C2 = (double*)ws.x_c2.get(mn8);
        if (inter->Q) ex.Q = (double*)ws.x_q.get(mn8);
        if (inter->Cpp64) ex.Cpp64 = (double*)ws.x_cpp64.get(mn8);
        if (inter->Cpp32 && prec == OZ2G_FP32) ex.Cpp32 = (float*)ws.x_cpp32.get(mn8 / 2);
    }
    const int ovb = crt_overlap_blocks();
    const bool overlap = ovb > 1 && !inter_mats && m >= 2048;
    if (overlap) ws.ensure_streams();
    // W holds one row block (all N planes) unless every plane of the whole
    // matrix is wanted (intermediates) or blocks overlap (side-stream CRT).
    // W per block only when the whole-matrix W would be large (more launches
    // cost more than the memory saves on mid-size problems)
    const int64_t w_block_min = (int64_t)opt(OPT_WBLOCK_MIN_MB) << 20;
    const bool w_full = (inter && inter->W) || overlap || (int64_t)N * m * ldw < w_block_min;
    const int64_t wrows = w_full ? m : std::min<int64_t>(m, kWBlockRows);
    int8_t* W = (int8_t*)ws.W.get((size_t)N * (size_t)(wrows * ldw));
    fill_gemm_moduli(gp, tab);
    const bool fused = fused_mode() >= 1 && !inter && !bo && !overlap && m * n > 0;
    // A residues streamed per row block (option "resid_stream"): block b + 1's
    // split runs on the side stream beside block b's residue GEMMs, so only the
    // first block's split precedes the GEMMs
    const bool rstream = opt(OPT_RESID_STREAM) != 0 && fork && !fused && m > kWBlockRows;
    struct Block { int64_t r0, rows; int chunk; };
    std::vector<Block> blocks;  // row blocks of C, one residue-GEMM + CRT launch each
    const int64_t max_block =
        (w_full && !rstream) ? (overlap ? round_up((m + ovb - 1) / ovb, 128) : m) : kWBlockRows;
    for (int c = 0; c < nchunks; ++c) {
        const int64_t r0 = c * chunk_rows, rc = std::min<int64_t>(chunk_rows, m - r0);
        if (rc <= 0) continue;
        const int64_t sub = (pipe && host && !spec2 && c == nchunks - 1 && rc >= 2 * 128)
                                ? std::min<int64_t>(max_block, round_up((rc + kTailSplit - 1) / kTailSplit, 128))
                                : max_block;
        for (int64_t q = r0; q < r0 + rc; q += sub) blocks.push_back({q, std::min<int64_t>(sub, r0 + rc - q), c});
    }
    const CUtensorMap tBres = make_plane_map_mn(bres, n, ldn, kp, N, kp * ldn);

    // Speculative column exponents (blocking host-pointer calls).  nu_j needs
    // the clearance maxima of column j over every row of A, i.e. the whole
    // upload, and every residue GEMM needs the B residues, which need nu.  nu
    // is a step function of those maxima (thresholds 4x apart), so it is taken
    // from the maxima of the first uploaded row chunk, and the B residues and
    // the residue GEMMs + CRT of each chunk run while the rest of A is still
    // uploading.  After every later chunk's clearance product the exponents
    // are re-derived from the maxima so far; where one moved, the B residues
    // are recomputed and the 256-column tiles holding moved columns are redone
    // for every block already computed (once that would exceed an eighth of
    // all block tiles, the remaining blocks wait for the final exponents and
    // the moved tiles are repaired once at the end).  After the last chunk nu is final, so C
    // is the unspeculated C bit for bit.  Status flags of the stages that read
    // nu (B residues, CRT) are kept per stage / block so that flags raised with
    // a superseded nu are dropped; a repaired block whose first CRT raised any
    // flag makes the call redo every stage after the upload unspeculated.
    const bool spec = spec_mode >= 1 && !spec2 && n > 0 && !async;
    const size_t nb = blocks.size();
    const int64_t ntiles = (n + 255) / 256;
    DevStatus* sx = nullptr;       // [0] discarded, [1] B residues, [2 + b] CRT of block b, [2 + nb + b] its repairs
    int32_t* changed_h = nullptr;  // [0] any column moved, [1 + t] a column of tile t moved (host view)
    int32_t* changed = nullptr;    // its device alias
    std::vector<char> repaired;
    int spec_state = (spec || spec2) ? 1 : 0;
    if (spec) {
        ws.ensure_streams();
        sx = (DevStatus*)ws.spec_st.get(sizeof(DevStatus) * (2 + 2 * nb));
        CUDA_TRY(cudaMemsetAsync(sx, 0, sizeof(DevStatus) * (2 + 2 * nb), stream));
        changed_h = ws.changed_flags((size_t)(1 + ntiles));
        CUDA_TRY(cudaHostGetDevicePointer((void**)&changed, changed_h, 0));
        repaired.assign(nb, 0);
    }
    const ChangeFlags cf1{changed, 0, 256, 0};
    bool defer1 = false;                    // columns-only speculation: blocks wait for the final exponents
    int64_t repair_work = 0;                // block tiles recomputed so far
    std::vector<char> dirty1((size_t)ntiles, 0);  // 256-column tiles whose exponents moved (to repair)

    // ---- K5 + K6 of one row block of C (columns c0 .. c0 + nc): residue GEMMs
    //      (fused signed mod p), CRT + unscale, download ----
    auto run_block = [&](size_t bi, int64_t c0, int64_t nc, DevStatus* sb) {
        const int64_t r0 = blocks[bi].r0, rc = blocks[bi].rows;
        if (nc <= 0) return;
        GemmParams g = gp;
        g.planes = N;
        g.ldw = ldw;
        g.wplane = wrows * ldw;
        g.n = (int)nc;
        g.tiles_n = (int)((nc + BN - 1) / BN);
        const CUtensorMap tA = make_plane_map(ares + r0 * kp, kp, rc, N, boxA, m * kp);
        const CUtensorMap tB = (c0 == 0 && nc == n) ? tBres : make_plane_map_mn(bres + c0, nc, ldn, kp, N, kp * ldn);
        int8_t* Wb = (w_full ? W + r0 * ldw : W) + c0;
        set_rows(g, rc);
        g.W = Wb;
        if (opt(OPT_GEMM_FENCE) == 1) {  // experiment: keep the persistent CTAs within one unit of each other
            g.fence = (unsigned long long*)ws.x_bmax.get(64) + 5;
            CUDA_TRY(cudaMemsetAsync(g.fence, 0, 8, stream));
        }
        tm.span(5, stream, [&] { CUDA_TRY(launch_gemm(EPI_RESID, tA, tB, g)); });
        ++launches;
        if (inter && inter->Cprod) {  // rows of this block of the m x n planes
            GemmParams g2 = g;
            g2.C32 = (int32_t*)ws.x_cprod.get(4 * (size_t)N * (size_t)(m * n)) + r0 * n;
            g2.ldc32 = n;
            g2.cplane = m * n;
            CUDA_TRY(launch_gemm(EPI_I32, tA, tB, g2)); ++launches;
        }
        cudaStream_t crt_stream = stream;
        if (overlap) {  // this block's CRT beside the next block's GEMM
            const cudaEvent_t eg = ws.pool_event(evn++);
            CUDA_TRY(cudaEventRecord(eg, stream));
            CUDA_TRY(cudaStreamWaitEvent(ws.s_aux, eg, 0));
            crt_stream = ws.s_aux;
        }
        // the CRT indexes rows from the block's first row: offset the optional
        // per-entry outputs and the per-row bound vectors to this block
        CrtExtra exb = ex;
        const int64_t eo = r0 * n;
        if (exb.C1) exb.C1 += eo;
        if (exb.C2) exb.C2 += eo;
        if (exb.Q) exb.Q += eo;
        if (exb.Cpp64) exb.Cpp64 += eo;
        if (exb.Cpp32) exb.Cpp32 += eo;
        if (exb.bnd.on) {
            exb.bnd.v.RA += r0;
            exb.bnd.v.PA += r0;
            exb.bnd.v.ea += r0;
            if (exb.bnd.cheap) exb.bnd.cheap += eo;
            if (exb.bnd.tight) exb.bnd.tight += eo;
            if (exb.bnd.ab_lo) exb.bnd.ab_lo += eo;
        }
        tm.span(6, crt_stream, [&] {
            CUDA_TRY(launch_crt(prec, Wb, ldw, wrows * ldw, rc, nc, cc, mu + r0, nu + c0,
                                (char*)dC + esz * (size_t)(r0 * ldc_d + c0), ldc_d, exb, sb, crt_stream));
        });
        ++launches;
        if (pipe && host) {  // download this C block while the next one computes
            const cudaEvent_t ec = ws.pool_event(evn++);
            CUDA_TRY(cudaEventRecord(ec, crt_stream));
            CUDA_TRY(cudaStreamWaitEvent(ws.s_d2h, ec, 0));
            tm.span(7, ws.s_d2h, [&] {
                CUDA_TRY(cudaMemcpy2DAsync((char*)C + esz * (size_t)(r0 * ldc + c0), esz * ldc,
                                           (const char*)dC + esz * (size_t)(r0 * n + c0), esz * n, esz * nc, rc,
                                           cudaMemcpyDeviceToHost, ws.s_d2h));
            });
        }
    };

    // mode 1: redo the dirty 256-column tiles of blocks [0, upto) (their CRT flags
    // go to the repair statuses; see the fallback after the final status read)
    auto repair_blocks = [&](size_t upto) {
        for (size_t bi = 0; bi < upto; ++bi) {
            bool any = false;
            for (int64_t t = 0; t < ntiles;) {
                if (!dirty1[(size_t)t]) { ++t; continue; }
                int64_t t1 = t + 1;
                while (t1 < ntiles && dirty1[(size_t)t1]) ++t1;
                run_block(bi, 256 * t, std::min<int64_t>(n, 256 * t1) - 256 * t, sx + 2 + nb + bi);
                any = true;
                t = t1;
            }
            if (any) ++repaired[bi];
        }
    };

    // ---- speculated row and column exponents (spec2) ----
    // A row chunks and B column chunks arrive alternately.  Each arrival is
    // scanned and its clearance products with everything already present are
    // formed; mu / nu of every row / column present are then re-derived from
    // the maxima so far (final after the last arrival).  The residues of a new
    // chunk, or of one whose exponents moved, are (re)computed, and every
    // tile (row chunk x column chunk) of C that is new or lies in a moved
    // chunk is (re)computed: residue GEMMs, CRT, download.  Status flags of
    // every stage that reads mu / nu are kept per chunk / tile and a tile's
    // are reset when it is redone, so only flags of the final exponents count.
    const int64_t nrs = spec2 ? nchunks : 0;
    const size_t nst2 = spec2 ? (size_t)(1 + nrs + ncc + nrs * nunits) : 0;
    auto run_spec2 = [&]() {
        ws.ensure_streams();
        // statuses: [0] discarded, [1 + r] A residues of row chunk r, [1 + nrs + c] B residues of
        // column chunk c, [1 + nrs + ncc + r * nunits + u] CRT of row chunk r x column unit u
        sx = (DevStatus*)ws.spec_st.get(sizeof(DevStatus) * nst2);
        CUDA_TRY(cudaMemsetAsync(sx, 0, sizeof(DevStatus) * nst2, stream));
        DevStatus* const st_tile = sx + 1 + nrs + ncc;
        changed_h = ws.changed_flags((size_t)(1 + nrs + nunits));
        CUDA_TRY(cudaHostGetDevicePointer((void**)&changed, changed_h, 0));
        const ChangeFlags cf{changed, chunk_rows, cu, nrs};
        volatile int32_t* const flags = changed_h;
        // W of one region launch, compact: [N][rows][round_up(cols, 16)]
        const int64_t wcap = (int64_t)N * std::max(chunk_rows * ldw, m * round_up(col_chunk, 16));
        int8_t* W2 = (int8_t*)ws.W.get((size_t)wcap);
        auto rows_of = [&](int r) { return std::min<int64_t>(chunk_rows, m - r * chunk_rows); };
        auto cols_of = [&](int c) { return cstart[(size_t)c + 1] - cstart[(size_t)c]; };
        auto unit_lo = [&](int c) { return cstart[(size_t)c] / cu; };
        auto unit_hi = [&](int c) { return (cstart[(size_t)c + 1] + cu - 1) / cu; };  // exclusive
        // GEMM + CRT + download of rows [r0, r0 + rc) x columns [c0, c0 + nc), whole tiles, in
        // pieces of at most one row chunk (each piece's download overlaps the next piece)
        auto run_region = [&](int64_t r0, int64_t rc, int64_t c0, int64_t nc) {
            const int64_t pitch = round_up(nc, 16);
            for (int64_t q = r0; q < r0 + rc;) {
                const int64_t rq = std::min<int64_t>(std::min<int64_t>(r0 + rc - q, chunk_rows), wcap / ((int64_t)N * pitch) / 128 * 128);
                GemmParams g = gp;
                g.planes = N;
                g.ldw = pitch;
                g.wplane = rq * pitch;
                g.n = (int)nc;
                g.tiles_n = (int)((nc + BN - 1) / BN);
                set_rows(g, rq);
                g.W = W2;
                const CUtensorMap tA = make_plane_map(ares + q * kp, kp, rq, N, boxA, m * kp);
                const CUtensorMap tB = make_plane_map_mn(bres + c0, nc, ldn, kp, N, kp * ldn);
                tm.span(5, stream, [&] { CUDA_TRY(launch_gemm(EPI_RESID, tA, tB, g)); });
                CrtExtra exr = ex;
                exr.sg = StatusGrid{st_tile, q, c0, chunk_rows, cu, nunits};
                tm.span(6, stream, [&] {
                    CUDA_TRY(launch_crt(prec, W2, pitch, rq * pitch, rq, nc, cc, mu + q, nu + c0,
                                        (char*)dC + esz * (size_t)(q * ldc_d + c0), ldc_d, exr, st, stream));
                });
                launches += 2;
                const cudaEvent_t ec = ws.pool_event(evn++);
                CUDA_TRY(cudaEventRecord(ec, stream));
                CUDA_TRY(cudaStreamWaitEvent(ws.s_d2h, ec, 0));
                tm.span(7, ws.s_d2h, [&] {
                    CUDA_TRY(cudaMemcpy2DAsync((char*)C + esz * (size_t)(q * ldc + c0), esz * ldc,
                                               (const char*)dC + esz * (size_t)(q * n + c0), esz * n, esz * nc, rq,
                                               cudaMemcpyDeviceToHost, ws.s_d2h));
                });
                q += rq;
            }
        };
        auto clearance = [&](int64_t r0, int64_t rc, int64_t c0, int64_t nc) {
            tm.span(2, stream, [&] {
                const CUtensorMap tA = make_plane_map(abar + r0 * kp, kp, rc, 1, boxA);
                const CUtensorMap tB = make_plane_map_mn(bbar + c0, nc, ldn, kp, 1, kp * ldn);
                GemmParams g = gp;
                g.n = (int)nc;
                g.tiles_n = (int)((nc + BN - 1) / BN);
                set_rows(g, rc);
                g.planes = 1;
                g.rowmax = cmax_row + r0;
                g.colmax = cmax_col + c0;
                CUDA_TRY(launch_gemm(EPI_MAX, tA, tB, g));
            });
            ++launches;
        };
        std::vector<char> haveA((size_t)nrs, 0), haveB((size_t)ncc, 0), done((size_t)(nrs * ncc), 0);
        int64_t invalidated = 0;  // tiles computed with exponents that later moved
        bool seen_move = false;
        bool give_up = false;     // defer every remaining tile to the final exponents
        int R = 0, Cn = 0;  // row / column chunks present (prefixes)
        for (const auto& a : arrivals) {
            if (a.first) {
                const int r = a.second;
                const int64_t r0 = r * chunk_rows, rc = rows_of(r);
                CUDA_TRY(cudaStreamWaitEvent(stream, ws.ev_a[r], 0));
                tm.span(1, stream, [&] {
                    CUDA_TRY(launch_row_scan_A(prec, (const char*)dA + esz * (size_t)(r0 * lda_d), lda_d, rc, k, kp,
                                               mup + r0, abar + r0 * kp, st, stream, r0));
                });
                ++launches;
                if (Cn) clearance(r0, rc, 0, cstart[(size_t)Cn]);
                ++R;
            } else {
                const int c = a.second;
                const int64_t c0 = cstart[(size_t)c], nc = cols_of(c);
                CUDA_TRY(cudaStreamWaitEvent(stream, ws.ev_bc[c], 0));
                tm.span(1, stream, [&] {
                    const char* Bc = (const char*)dB + esz * (size_t)c0;
                    CUDA_TRY(launch_col_max_B(prec, Bc, ldb_d, k, nc, bmax + c0, st, stream));
                    CUDA_TRY(launch_col_exp_B(bmax + c0, nc, nup + c0, st, stream, c0));
                    CUDA_TRY(launch_bbar_rows(prec, Bc, ldb_d, k, nc, kp, ldn, nup + c0, bbar + c0, st, stream,
                                              c == ncc - 1 ? ldn - c0 : nc));
                });
                launches += 3;
                if (R) clearance(0, std::min<int64_t>(m, R * chunk_rows), c0, nc);
                ++Cn;
            }
            if (R == 0 || Cn == 0) continue;
            const bool last = R == nrs && Cn == ncc;
            const int64_t mr = std::min<int64_t>(m, R * chunk_rows), nr = cstart[(size_t)Cn];
            std::memset(changed_h, 0, 4 * (size_t)(1 + nrs + nunits));  // idle: the last check was read
            tm.span(3, stream, [&] {
                CUDA_TRY(launch_exponents(cmax_row, mr, cmax_col, nr, mup, nup, tab.shift0, tab.nthr, tab.thr, mu,
                                          nu, ev, fv, last ? st : sx, stream, &cf));
            });
            ++launches;
            CUDA_TRY(cudaEventRecord(ws.ev_check, stream));
            CUDA_TRY(cudaEventSynchronize(ws.ev_check));
            // moved: exponents changed at this check; new: first exponents of the chunk
            std::vector<char> movR((size_t)R), movC((size_t)Cn), newR((size_t)R), newC((size_t)Cn);
            for (int r = 0; r < R; ++r) {
                newR[(size_t)r] = !haveA[(size_t)r];
                movR[(size_t)r] = flags[1 + r] != 0 && haveA[(size_t)r];
            }
            for (int c = 0; c < Cn; ++c) {
                bool mv = false;
                for (int64_t u = unit_lo(c); u < unit_hi(c); ++u) mv |= flags[1 + nrs + u] != 0;
                newC[(size_t)c] = !haveB[(size_t)c];
                movC[(size_t)c] = mv && haveB[(size_t)c];
            }
            // residues of new chunks and of chunks whose exponents moved
            tm.span(4, stream, [&] {
                for (int r = 0; r < R; ++r) {
                    if (!movR[(size_t)r] && !newR[(size_t)r]) continue;
                    const int64_t r0 = r * chunk_rows;
                    CUDA_TRY(cudaMemsetAsync(sx + 1 + r, 0, sizeof(DevStatus), stream));
                    CUDA_TRY(launch_resid_A(prec, (const char*)dA + esz * (size_t)(r0 * lda_d), lda_d, rows_of(r), k,
                                            kp, mu + r0, rc_dev, N, ares + r0 * kp, m * kp, sx + 1 + r, stream));
                    haveA[(size_t)r] = 1;
                    ++launches;
                }
                for (int c = 0; c < Cn; ++c) {
                    if (!movC[(size_t)c] && !newC[(size_t)c]) continue;
                    const int64_t c0 = cstart[(size_t)c];
                    CUDA_TRY(cudaMemsetAsync(sx + 1 + nrs + c, 0, sizeof(DevStatus), stream));
                    CUDA_TRY(launch_resid_B_rows(prec, (const char*)dB + esz * (size_t)c0, ldb_d, k, cols_of(c), kp,
                                                 ldn, nu + c0, rc_dev, N, bres + c0, sx + 1 + nrs + c, stream,
                                                 c == ncc - 1 ? ldn - c0 : cols_of(c)));
                    haveB[(size_t)c] = 1;
                    ++launches;
                }
            });
            // tiles.  A tile computed with an exponent that has since moved is
            // invalid.  Tiles are (re)computed when their row and column chunks
            // held still at this check (new chunks count as still until anything
            // has moved) or at the last arrival, so inputs whose maxima keep
            // moving (wide exponent spreads) are not recomputed at every arrival;
            // once an eighth of all tiles was invalidated, the rest wait for the
            // final exponents.
            for (int r = 0; r < R; ++r)
                for (int c = 0; c < Cn; ++c) {
                    const size_t t = (size_t)(r * ncc + c);
                    if (done[t] && (movR[(size_t)r] || movC[(size_t)c])) {
                        done[t] = 0;
                        ++invalidated;
                        spec_state = 2;
                    }
                }
            for (int r = 0; r < R; ++r) seen_move |= movR[(size_t)r] != 0;
            for (int c = 0; c < Cn; ++c) seen_move |= movC[(size_t)c] != 0;
            // once anything moved, a new chunk also has to hold still for one check
            auto still_r = [&](int r) { return !movR[(size_t)r] && !(seen_move && newR[(size_t)r]); };
            auto still_c = [&](int c) { return !movC[(size_t)c] && !(seen_move && newC[(size_t)c]); };
            auto ready = [&](int r, int c) {
                if (done[(size_t)(r * ncc + c)]) return false;
                return last || (!give_up && still_r(r) && still_c(c));
            };
            for (int r = 0; r < R; ++r) {
                for (int c = 0; c < Cn;) {
                    if (!ready(r, c)) { ++c; continue; }
                    int c1 = c + 1;
                    while (c1 < Cn && ready(r, c1)) ++c1;
                    for (int cc2 = c; cc2 < c1; ++cc2) done[(size_t)(r * ncc + cc2)] = 1;
                    CUDA_TRY(cudaMemsetAsync(st_tile + r * nunits + unit_lo(c), 0,
                                             sizeof(DevStatus) * (size_t)(unit_hi(c1 - 1) - unit_lo(c)), stream));
                    run_region(r * chunk_rows, rows_of(r), cstart[(size_t)c], cstart[(size_t)c1] - cstart[(size_t)c]);
                    c = c1;
                }
            }
            give_up |= 8 * invalidated >= nrs * ncc;
        }
        // flags of every chunk's residues and every tile's CRT (each from its final computation)
        CUDA_TRY(launch_merge_status(st, sx + 1, (int64_t)nst2 - 1, stream));
        ++launches;
    };

    // ---- K1 (A) + K2 per row chunk: row pre-exponents, Abar, clearance product with fused maxima ----
    // Pipelined: B is complete before the first chunk, so a chunk's row maxima
    // are final after its clearance GEMM and its mu and A residues follow at
    // once, overlapping the upload of the next chunks.
    if (spec2) run_spec2();
    size_t next_block = 0;
    for (int c = 0; c < (scan && !spec2 ? nchunks : 0); ++c) {
        const int64_t r0 = c * chunk_rows, rc = std::min<int64_t>(chunk_rows, m - r0);
        if (pipe) CUDA_TRY(cudaStreamWaitEvent(stream, arr ? arr->a[c] : ws.ev_a[c], 0));
        tm.span(1, stream, [&] {
            CUDA_TRY(launch_row_scan_A(prec, (const char*)dA + esz * (size_t)(r0 * lda_d), lda_d, rc, k, kp,
                                       mup + r0, abar + r0 * kp, st, stream, r0));
        });
        launches += rc > 0;
        if (ev_bdone) CUDA_TRY(cudaStreamWaitEvent(stream, ev_bdone, 0));  // join: Bbar and nu' are ready
        if (rc > 0 && n > 0) tm.span(2, stream, [&] {
            const CUtensorMap tA = make_plane_map(abar + r0 * kp, kp, rc, 1, boxA);
            const CUtensorMap tB = make_plane_map_mn(bbar, n, ldn, kp, 1, kp * ldn);
            GemmParams g = gp;
            set_rows(g, rc);
            g.planes = 1;
            g.rowmax = cmax_row + r0;
            g.colmax = cmax_col;
            CUDA_TRY(launch_gemm(EPI_MAX, tA, tB, g)); ++launches;
            if (inter && inter->Cbar) {
                GemmParams g2 = g;
                g2.C32 = (int32_t*)ws.x_cbar.get(4 * (size_t)(m * n));
                g2.ldc32 = n;
                g2.cplane = m * n;
                CUDA_TRY(launch_gemm(EPI_I32, tA, tB, g2)); ++launches;
            }
        });
        if (pipe && !hooked && rc > 0) {
            tm.span(3, stream, [&] {
                CUDA_TRY(launch_exponents(cmax_row + r0, rc, cmax_col, 0, mup + r0, nup, tab.shift0, tab.nthr,
                                          tab.thr, mu + r0, nu, ev + r0, fv, st, stream));
                if (spec) {  // column exponents from the maxima so far (final after the last chunk)
                    if (c > 0) std::memset(changed_h, 0, 4 * (size_t)(1 + ntiles));  // idle: last check was read
                    CUDA_TRY(launch_exponents(cmax_row, 0, cmax_col, n, mup, nup, tab.shift0, tab.nthr, tab.thr, mu,
                                              nu, ev, fv, c == nchunks - 1 ? st : sx, stream,
                                              c > 0 ? &cf1 : nullptr));
                    ++launches;
                }
            });
            tm.span(4, stream, [&] {
                CUDA_TRY(launch_resid_A(prec, (const char*)dA + esz * (size_t)(r0 * lda_d), lda_d, rc, k, kp,
                                        mu + r0, rc_dev, N, ares + r0 * kp, m * kp, st, stream));
            });
            launches += 2;
        }
        if (spec) {
            bool moved = c == 0;
            if (c > 0) {
                CUDA_TRY(cudaEventRecord(ws.ev_check, stream));
                CUDA_TRY(cudaEventSynchronize(ws.ev_check));
                moved = ((volatile int32_t*)changed_h)[0] != 0;
            }
            volatile int32_t* const fl = changed_h;
            if (c > 0 && moved) {
                spec_state = 2;
                int64_t nmoved = 0;
                for (int64_t t = 0; t < ntiles; ++t) nmoved += fl[1 + t] != 0;
                // repairs cost (blocks done) x (moved tiles); past an eighth of all
                // block tiles, stop computing blocks before the final exponents
                const bool was_deferred = defer1;
                if (!defer1 && 8 * (repair_work + (int64_t)next_block * nmoved) > (int64_t)nb * ntiles) defer1 = true;
                for (int64_t t = 0; t < ntiles; ++t)  // tiles to repair (accumulated while deferred)
                    dirty1[(size_t)t] = (was_deferred && dirty1[(size_t)t]) || fl[1 + t] != 0;
                if (!defer1) repair_work += (int64_t)next_block * nmoved;
            }
            if (moved && !defer1) {  // B residues with the exponents so far, then the repairs
                tm.span(4, stream, [&] {
                    CUDA_TRY(cudaMemsetAsync(sx + 1, 0, sizeof(DevStatus), stream));
                    CUDA_TRY(launch_resid_B_rows(prec, dB, ldb_d, k, n, kp, ldn, nu, rc_dev, N, bres, sx + 1, stream));
                });
                ++launches;
                if (c > 0) repair_blocks(next_block);
            }
            if (!defer1)
                for (; next_block < nb && blocks[next_block].chunk <= c; ++next_block)
                    run_block(next_block, 0, n, sx + 2 + next_block);
        }
    }
    if (spec && defer1) {
        // the exponents are final: B residues, then the moved tiles of the blocks
        // computed before deferring, then every remaining block
        tm.span(4, stream, [&] {
            CUDA_TRY(cudaMemsetAsync(sx + 1, 0, sizeof(DevStatus), stream));
            CUDA_TRY(launch_resid_B_rows(prec, dB, ldb_d, k, n, kp, ldn, nu, rc_dev, N, bres, sx + 1, stream));
        });
        ++launches;
        repair_blocks(next_block);
        for (; next_block < nb; ++next_block) run_block(next_block, 0, n, sx + 2 + next_block);
    }
    if (reduce_fn) {
        if (reduce_fn(cmax_row, m, cmax_col, n, (void*)stream, reduce_user) != 0)
        {
            Fail f{OZ2G_CUDA_ERROR, "oz2g_gemm: reduce_maxima callback failed"};
            f.order = 201;  // a peer's own failure (multi-device) is the one to report
            throw f;
        }
    }

    if (spec || spec2) {
        if (ws.ev_inputs_free) CUDA_TRY(cudaEventRecord(ws.ev_inputs_free, stream));
    } else {
        // ---- K3: scaling exponents; K4: residue planes ----
        // (pipelined: row exponents and A residues were produced per chunk during the upload)
        tm.span(3, stream, [&] {
            CUDA_TRY(launch_exponents(cmax_row, (pipe && !hooked) ? 0 : m, cmax_col, n, mup, nup, tab.shift0, tab.nthr,
                                      tab.thr,
                                      mu, nu, ev, fv, st, stream));
        });
        ++launches;
        if (fork) {  // B residues beside the A residues
            const cudaEvent_t ef = ws.pool_event(evn++);
            CUDA_TRY(cudaEventRecord(ef, stream));
            CUDA_TRY(cudaStreamWaitEvent(sB, ef, 0));
        }
        tm.span(4, stream, [&] {
            if (!pipe || hooked) {  // (streamed: the first row block only)
                const int64_t ra = rstream ? blocks[0].rows : m;
                CUDA_TRY(launch_resid_A(prec, dA, lda_d, ra, k, kp, mu, rc_dev, N, ares, m * kp, st, stream));
                launches += m > 0;
            }
        });
        tm.span(4, sB, [&] {
            CUDA_TRY(launch_resid_B_rows(prec, dB, ldb_d, k, n, kp, ldn, nu, rc_dev, N, bres, st, sB));
            launches += n > 0;
        });
        if (fork) {
            const cudaEvent_t ej = ws.pool_event(evn++);
            CUDA_TRY(cudaEventRecord(ej, sB));
            CUDA_TRY(cudaStreamWaitEvent(stream, ej, 0));
        }

        if (bo && m * n) {
            // bounds.hpp:143-206 evaluated in the CRT pass
            const BoundScalars bs = bound_scalars(tab, k);
            double* vec = (double*)ws.x_bvec.get(8 * (size_t)(2 * (m + n)) + 4 * (size_t)(m + n) + 16);
            BoundVecs v;
            v.RA = vec; v.PA = vec + m; v.CB = vec + 2 * m; v.PB = vec + 2 * m + n;
            v.ea = reinterpret_cast<int32_t*>(vec + 2 * (m + n));
            v.eb = v.ea + m;
            double* scratch = (double*)ws.x_bscr.get(8 * bound_scratch_doubles(m, n, k));
            CUDA_TRY(launch_bound_vectors(prec, dA, lda_d, m, dB, ldb_d, k, n, cmax_row, cmax_col, mup, nup, bs.t_up,
                                          scratch, v, stream));
            launches += 5;
            if (bo->relative && !ws.lo_ready)
                compute_relative_operands(ws, prec, dA, lda_d, dB, ldb_d, m, n, k, mup, nup, stream, launches);
            bmax_dev = (unsigned long long*)ws.x_bmax.get(32);
            CUDA_TRY(cudaMemsetAsync(bmax_dev, 0, 24, stream));
            ex.bnd.ab_lo = bo->relative ? (const double*)ws.ab_lo.p : nullptr;
            ex.bnd.on = 1;
            ex.bnd.v = v;
            ex.bnd.t2_up = bs.t2_up;
            ex.bnd.rconst_up = bs.rconst_up;
            ex.bnd.ucoef = bs.ucoef;
            ex.bnd.kpr_cheap_up = bs.kpr_cheap_up;
            ex.bnd.k_rconst_up = bs.k_rconst_up;
            ex.bnd.max_bits = bmax_dev;
            if (bo->cheap) ex.bnd.cheap = bo->device ? bo->cheap : (double*)ws.x_bcheap.get(mn8);
            if (bo->tight) ex.bnd.tight = bo->device ? bo->tight : (double*)ws.x_btight.get(mn8);
        }
        // every read of the device copies of A and B is enqueued by now
        if (host && ws.ev_inputs_free) CUDA_TRY(cudaEventRecord(ws.ev_inputs_free, stream));
        if (fused) {
            // the N residue GEMMs with the CRT and the inverse scaling in their epilogue:
            // one launch over every 128 x 128 tile of C, no W
            FusedParams fp;
            std::memset(&fp, 0, sizeof fp);
            fp.g = gp;
            fp.g.planes = N;
            fp.g.m = (int)m;
            fp.g.n = (int)n;
            fp.g.tiles_m = (int)((m + fused_tile_m() - 1) / fused_tile_m());
            fp.g.tiles_n = (int)((n + fused_tile_n() - 1) / fused_tile_n());
            // the fused kernel rasters by tile-rows only (a "group_n" request
            // falls back to the default tile-row groups)
            const int gm = group_m_for(fp.g.tiles_m, fp.g.tiles_n);
            fp.g.group_m = gm > 0 ? gm : std::max(1, std::min(16, fp.g.tiles_m));
            for (int l = 0; l < N; ++l) { fp.s1[l] = tab.s1[l]; fp.s2[l] = tab.s2[l]; }
            fp.P1 = tab.P1; fp.P2 = tab.P2; fp.P_inv = tab.P_inv;
            fp.mode = tab.mode;
            fp.probe = fused_mode() == 2 ? 1 : 0;
            fp.dbg = opt(OPT_DEBUG_SYNC) ? 1 : 0;
            if (opt(OPT_FUSED_FENCE) != 0) {
                fp.plane_sync = (unsigned long long*)ws.x_bmax.get(64) + 4;
                CUDA_TRY(cudaMemsetAsync(fp.plane_sync, 0, 8, stream));
            }
            fp.mu = mu;
            fp.nu = nu;
            fp.C = dC;
            fp.ldc = ldc_d;
            fp.st = st;
            // option "fused_mc" 1: CTA pairs sharing a multicast B tile (default 0: one CTA per tile)
            const bool mc = opt(OPT_FUSED_MC) != 0;
            const CUtensorMap tA = make_plane_map(ares, kp, m, N, fused_tile_m(), m * kp);
            const CUtensorMap tB = make_plane_map_mn(bres, n, ldn, kp, N, kp * ldn, fused_b_box_rows(mc));
            tm.span(5, stream, [&] { CUDA_TRY(launch_gemm_crt_fused(prec, tA, tB, fp, ws.num_sms, mc, stream)); });
            ++launches;
            if (pipe && host) {  // the pipelined path downloads on its D2H stream (joined below)
                const cudaEvent_t ec = ws.pool_event(evn++);
                CUDA_TRY(cudaEventRecord(ec, stream));
                CUDA_TRY(cudaStreamWaitEvent(ws.s_d2h, ec, 0));
                tm.span(7, ws.s_d2h, [&] {
                    CUDA_TRY(cudaMemcpy2DAsync(C, esz * ldc, dC, esz * n, esz * n, m, cudaMemcpyDeviceToHost, ws.s_d2h));
                });
            }
        } else if (rstream) {
            size_t ev_res = 0;  // event after the A residues of block bi
            for (size_t bi = 0; bi < nb; ++bi) {
                if (bi > 0) CUDA_TRY(cudaStreamWaitEvent(stream, ws.pool_event(ev_res), 0));
                if (bi + 1 < nb) {
                    const int64_t r0 = blocks[bi + 1].r0, rb = blocks[bi + 1].rows;
                    tm.span(4, sB, [&] {
                        CUDA_TRY(launch_resid_A(prec, (const char*)dA + esz * (size_t)(r0 * lda_d), lda_d, rb, k, kp,
                                                mu + r0, rc_dev, N, ares + r0 * kp, m * kp, st, sB));
                    });
                    ++launches;
                    ev_res = evn++;
                    CUDA_TRY(cudaEventRecord(ws.pool_event(ev_res), sB));
                }
                run_block(bi, 0, n, st);
            }
        } else {
            for (size_t bi = 0; bi < nb; ++bi) run_block(bi, 0, n, st);
        }
    }
    if (overlap) {  // join the side stream
        const cudaEvent_t ej = ws.pool_event(evn++);
        CUDA_TRY(cudaEventRecord(ej, ws.s_aux));
        CUDA_TRY(cudaStreamWaitEvent(stream, ej, 0));
    }
    if (pipe && host) {
        CUDA_TRY(cudaEventRecord(ws.ev_done, ws.s_d2h));
        CUDA_TRY(cudaStreamWaitEvent(stream, ws.ev_done, 0));
    } else if (host && m * n) {
        tm.span(7, stream, [&] {
            CUDA_TRY(cudaMemcpy2DAsync(C, esz * ldc, dC, esz * n, esz * n, m, cudaMemcpyDeviceToHost, stream));
        });
    }

    // ---- intermediates (host copies) ----
    std::vector<int32_t> tmp32;
    if (inter) {
        auto get_i16 = [&](int16_t* dst, const int32_t* src, int64_t cnt) {
            if (!dst || cnt == 0) return;
            tmp32.resize((size_t)cnt);
            CUDA_TRY(cudaMemcpyAsync(tmp32.data(), src, 4 * (size_t)cnt, cudaMemcpyDeviceToHost, stream));
            CUDA_TRY(cudaStreamSynchronize(stream));
            for (int64_t i = 0; i < cnt; ++i) dst[i] = (int16_t)tmp32[(size_t)i];
        };
        get_i16(inter->mu, mu, m);
        get_i16(inter->nu, nu, n);
        get_i16(inter->mu_prime, mup, m);
        get_i16(inter->nu_prime, nup, n);
        if (inter->e && m) CUDA_TRY(cudaMemcpyAsync(inter->e, ev, 4 * (size_t)m, cudaMemcpyDeviceToHost, stream));
        if (inter->f && n) CUDA_TRY(cudaMemcpyAsync(inter->f, fv, 4 * (size_t)n, cudaMemcpyDeviceToHost, stream));
        if (inter->cmax_row && m) CUDA_TRY(cudaMemcpyAsync(inter->cmax_row, cmax_row, 4 * (size_t)m, cudaMemcpyDeviceToHost, stream));
        if (inter->cmax_col && n) CUDA_TRY(cudaMemcpyAsync(inter->cmax_col, cmax_col, 4 * (size_t)n, cudaMemcpyDeviceToHost, stream));
        if (inter->Aprime && m * k) {
            double* d = (double*)ws.x_ap.get(8 * (size_t)(m * k));
            CUDA_TRY(launch_trunc_scaled(prec, dA, lda_d, m, k, mu, 0, d, stream)); ++launches;
            CUDA_TRY(cudaMemcpyAsync(inter->Aprime, d, 8 * (size_t)(m * k), cudaMemcpyDeviceToHost, stream));
        }
        if (inter->Bprime && k * n) {
            double* d = (double*)ws.x_bp.get(8 * (size_t)(k * n));
            CUDA_TRY(launch_trunc_scaled(prec, dB, ldb_d, k, n, nu, 1, d, stream)); ++launches;
            CUDA_TRY(cudaMemcpyAsync(inter->Bprime, d, 8 * (size_t)(k * n), cudaMemcpyDeviceToHost, stream));
        }
        if (m * n) {
            if (inter->Cbar) CUDA_TRY(cudaMemcpyAsync(inter->Cbar, ws.x_cbar.p, 4 * (size_t)(m * n), cudaMemcpyDeviceToHost, stream));
            if (inter->W)
                for (int l = 0; l < N; ++l)
                    CUDA_TRY(cudaMemcpy2DAsync(inter->W + (size_t)l * (size_t)(m * n), (size_t)n, W + (size_t)l * (size_t)(m * ldw),
                                               (size_t)ldw, (size_t)n, (size_t)m, cudaMemcpyDeviceToHost, stream));
            if (inter->Cprod) CUDA_TRY(cudaMemcpyAsync(inter->Cprod, ws.x_cprod.p, 4 * (size_t)N * (size_t)(m * n), cudaMemcpyDeviceToHost, stream));
            if (ex.C1) CUDA_TRY(cudaMemcpyAsync(inter->C1, ex.C1, mn8, cudaMemcpyDeviceToHost, stream));
            if (ex.C2) CUDA_TRY(cudaMemcpyAsync(inter->C2, ex.C2, mn8, cudaMemcpyDeviceToHost, stream));
            if (ex.Q) CUDA_TRY(cudaMemcpyAsync(inter->Q, ex.Q, mn8, cudaMemcpyDeviceToHost, stream));
            if (ex.Cpp64) CUDA_TRY(cudaMemcpyAsync(inter->Cpp64, ex.Cpp64, mn8, cudaMemcpyDeviceToHost, stream));
            if (ex.Cpp32) CUDA_TRY(cudaMemcpyAsync(inter->Cpp32, ex.Cpp32, mn8 / 2, cudaMemcpyDeviceToHost, stream));
        }
        if (inter->Ares && m * k)
            for (int l = 0; l < N; ++l)
                CUDA_TRY(cudaMemcpy2DAsync(inter->Ares + (size_t)l * (size_t)(m * k), (size_t)k, ares + (size_t)l * (size_t)(m * kp),
                                           (size_t)kp, (size_t)k, (size_t)m, cudaMemcpyDeviceToHost, stream));
        if (inter->Bres && k * n)  // device planes are [kp][ldn], the reference layout k x n
            for (int l = 0; l < N; ++l)
                CUDA_TRY(cudaMemcpy2DAsync(inter->Bres + (size_t)l * (size_t)(k * n), (size_t)n,
                                           bres + (size_t)l * (size_t)(kp * ldn), (size_t)ldn, (size_t)n, (size_t)k,
                                           cudaMemcpyDeviceToHost, stream));
    }

    if (async) {
        if (!ws.ev_last_async) CUDA_TRY(cudaEventCreateWithFlags(&ws.ev_last_async, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(ws.ev_last_async, stream));
        ws.last_async_stream = stream;
        CUDA_TRY(cudaGetLastError());
        ws.pending.push_back({ring_slot, row_base, col_base, stream});
        if (diag) diag->kernels_launched = launches;
        return OZ2G_OK;
    }

    if (g_capture) {  // run_gemm_graph reads the status after the replay
        if (diag) diag->kernels_launched = launches;
        return OZ2G_OK;
    }
    unsigned long long bmax_host[3] = {0, 0, 0};
    if (bo && bmax_dev) {
        CUDA_TRY(cudaMemcpyAsync(bmax_host, bmax_dev, 24, cudaMemcpyDeviceToHost, stream));
        if (!bo->device && bo->cheap) CUDA_TRY(cudaMemcpyAsync(bo->cheap, ex.bnd.cheap, mn8, cudaMemcpyDeviceToHost, stream));
        if (!bo->device && bo->tight) CUDA_TRY(cudaMemcpyAsync(bo->tight, ex.bnd.tight, mn8, cudaMemcpyDeviceToHost, stream));
    }
    DevStatus hs;
    CUDA_TRY(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaGetLastError());
    if (spec) {
        std::vector<DevStatus> hx(2 + 2 * nb);
        CUDA_TRY(cudaMemcpy(hx.data(), sx, sizeof(DevStatus) * hx.size(), cudaMemcpyDeviceToHost));
        bool redo = false;
        for (size_t bi = 0; bi < nb; ++bi) {
            // a block whose first CRT, or (repaired more than once) an earlier repair,
            // raised a flag under exponents that later moved
            redo |= repaired[bi] && (hx[2 + bi].err || hx[2 + bi].subnormal);
            redo |= repaired[bi] > 1 && (hx[2 + nb + bi].err || hx[2 + nb + bi].subnormal);
        }
        if (redo) {
            // a block computed with a superseded nu raised a flag that may not
            // hold for the final nu: redo every stage after the upload from the
            // device copies of A and B (the unspeculated device path, which also
            // reports this call's errors) and download C again
            const int outer = launches;
            run_gemm(prec, m, n, k, dA, lda_d, dB, ldb_d, dC, ldc_d, nmod, OZ2G_DEVICE_PTRS | (flags & OZ2G_TIMING),
                     stream, inter, diag, nullptr, nullptr, row_base, col_base, slot, false);
            if (m * n)
                CUDA_TRY(cudaMemcpy2DAsync(C, esz * ldc, dC, esz * n, esz * n, m, cudaMemcpyDeviceToHost, stream));
            CUDA_TRY(cudaStreamSynchronize(stream));
            if (diag) {
                diag->kernels_launched += outer;
                diag->speculation = 3;
            }
            return OZ2G_OK;
        }
        // flags of the B residues (last run, final nu) and of every CRT
        for (size_t i = 1; i < hx.size(); ++i) {
            hs.err |= hx[i].err;
            hs.subnormal |= hx[i].subnormal;
        }
    }
    if (bo) {
        double v0, v1;
        std::memcpy(&v0, &bmax_host[0], 8);
        std::memcpy(&v1, &bmax_host[1], 8);
        bo->cheap_max = v0;
        bo->tight_max = v1;
        if (bo->relative) std::memcpy(&bo->tight_rel_max, &bmax_host[2], 8);
    }

    if (inter && inter->Dbar && inter->Cbar)
        for (int64_t i = 0; i < m * n; ++i) inter->Dbar[i] = fp32_round_up(inter->Cbar[i]);

    if (diag) {
        diag->subnormal = hs.subnormal ? 1 : 0;
        diag->kernels_launched = launches;
        diag->speculation = spec_state;
        if (tm.on) {
            // stage order: 0 H2D, 1 K1 scale, 2 clearance GEMM, 3 exponents, 4 residues,
            //              5 residue GEMMs, 6 CRT, 7 D2H
            tm.collect(diag->stage_ms);
        }
    }

    Fail f{OZ2G_OK, ""};
    if (status_failure(hs, row_base, col_base, f)) throw f;
    return OZ2G_OK;
}

}  // namespace oz2g
