// api_ext.cu — the C ABI (include/oz2g.h) and the runners built on run_gemm:
// CUDA-graph replays of repeated device-pointer calls, suggest_n (cheap and
// tight), the single-process multi-device tiling and the N sweep.
#include "api_internal.h"

#include <condition_variable>
#include <cstdio>
#include <thread>

namespace oz2g {
namespace {
// Device-pointer calls repeated with the same shape, pointers, N and stream
// replay a CUDA graph of the whole pipeline (memsets, every kernel) instead of
// re-enqueuing ~20 launches: the first call runs normally (and allocates), the
// second captures, later ones replay; a workspace reallocation anywhere
// (g_alloc_gen) invalidates the graphs.  The status word is read after the
// replay from pinned memory, so errors are reported exactly as run_gemm does.
// Option "graph" 0 disables.
bool graph_enabled() { return opt(OPT_GRAPH) != 0; }

int run_gemm_graph(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                   void* C, int64_t ldc, int nmod, unsigned flags, cudaStream_t stream, oz2g_diag* diag) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    Workspace& ws = workspace(dev, 0);
    std::lock_guard<std::recursive_mutex> dev_lock(ws.mtx);
    // OZ2G_ASYNC: the replay is followed by a copy of the call's status into
    // its ring slot and joins the pending list (complete_pending checks it)
    const bool async = (flags & OZ2G_ASYNC) != 0;
    if (!async && !ws.pending.empty()) {
        Fail f{OZ2G_OK, ""};
        if (complete_pending(ws, f)) throw f;
    }
    const std::vector<int64_t> key{prec, m, n, k, (int64_t)(uintptr_t)A, lda, (int64_t)(uintptr_t)B, ldb,
                                   (int64_t)(uintptr_t)C, ldc, nmod, (int64_t)(uintptr_t)stream, fused_mode(),
                                   (int64_t)flags};
    Workspace::GraphEntry& e = ws.graphs[key];
    const uint64_t gen = g_alloc_gen.load();
    if (!e.exec || e.gen != gen) {
        if (e.exec) { cudaGraphExecDestroy(e.exec); e.exec = nullptr; }
        if (e.plain || e.seen++ == 0 || ws.graphs.size() > 64) {  // first sight: a plain call (allocates, uploads)
            if (ws.graphs.size() > 64) ws.drop_graphs();
            return run_gemm(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, stream, nullptr, diag, nullptr,
                            nullptr);
        }
        if (!ws.pending.empty()) {  // (async key) earlier calls complete before the capture
            Fail f{OZ2G_OK, ""};
            if (complete_pending(ws, f)) throw f;
        }
        oz2g_diag d;
        std::memset(&d, 0, sizeof d);
        if (!ws.s_cap) CUDA_TRY(cudaStreamCreateWithFlags(&ws.s_cap, cudaStreamNonBlocking));
        if (!ws.status_host) CUDA_TRY(cudaHostAlloc((void**)&ws.status_host, sizeof(DevStatus), cudaHostAllocDefault));
        // capture; any failure (an operation the capture does not allow, instantiation)
        // leaves this entry plain and the call runs uncaptured
        auto capture = [&]() -> bool {
            cudaGraph_t g = nullptr;
            if (cudaStreamBeginCapture(ws.s_cap, cudaStreamCaptureModeRelaxed) != cudaSuccess) return false;
            g_capture = true;
            bool ok = true;
            try {
                run_gemm(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags & ~OZ2G_ASYNC, ws.s_cap, nullptr, &d,
                         nullptr, nullptr);
            } catch (...) {
                ok = false;
            }
            g_capture = false;
            // the status read-back is the graph's last node
            if (ok && cudaMemcpyAsync(ws.status_host, ws.status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                                      ws.s_cap) != cudaSuccess)
                ok = false;
            if (cudaStreamEndCapture(ws.s_cap, &g) != cudaSuccess) ok = false;
            if (ok && g && cudaGraphInstantiate(&e.exec, g, 0) != cudaSuccess) {
                e.exec = nullptr;
                ok = false;
            }
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();  // clear a capture error
            return ok && e.exec;
        };
        if (!capture()) {
            e.plain = true;
            return run_gemm(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, stream, nullptr, diag, nullptr,
                            nullptr);
        }
        e.gen = g_alloc_gen.load();
        e.launches = d.kernels_launched;
    }
    if (diag) std::memset(diag, 0, sizeof *diag);
    if (async) {
        if ((int)ws.pending.size() >= kStatusRing) {  // ring full: complete the oldest calls first
            Fail f{OZ2G_OK, ""};
            if (complete_pending(ws, f)) throw f;
        }
        if (!ws.pending.empty() && ws.last_async_stream != stream)
            CUDA_TRY(cudaStreamWaitEvent(stream, ws.ev_last_async, 0));
        const int slot = ws.ring_next;
        ws.ring_next = (ws.ring_next + 1) % kStatusRing;
        DevStatus* ring = (DevStatus*)ws.status_ring.get(sizeof(DevStatus) * kStatusRing);
        CUDA_TRY(cudaGraphLaunch(e.exec, stream));
        CUDA_TRY(cudaMemcpyAsync(ring + slot, ws.status.p, sizeof(DevStatus), cudaMemcpyDeviceToDevice, stream));
        if (!ws.ev_last_async) CUDA_TRY(cudaEventCreateWithFlags(&ws.ev_last_async, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(ws.ev_last_async, stream));
        ws.last_async_stream = stream;
        ws.pending.push_back({slot, 0, 0, stream});
        if (diag) diag->kernels_launched = e.launches;
        return OZ2G_OK;
    }
    CUDA_TRY(cudaGraphLaunch(e.exec, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (diag) {
        diag->kernels_launched = e.launches;
        diag->subnormal = ws.status_host->subnormal != 0;
    }
    Fail f{OZ2G_OK, ""};
    if (status_failure(*ws.status_host, 0, 0, f)) throw f;
    return OZ2G_OK;
}

// suggest_n (bounds.hpp:217-243): one clearance pass (Cbar does not depend on
// N), then the cheap bound's maximum for N = 2, 3, ... until it meets the
// absolute target.  fp32 candidates stop at the format's safe ceiling.
int run_suggest_n(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                  double target, unsigned flags, cudaStream_t stream, int* n_out, double* bound_out) {
    if (prec != OZ2G_FP32 && prec != OZ2G_FP64) throw Fail{OZ2G_INVALID_ARGUMENT, "suggest_n: bad precision"};
    if (!(target > 0)) throw Fail{OZ2G_DOMAIN_ERROR, "suggest_n: target must be positive"};
    if (m < 0 || n < 0 || k < 0 || lda < k || ldb < n) throw Fail{OZ2G_INVALID_ARGUMENT, "dimension mismatch: suggest_n"};
    if (k > OZ2G_MAX_INNER_DIM) throw Fail{OZ2G_DOMAIN_ERROR, "os_ii: k exceeds 2^17"};
    if (k == 0 && m > 0) throw Fail{OZ2G_DOMAIN_ERROR, "row_pre_exponents: zero row 0"};
    if (k == 0 && n > 0) throw Fail{OZ2G_DOMAIN_ERROR, "col_pre_exponents: zero column 0"};
    *n_out = 0;
    *bound_out = 0.0;
    if (m == 0 || n == 0) return OZ2G_OK;
    const bool host = (flags & OZ2G_DEVICE_PTRS) == 0;
    const size_t esz = prec ? 8 : 4;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    Workspace& ws = workspace(dev);
    std::lock_guard<std::recursive_mutex> dev_lock(ws.mtx);
    if (!ws.pending.empty()) {  // complete earlier OZ2G_ASYNC calls (they may still read ws.A / ws.B)
        Fail f{OZ2G_OK, ""};
        if (complete_pending(ws, f)) throw f;
    }
    const int64_t kp = round_up(k, 128);
    const void* dA = A;
    const void* dB = B;
    int64_t lda_d = lda, ldb_d = ldb;
    if (host) {
        dA = ws.A.get(esz * (size_t)(m * k));
        dB = ws.B.get(esz * (size_t)(k * n));
        lda_d = k; ldb_d = n;
        CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dA), esz * k, A, esz * lda, esz * k, m, cudaMemcpyHostToDevice, stream));
        CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dB), esz * n, B, esz * ldb, esz * n, k, cudaMemcpyHostToDevice, stream));
    }
    DevStatus* st = (DevStatus*)ws.status.get(sizeof(DevStatus));
    CUDA_TRY(cudaMemsetAsync(st, 0, 8, stream));
    CUDA_TRY(cudaMemsetAsync(&st->first_row, 0x7f, 16, stream));
    int32_t* mup = (int32_t*)ws.mup.get(4 * (size_t)m);
    int32_t* nup = (int32_t*)ws.nup.get(4 * (size_t)n);
    unsigned long long* bmax = (unsigned long long*)ws.bmax.get(8 * (size_t)n);
    int32_t* cmax_row = (int32_t*)ws.cmax_row.get(4 * (size_t)m);
    int32_t* cmax_col = (int32_t*)ws.cmax_col.get(4 * (size_t)n);
    int8_t* abar = (int8_t*)ws.abar.get((size_t)(m * kp));
    const int64_t ldn = round_up(n, 16);
    int8_t* bbar = (int8_t*)ws.bbar.get((size_t)(kp * ldn));
    CUDA_TRY(cudaMemsetAsync(bmax, 0, 8 * (size_t)n, stream));
    CUDA_TRY(cudaMemsetAsync(cmax_row, 0, 4 * (size_t)m, stream));
    CUDA_TRY(cudaMemsetAsync(cmax_col, 0, 4 * (size_t)n, stream));
    CUDA_TRY(launch_col_max_B(prec, dB, ldb_d, k, n, bmax, st, stream));
    CUDA_TRY(launch_col_exp_B(bmax, n, nup, st, stream));
    CUDA_TRY(launch_bbar_rows(prec, dB, ldb_d, k, n, kp, ldn, nup, bbar, st, stream));
    CUDA_TRY(launch_row_scan_A(prec, dA, lda_d, m, k, kp, mup, abar, st, stream, 0));
    GemmParams gp;
    std::memset(&gp, 0, sizeof gp);
    gp.m = (int)m;
    gp.n = (int)n;
    gp.kblocks = (int)(kp / 128);
    gp.tiles_m = (int)((m + gemm_tile_m() - 1) / gemm_tile_m());
    gp.tiles_n = (int)((n + gemm_tile_n() - 1) / gemm_tile_n());
    gp.group_m = group_m_for(gp.tiles_m, gp.tiles_n);
    set_l2_hints(gp);
    gp.planes = 1;
    gp.rowmax = cmax_row;
    gp.colmax = cmax_col;
    CUDA_TRY(launch_gemm_i8(EPI_MAX, make_plane_map(abar, kp, m, 1, gemm_tile_m()),
                            make_plane_map_mn(bbar, n, ldn, kp, 1, kp * ldn), gp, ws.num_sms, stream));
    // exponent_stats (bounds.hpp:32-60) as the per-row / per-column factors with t = 1
    double* vec = (double*)ws.x_bvec.get(8 * (size_t)(2 * (m + n)) + 4 * (size_t)(m + n) + 16);
    BoundVecs v;
    v.RA = vec; v.PA = vec + m; v.CB = vec + 2 * m; v.PB = vec + 2 * m + n;
    v.ea = reinterpret_cast<int32_t*>(vec + 2 * (m + n));
    v.eb = v.ea + m;
    double* scratch = (double*)ws.x_bscr.get(8 * bound_scratch_doubles(m, n, k));
    CUDA_TRY(launch_bound_vectors(prec, dA, lda_d, m, dB, ldb_d, k, n, cmax_row, cmax_col, mup, nup, 1.0, scratch, v,
                                  stream));
    DevStatus hs;
    CUDA_TRY(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (hs.err & (ERR_A_NONFINITE | ERR_B_NONFINITE)) throw Fail{OZ2G_DOMAIN_ERROR, "matrix entry is not finite"};
    if (hs.err & (ERR_A_ZERO_ROW | ERR_B_ZERO_COL)) throw Fail{OZ2G_DOMAIN_ERROR, "exponent_stats: zero row"};
    unsigned long long* bits = (unsigned long long*)ws.x_bmax.get(16);
    const int n_max = prec == OZ2G_FP32 ? fp32_safe_moduli_max() : kMaxModuli;
    for (int nm = 2; nm <= n_max; ++nm) {
        const BoundScalars bs = bound_scalars(table_for(nm, prec), k);
        CUDA_TRY(cudaMemsetAsync(bits, 0, 8, stream));
        CUDA_TRY(launch_cheap_bound_max(v, m, n, bs.t_up, __builtin_nextafter(bs.kpr_cheap_up * bs.t2_up, 1e308), bits,
                                        ws.num_sms, stream));
        unsigned long long hb = 0;
        CUDA_TRY(cudaMemcpyAsync(&hb, bits, 8, cudaMemcpyDeviceToHost, stream));
        CUDA_TRY(cudaStreamSynchronize(stream));
        double mx;
        std::memcpy(&mx, &hb, 8);
        *bound_out = mx;
        if (mx <= target) {
            *n_out = nm;
            return OZ2G_OK;
        }
    }
    return OZ2G_OK;  // not achievable: n_out = 0, bound_out = bound max at the cap
}

// suggest_n with the TIGHT bound (bounds.hpp:182-195), absolute or relative
// to (|A||B|)_ij: the smallest N whose device tight-bound maximum (the sound
// |A'B'| <= (|C''| + r_const) / (1 - u_coef) form, bounds.cu) meets `target`.
// The tight bound needs C'' at that N, i.e. a full emulation, so:
//  1. one scaling + clearance pass and the N-independent bound factors;
//  2. N = 2, 3, ...: a lower estimate of the tight bound (tight without its
//     |A'B'| term, over an upper bound of |A||B|) proves N too small while it
//     exceeds the target; the first N it does not exclude is N0;
//  3. N = N0, N0 + 1, ...: the emulation with the bounds evaluated in its CRT
//     pass (the N sweep: scaling reused) until the maximum meets the target.
// So every N below the answer is shown to fail — by the lower estimate or by
// its own emulation.
int run_suggest_tight(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                      int64_t ldb, double target, int relative, unsigned flags, cudaStream_t stream,
                      oz2g_suggest* out) {
    if (!out) throw Fail{OZ2G_INVALID_ARGUMENT, "suggest_n: null result"};
    std::memset(out, 0, sizeof *out);
    int n_cheap = 0;
    double cheap_max = 0.0;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    Workspace& ws = workspace(dev, 0);
    std::lock_guard<std::recursive_mutex> dev_lock(ws.mtx);
    // steps 1 (the cheap search's scaling pass leaves mu', nu', the clearance
    // maxima and the bound factors with t = 1 in the workspace)
    run_suggest_n(prec, m, n, k, A, lda, B, ldb, target, flags, stream, &n_cheap, &cheap_max);
    out->cheap_n = n_cheap;
    if (m == 0 || n == 0) return OZ2G_OK;
    const bool host = (flags & OZ2G_DEVICE_PTRS) == 0;
    const size_t esz = prec ? 8 : 4;
    const void* dA = host ? ws.A.p : A;
    const void* dB = host ? ws.B.p : B;
    const int64_t lda_d = host ? k : lda, ldb_d = host ? n : ldb;
    int launches = 0;
    int32_t* mup = (int32_t*)ws.mup.p;
    int32_t* nup = (int32_t*)ws.nup.p;
    if (relative) compute_relative_operands(ws, prec, dA, lda_d, dB, ldb_d, m, n, k, mup, nup, stream, launches);
    const double* vec = (const double*)ws.x_bvec.p;
    BoundVecs v;
    v.RA = const_cast<double*>(vec); v.PA = v.RA + m; v.CB = v.RA + 2 * m; v.PB = v.RA + 2 * m + n;
    v.ea = reinterpret_cast<int32_t*>(v.RA + 2 * (m + n));
    v.eb = v.ea + m;
    const int32_t* sums = (const int32_t*)ws.lo_sum.p;
    unsigned long long* bits = (unsigned long long*)ws.x_bmax.get(32);
    const int n_max = prec == OZ2G_FP32 ? fp32_safe_moduli_max() : kMaxModuli;
    int n0 = 0;
    for (int nm = 2; nm <= n_max && !n0; ++nm) {
        const BoundScalars bs = bound_scalars(table_for(nm, prec), k);
        CUDA_TRY(cudaMemsetAsync(bits, 0, 8, stream));
        CUDA_TRY(launch_tight_lower_max(v, m, n, k, bs.t_up, __builtin_nextafter(bs.k_rconst_up * bs.t2_up, 1e308),
                                        relative ? (const int32_t*)ws.lo_ab.p : nullptr, relative ? sums : nullptr,
                                        relative ? sums + m : nullptr, bits, ws.num_sms, stream));
        unsigned long long hb = 0;
        CUDA_TRY(cudaMemcpyAsync(&hb, bits, 8, cudaMemcpyDeviceToHost, stream));
        CUDA_TRY(cudaStreamSynchronize(stream));
        double lower;
        std::memcpy(&lower, &hb, 8);
        if (!(lower > target)) n0 = nm;
        else out->excluded_below = nm + 1;
    }
    if (!n0) return OZ2G_OK;  // every N excluded: not achievable
    // step 3: emulations on the kept scaling (lo_ready survives reuse_scaling calls)
    DevBuf cbuf;
    struct Rel { DevBuf* b; ~Rel() { b->release(); } } rel{&cbuf};
    void* dC = cbuf.get(esz * (size_t)(m * n));
    for (int nm = n0; nm <= n_max; ++nm) {
        oz2g_bounds bo;
        std::memset(&bo, 0, sizeof bo);
        bo.relative = relative;
        oz2g_intermediates in;
        std::memset(&in, 0, sizeof in);
        in.bounds = &bo;
        oz2g_diag d;
        run_gemm(prec, m, n, k, dA, lda_d, dB, ldb_d, dC, n, nm, OZ2G_DEVICE_PTRS, stream, &in, &d, nullptr, nullptr,
                 0, 0, 0, /*reuse_scaling=*/true);
        ++out->emulations;
        const double val = relative ? bo.tight_rel_max : bo.tight_max;
        out->bound_max = val;
        out->tight_max = bo.tight_max;
        out->tight_rel_max = bo.tight_rel_max;
        if (val <= target) {
            out->n = nm;
            return OZ2G_OK;
        }
    }
    return OZ2G_OK;
}

// ---------------------------------------------------------------------------
// Single-process multi-device tiling (oz2g_gemm_multi): the C grid
// R x Cg over the listed devices (1 -> 1x1, 2 -> 2x1, 4 -> 2x2, 8 -> 2x4, else
// count x 1; the same grid as paper_2602_02549_b200/dist.py), one host thread
// per tile.  Tile (r, c) gets the row block r of A and the column block c of B
// (all of k).  The clearance maxima are max-reduced across tiles on the host
// between the clearance product and the scaling exponents — the reduce hook of
// oz2g_gemm — so every tile scales exactly as the single-device call does and
// C is bit-identical.  Inputs are host pointers (each device uploads its own
// blocks over its own link).
// ---------------------------------------------------------------------------
void grid_shape(int count, int& R, int& Cg) {
    switch (count) {
        case 1: R = 1; Cg = 1; break;
        case 2: R = 2; Cg = 1; break;
        case 4: R = 2; Cg = 2; break;
        case 8: R = 2; Cg = 4; break;
        default: R = count; Cg = 1; break;
    }
}

struct MultiCtx {
    std::mutex mtx;
    std::condition_variable cv;
    int count = 0, arrived = 0, generation = 0;
    bool broken = false;
    std::vector<int32_t> rowmax, colmax;  // global clearance maxima
    // barrier that a failing tile can break (the others then fail fast)
    bool wait() {
        std::unique_lock<std::mutex> lk(mtx);
        if (broken) return false;
        const int gen = generation;
        if (++arrived == count) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return true;
        }
        cv.wait(lk, [&] { return broken || generation != gen; });
        return generation != gen;
    }
    void breakit() {
        std::lock_guard<std::mutex> lk(mtx);
        broken = true;
        cv.notify_all();
    }
};

struct MultiTile {
    MultiCtx* ctx;
    int64_t r0, c0;
};

int multi_reduce_hook(int32_t* rowp, int64_t m, int32_t* colp, int64_t n, void* stream, void* user) {
    MultiTile* t = static_cast<MultiTile*>(user);
    MultiCtx* x = t->ctx;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<int32_t> hr((size_t)m), hc((size_t)n);
    bool ok = true;
    if (m) ok &= cudaMemcpyAsync(hr.data(), rowp, 4 * (size_t)m, cudaMemcpyDeviceToHost, s) == cudaSuccess;
    if (n) ok &= cudaMemcpyAsync(hc.data(), colp, 4 * (size_t)n, cudaMemcpyDeviceToHost, s) == cudaSuccess;
    ok &= cudaStreamSynchronize(s) == cudaSuccess;
    if (!ok) { x->breakit(); return -1; }
    {
        std::lock_guard<std::mutex> lk(x->mtx);
        for (int64_t i = 0; i < m; ++i) x->rowmax[(size_t)(t->r0 + i)] = std::max(x->rowmax[(size_t)(t->r0 + i)], hr[(size_t)i]);
        for (int64_t j = 0; j < n; ++j) x->colmax[(size_t)(t->c0 + j)] = std::max(x->colmax[(size_t)(t->c0 + j)], hc[(size_t)j]);
    }
    if (!x->wait()) return -1;
    {
        std::lock_guard<std::mutex> lk(x->mtx);
        for (int64_t i = 0; i < m; ++i) hr[(size_t)i] = x->rowmax[(size_t)(t->r0 + i)];
        for (int64_t j = 0; j < n; ++j) hc[(size_t)j] = x->colmax[(size_t)(t->c0 + j)];
    }
    if (m) ok &= cudaMemcpyAsync(rowp, hr.data(), 4 * (size_t)m, cudaMemcpyHostToDevice, s) == cudaSuccess;
    if (n) ok &= cudaMemcpyAsync(colp, hc.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, s) == cudaSuccess;
    ok &= cudaStreamSynchronize(s) == cudaSuccess;
    return ok ? 0 : -1;
}

int run_gemm_multi(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                   void* C, int64_t ldc, int nmod, unsigned flags, const int* devices, int count, oz2g_diag* diag) {
    if (!devices || count < 1) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_multi: empty device list"};
    if (count > 256) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_multi: at most 256 tiles"};
    if (flags & OZ2G_DEVICE_PTRS) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_multi: host pointers required"};
    if (prec != OZ2G_FP32 && prec != OZ2G_FP64) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: prec must be OZ2G_FP32 or OZ2G_FP64"};
    if (m < 0 || n < 0 || k < 0) throw Fail{OZ2G_INVALID_ARGUMENT, "Matrix: negative dimension"};
    if (lda < k || ldb < n || ldc < n) throw Fail{OZ2G_INVALID_ARGUMENT, "dimension mismatch: leading dimension"};
    if (k > OZ2G_MAX_INNER_DIM) throw Fail{OZ2G_DOMAIN_ERROR, "os_ii: k exceeds 2^17"};
    (void)table_for(nmod, prec);  // std::domain_error for N outside [2, 49]
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    for (int t = 0; t < count; ++t)
        if (devices[t] < 0 || devices[t] >= ndev) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_multi: no such device"};
    if (diag) std::memset(diag, 0, sizeof *diag);
    // every tile thread holds its workspace lock while it waits at the
    // cross-tile barrier of the maxima exchange: two multi calls interleaving
    // their tiles over the same (device, slot) workspaces could each hold a
    // lock the other's barrier waits on, so multi calls run one at a time
    static std::mutex multi_mtx;
    std::lock_guard<std::mutex> multi_lock(multi_mtx);
    const size_t esz = prec ? 8 : 4;
    int R = 1, Cg = 1;
    grid_shape(count, R, Cg);
    const int64_t mb = (m + R - 1) / R, nb = (n + Cg - 1) / Cg;
    MultiCtx ctx;
    ctx.count = count;
    ctx.rowmax.assign((size_t)m, 0);
    ctx.colmax.assign((size_t)n, 0);
    std::vector<MultiTile> tiles((size_t)count);
    std::vector<Fail> fails((size_t)count, Fail{OZ2G_OK, ""});
    std::vector<oz2g_diag> diags((size_t)count);
    int caller_dev = 0;
    CUDA_TRY(cudaGetDevice(&caller_dev));
    auto body = [&](int t) {
        const int r = t / Cg, c = t % Cg;
        const int64_t r0 = std::min(m, r * mb), r1 = std::min(m, (r + 1) * mb);
        const int64_t c0 = std::min(n, c * nb), c1 = std::min(n, (c + 1) * nb);
        tiles[(size_t)t] = MultiTile{&ctx, r0, c0};
        try {
            CUDA_TRY(cudaSetDevice(devices[t]));
            Workspace& ws = workspace(devices[t], t);
            {
                std::lock_guard<std::recursive_mutex> lk(ws.mtx);
                ws.ensure_streams();
            }
            run_gemm(prec, r1 - r0, c1 - c0, k, (const char*)A + esz * (size_t)(r0 * lda), lda,
                     (const char*)B + esz * (size_t)c0, ldb, (char*)C + esz * (size_t)(r0 * ldc + c0), ldc, nmod,
                     flags & OZ2G_TIMING, ws.s_main, nullptr, diag ? &diags[(size_t)t] : nullptr, multi_reduce_hook,
                     &tiles[(size_t)t], r0, c0, t);
        } catch (const Fail& f) {
            fails[(size_t)t] = f;
            ctx.breakit();
        } catch (const std::exception& e) {
            fails[(size_t)t] = Fail{OZ2G_CUDA_ERROR, e.what()};
            ctx.breakit();
        }
    };
    if (count == 1) {
        body(0);
    } else {
        std::vector<std::thread> th;
        th.reserve((size_t)count);
        for (int t = 0; t < count; ++t) th.emplace_back(body, t);
        for (auto& x : th) x.join();
    }
    cudaSetDevice(caller_dev);
    const Fail* worst = nullptr;
    for (const Fail& f : fails)
        if (f.code != OZ2G_OK && (!worst || f.order < worst->order || (f.order == worst->order && f.index < worst->index)))
            worst = &f;
    if (worst) throw *worst;
    if (diag) {
        for (const oz2g_diag& d : diags) {
            diag->subnormal |= d.subnormal;
            diag->kernels_launched += d.kernels_launched;
            for (int q = 0; q < 8; ++q) diag->stage_ms[q] = std::max(diag->stage_ms[q], d.stage_ms[q]);
        }
    }
    return OZ2G_OK;
}

// Several N on the same A, B (the cfg3 sweep): the pre-exponents,
// Abar / Bbar and the clearance maxima do not depend on N, so they are
// computed once; each N then runs exponents, residues, residue GEMMs and CRT.
// C[i] (ldc) receives the result for nmods[i]; every C[i] equals
// oz2g_gemm(..., nmods[i]) bit for bit.
int run_gemm_sweep(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                   void* const* C, int64_t ldc, const int* nmods, int count, unsigned flags, cudaStream_t stream,
                   oz2g_diag* diag) {
    if (count < 1 || !nmods || !C) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_sweep: empty moduli list"};
    if (flags & (OZ2G_ASYNC | OZ2G_TIMING)) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_sweep: no async / timing"};
    if (prec != OZ2G_FP32 && prec != OZ2G_FP64) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: prec must be OZ2G_FP32 or OZ2G_FP64"};
    if (m < 0 || n < 0 || k < 0) throw Fail{OZ2G_INVALID_ARGUMENT, "Matrix: negative dimension"};
    if (lda < k || ldb < n || ldc < n) throw Fail{OZ2G_INVALID_ARGUMENT, "dimension mismatch: leading dimension"};
    for (int i = 0; i < count; ++i) (void)table_for(nmods[i], prec);  // every N valid before any work
    const bool host = (flags & OZ2G_DEVICE_PTRS) == 0;
    const size_t esz = prec ? 8 : 4;
    if (diag) std::memset(diag, 0, sizeof *diag);
    const void* dA = A;
    const void* dB = B;
    void* dC = nullptr;
    int64_t lda_d = lda, ldb_d = ldb, ldc_d = ldc;
    DevBuf bufA, bufB, bufC;  // sweep-private device copies for host inputs / outputs
    if (host) {
        dA = bufA.get(esz * (size_t)(m * k));
        dB = bufB.get(esz * (size_t)(k * n));
        dC = bufC.get(esz * (size_t)(m * n));
        lda_d = k; ldb_d = n; ldc_d = n;
        if (m * k) CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dA), esz * k, A, esz * lda, esz * k, m, cudaMemcpyHostToDevice, stream));
        if (k * n) CUDA_TRY(cudaMemcpy2DAsync(const_cast<void*>(dB), esz * n, B, esz * ldb, esz * n, k, cudaMemcpyHostToDevice, stream));
    }
    struct Release {
        DevBuf *a, *b, *c;
        ~Release() { a->release(); b->release(); c->release(); }
    } rel{&bufA, &bufB, &bufC};
    // later iterations reuse mu', nu' and the clearance maxima left in the
    // device workspace by the first: hold its lock for the whole sweep so no
    // concurrent call on this device can overwrite them in between
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::recursive_mutex> sweep_lock(workspace(dev, 0).mtx);
    for (int i = 0; i < count; ++i) {
        void* Ci = host ? dC : C[i];
        oz2g_diag d;
        run_gemm(prec, m, n, k, dA, lda_d, dB, ldb_d, Ci, ldc_d, nmods[i], OZ2G_DEVICE_PTRS, stream, nullptr,
                 diag ? &d : nullptr, nullptr, nullptr, 0, 0, 0, /*reuse_scaling=*/i > 0);
        if (diag) {
            diag->subnormal |= d.subnormal;
            diag->kernels_launched += d.kernels_launched;
        }
        if (host && m * n)
            CUDA_TRY(cudaMemcpy2DAsync(C[i], esz * ldc, dC, esz * n, esz * n, m, cudaMemcpyDeviceToHost, stream));
    }
    CUDA_TRY(cudaStreamSynchronize(stream));
    return OZ2G_OK;
}

template <class F>
int guarded(F&& f) {
    g_last_error.clear();
    try {
        return f();
    } catch (const Fail& x) {
        g_last_error = x.what;
        return x.code;
    } catch (const std::invalid_argument& x) {
        g_last_error = x.what();
        return OZ2G_INVALID_ARGUMENT;
    } catch (const std::domain_error& x) {
        g_last_error = x.what();
        return OZ2G_DOMAIN_ERROR;
    } catch (const std::range_error& x) {
        g_last_error = x.what();
        return OZ2G_RANGE_ERROR;
    } catch (const std::logic_error& x) {
        g_last_error = x.what();
        return OZ2G_LOGIC_ERROR;
    } catch (const std::exception& x) {
        g_last_error = x.what();
        return OZ2G_CUDA_ERROR;
    }
}

}  // namespace
}  // namespace oz2g

using namespace oz2g;

extern "C" {

int oz2g_gemm(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
              void* C, int64_t ldc, int nmod, unsigned flags, void* stream, oz2g_intermediates* inter,
              oz2g_diag* diag, oz2g_reduce_maxima_fn reduce_fn, void* reduce_user) {
    return guarded([&] {
        if ((flags & ~OZ2G_ASYNC) == OZ2G_DEVICE_PTRS && !inter && !reduce_fn && graph_enabled() && m > 0 && n > 0 &&
            k > 0)
            return run_gemm_graph(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, (cudaStream_t)stream, diag);
        return run_gemm(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, (cudaStream_t)stream, inter, diag,
                        reduce_fn, reduce_user);
    });
}

int oz2g_dgemm(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
               double* C, int64_t ldc, int nmod, unsigned flags, void* stream, oz2g_diag* diag) {
    return oz2g_gemm(OZ2G_FP64, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, stream, nullptr, diag, nullptr, nullptr);
}

int oz2g_sgemm(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B, int64_t ldb,
               float* C, int64_t ldc, int nmod, unsigned flags, void* stream, oz2g_diag* diag) {
    return oz2g_gemm(OZ2G_FP32, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, stream, nullptr, diag, nullptr, nullptr);
}

int oz2g_gemm_multi(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                    void* C, int64_t ldc, int nmod, unsigned flags, const int* devices, int count, oz2g_diag* diag) {
    return guarded([&] {
        return run_gemm_multi(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, devices, count, diag);
    });
}

int oz2g_gemm_sweep(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                    void* const* C, int64_t ldc, const int* nmods, int count, unsigned flags, void* stream,
                    oz2g_diag* diag) {
    return guarded([&] {
        return run_gemm_sweep(prec, m, n, k, A, lda, B, ldb, C, ldc, nmods, count, flags, (cudaStream_t)stream, diag);
    });
}

int oz2g_grid_shape(int count, int* rows, int* cols) {
    if (count < 1 || !rows || !cols) return OZ2G_INVALID_ARGUMENT;
    grid_shape(count, *rows, *cols);
    return OZ2G_OK;
}

int oz2g_init(const int* devices, int count) {
    return guarded([&] {
        if (count < 0 || (count > 0 && !devices)) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_init: bad device list"};
        int caller = 0;
        CUDA_TRY(cudaGetDevice(&caller));
        for (int t = 0; t < count; ++t) {
            CUDA_TRY(cudaSetDevice(devices[t]));
            Workspace& ws = workspace(devices[t], 0);
            std::lock_guard<std::recursive_mutex> lk(ws.mtx);
            ws.ensure_streams();
            for (int mode : {OZ2G_FP32, OZ2G_FP64})
                for (int nm = 2; nm <= 49; ++nm) {
                    const Table& tab = table_for(nm, mode);
                    const auto key = std::make_pair(tab.n, tab.mode);
                    if (ws.rc.count(key)) continue;
                    const std::vector<uint8_t> h = build_resid_consts(tab);
                    ResidConsts* d = nullptr;
                    CUDA_TRY(cudaMalloc(&d, h.size()));
                    CUDA_TRY(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
                    ws.rc[key] = d;
                }
        }
        CUDA_TRY(cudaSetDevice(caller));
        return OZ2G_OK;
    });
}

int oz2g_synchronize(void) {
    return guarded([&] {
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        Workspace& ws = workspace(dev, 0);
        std::lock_guard<std::recursive_mutex> lk(ws.mtx);
        Fail f{OZ2G_OK, ""};
        if (complete_pending(ws, f)) throw f;
        return OZ2G_OK;
    });
}

const char* oz2g_last_error(void) { return g_last_error.c_str(); }

int oz2g_table_for(int n, int mode, oz2g_table* out) {
    return guarded([&] {
        if (mode != OZ2G_FP32 && mode != OZ2G_FP64) throw Fail{OZ2G_INVALID_ARGUMENT, "table_for: bad mode"};
        const Table& t = table_for(n, mode);
        std::memset(out, 0, sizeof *out);
        out->n = t.n;
        out->mode = t.mode;
        for (int l = 0; l < t.n; ++l) {
            out->p[l] = t.p[l];
            out->q[l] = t.q[l];
            out->beta[l] = t.beta[l];
            out->s1[l] = t.s1[l];
            out->s2[l] = t.s2[l];
        }
        out->rho = t.rho;
        out->P1 = t.P1;
        out->P2 = t.P2;
        out->P_inv = t.P_inv;
        out->P_prime = t.P_prime;
        std::snprintf(out->P_dec, sizeof out->P_dec, "%s", t.P_dec.c_str());
        out->shift0 = t.shift0;
        out->nthr = t.nthr;
        for (int q = 0; q < t.nthr; ++q) out->thr[q] = t.thr[q];
        return OZ2G_OK;
    });
}

int oz2g_fp32_safe_moduli_max(void) { return fp32_safe_moduli_max(); }

int oz2g_shift_of_cmax(int n, int64_t c) {
    const Table& t = table_for(n < 2 ? 2 : (n > 49 ? 49 : n), OZ2G_FP64);
    return shift_of_cmax(t.P_prime, c, nullptr);
}

int oz2g_device_log2f(const float* x_dev, float* out_dev, int64_t count, void* stream) {
    return guarded([&] {
        CUDA_TRY(launch_log2f(x_dev, out_dev, count, (cudaStream_t)stream));
        return OZ2G_OK;
    });
}

int oz2g_suggest_n(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                   double target, unsigned flags, void* stream, int* n_out, double* bound_max) {
    return guarded([&] {
        return run_suggest_n(prec, m, n, k, A, lda, B, ldb, target, flags, (cudaStream_t)stream, n_out, bound_max);
    });
}

int oz2g_suggest_n_tight(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                         int64_t ldb, double target, int relative, unsigned flags, void* stream, oz2g_suggest* out) {
    return guarded([&] {
        return run_suggest_tight(prec, m, n, k, A, lda, B, ldb, target, relative, flags, (cudaStream_t)stream, out);
    });
}

int oz2g_dd_gemm(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                 double* Chi, double* Clo, int64_t ldc, void* stream) {
    return guarded([&] {
        if (m < 0 || n < 0 || k < 0 || lda < k || ldb < n || ldc < n)
            throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_dd_gemm: bad dimensions"};
        CUDA_TRY(launch_dd_gemm(A, lda, B, ldb, m, n, k, Chi, Clo, ldc, (cudaStream_t)stream));
        return OZ2G_OK;
    });
}

int oz2g_native_gemm(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                     int64_t ldb, void* C, int64_t ldc, void* stream) {
    return guarded([&] {
        if (m < 0 || n < 0 || k < 0 || lda < k || ldb < n || ldc < n)
            throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_native_gemm: bad dimensions"};
        CUDA_TRY(launch_native_gemm(prec, A, lda, B, ldb, m, n, k, C, ldc, (cudaStream_t)stream));
        return OZ2G_OK;
    });
}

}  // extern "C"

namespace oz2g {

int gemm_arrivals(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, int nmod, unsigned flags, cudaStream_t stream, oz2g_diag* diag,
                  oz2g_reduce_maxima_fn reduce_fn, void* reduce_user, const Arrivals& arr, std::string* err) {
    const int rc = guarded([&] {
        if ((flags & ~OZ2G_TIMING) != OZ2G_DEVICE_PTRS)
            throw Fail{OZ2G_INVALID_ARGUMENT, "gemm_arrivals: device pointers, C only"};
        return run_gemm(prec, m, n, k, A, lda, B, ldb, C, ldc, nmod, flags, stream, nullptr, diag, reduce_fn,
                        reduce_user, 0, 0, 0, false, &arr);
    });
    if (rc != OZ2G_OK && err) *err = g_last_error;
    return rc;
}

}  // namespace oz2g

extern "C" {

int oz2g_set_option(const char* name, long long value) {
    return guarded([&] {
        const int i = opt_index(name);
        if (i < 0) throw Fail{OZ2G_INVALID_ARGUMENT, std::string("oz2g_set_option: unknown option ") + (name ? name : "(null)")};
        if (!opt_set(i, value))
            throw Fail{OZ2G_INVALID_ARGUMENT, std::string("oz2g_set_option: value out of range for ") + name};
        ++g_alloc_gen;  // captured graphs embed the old choice
        return OZ2G_OK;
    });
}

int oz2g_get_option(const char* name, long long* value) {
    return guarded([&] {
        const int i = opt_index(name);
        if (i < 0 || !value) throw Fail{OZ2G_INVALID_ARGUMENT, std::string("oz2g_get_option: unknown option ") + (name ? name : "(null)")};
        *value = opt((Opt)i);
        return OZ2G_OK;
    });
}

const char* oz2g_option_name(int index) { return opt_name(index); }

int oz2g_i8_peak(long long iters, int launches, int random, double* ms_out, double* ops_out) {
    return guarded([&] {
        if (iters < 1 || launches < 1) throw Fail{OZ2G_INVALID_ARGUMENT, "oz2g_i8_peak: iters, launches >= 1"};
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        Workspace& ws = workspace(dev, 0);
        std::lock_guard<std::recursive_mutex> lk(ws.mtx);
        int* sink = (int*)ws.x_bmax.get(32);
        cudaStream_t s = nullptr;
        cudaEvent_t e0, e1;
        CUDA_TRY(cudaEventCreate(&e0));
        CUDA_TRY(cudaEventCreate(&e1));
        double ops = 0, one = 0;
        CUDA_TRY(launch_i8_peak(iters, random, ws.num_sms, sink, s, &one));  // warm-up
        CUDA_TRY(cudaEventRecord(e0, s));
        for (int i = 0; i < launches; ++i) {
            CUDA_TRY(launch_i8_peak(iters, random, ws.num_sms, sink, s, &one));
            ops += one;
        }
        CUDA_TRY(cudaEventRecord(e1, s));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms_out) *ms_out = ms;
        if (ops_out) *ops_out = ops;
        return OZ2G_OK;
    });
}

int oz2g_version(void) { return OZ2G_API_VERSION; }

void oz2g_release_workspace(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_ws_mtx);
    for (auto& kv : g_ws)
        if (kv.first / 256 == dev) {
            std::lock_guard<std::recursive_mutex> wl(kv.second->mtx);
            for (const auto& p : kv.second->pending) cudaStreamSynchronize(p.stream);
            kv.second->pending.clear();
            kv.second->release();
        }
}

}  // extern "C"
