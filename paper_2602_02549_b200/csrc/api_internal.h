// api_internal.h — shared internals of the host orchestration (api.cu, api_ext.cu):
// the error type, device buffers, per-device workspaces, launch helpers and the
// single-device pipeline run_gemm.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/oz2g.h"
#include "arrivals.h"
#include "device_common.cuh"
#include "kernels.h"
#include "tables.h"

namespace oz2g {


extern thread_local std::string g_last_error;

struct Fail {
    int code;
    std::string what;
    // multi-device calls report the failure the single-device call would:
    // the smallest (order, index) — order = position in the reference's
    // pipeline, index = the global row / column for zero-row / zero-column errors
    int order = 200;
    int64_t index = 0;
};

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            throw Fail{OZ2G_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)};    \
    } while (0)

// Bumped whenever any workspace buffer is (re)allocated: a captured CUDA
// graph (run_gemm_graph) embeds buffer addresses and is valid only while this
// is unchanged.
extern std::atomic<uint64_t> g_alloc_gen;

// run_gemm enqueues only (no final status read-back) while a graph is captured.
extern thread_local bool g_capture;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            ++g_alloc_gen;
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CUDA_TRY(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Host-pointer calls on large problems are pipelined in row chunks of A / C
// (see run_gemm): uploads of A overlap the row scan and the clearance GEMM,
// and the download of each finished C row block overlaps the next block.
constexpr int kPipeChunks = 8;
constexpr int kMaxColChunks = kPipeChunks + 4;  // spec2 column chunks: regular ones + a halving tail
// The last C row block is split in this many pieces so that only a small
// download follows the last kernel.
constexpr int kTailSplit = 4;

struct Workspace {
    DevBuf A, B, C, abar, bbar, ares, bres, W, mup, nup, mu, nu, bmax, cmax_row, cmax_col, e, f, status;
    DevBuf x_cbar, x_cprod, x_c1, x_c2, x_q, x_cpp64, x_cpp32, x_ap, x_bp, x_bvec, x_bscr, x_bmax, x_bcheap, x_btight;
    DevBuf spec_st;  // speculated column exponents: per-stage statuses
    // relative error criterion (suggest_n tight / relative): floor operands, their
    // row / column sums and product (launch_floor_operands); valid for the
    // inputs of the last scan that computed them
    DevBuf lo_a, lo_b, lo_sum, lo_ab, ab_lo;
    bool lo_ready = false;
    // changed-tile flags of the speculation checks: mapped pinned host memory
    // written by the check kernel, read by the host after an event
    int32_t* spec_changed = nullptr;
    size_t spec_changed_cap = 0;
    cudaEvent_t ev_check = nullptr;
    int32_t* changed_flags(size_t count) {
        if (count > spec_changed_cap) {
            if (spec_changed) cudaFreeHost(spec_changed);
            spec_changed = nullptr;
            spec_changed_cap = 0;
            CUDA_TRY(cudaHostAlloc((void**)&spec_changed, 4 * count, cudaHostAllocMapped));
            spec_changed_cap = count;
        }
        if (!ev_check) CUDA_TRY(cudaEventCreateWithFlags(&ev_check, cudaEventDisableTiming));
        return spec_changed;
    }
    std::map<std::pair<int, int>, ResidConsts*> rc;  // device copies of residue constants
    // CUDA graphs of device-pointer calls (run_gemm_graph), keyed by the call's
    // shape, pointers, N, stream and path; valid for one allocation generation
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        uint64_t gen = 0;
        int launches = 0;
        int seen = 0;
        bool plain = false;  // capture failed once: always run plainly
    };
    std::map<std::vector<int64_t>, GraphEntry> graphs;
    DevStatus* status_host = nullptr;  // pinned copy of the status word read after a replay
    cudaStream_t s_cap = nullptr;      // graphs are captured on this stream (the legacy stream cannot be)
    void drop_graphs() {
        for (auto& kv : graphs)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        graphs.clear();
    }
    int num_sms = 0;
    std::recursive_mutex mtx;           // calls on one workspace are serialised (re-entered by the
                                        // speculation fallback of run_gemm)
    cudaStream_t s_main = nullptr;      // compute stream of oz2g_gemm_multi tiles
    // copy streams / events of the pipelined host-pointer path
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr, s_aux = nullptr;
    // OZ2G_ASYNC: one status slot per call in flight, completed by oz2g_synchronize
    struct Pending { int slot; int64_t row_base, col_base; cudaStream_t stream; };
    DevBuf status_ring;
    int ring_next = 0;
    std::vector<Pending> pending;
    cudaEvent_t ev_inputs_free = nullptr;  // the last read of the device copies of A and B
    // end of the last OZ2G_ASYNC call and its stream: an asynchronous call on
    // another stream waits for it (every call shares this workspace's buffers)
    cudaEvent_t ev_last_async = nullptr;
    cudaStream_t last_async_stream = nullptr;
    std::vector<cudaEvent_t> ev_pool;  // per-block events of the overlapped CRT
    cudaEvent_t pool_event(size_t i) {
        while (ev_pool.size() <= i) {
            cudaEvent_t e = nullptr;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev_pool.push_back(e);
        }
        return ev_pool[i];
    }
    cudaEvent_t ev_start = nullptr, ev_b = nullptr, ev_done = nullptr;
    cudaEvent_t ev_a[kPipeChunks] = {}, ev_bc[kMaxColChunks] = {}, ev_c[kPipeChunks + kTailSplit] = {};
    void ensure_streams() {
        if (s_h2d) return;
        CUDA_TRY(cudaStreamCreateWithFlags(&s_main, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&s_aux, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&ev_start, &ev_b, &ev_done, &ev_inputs_free})
            CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        for (int c = 0; c < kPipeChunks; ++c) CUDA_TRY(cudaEventCreateWithFlags(&ev_a[c], cudaEventDisableTiming));
        for (int c = 0; c < kMaxColChunks; ++c) CUDA_TRY(cudaEventCreateWithFlags(&ev_bc[c], cudaEventDisableTiming));
        for (int c = 0; c < kPipeChunks + kTailSplit; ++c)
            CUDA_TRY(cudaEventCreateWithFlags(&ev_c[c], cudaEventDisableTiming));
    }
    void release() {
        for (DevBuf* b : {&A, &B, &C, &abar, &bbar, &ares, &bres, &W, &mup, &nup, &mu, &nu, &bmax, &cmax_row,
                          &cmax_col, &e, &f, &status, &x_cbar, &x_cprod, &x_c1, &x_c2, &x_q, &x_cpp64, &x_cpp32,
                          &x_ap, &x_bp, &x_bvec, &x_bscr, &x_bmax, &x_bcheap, &x_btight, &status_ring, &spec_st,
                          &lo_a, &lo_b, &lo_sum, &lo_ab, &ab_lo})
            b->release();
        if (spec_changed) cudaFreeHost(spec_changed);
        spec_changed = nullptr;
        spec_changed_cap = 0;
        for (auto& kv : rc) cudaFree(kv.second);
        rc.clear();
        drop_graphs();
        if (status_host) cudaFreeHost(status_host);
        status_host = nullptr;
        lo_ready = false;
    }
};


extern std::mutex g_ws_mtx;
extern std::map<int, Workspace*> g_ws;  // key device * 256 + slot

constexpr int kStatusRing = 64;
constexpr double kPdlMaxWork = 2048.0 * 2048.0 * 2048.0;  // m n k up to which run_gemm uses PDL
// Row block of the residue GEMMs + CRT: one raster group (16 x 128 rows), so
// W (N int8 planes) is held for one block only.
constexpr int64_t kWBlockRows = 2048;

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Per-stage device time (OZ2G_TIMING): every launch or copy is bracketed by
// events on the stream it runs on and the intervals are summed per stage, so
// the numbers are right for row-blocked and pipelined calls too (where stages
// overlap, a stage's figure is its busy time).
struct Timer {
    bool on = false;
    struct Interval { int stage; cudaEvent_t a, b; };
    std::vector<Interval> iv;
    std::vector<cudaEvent_t> owned;
    cudaEvent_t rec(cudaStream_t s) {
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        owned.push_back(e);
        return e;
    }
    template <class F>
    void span(int stage, cudaStream_t s, F&& f) {
        if (opt(OPT_DEBUG_SYNC)) {  // diagnostics: each stage completes before the next is enqueued
            std::fprintf(stderr, "oz2g: stage %d ...\n", stage);
            f();
            const cudaError_t e = cudaStreamSynchronize(s);
            std::fprintf(stderr, "oz2g: stage %d done (%s)\n", stage, cudaGetErrorString(e));
            return;
        }
        if (!on) { f(); return; }
        cudaEvent_t a = rec(s);
        f();
        iv.push_back({stage, a, rec(s)});
    }
    void collect(double* out) {
        for (const Interval& x : iv) {
            float ms = 0;
            if (cudaEventElapsedTime(&ms, x.a, x.b) == cudaSuccess) out[x.stage] += ms;
        }
    }
    ~Timer() {
        for (auto e : owned) cudaEventDestroy(e);
    }
};

PFN_cuTensorMapEncodeTiled_v12000 get_encode();
// 3-D uint8 tensor [planes][rows][kp] (kp contiguous), box {128, box_rows, 1}, 128-B swizzle;
// plane_stride (bytes) defaults to rows * kp.
CUtensorMap make_plane_map(const void* base, int64_t kp, int64_t rows, int64_t planes, int box_rows,
                           int64_t plane_stride = 0);
// 3-D uint8 tensor [planes][rows][cols] read as MN-major B tiles: box {128 columns, box_rows rows, 1}.
CUtensorMap make_plane_map_mn(const void* base, int64_t cols, int64_t pitch, int64_t rows, int64_t planes,
                              int64_t plane_stride, int box_rows = 128);
std::vector<uint8_t> build_resid_consts(const Table& t);
void fill_gemm_moduli(GemmParams& P, const Table& t);
Workspace& workspace(int dev, int slot = 0);
int gemm_variant();
void set_l2_hints(GemmParams& g);
int crt_overlap_blocks();
int fused_mode();
int speculation_mode(size_t input_bytes);
int group_m_for(int tiles_m, int tiles_n);
bool status_failure(const DevStatus& hs, int64_t row_base, int64_t col_base, Fail& out);
bool complete_pending(Workspace& ws, Fail& first);
void compute_relative_operands(Workspace& ws, int prec, const void* dA, int64_t lda, const void* dB, int64_t ldb,
                               int64_t m, int64_t n, int64_t k, const int32_t* mup, const int32_t* nup,
                               cudaStream_t stream, int& launches);
// The single-device pipeline (api.cu): oz2::os_ii<T> (emulate.hpp:54-88).
int run_gemm(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
             void* C, int64_t ldc, int nmod, unsigned flags, cudaStream_t stream, oz2g_intermediates* inter,
             oz2g_diag* diag, oz2g_reduce_maxima_fn reduce_fn, void* reduce_user, int64_t row_base = 0,
             int64_t col_base = 0, int slot = 0, bool reuse_scaling = false, const Arrivals* arr = nullptr);

}  // namespace oz2g
