// comm.cpp — one emulated GEMM across the GPUs of one node, one process per
// GPU, with NCCL driven from the library (the reference's only
// partition is the row-wise parallel_for of parallel.hpp:22-40 / crt.hpp:60).
//
// C is tiled R x C over the P ranks (oz2g_grid_shape: 2 -> 2x1, 4 -> 2x2,
// 8 -> 2x4), rank q = r * C + c owns tile (r, c).  Communicators: the world
// comm and two ncclCommSplit children — the row comm (the C ranks of grid row
// r, which share A's row block r and C's rows) and the column comm (the R
// ranks of grid column c, sharing B's column block c).
//
// Per call (oz2g_gemm_dist):
//  1. inputs: with OZ2G_DIST_SHARDS the caller holds 1-D shards — A rows
//     [q m/P, (q+1) m/P) and B columns of shard s = c R + r (width n/P), both
//     row-major — and the blocks are assembled over NVLink: an all-gather of
//     the A shards in the row comm IS A's row block r (the shards of grid row
//     r are consecutive), an all-gather of the B shards in the column comm
//     gives B's column block c as R column panels, interleaved into row-major
//     by 2-D device copies.  With OZ2G_DIST_TILES the caller already holds
//     the blocks.
//  2. the single-device pipeline on the tile (oz2g_gemm, device pointers)
//     with the exchange step as its reduce hook: ncclAllReduce(MAX, int32)
//     of the clearance row maxima in the row comm and of the column maxima in
//     the column comm, on the library's stream — the one exchange the tiled
//     result needs to equal the single-GPU result bit for bit.
// NCCL is loaded at run time (dlopen libnccl.so.2 — the copy torch already
// loaded when there is one), so the library itself has no link dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/oz2g.h"
#include "arrivals.h"
#include "options.h"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p && api.why.empty()) api.why = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommSplit = (decltype(api.CommSplit))sym("ncclCommSplit");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
        api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.GetVersion = (decltype(api.GetVersion))sym("ncclGetVersion");
        api.ok = api.why.empty();
    });
    return api;
}

thread_local std::string g_comm_error;

struct CommFail {
    int code;
    std::string what;
};

#define NCCL_TRY(expr)                                                                                \
    do {                                                                                              \
        ncclResult_t r_ = (expr);                                                                     \
        if (r_ != ncclSuccess)                                                                        \
            throw CommFail{OZ2G_CUDA_ERROR, std::string(#expr) + ": " + nccl().GetErrorString(r_)};   \
    } while (0)
#define CU_TRY(expr)                                                                                  \
    do {                                                                                              \
        cudaError_t e_ = (expr);                                                                      \
        if (e_ != cudaSuccess) throw CommFail{OZ2G_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CU_TRY(cudaMalloc(&p, bytes));
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

template <class F>
int guard(F&& f) {
    g_comm_error.clear();
    try {
        return f();
    } catch (const CommFail& x) {
        g_comm_error = x.what;
        return x.code;
    }
}

}  // namespace

struct oz2g_comm {
    ncclComm_t world = nullptr, row = nullptr, col = nullptr;
    int P = 1, rank = 0, R = 1, C = 1, r = 0, c = 0, device = 0;
    Buf a_blk, b_stage, b_blk;
    // the input exchange's own stream and events (overlapped path)
    cudaStream_t s_in = nullptr;
    cudaEvent_t ev_start = nullptr;
    oz2g::Arrivals arr;
    std::mutex mtx;
    void ensure_stream() {
        if (s_in) return;
        CU_TRY(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
        CU_TRY(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
        CU_TRY(cudaEventCreateWithFlags(&arr.b, cudaEventDisableTiming));
        for (cudaEvent_t& e : arr.a) CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    void release_stream() {
        if (!s_in) return;
        cudaStreamSynchronize(s_in);
        cudaStreamDestroy(s_in);
        cudaEventDestroy(ev_start);
        cudaEventDestroy(arr.b);
        for (cudaEvent_t& e : arr.a) cudaEventDestroy(e);
        s_in = nullptr;
    }
};

namespace {

// The exchange step of the tiled pipeline (oz2g_reduce_maxima_fn): the row
// maxima of C̄ over the ranks sharing these rows, the column maxima over the
// ranks sharing these columns, in place on the pipeline's stream.
int nccl_reduce_hook(int32_t* cmax_row, int64_t m, int32_t* cmax_col, int64_t n, void* stream, void* user) {
    oz2g_comm* cm = static_cast<oz2g_comm*>(user);
    NcclApi& a = nccl();
    cudaStream_t s = (cudaStream_t)stream;
    if (a.GroupStart() != ncclSuccess) return 1;
    ncclResult_t r1 = ncclSuccess, r2 = ncclSuccess;
    if (m) r1 = a.AllReduce(cmax_row, cmax_row, (size_t)m, ncclInt32, ncclMax, cm->row, s);
    if (n) r2 = a.AllReduce(cmax_col, cmax_col, (size_t)n, ncclInt32, ncclMax, cm->col, s);
    const ncclResult_t r3 = a.GroupEnd();
    return (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess) ? 1 : 0;
}

}  // namespace

extern "C" {

const char* oz2g_comm_last_error(void) { return g_comm_error.c_str(); }

int oz2g_comm_available(void) { return nccl().ok ? 1 : 0; }

int oz2g_comm_unique_id(unsigned char* id_out) {
    return guard([&] {
        if (!nccl().ok) throw CommFail{OZ2G_CUDA_ERROR, nccl().why};
        ncclUniqueId id;
        NCCL_TRY(nccl().GetUniqueId(&id));
        std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
        return OZ2G_OK;
    });
}

int oz2g_comm_init(const unsigned char* id_in, int nranks, int rank, oz2g_comm** out) {
    return guard([&] {
        if (!out || !id_in) throw CommFail{OZ2G_INVALID_ARGUMENT, "oz2g_comm_init: null argument"};
        if (nranks < 1 || rank < 0 || rank >= nranks) throw CommFail{OZ2G_INVALID_ARGUMENT, "oz2g_comm_init: bad rank"};
        if (!nccl().ok) throw CommFail{OZ2G_CUDA_ERROR, nccl().why};
        ncclUniqueId id;
        std::memcpy(id.internal, id_in, NCCL_UNIQUE_ID_BYTES);
        oz2g_comm* cm = new oz2g_comm();
        try {
            CU_TRY(cudaGetDevice(&cm->device));
            cm->P = nranks;
            cm->rank = rank;
            oz2g_grid_shape(nranks, &cm->R, &cm->C);
            cm->r = rank / cm->C;
            cm->c = rank % cm->C;
            NCCL_TRY(nccl().CommInitRank(&cm->world, nranks, id, rank));
            NCCL_TRY(nccl().CommSplit(cm->world, cm->r, cm->c, &cm->row, nullptr));
            NCCL_TRY(nccl().CommSplit(cm->world, cm->c, cm->r, &cm->col, nullptr));
        } catch (...) {
            if (cm->row) nccl().CommDestroy(cm->row);
            if (cm->col) nccl().CommDestroy(cm->col);
            if (cm->world) nccl().CommDestroy(cm->world);
            delete cm;
            throw;
        }
        *out = cm;
        return OZ2G_OK;
    });
}

int oz2g_comm_grid(const oz2g_comm* cm, int* R, int* C, int* r, int* c) {
    if (!cm) return OZ2G_INVALID_ARGUMENT;
    if (R) *R = cm->R;
    if (C) *C = cm->C;
    if (r) *r = cm->r;
    if (c) *c = cm->c;
    return OZ2G_OK;
}

int oz2g_comm_destroy(oz2g_comm* cm) {
    if (!cm) return OZ2G_OK;
    if (nccl().ok) {
        if (cm->row) nccl().CommDestroy(cm->row);
        if (cm->col) nccl().CommDestroy(cm->col);
        if (cm->world) nccl().CommDestroy(cm->world);
    }
    cm->release_stream();
    cm->a_blk.release();
    cm->b_stage.release();
    cm->b_blk.release();
    delete cm;
    return OZ2G_OK;
}

int oz2g_dist_layout(int nranks, int rank, int64_t m, int64_t n, oz2g_dist_tile* out) {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks || m < 0 || n < 0) return OZ2G_INVALID_ARGUMENT;
    int R = 1, C = 1;
    oz2g_grid_shape(nranks, &R, &C);
    const int r = rank / C, c = rank % C;
    const int64_t mb = (m + R - 1) / R, nb = (n + C - 1) / C;
    out->R = R;
    out->C = C;
    out->r = r;
    out->c = c;
    out->row0 = std::min<int64_t>(m, r * mb);
    out->rows = std::min<int64_t>(m, (r + 1) * mb) - out->row0;
    out->col0 = std::min<int64_t>(n, c * nb);
    out->cols = std::min<int64_t>(n, (c + 1) * nb) - out->col0;
    // 1-D shards (OZ2G_DIST_SHARDS; m and n multiples of nranks)
    out->a_shard_row0 = (m / nranks) * rank;
    out->a_shard_rows = m / nranks;
    out->b_shard_col0 = (n / nranks) * ((int64_t)c * R + r);
    out->b_shard_cols = n / nranks;
    return OZ2G_OK;
}

int oz2g_gemm_dist(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                   int64_t ldb, void* C, int64_t ldc, int nmod, unsigned flags, void* stream, oz2g_comm* cm,
                   oz2g_diag* diag) {
    const int rc = guard([&] {
        if (!cm) throw CommFail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_dist: null communicator"};
        if (prec != OZ2G_FP32 && prec != OZ2G_FP64)
            throw CommFail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm: prec must be OZ2G_FP32 or OZ2G_FP64"};
        if (m < 0 || n < 0 || k < 0) throw CommFail{OZ2G_INVALID_ARGUMENT, "Matrix: negative dimension"};
        const bool shards = (flags & OZ2G_DIST_TILES) == 0;
        std::lock_guard<std::mutex> lk(cm->mtx);
        oz2g_dist_tile t;
        oz2g_dist_layout(cm->P, cm->rank, m, n, &t);
        const size_t esz = prec ? 8 : 4;
        cudaStream_t s = (cudaStream_t)stream;
        const void* dA = A;
        const void* dB = B;
        int64_t lda_t = lda, ldb_t = ldb;
        // Overlapped input exchange (option "dist_pipeline", default on): on the
        // comm's own stream, B's column block first (all-gather in the column
        // comm + interleave), then A's row block in row chunks — one
        // ncclBroadcast per chunk from the rank whose shard holds it — each
        // chunk's row scans and clearance products (run_gemm's chunked path)
        // overlapping the broadcasts of the next ones.  Off: both blocks are
        // all-gathered before the pipeline starts.
        bool overlapped = false;
        int64_t chunk_rows = 0;
        int nchunks = 0;
        if (shards) {
            if (m % cm->P || n % cm->P)
                throw CommFail{OZ2G_INVALID_ARGUMENT, "oz2g_gemm_dist: m and n must be multiples of the rank count"};
            const int64_t ms = m / cm->P, ns = n / cm->P;
            if (lda < k || ldb < ns) throw CommFail{OZ2G_INVALID_ARGUMENT, "dimension mismatch: leading dimension"};
            // A row block r: the C consecutive row shards of grid row r
            char* ablk = (char*)cm->a_blk.get(esz * (size_t)(t.rows * k));
            char* bstg = (char*)cm->b_stage.get(esz * (size_t)(cm->R * k * ns));
            char* bblk = (char*)cm->b_blk.get(esz * (size_t)(k * t.cols));
            char* own_a = ablk + esz * (size_t)(cm->c * ms * k);   // in place: this rank's slot
            char* own_b = bstg + esz * (size_t)(cm->r * k * ns);
            // chunks: whole shards, split in two or four when a grid row has
            // fewer than four shards (one shard: ragged last chunk allowed)
            int per = cm->C >= 4 ? 1 : 4 / cm->C;
            if (cm->C > 1 && ms % per) per = 1;
            chunk_rows = cm->C == 1 ? (ms + per - 1) / per : ms / per;
            nchunks = chunk_rows > 0 ? (int)((t.rows + chunk_rows - 1) / chunk_rows) : 0;
            overlapped = oz2g::opt(oz2g::OPT_DIST_PIPELINE) != 0 && nchunks >= 1 &&
                         nchunks <= oz2g::kMaxArrivalChunks && t.rows > 0 && t.cols > 0 && k > 0;
            cudaStream_t si = s;
            if (overlapped) {
                cm->ensure_stream();
                si = cm->s_in;
                CU_TRY(cudaEventRecord(cm->ev_start, s));  // the shards are ready on the caller's stream
                CU_TRY(cudaStreamWaitEvent(si, cm->ev_start, 0));
            }
            if (ms * k) CU_TRY(cudaMemcpy2DAsync(own_a, esz * k, A, esz * lda, esz * k, ms, cudaMemcpyDeviceToDevice, si));
            if (k * ns) CU_TRY(cudaMemcpy2DAsync(own_b, esz * ns, B, esz * ldb, esz * ns, k, cudaMemcpyDeviceToDevice, si));
            if (!overlapped) {
                NCCL_TRY(nccl().GroupStart());
                NCCL_TRY(nccl().AllGather(own_a, ablk, esz * (size_t)(ms * k), ncclUint8, cm->row, si));
                NCCL_TRY(nccl().AllGather(own_b, bstg, esz * (size_t)(k * ns), ncclUint8, cm->col, si));
                NCCL_TRY(nccl().GroupEnd());
            } else {
                NCCL_TRY(nccl().AllGather(own_b, bstg, esz * (size_t)(k * ns), ncclUint8, cm->col, si));
            }
            // B column block c: the R gathered panels [r][k][ns] interleaved into row-major k x (R ns)
            for (int rr = 0; rr < cm->R && k * ns; ++rr)
                CU_TRY(cudaMemcpy2DAsync(bblk + esz * (size_t)(rr * ns), esz * (size_t)t.cols,
                                         bstg + esz * (size_t)(rr * k * ns), esz * ns, esz * ns, k,
                                         cudaMemcpyDeviceToDevice, si));
            if (overlapped) {
                CU_TRY(cudaEventRecord(cm->arr.b, si));
                for (int q = 0; q < nchunks; ++q) {
                    const int64_t r0 = q * chunk_rows, rc = std::min<int64_t>(chunk_rows, t.rows - r0);
                    char* p = ablk + esz * (size_t)(r0 * k);
                    NCCL_TRY(nccl().Broadcast(p, p, esz * (size_t)(rc * k), ncclUint8, (int)(r0 / ms), cm->row, si));
                    CU_TRY(cudaEventRecord(cm->arr.a[q], si));
                }
                cm->arr.chunk_rows = chunk_rows;
                cm->arr.nchunks = nchunks;
            }
            dA = ablk;
            dB = bblk;
            lda_t = k;
            ldb_t = t.cols;
        }
        if (overlapped) {
            std::string err;
            const int r = oz2g::gemm_arrivals(prec, t.rows, t.cols, k, dA, lda_t, dB, ldb_t, C, ldc, nmod,
                                              OZ2G_DEVICE_PTRS | (flags & OZ2G_TIMING), s, diag, nccl_reduce_hook, cm,
                                              cm->arr, &err);
            if (r != OZ2G_OK) throw CommFail{r, err};
            return OZ2G_OK;
        }
        const unsigned f = OZ2G_DEVICE_PTRS | (flags & OZ2G_TIMING);
        int r = oz2g_gemm(prec, t.rows, t.cols, k, dA, lda_t, dB, ldb_t, C, ldc, nmod, f, stream, nullptr, diag,
                          nccl_reduce_hook, cm);
        if (r != OZ2G_OK) throw CommFail{r, oz2g_last_error()};
        return OZ2G_OK;
    });
    return rc;
}

}  // extern "C"
