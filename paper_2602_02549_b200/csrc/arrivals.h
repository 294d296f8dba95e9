// arrivals.h — inputs that arrive on another stream while the pipeline runs
// (the multi-GPU input exchange of comm.cpp): run_gemm's chunked path waits
// on these events instead of issuing host uploads — B first, then A in row
// chunks, each chunk's row scans and clearance products overlapping the
// arrival of the next.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/oz2g.h"

namespace oz2g {

constexpr int kMaxArrivalChunks = 8;

struct Arrivals {
    cudaEvent_t b = nullptr;                // all of B is in place
    cudaEvent_t a[kMaxArrivalChunks] = {};  // row chunk c of A is in place
    int64_t chunk_rows = 0;                 // rows per chunk (the last one may be shorter)
    int nchunks = 0;
};

// oz2g_gemm on device pointers (C only) whose inputs arrive per `arr`, with
// the multi-rank reduce hook; returns an oz2g status, *err its message.
int gemm_arrivals(int prec, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, int nmod, unsigned flags, cudaStream_t stream, oz2g_diag* diag,
                  oz2g_reduce_maxima_fn reduce_fn, void* reduce_user, const Arrivals& arr, std::string* err);

}  // namespace oz2g
