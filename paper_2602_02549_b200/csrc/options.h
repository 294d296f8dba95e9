// options.h — the library's tuning options.  Every default is the measured
// best; an option is set per process through
// oz2g_set_option (C ABI) / set_option (Python), and otherwise taken from the
// OZ2G_<NAME> environment variable at first use.  Setting one invalidates the
// captured CUDA graphs, so the next call runs with it.
#pragma once

namespace oz2g {

enum Opt : int {
    OPT_GEMM,             // residue-GEMM kernel: 0 single-CTA 128x256 tiles, 1 CTA pair, 2 multicast cluster
    OPT_FUSED,            // 0 two-pass (GEMM epilogue + CRT pass), 1 CRT fused into the GEMM, 2 fused probe
    OPT_FUSED_MC,         // fused kernel: 0 one CTA per tile, 1 B-tile multicast in CTA pairs
    OPT_FUSED_FENCE,      // fused kernel: 1 plane fence, 0 off
    OPT_SPEC,             // host-pointer speculation: -1 by size, 0 off, 1 columns, 2 rows + columns
    OPT_GRAPH,            // CUDA-graph replays of repeated device-pointer calls: 1 on, 0 off
    OPT_PDL,              // programmatic dependent launch: 1 small calls, 0 never, 2 always
    OPT_GROUP_M,          // raster group height in tile-rows (0: 16)
    OPT_GROUP_N,          // > 0: raster groups of tile-columns instead
    OPT_L2HINT,           // TMA eviction hints: 0 normal, 1 A last / B first, 2 A last, 3 B first
    OPT_CRT_OVERLAP,      // > 1: CRT of a row block on a side stream beside the next block's GEMM
    OPT_CRT_CV,           // columns per CRT thread: 8 or 4
    OPT_WBLOCK_MIN_MB,    // W size (MiB) from which W is held per 2048-row block
    OPT_GEMM_FENCE,       // 1: persistent GEMM CTAs kept within one unit of each other
    OPT_EPI_WARPS,        // GEMM epilogue warps: 0 by k, 4 or 8
    OPT_PAIR_STAGES,      // CTA-pair GEMM pipeline depth: 4, 5 or 6
    OPT_ROWSCAN_THREADS,  // row-scan CTA size: 0 by row length, 256, 512 or 1024
    OPT_RESID_STREAM,     // 1: A residues per row block on a side stream beside the previous block's GEMMs
    OPT_SPEC_TAIL,        // host pipeline, rows + columns: halvings of the last column chunks (1..3)
    OPT_DIST_PIPELINE,    // oz2g_gemm_dist: 1 A row chunks broadcast under the scans, 0 all-gathers first
    OPT_DEBUG_SYNC,       // diagnostics: 1 synchronises and reports after every stage (stderr)
    OPT_RESID_FAST,       // residue splits: 1 balanced digits for |A'| < 2^62 (exponent buckets otherwise), 0 buckets only
    OPT_COUNT
};

// Current value of an option (lock-free read).
long long opt(Opt o);

// Name ("gemm", "fused", ... — the OZ2G_ variable without the prefix, lower
// case) -> option; -1 when unknown.
int opt_index(const char* name);
const char* opt_name(int index);

// Set (validated against the option's range; false when out of range).
bool opt_set(int index, long long value);

}  // namespace oz2g
