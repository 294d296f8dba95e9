"""ctypes binding of the native C ABI (include/oz2g.h) — the product path.

There is no fallback: if liboz2g.so is missing or fails to load, every entry
point raises.  The library is built in-tree by paper_2602_02549_b200.build.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboz2g.so")

OZ2G_OK, OZ2G_INVALID_ARGUMENT, OZ2G_DOMAIN_ERROR, OZ2G_RANGE_ERROR, OZ2G_LOGIC_ERROR, OZ2G_CUDA_ERROR = range(6)
OZ2G_FP32, OZ2G_FP64 = 0, 1
OZ2G_HOST_PTRS, OZ2G_DEVICE_PTRS, OZ2G_TIMING, OZ2G_ASYNC = 0, 1, 2, 4


class Intermediates(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "mu", "nu", "mu_prime", "nu_prime", "e", "f", "Aprime", "Bprime", "Cbar", "Dbar", "W",
        "C1", "C2", "Q", "Cpp64", "Cpp32", "Ares", "Bres", "Cprod", "cmax_row", "cmax_col", "bounds")]


class Bounds(C.Structure):
    _fields_ = [("cheap", C.c_void_p), ("tight", C.c_void_p), ("device", C.c_int),
                ("cheap_max", C.c_double), ("tight_max", C.c_double), ("relative", C.c_int),
                ("tight_rel_max", C.c_double)]


class DistTile(C.Structure):
    _fields_ = [("R", C.c_int), ("C", C.c_int), ("r", C.c_int), ("c", C.c_int), ("row0", C.c_int64),
                ("rows", C.c_int64), ("col0", C.c_int64), ("cols", C.c_int64), ("a_shard_row0", C.c_int64),
                ("a_shard_rows", C.c_int64), ("b_shard_col0", C.c_int64), ("b_shard_cols", C.c_int64)]


OZ2G_DIST_SHARDS, OZ2G_DIST_TILES = 0, 8


class Suggest(C.Structure):
    _fields_ = [("n", C.c_int), ("cheap_n", C.c_int), ("excluded_below", C.c_int), ("emulations", C.c_int),
                ("bound_max", C.c_double), ("tight_max", C.c_double), ("tight_rel_max", C.c_double)]


class Diag(C.Structure):
    _fields_ = [("subnormal", C.c_int), ("kernels_launched", C.c_int), ("stage_ms", C.c_double * 8),
                ("speculation", C.c_int)]


class TableC(C.Structure):
    _fields_ = [("n", C.c_int), ("mode", C.c_int), ("p", C.c_int * 49), ("q", C.c_int * 49),
                ("beta", C.c_int * 49), ("s1", C.c_double * 49), ("s2", C.c_double * 49), ("rho", C.c_long),
                ("P1", C.c_double), ("P2", C.c_double), ("P_inv", C.c_double), ("P_prime", C.c_float),
                ("P_dec", C.c_char * 160), ("shift0", C.c_int), ("nthr", C.c_int), ("thr", C.c_int32 * 64)]


REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)

EXPORTED = ("oz2g_gemm", "oz2g_dgemm", "oz2g_sgemm", "oz2g_last_error", "oz2g_table_for",
            "oz2g_fp32_safe_moduli_max", "oz2g_shift_of_cmax", "oz2g_device_log2f", "oz2g_version",
            "oz2g_release_workspace", "oz2g_dd_gemm", "oz2g_suggest_n", "oz2g_gen_matrix", "oz2g_derive_seed",
            "oz2g_native_gemm", "oz2g_gemm_multi", "oz2g_grid_shape", "oz2g_init", "oz2g_synchronize",
            "oz2g_gemm_sweep", "oz2g_suggest_n_tight", "oz2g_i8_peak", "oz2g_comm_available", "oz2g_comm_unique_id",
            "oz2g_comm_init", "oz2g_comm_grid", "oz2g_comm_destroy", "oz2g_comm_last_error", "oz2g_dist_layout",
            "oz2g_gemm_dist", "oz2g_set_option", "oz2g_get_option", "oz2g_option_name")

_LIB = None


def load() -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise OSError(f"oz2g: native library {LIB_PATH} is missing — run "
                      "`python -m paper_2602_02549_b200.build` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.oz2g_gemm.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                            C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_uint, C.c_void_p,
                            C.POINTER(Intermediates), C.POINTER(Diag), REDUCE_FN, C.c_void_p]
    L.oz2g_gemm.restype = C.c_int
    L.oz2g_dgemm.argtypes = [C.c_int64] * 3 + [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                               C.c_int64, C.c_int, C.c_uint, C.c_void_p, C.POINTER(Diag)]
    L.oz2g_sgemm.argtypes = L.oz2g_dgemm.argtypes
    L.oz2g_last_error.restype = C.c_char_p
    L.oz2g_table_for.argtypes = [C.c_int, C.c_int, C.POINTER(TableC)]
    L.oz2g_shift_of_cmax.argtypes = [C.c_int, C.c_int64]
    L.oz2g_device_log2f.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    L.oz2g_dd_gemm.argtypes = [C.c_int64] * 3 + [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                                 C.c_void_p, C.c_int64, C.c_void_p]
    L.oz2g_suggest_n.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_int64, C.c_double, C.c_uint, C.c_void_p, C.POINTER(C.c_int),
                                 C.POINTER(C.c_double)]
    L.oz2g_suggest_n_tight.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_double, C.c_int, C.c_uint, C.c_void_p, C.POINTER(Suggest)]
    L.oz2g_i8_peak.argtypes = [C.c_longlong, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.oz2g_set_option.argtypes = [C.c_char_p, C.c_longlong]
    L.oz2g_get_option.argtypes = [C.c_char_p, C.POINTER(C.c_longlong)]
    L.oz2g_option_name.argtypes = [C.c_int]
    L.oz2g_option_name.restype = C.c_char_p
    L.oz2g_comm_unique_id.argtypes = [C.c_void_p]
    L.oz2g_comm_init.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.oz2g_comm_grid.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 4
    L.oz2g_comm_destroy.argtypes = [C.c_void_p]
    L.oz2g_comm_last_error.restype = C.c_char_p
    L.oz2g_dist_layout.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.POINTER(DistTile)]
    L.oz2g_gemm_dist.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_uint, C.c_void_p, C.c_void_p,
                                 C.POINTER(Diag)]
    L.oz2g_gen_matrix.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_void_p]
    L.oz2g_derive_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    L.oz2g_derive_seed.restype = C.c_uint64
    L.oz2g_native_gemm.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
    L.oz2g_gemm_multi.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_uint, C.POINTER(C.c_int), C.c_int,
                                  C.POINTER(Diag)]
    L.oz2g_grid_shape.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.oz2g_gemm_sweep.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_int64, C.POINTER(C.c_void_p), C.c_int64, C.POINTER(C.c_int), C.c_int, C.c_uint,
                                  C.c_void_p, C.POINTER(Diag)]
    L.oz2g_init.argtypes = [C.POINTER(C.c_int), C.c_int]
    _LIB = L
    return L
