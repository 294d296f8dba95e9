"""B200-native Ozaki-II (accurate mode) emulated DGEMM/SGEMM.

Drop-in for the reference's hot path `oz2::os_ii<T>`
(/root/reference/proj/include/oz2/emulate.hpp:54-88): hand-written sm_100a
kernels (tcgen05 kind::i8 GEMMs with TMEM accumulators fed by TMA, fused
scaling / residue / CRT stages) behind the C ABI in include/oz2g.h.
"""
from .emulate import (CudaError, DomainError, EmulationResult, InvalidArgument, LogicError, ModuliTable,
                      RangeError, F32, F64, SuggestResult, dd_gemm, device_log2f, fp32_safe_moduli_max, get_option,
                      option_names, options, os_ii, os_ii_sweep, set_option, suggest_n, synchronize, table_for)
from ._lib import LIB_PATH, load as load_library

__all__ = ["os_ii", "table_for", "fp32_safe_moduli_max", "EmulationResult", "ModuliTable", "InvalidArgument",
           "DomainError", "RangeError", "LogicError", "CudaError", "F32", "F64", "device_log2f", "dd_gemm", "LIB_PATH",
           "load_library", "suggest_n", "SuggestResult", "synchronize", "os_ii_sweep", "set_option", "get_option",
           "option_names", "options"]
