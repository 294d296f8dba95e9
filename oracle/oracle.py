"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, bench.py's cpu_baseline / --impl reference legs and
__graft_entry__.smoke() may import this module, and only as the checker or the
timed CPU baseline — the product package (paper_2602_02549_b200) never does.

`os_ii(A, B, n, keep_intermediates)` restates the reference's
`oz2::os_ii<T>` (/root/reference/proj/include/oz2/emulate.hpp:54-88) via
oz2_oracle.c, with constants from moduli.py (moduli.hpp:93-142).  Exceptions
mirror the reference's classes (emulate.hpp:59, scaling.hpp:90, crt.hpp:144).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

from . import moduli as M

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None


class OracleDomainError(ValueError):
    """std::domain_error"""


class OracleRangeError(ArithmeticError):
    """std::range_error"""


class OracleLogicError(RuntimeError):
    """std::logic_error"""


class OracleInvalidArgument(ValueError):
    """std::invalid_argument"""


_EXC = {1: OracleInvalidArgument, 2: OracleDomainError, 3: OracleRangeError, 4: OracleLogicError}


class _Table(C.Structure):
    _fields_ = [("n", C.c_int), ("mode", C.c_int), ("p", C.c_int * 49), ("s1", C.c_double * 49),
                ("s2", C.c_double * 49), ("P1", C.c_double), ("P2", C.c_double), ("P_inv", C.c_double),
                ("P_prime", C.c_float), ("coeff", C.c_float)]


class _Out(C.Structure):
    _fields_ = [("mu", C.c_void_p), ("nu", C.c_void_p), ("mu_prime", C.c_void_p), ("nu_prime", C.c_void_p),
                ("e", C.c_void_p), ("f", C.c_void_p), ("Aprime", C.c_void_p), ("Bprime", C.c_void_p),
                ("Cbar", C.c_void_p), ("Dbar", C.c_void_p), ("W", C.c_void_p), ("C1", C.c_void_p),
                ("C2", C.c_void_p), ("Q", C.c_void_p), ("Cpp64", C.c_void_p), ("Cpp32", C.c_void_p),
                ("Ares", C.c_void_p), ("Bres", C.c_void_p), ("Cprod", C.c_void_p),
                ("cmax_row", C.c_void_p), ("cmax_col", C.c_void_p),
                ("ext_cmax_row", C.c_void_p), ("ext_cmax_col", C.c_void_p),
                ("subnormal", C.c_int), ("msg", C.c_char * 256)]


def build() -> None:
    """Compile liboz2_oracle.so (and _ref/ when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboz2_oracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.ora_os_ii.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.POINTER(_Table), C.POINTER(_Out)]
        L.ora_os_ii.restype = C.c_int
        L.ora_gen_matrix_f64.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_void_p]
        L.ora_gen_matrix_f32.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_void_p]
        L.ora_derive_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ora_derive_seed.restype = C.c_uint64
        L.ora_gemm_i8_wrap.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ora_residue_of.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_int8)]
        L.ora_fp32_round_up.argtypes = [C.c_int64]
        L.ora_fp32_round_up.restype = C.c_float
        L.ora_log2_fp32.argtypes = [C.c_float]
        L.ora_log2_fp32.restype = C.c_float
        L.ora_fma_fp32_down.argtypes = [C.c_float, C.c_float, C.c_float]
        L.ora_fma_fp32_down.restype = C.c_float
        L.ora_shift_of_cmax.argtypes = [C.c_int64, C.c_float, C.c_float, C.POINTER(C.c_float)]
        L.ora_shift_of_cmax.restype = C.c_long
        L.ora_set_threads.argtypes = [C.c_int]
        L.ora_xoshiro_next.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.ora_log2f_monotone_violations.restype = C.c_int64
        L.ora_log2f_array.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.ora_ceil_abs_scaled.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_int8)]
        L.ora_signed_mod.argtypes = [C.c_longlong, C.c_longlong]
        L.ora_signed_mod.restype = C.c_longlong
        L.ora_round_nearest_even.argtypes = [C.c_double]
        L.ora_round_nearest_even.restype = C.c_double
        _LIB = L
    return _LIB


def ref_lib():
    """The reference's own GMP-free headers compiled in place (oracle/_ref), or None."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "liboz2_ref.so")
        if not os.path.exists(path):
            return None
        L = C.CDLL(path)
        L.ref_gen_matrix_f64.argtypes = [C.c_longlong, C.c_longlong, C.c_double, C.c_ulonglong, C.c_void_p]
        L.ref_gen_matrix_f32.argtypes = [C.c_longlong, C.c_longlong, C.c_double, C.c_ulonglong, C.c_void_p]
        L.ref_gemm_i8_wrap.argtypes = [C.c_longlong] * 3 + [C.c_void_p] * 3
        L.ref_xoshiro_next.argtypes = [C.c_ulonglong, C.c_longlong, C.c_void_p]
        L.ref_set_threads.argtypes = [C.c_int]
        _REF = L
    return _REF


def set_threads(t: int) -> None:
    lib().ora_set_threads(int(t))


def table(n: int, mode: int) -> _Table:
    t = M.build_table(n, mode)
    tab = _Table()
    tab.n, tab.mode = n, mode
    for l in range(n):
        tab.p[l] = t["p"][l]
        tab.s1[l] = t["s1"][l]
        tab.s2[l] = t["s2"][l]
    tab.P1, tab.P2, tab.P_inv = t["P1"], t["P2"], t["P_inv"]
    tab.P_prime = t["P_prime"]
    tab.coeff = M.scaling_coeff_fp32()
    return tab


def gen_matrix(rows: int, cols: int, phi: float, seed: int, dtype=np.float64) -> np.ndarray:
    """gen.hpp:15-31 (restated in C; identical stream to the reference)."""
    out = np.empty((rows, cols), dtype=dtype)
    fn = lib().ora_gen_matrix_f64 if dtype == np.float64 else lib().ora_gen_matrix_f32
    if fn(rows, cols, float(phi), seed, out.ctypes.data) != 0:
        raise OracleDomainError("gen_matrix: phi must be nonnegative")
    return out


def derive_seed(seed: int, trial: int, role: int) -> int:
    """experiment.hpp:83-88."""
    return int(lib().ora_derive_seed(seed, trial, role))


def gemm_i8_wrap(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int8)
    b = np.ascontiguousarray(b, dtype=np.int8)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise OracleInvalidArgument("dimension mismatch: gemm_i8_wrap inner dimension")
    c = np.empty((m, n), dtype=np.int32)
    if lib().ora_gemm_i8_wrap(m, k, n, a.ctypes.data, b.ctypes.data, c.ctypes.data) != 0:
        raise OracleDomainError("gemm_i8_wrap: k exceeds 2^17")
    return c


def residue_of(x: float, p: int) -> int:
    r = C.c_int8()
    if lib().ora_residue_of(float(x), int(p), C.byref(r)) != 0:
        raise OracleDomainError("residue_of: non-finite or non-integer entry")
    return int(r.value)


def ceil_abs_scaled(a: float, sft: int) -> int:
    r = C.c_int8()
    if lib().ora_ceil_abs_scaled(float(a), int(sft), C.byref(r)) != 0:
        raise OracleLogicError("ceil_abs_scaled: entry above row/column max")
    return int(r.value)


def signed_mod(x: int, p: int) -> int:
    return int(lib().ora_signed_mod(int(x), int(p)))


def round_nearest_even(x: float) -> float:
    return float(lib().ora_round_nearest_even(float(x)))


def shift_of_cmax(c: int, n: int) -> tuple[int, float]:
    t = M.build_table(n, M.F64)
    e = C.c_float()
    s = lib().ora_shift_of_cmax(int(c), M.scaling_coeff_fp32(), t["P_prime"], C.byref(e))
    return int(s), float(e.value)


@dataclass
class OracleResult:
    C: np.ndarray
    subnormal: bool
    table: dict
    inter: dict = field(default_factory=dict)


def os_ii(A: np.ndarray, B: np.ndarray, n: int, keep_intermediates: bool = False,
          residues: bool = False, ext_cmax_row=None, ext_cmax_col=None,
          want_cmax: bool = False) -> OracleResult:
    """emulate.hpp:54-88 os_ii<T>; T from A.dtype (float32 or float64)."""
    if A.dtype != B.dtype or A.dtype not in (np.float32, np.float64):
        raise TypeError("os_ii: A and B must both be float32 or float64")
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise OracleInvalidArgument("dimension mismatch: os_ii inner dimension")
    if not (2 <= n <= 49):
        if A.shape[1] > (1 << 17):
            raise OracleDomainError("os_ii: k exceeds 2^17")
        raise OracleDomainError("build_table: N out of [2, 49]")
    prec = 1 if A.dtype == np.float64 else 0
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    m, k = A.shape
    nn = B.shape[1]
    Cm = np.empty((m, nn), dtype=A.dtype)
    out = _Out()
    inter = {}
    if keep_intermediates:
        spec = dict(mu=((m,), np.int16), nu=((nn,), np.int16), mu_prime=((m,), np.int16),
                    nu_prime=((nn,), np.int16), e=((m,), np.float32), f=((nn,), np.float32),
                    Aprime=((m, k), np.float64), Bprime=((k, nn), np.float64),
                    Cbar=((m, nn), np.int32), Dbar=((m, nn), np.float32), W=((n, m, nn), np.int8),
                    C1=((m, nn), np.float64), C2=((m, nn), np.float64), Q=((m, nn), np.float64),
                    Cpp64=((m, nn), np.float64))
        if prec == 0:
            spec["Cpp32"] = ((m, nn), np.float32)
        if residues:
            spec.update(Ares=((n, m, k), np.int8), Bres=((n, k, nn), np.int8),
                        Cprod=((n, m, nn), np.int32))
        for name, (shape, dt) in spec.items():
            arr = np.zeros(shape, dtype=dt)
            inter[name] = arr
            setattr(out, name, arr.ctypes.data)
    if want_cmax or keep_intermediates:
        for name, cnt in (("cmax_row", m), ("cmax_col", nn)):
            arr = np.zeros(cnt, dtype=np.int32)
            inter[name] = arr
            setattr(out, name, arr.ctypes.data)
    keep_alive = []
    for name, arr in (("ext_cmax_row", ext_cmax_row), ("ext_cmax_col", ext_cmax_col)):
        if arr is not None:
            arr = np.ascontiguousarray(arr, dtype=np.int32)
            keep_alive.append(arr)
            setattr(out, name, arr.ctypes.data)
    tab = table(n, prec)
    rc = lib().ora_os_ii(prec, m, k, nn, A.ctypes.data, B.ctypes.data, Cm.ctypes.data,
                         C.byref(tab), C.byref(out))
    if rc != 0:
        raise _EXC.get(rc, RuntimeError)(out.msg.decode())
    return OracleResult(C=Cm, subnormal=bool(out.subnormal), table=M.build_table(n, prec), inter=inter)


# ---------------------------------------------------------------- sampled full-size checks
def _setup_sampled():
    L = lib()
    if getattr(L, "_sampled_ready", False):
        return L
    L.ora_pre_exponents.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    L.ora_ceil_scale.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
    L.ora_cbar_row_max.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
    L.ora_cbar_col_max.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                   C.c_void_p]
    L.ora_entries.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(_Table), C.c_void_p]
    L._sampled_ready = True
    return L


def pre_exponents(X: np.ndarray, by_col: bool) -> np.ndarray:
    """scaling.hpp:86-107 (mu' of every row, or nu' of every column)."""
    L = _setup_sampled()
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty(X.shape[1] if by_col else X.shape[0], dtype=np.int16)
    if L.ora_pre_exponents(X.ctypes.data, X.shape[0], X.shape[1], int(by_col), out.ctypes.data) != 0:
        raise OracleDomainError("zero row/column or non-finite entry")
    return out


def ceil_scale(X: np.ndarray, sft: np.ndarray, by_col: bool) -> np.ndarray:
    """Abar / Bbar, scaling.hpp:111-131."""
    L = _setup_sampled()
    X = np.ascontiguousarray(X, dtype=np.float64)
    sft = np.ascontiguousarray(sft, dtype=np.int16)
    out = np.empty(X.shape, dtype=np.int8)
    if L.ora_ceil_scale(X.ctypes.data, X.shape[0], X.shape[1], sft.ctypes.data, int(by_col), out.ctypes.data) != 0:
        raise OracleLogicError("ceil_abs_scaled")
    return out


def cbar_row_max(abar, bbar, rows) -> np.ndarray:
    L = _setup_sampled()
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(len(rows), dtype=np.int32)
    L.ora_cbar_row_max(abar.ctypes.data, bbar.ctypes.data, abar.shape[1], bbar.shape[1], rows.ctypes.data,
                       len(rows), out.ctypes.data)
    return out


def cbar_col_max(abar, bbar, cols) -> np.ndarray:
    L = _setup_sampled()
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(len(cols), dtype=np.int32)
    L.ora_cbar_col_max(abar.ctypes.data, bbar.ctypes.data, abar.shape[0], abar.shape[1], bbar.shape[1],
                       cols.ctypes.data, len(cols), out.ctypes.data)
    return out


def entries(A, B, n, mu, nu, rows, cols, prec=1) -> np.ndarray:
    """C_ij of os_ii for the given (i, j) pairs, with the given mu / nu."""
    L = _setup_sampled()
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.int16)
    nu = np.ascontiguousarray(nu, dtype=np.int16)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(len(rows), dtype=np.float64 if prec else np.float32)
    tab = table(n, prec)
    rc = L.ora_entries(prec, A.ctypes.data, B.ctypes.data, A.shape[1], B.shape[1], mu.ctypes.data, nu.ctypes.data,
                       rows.ctypes.data, cols.ctypes.data, len(rows), C.byref(tab), out.ctypes.data)
    if rc != 0:
        raise _EXC.get(rc, RuntimeError)("ora_entries")
    return out
