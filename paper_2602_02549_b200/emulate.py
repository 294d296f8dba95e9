"""Python mirror of the reference's public interface for the hot path.

    os_ii(a, b, n, keep_intermediates=False) -> EmulationResult
        /root/reference/proj/include/oz2/emulate.hpp:54-88
    table_for(n, mode) -> ModuliTable            moduli.hpp:145-153
    fp32_safe_moduli_max() -> int                moduli.hpp:157-170

Same names, argument meaning and error behaviour as the reference: the
exception classes below correspond one-to-one to std::invalid_argument,
std::domain_error, std::range_error and std::logic_error.  Everything is
computed by the native library (liboz2g.so, CUDA on sm_100a) through the C ABI;
inputs may be host numpy arrays (copied in and out inside the call) or CUDA
torch tensors (device pointers, no copies).
"""
from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib

F32, F64 = _lib.OZ2G_FP32, _lib.OZ2G_FP64
K_MAX_INNER_DIM = 1 << 17
K_MAX_MODULI = 49


class InvalidArgument(ValueError):
    """std::invalid_argument (matrix.hpp:47-49)."""


class DomainError(ValueError):
    """std::domain_error (emulate.hpp:59, scaling.hpp:90/102, moduli.hpp:94)."""


class RangeError(ArithmeticError):
    """std::range_error (scaling.hpp:145/206/220, crt.hpp:144, emulate.hpp:39)."""


class LogicError(RuntimeError):
    """std::logic_error (scaling.hpp:67/77/179/189)."""


class CudaError(RuntimeError):
    """Device or driver failure (no reference counterpart)."""


_EXC = {1: InvalidArgument, 2: DomainError, 3: RangeError, 4: LogicError, 5: CudaError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.load().oz2g_last_error().decode()
        raise _EXC.get(rc, CudaError)(msg)


_GEMM_VARIANTS = {"single": 0, "pair": 1, "mcast": 2}


def set_option(name: str, value) -> None:
    """Set a tuning option for this process (oz2g_set_option: "gemm", "fused",
    "spec", "graph", "pdl", ...; `option_names()` lists them).  "gemm" also
    takes "single" / "pair" / "mcast".  Applies from the next call."""
    if name == "gemm" and isinstance(value, str):
        if value not in _GEMM_VARIANTS:
            raise InvalidArgument(f"set_option: gemm must be one of {sorted(_GEMM_VARIANTS)}")
        value = _GEMM_VARIANTS[value]
    _check(_lib.load().oz2g_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = C.c_longlong()
    _check(_lib.load().oz2g_get_option(name.encode(), C.byref(v)))
    return v.value


def option_names() -> list:
    L = _lib.load()
    out, i = [], 0
    while (nm := L.oz2g_option_name(i)) is not None:
        out.append(nm.decode())
        i += 1
    return out


@contextmanager
def options(**kw):
    """Temporarily set options: `with options(spec=0, fused=1): ...`."""
    old = {k: get_option(k) for k in kw}
    try:
        for k, v in kw.items():
            set_option(k, v)
        yield
    finally:
        for k, v in old.items():
            set_option(k, v)


@dataclass
class ModuliTable:
    """moduli.hpp:78-91 (P as a Python int)."""
    n: int
    mode: int
    p: list
    q: list
    P: int
    rho: int
    P1: float
    P2: float
    P_inv: float
    beta: list
    s1: list
    s2: list
    P_prime: float
    shift0: int = 0
    thresholds: list = field(default_factory=list)


def table_for(n: int, mode: int = F64) -> ModuliTable:
    """moduli.hpp:145-153: built once per (n, mode) and cached (immutable)."""
    key = (int(n), int(mode))
    t = _TABLES.get(key)
    if t is None:
        t = _TABLES[key] = _table_for(*key)
    return t


_TABLES: dict = {}


def _table_for(n: int, mode: int) -> ModuliTable:
    t = _lib.TableC()
    _check(_lib.load().oz2g_table_for(int(n), int(mode), C.byref(t)))
    k = t.n
    return ModuliTable(n=k, mode=t.mode, p=list(t.p[:k]), q=list(t.q[:k]), P=int(t.P_dec.decode()), rho=t.rho,
                       P1=t.P1, P2=t.P2, P_inv=t.P_inv, beta=list(t.beta[:k]), s1=list(t.s1[:k]),
                       s2=list(t.s2[:k]), P_prime=t.P_prime, shift0=t.shift0, thresholds=list(t.thr[:t.nthr]))


def fp32_safe_moduli_max() -> int:
    return int(_lib.load().oz2g_fp32_safe_moduli_max())


@dataclass
class ScalingOutput:
    """scaling.hpp:20-28 (+ the clearance maxima the device actually keeps)."""
    mu: np.ndarray = None
    nu: np.ndarray = None
    mu_prime: np.ndarray = None
    nu_prime: np.ndarray = None
    e: np.ndarray = None
    f: np.ndarray = None
    Aprime: np.ndarray = None
    Bprime: np.ndarray = None
    Cbar: np.ndarray = None
    Dbar: np.ndarray = None
    cmax_row: np.ndarray = None
    cmax_col: np.ndarray = None


@dataclass
class CrtIntermediates:
    """crt.hpp:81-87 (+ residue planes and wrapped INT32 products)."""
    W: np.ndarray = None
    C1: np.ndarray = None
    C2: np.ndarray = None
    Q: np.ndarray = None
    Cpp64: np.ndarray = None
    Cpp32: np.ndarray = None
    Ares: np.ndarray = None
    Bres: np.ndarray = None
    Cprod: np.ndarray = None


@dataclass
class EmulationResult:
    """emulate.hpp:17-24."""
    C: object
    scaling: ScalingOutput
    crt: CrtIntermediates
    table: ModuliTable
    subnormal: bool
    kernels_launched: int = 0
    stage_ms: tuple = ()
    bounds: Optional[dict] = None
    speculation: int = 0  # 0 none, 1 speculated column exponents confirmed, 2 missed and redone


_NO_HOOK = _lib.REDUCE_FN()  # the null oz2g_reduce_maxima_fn


def _current_stream(t) -> int:
    """The caller's current CUDA stream on the device of tensor `t` (raw
    handle; torch's internal accessor is ~30x cheaper than
    torch.cuda.current_stream(...).cuda_stream, which is the fallback)."""
    import torch
    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return int(get(t.get_device()))
    return torch.cuda.current_stream(t.device).cuda_stream


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def os_ii(a, b, n: int, keep_intermediates: bool = False, *, evidence: bool = False, out=None,
          stream=None, timing: bool = False, bounds=False, vectors: bool = False,
          reduce_maxima: Optional[Callable] = None, devices=None, blocking: bool = True,
          relative: bool = False) -> EmulationResult:
    """C ~ A*B by Ozaki-II accurate mode with `n` moduli (emulate.hpp:54-88).

    `a`, `b`: 2-D float32/float64 numpy arrays (host) or CUDA torch tensors
    (row-major, unit column stride).  The precision of the call follows the
    dtype, like os_ii<float> / os_ii<double>.  `keep_intermediates` returns the
    reference's ScalingOutput/CrtIntermediates fields; `evidence` also returns
    the residue planes and wrapped INT32 products; `vectors` returns only the
    O(m+n) scaling vectors (mu, nu, mu', nu', e, f, clearance maxima).
    `bounds=True` evaluates the
    paper's error bounds (bounds.hpp) and returns their maxima;
    `bounds="full"` also returns the m x n cheap / tight bound matrices (same
    memory space as the inputs); with `relative=True` also
    bounds["tight_rel_max"] = max_ij tight_ij / (|A||B|)_ij (a certificate:
    against a lower bound of |A||B|).  `reduce_maxima(row_ptr, m, col_ptr, n,
    stream)` is the multi-GPU hook of oz2g.h.  `devices=[d0, d1, ...]` tiles
    one call over those devices of this process (oz2g_gemm_multi; host arrays,
    C only) with a result identical to the single-device call.
    `blocking=False` enqueues the call and returns at once (C only): A, B and
    the output must stay alive and C must not be read until `synchronize()`,
    which raises the first failure among the pending calls.  Back-to-back
    host-array calls then overlap the next upload with the previous GEMMs.
    """
    L = _lib.load()
    dev = _is_torch_cuda(a)
    if dev != _is_torch_cuda(b):
        raise InvalidArgument("os_ii: A and B must both be host arrays or both CUDA tensors")
    if dev:
        import torch
        if a.dtype != b.dtype or a.dtype not in (torch.float32, torch.float64):
            raise TypeError("os_ii: A and B must both be float32 or float64")
        if a.dim() != 2 or b.dim() != 2:
            raise InvalidArgument("os_ii: 2-D matrices expected")
        if a.stride(1) != 1 or b.stride(1) != 1:
            raise InvalidArgument("os_ii: unit column stride required (row-major)")
        prec = F64 if a.dtype == torch.float64 else F32
        m, k = a.shape
        k2, nn = b.shape
        if k != k2:
            raise InvalidArgument("dimension mismatch: os_ii inner dimension")
        if out is not None:
            if not _is_torch_cuda(out) or out.device != a.device:
                raise InvalidArgument("os_ii: out must be a CUDA tensor on the device of A and B")
            if out.dtype != a.dtype or tuple(out.shape) != (m, nn):
                raise InvalidArgument(f"os_ii: out must be {m}x{nn} {a.dtype}")
            if nn > 1 and out.stride(1) != 1 or m > 1 and out.stride(0) < nn:
                raise InvalidArgument("os_ii: out must be row-major with unit column stride")
        C_out = out if out is not None else torch.empty((m, nn), dtype=a.dtype, device=a.device)
        pa, pb, pc = a.data_ptr(), b.data_ptr(), C_out.data_ptr()
        lda, ldb, ldc = max(a.stride(0), k), max(b.stride(0), nn), max(C_out.stride(0), nn)
        flags = _lib.OZ2G_DEVICE_PTRS
        if stream is None:
            stream = _current_stream(a)
    else:
        a = np.asarray(a)
        b = np.asarray(b)
        if a.dtype != b.dtype or a.dtype not in (np.float32, np.float64):
            raise TypeError("os_ii: A and B must both be float32 or float64")
        if a.ndim != 2 or b.ndim != 2:
            raise InvalidArgument("os_ii: 2-D matrices expected")
        if a.shape[1] != b.shape[0]:
            raise InvalidArgument("dimension mismatch: os_ii inner dimension")
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        prec = F64 if a.dtype == np.float64 else F32
        m, k = a.shape
        nn = b.shape[1]
        ldc = nn
        if out is not None:
            if not isinstance(out, np.ndarray):
                raise InvalidArgument("os_ii: out must be a numpy array for host inputs")
            if out.dtype != a.dtype or out.shape != (m, nn):
                raise InvalidArgument(f"os_ii: out must be {m}x{nn} {a.dtype}")
            isz = out.itemsize
            if (nn > 1 and out.strides[1] != isz) or (m > 1 and (out.strides[0] % isz or out.strides[0] < nn * isz)):
                raise InvalidArgument("os_ii: out must be row-major with unit column stride")
            if not out.flags.writeable:
                raise InvalidArgument("os_ii: out is read-only")
            if m > 1:
                ldc = out.strides[0] // isz
        C_out = np.empty((m, nn), dtype=a.dtype) if out is None else out
        pa, pb, pc = a.ctypes.data, b.ctypes.data, C_out.ctypes.data
        lda, ldb = k, nn
        flags = _lib.OZ2G_HOST_PTRS
    if timing:
        flags |= _lib.OZ2G_TIMING
    if not blocking:
        if keep_intermediates or evidence or vectors or bounds or reduce_maxima is not None or timing:
            raise InvalidArgument("os_ii: blocking=False returns C only (no intermediates, bounds, hook or timing)")
        if devices is not None:
            raise InvalidArgument("os_ii: blocking=False is single-device")
        flags |= _lib.OZ2G_ASYNC
        diag = _lib.Diag()
        _check(L.oz2g_gemm(prec, m, nn, k, pa, lda, pb, ldb, pc, ldc, int(n), flags,
                           C.c_void_p(int(stream) if stream else 0), None, C.byref(diag), _lib.REDUCE_FN(), None))
        return EmulationResult(C=C_out, scaling=ScalingOutput(), crt=CrtIntermediates(), table=table_for(n, prec),
                               subnormal=False, kernels_launched=diag.kernels_launched)
    if devices is not None:
        if dev:
            raise InvalidArgument("os_ii: devices= takes host arrays (each device uploads its own blocks)")
        if keep_intermediates or evidence or vectors or bounds or reduce_maxima is not None:
            raise InvalidArgument("os_ii: devices= returns C only")
        devs = [int(d) for d in devices]
        ds = (C.c_int * max(1, len(devs)))(*devs)
        diag = _lib.Diag()
        _check(L.oz2g_gemm_multi(prec, m, nn, k, pa, lda, pb, ldb, pc, ldc, int(n), flags, ds, len(devs),
                                 C.byref(diag)))
        return EmulationResult(C=C_out, scaling=ScalingOutput(), crt=CrtIntermediates(), table=table_for(n, prec),
                               subnormal=bool(diag.subnormal), kernels_launched=diag.kernels_launched,
                               stage_ms=tuple(diag.stage_ms))

    inter_c = None
    sc, cr = ScalingOutput(), CrtIntermediates()
    keep = {}
    if keep_intermediates or evidence or vectors:
        inter_c = _lib.Intermediates()
        N = int(n)
        spec = dict(mu=(sc, (m,), np.int16), nu=(sc, (nn,), np.int16), mu_prime=(sc, (m,), np.int16),
                    nu_prime=(sc, (nn,), np.int16), e=(sc, (m,), np.float32), f=(sc, (nn,), np.float32),
                    cmax_row=(sc, (m,), np.int32), cmax_col=(sc, (nn,), np.int32))
        if keep_intermediates:
            spec.update(Aprime=(sc, (m, k), np.float64), Bprime=(sc, (k, nn), np.float64),
                        Cbar=(sc, (m, nn), np.int32), Dbar=(sc, (m, nn), np.float32),
                        W=(cr, (N, m, nn), np.int8), C1=(cr, (m, nn), np.float64), C2=(cr, (m, nn), np.float64),
                        Q=(cr, (m, nn), np.float64), Cpp64=(cr, (m, nn), np.float64))
            if prec == F32:
                spec["Cpp32"] = (cr, (m, nn), np.float32)
        if evidence:
            spec.update(W=(cr, (N, m, nn), np.int8), Ares=(cr, (N, m, k), np.int8),
                        Bres=(cr, (N, k, nn), np.int8), Cprod=(cr, (N, m, nn), np.int32))
        if 2 <= N <= K_MAX_MODULI:
            for name, (holder, shape, dt) in spec.items():
                arr = np.zeros(shape, dtype=dt)
                keep[name] = (holder, arr)
                setattr(inter_c, name, arr.ctypes.data)
    bnd_c, bnd_arrays = None, {}
    if bounds and 2 <= int(n) <= K_MAX_MODULI:
        if inter_c is None:
            inter_c = _lib.Intermediates()
        bnd_c = _lib.Bounds()
        bnd_c.relative = 1 if relative else 0
        if bounds == "full":
            for name in ("cheap", "tight"):
                if dev:
                    import torch
                    arr = torch.empty((m, nn), dtype=torch.float64, device=a.device)
                    setattr(bnd_c, name, arr.data_ptr())
                else:
                    arr = np.zeros((m, nn), dtype=np.float64)
                    setattr(bnd_c, name, arr.ctypes.data)
                bnd_arrays[name] = arr
            bnd_c.device = 1 if dev else 0
        inter_c.bounds = C.cast(C.pointer(bnd_c), C.c_void_p)

    diag = _lib.Diag()
    if reduce_maxima is not None:
        def _cb(rp, mm, cp, nn2, st, user):
            try:
                reduce_maxima(rp, mm, cp, nn2, st)
                return 0
            except Exception:  # pragma: no cover - reported as a status code
                import traceback
                traceback.print_exc()
                return 1
        cb = _lib.REDUCE_FN(_cb)
    else:
        cb = _NO_HOOK
    rc = L.oz2g_gemm(prec, m, nn, k, pa, lda, pb, ldb, pc, ldc, int(n), flags,
                     C.c_void_p(int(stream) if stream else 0),
                     C.byref(inter_c) if inter_c is not None else None, C.byref(diag), cb, None)
    _check(rc)
    for name, (holder, arr) in keep.items():
        setattr(holder, name, arr)
    bres = None
    if bnd_c is not None:
        bres = dict(cheap_max=bnd_c.cheap_max, tight_max=bnd_c.tight_max, **bnd_arrays)
        if relative:
            bres["tight_rel_max"] = bnd_c.tight_rel_max
    return EmulationResult(C=C_out, scaling=sc, crt=cr, table=table_for(n, prec), subnormal=bool(diag.subnormal),
                           kernels_launched=diag.kernels_launched, stage_ms=tuple(diag.stage_ms), bounds=bres,
                           speculation=diag.speculation)


def os_ii_sweep(a, b, ns, stream=None) -> list:
    """os_ii(a, b, n).C for every n in `ns` with the scaling scans and the
    clearance product computed once (they do not depend on N): the N sweep of
    the paper's experiments (oz2g_gemm_sweep).  Host arrays or CUDA tensors;
    returns the list of C, each bit-identical to os_ii(a, b, n).C."""
    L = _lib.load()
    ns = [int(x) for x in ns]
    dev = _is_torch_cuda(a)
    if dev != _is_torch_cuda(b):
        raise InvalidArgument("os_ii_sweep: A and B must both be host arrays or both CUDA tensors")
    if dev:
        import torch
        if a.dtype != b.dtype or a.dtype not in (torch.float32, torch.float64):
            raise TypeError("os_ii_sweep: A and B must both be float32 or float64")
        if a.stride(1) != 1 or b.stride(1) != 1:
            raise InvalidArgument("os_ii_sweep: unit column stride required (row-major)")
        prec = F64 if a.dtype == torch.float64 else F32
        m, k = a.shape
        nn = b.shape[1]
        if b.shape[0] != k:
            raise InvalidArgument("dimension mismatch: os_ii inner dimension")
        outs = [torch.empty((m, nn), dtype=a.dtype, device=a.device) for _ in ns]
        pa, pb, lda, ldb = a.data_ptr(), b.data_ptr(), max(a.stride(0), k), max(b.stride(0), nn)
        ptrs = [o.data_ptr() for o in outs]
        flags = _lib.OZ2G_DEVICE_PTRS
        if stream is None:
            stream = torch.cuda.current_stream(a.device).cuda_stream
    else:
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        if a.dtype != b.dtype or a.dtype not in (np.float32, np.float64):
            raise TypeError("os_ii_sweep: A and B must both be float32 or float64")
        if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
            raise InvalidArgument("dimension mismatch: os_ii inner dimension")
        prec = F64 if a.dtype == np.float64 else F32
        m, k = a.shape
        nn = b.shape[1]
        outs = [np.empty((m, nn), dtype=a.dtype) for _ in ns]
        pa, pb, lda, ldb = a.ctypes.data, b.ctypes.data, k, nn
        ptrs = [o.ctypes.data for o in outs]
        flags = _lib.OZ2G_HOST_PTRS
    cp = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
    cn = (C.c_int * max(1, len(ns)))(*ns)
    _check(L.oz2g_gemm_sweep(prec, m, nn, k, pa, lda, pb, ldb, cp, nn, cn, len(ns), flags,
                             C.c_void_p(int(stream) if stream else 0), None))
    return outs


def synchronize() -> None:
    """Complete every blocking=False call on the current device and raise the
    first failure among them in call order (oz2g_synchronize)."""
    _check(_lib.load().oz2g_synchronize())


def dd_gemm(a, b):
    """Double-double reference product (hi, lo) of CUDA fp64 tensors on the
    device (oz2g_dd_gemm); used to measure the emulation error."""
    import torch
    m, k = a.shape
    nn = b.shape[1]
    hi = torch.empty((m, nn), dtype=torch.float64, device=a.device)
    lo = torch.empty_like(hi)
    st = torch.cuda.current_stream(a.device).cuda_stream
    _check(_lib.load().oz2g_dd_gemm(m, nn, k, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
                                    hi.data_ptr(), lo.data_ptr(), nn, C.c_void_p(int(st))))
    return hi, lo


def device_log2f(x_dev, out_dev, stream=None) -> None:
    """Device log2f used for the e/f diagnostics (tests compare it with libm)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(x_dev.device).cuda_stream
    _check(_lib.load().oz2g_device_log2f(x_dev.data_ptr(), out_dev.data_ptr(), x_dev.numel(),
                                         C.c_void_p(int(stream))))


@dataclass
class SuggestResult:
    """bounds.hpp:208-212 (+ the tight search's bookkeeping)."""
    achievable: bool
    n: int
    bound_max: float
    bound: str = "cheap"
    relative: bool = False
    excluded_below: int = 0      # tight: every N below this excluded by the lower estimate
    emulations: int = 0          # tight: full emulations run to settle N
    tight_max: float = 0.0
    tight_rel_max: float = 0.0


def suggest_n(a, b, target: float, bound: str = "cheap", relative: bool = False) -> SuggestResult:
    """Smallest N whose error bound is <= `target` everywhere.

    bound="cheap" (default, the reference's suggest_n, bounds.hpp:217-243):
    the cheap bound (bounds.hpp:198-206), absolute target.
    bound="tight": the tight bound (bounds.hpp:182-195) with the sound device
    |A'B'| <= (|C''| + r_const)/(1 - u_coef); `relative=True` measures it
    against (|A||B|)_ij (the north star's "N from the paper's bound for 1e-15
    relative accuracy").  Every smaller N is shown to fail.  Host numpy arrays
    or CUDA tensors."""
    if bound not in ("cheap", "tight"):
        raise InvalidArgument("suggest_n: bound must be 'cheap' or 'tight'")
    if relative and bound != "tight":
        raise InvalidArgument("suggest_n: relative=True needs bound='tight'")
    L = _lib.load()
    if _is_torch_cuda(a):
        import torch
        if a.dtype != b.dtype or a.dtype not in (torch.float32, torch.float64):
            raise TypeError("suggest_n: A and B must both be float32 or float64")
        if a.stride(1) != 1 or b.stride(1) != 1:
            raise InvalidArgument("suggest_n: unit column stride required (row-major)")
        prec = F64 if a.dtype == torch.float64 else F32
        m, k = a.shape
        nn = b.shape[1]
        pa, pb, lda, ldb = a.data_ptr(), b.data_ptr(), max(a.stride(0), k), max(b.stride(0), nn)
        flags = _lib.OZ2G_DEVICE_PTRS
        stream = torch.cuda.current_stream(a.device).cuda_stream
    else:
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        if a.dtype != b.dtype or a.dtype not in (np.float32, np.float64):
            raise TypeError("suggest_n: A and B must both be float32 or float64")
        prec = F64 if a.dtype == np.float64 else F32
        m, k = a.shape
        nn = b.shape[1]
        pa, pb, lda, ldb = a.ctypes.data, b.ctypes.data, k, nn
        flags = _lib.OZ2G_HOST_PTRS
        stream = 0
    if a.shape[1] != b.shape[0]:
        raise InvalidArgument("dimension mismatch: suggest_n inner dimension")
    if bound == "tight":
        res = _lib.Suggest()
        _check(L.oz2g_suggest_n_tight(prec, m, nn, k, pa, lda, pb, ldb, float(target), 1 if relative else 0, flags,
                                      C.c_void_p(int(stream)), C.byref(res)))
        return SuggestResult(achievable=res.n > 0, n=res.n, bound_max=res.bound_max, bound="tight",
                             relative=bool(relative), excluded_below=res.excluded_below, emulations=res.emulations,
                             tight_max=res.tight_max, tight_rel_max=res.tight_rel_max)
    n_out = C.c_int()
    bmax = C.c_double()
    _check(L.oz2g_suggest_n(prec, m, nn, k, pa, lda, pb, ldb, float(target), flags, C.c_void_p(int(stream)),
                            C.byref(n_out), C.byref(bmax)))
    return SuggestResult(achievable=n_out.value > 0, n=n_out.value, bound_max=bmax.value)
