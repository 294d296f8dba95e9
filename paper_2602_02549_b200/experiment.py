"""The error-vs-bound sweep of the reference (experiment.hpp), on the GPU.

run_experiment(cfg) mirrors experiment.hpp:90-143 row for row:
  * inputs from the reference stream (gen_matrix + derive_seed, bit-identical);
  * per N: os_ii on the device, the tight and cheap bounds evaluated on the
    device (bounds.hpp:182-206; the tight form uses the sound device estimate
    of |A'B'|, so est_* is >= the reference's), the error |AB - C| against a
    double-double product (exact products, dd sums: within ~k 2^-104 |A||B| of
    the reference's exact GMP product), and the native working-precision GEMM
    error (experiment.hpp:55-68 semantics, sequential RN loop on the device);
  * CSV in the reference's format (experiment.hpp:147-156).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .emulate import DomainError, F32, F64, _check, fp32_safe_moduli_max, os_ii, dd_gemm
from .matrix_io import hexfloat


@dataclass
class ExperimentConfig:
    """experiment.hpp:22-29."""
    m: int = 64
    n: int = 64
    k: int = 1024
    phi: float = 0.5
    mode: int = F64
    n_list: list = field(default_factory=list)
    seed: int = 1
    trials: int = 1


@dataclass
class ExperimentRow:
    """experiment.hpp:31-37."""
    n: int
    est_max: float = -np.inf
    est_min: float = np.inf
    est2_max: float = -np.inf
    est2_min: float = np.inf
    err_max: float = -np.inf
    err_min: float = np.inf
    err_native_max: float = -np.inf


def validate_config(cfg: ExperimentConfig) -> None:
    """experiment.hpp:39-53."""
    if cfg.m < 1 or cfg.n < 1 or cfg.k < 1:
        raise DomainError("experiment: dims must be positive")
    if cfg.k > (1 << 17):
        raise DomainError("experiment: k exceeds 2^17")
    if cfg.phi < 0:
        raise DomainError("experiment: phi must be nonnegative")
    if cfg.trials < 1:
        raise DomainError("experiment: trials must be >= 1")
    if not cfg.n_list:
        raise DomainError("experiment: empty n-list")
    for n in cfg.n_list:
        if n < 2 or n > 49:
            raise DomainError("experiment: n-list entry out of [2, 49]")
        if cfg.mode == F32 and n > fp32_safe_moduli_max():
            raise DomainError(f"experiment: N={n} exceeds the fp32-safe ceiling {fp32_safe_moduli_max()} "
                              "(mode/moduli-count mismatch)")


def gen_matrix(rows: int, cols: int, phi: float, seed: int, mode: int = F64) -> np.ndarray:
    """gen.hpp:15-31 (the reference stream, via the library)."""
    out = np.empty((rows, cols), dtype=np.float64 if mode == F64 else np.float32)
    _check(_lib.load().oz2g_gen_matrix(mode, rows, cols, float(phi), seed, out.ctypes.data))
    return out


def derive_seed(seed: int, trial: int, role: int) -> int:
    """experiment.hpp:83-88."""
    return int(_lib.load().oz2g_derive_seed(seed, trial, role))


def _native_gemm(dA, dB):
    import torch
    m, k = dA.shape
    n = dB.shape[1]
    C_ = torch.empty((m, n), dtype=dA.dtype, device=dA.device)
    st = torch.cuda.current_stream(dA.device).cuda_stream
    _check(_lib.load().oz2g_native_gemm(F64 if dA.dtype == torch.float64 else F32, m, n, k, dA.data_ptr(), k,
                                        dB.data_ptr(), n, C_.data_ptr(), n, C.c_void_p(int(st))))
    return C_


def run_experiment(cfg: ExperimentConfig) -> list:
    """experiment.hpp:90-143."""
    import torch
    validate_config(cfg)
    rows = [ExperimentRow(n=n) for n in cfg.n_list]
    for trial in range(cfg.trials):
        a = gen_matrix(cfg.m, cfg.k, cfg.phi, derive_seed(cfg.seed, trial, 0), cfg.mode)
        b = gen_matrix(cfg.k, cfg.n, cfg.phi, derive_seed(cfg.seed, trial, 1), cfg.mode)
        dA, dB = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        hi, lo = dd_gemm(dA.double(), dB.double())          # the product reference
        native = _native_gemm(dA, dB).double()
        native_err_max = float(((native - hi) - lo).abs().max().item())
        for row in rows:
            res = os_ii(dA, dB, row.n, bounds="full")
            err = ((res.C.double() - hi) - lo).abs()
            tight, cheap = res.bounds["tight"], res.bounds["cheap"]
            row.est_max = max(row.est_max, float(tight.max().item()))
            row.est_min = min(row.est_min, float(tight.min().item()))
            row.est2_max = max(row.est2_max, float(cheap.max().item()))
            row.est2_min = min(row.est2_min, float(cheap.min().item()))
            row.err_max = max(row.err_max, float(err.max().item()))
            row.err_min = min(row.err_min, float(err.min().item()))
            row.err_native_max = max(row.err_native_max, native_err_max)
    return rows


def write_experiment_csv(path: str, rows: list) -> None:
    """experiment.hpp:147-156."""
    with open(path, "w") as f:
        f.write("n,est_max,est_min,est2_max,est2_min,err_max,err_min,err_native_max,err_max_dec\n")
        for r in rows:
            f.write(",".join([str(r.n)] + [hexfloat(v) for v in (r.est_max, r.est_min, r.est2_max, r.est2_min,
                                                                    r.err_max, r.err_min, r.err_native_max)])
                    + f",{r.err_max:.17g}\n")
