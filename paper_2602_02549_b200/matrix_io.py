"""Text matrix format of the reference CLI (matrix_io.hpp:1-81).

Header line "rows cols {fp32|fp64}", then one C99 hex-float per line,
row-major.  Hex-floats round-trip bit-exactly.
"""
from __future__ import annotations

import numpy as np


def hexfloat(v: float) -> str:
    """C printf("%a") spelling (matrix_io.hpp:19-23): minimal hex digits."""
    s = float(v).hex()
    if s in ("inf", "-inf", "nan"):
        return s
    sign = "-" if s.startswith("-") else ""
    body = s.lstrip("-")[2:]                      # "1.8000000000000p+1"
    mant, exp = body.split("p")
    if "." in mant:
        head, frac = mant.split(".")
        frac = frac.rstrip("0")
        mant = head + ("." + frac if frac else "")
    return f"{sign}0x{mant}p{exp}"


def write_matrix(path: str, m: np.ndarray) -> None:
    """matrix_io.hpp:26-39."""
    mode = "fp32" if m.dtype == np.float32 else "fp64"
    with open(path, "w") as f:
        f.write(f"{m.shape[0]} {m.shape[1]} {mode}\n")
        for v in m.reshape(-1):
            f.write(hexfloat(float(v)) + "\n")


def read_matrix(path: str) -> np.ndarray:
    """matrix_io.hpp:47-79: values parsed as doubles then narrowed for fp32."""
    with open(path) as f:
        toks = f.read().split()
    if len(toks) < 3:
        raise RuntimeError(f"bad matrix header in {path}")
    rows, cols, mode = int(toks[0]), int(toks[1]), toks[2]
    if mode not in ("fp32", "fp64"):
        raise RuntimeError(f"bad precision '{mode}' in {path}")
    vals = toks[3:]
    if len(vals) < rows * cols:
        raise RuntimeError(f"truncated matrix data in {path}")
    data = np.array([float.fromhex(t) if "x" in t.lower() else float(t) for t in vals[:rows * cols]],
                    dtype=np.float64).reshape(rows, cols)
    return data.astype(np.float32) if mode == "fp32" else data
