"""High-precision restatement of the reference's error bounds (TEST ONLY).

Restates /root/reference/proj/include/oz2/bounds.hpp:
  exponent_stats   :32-60   alpha_i = ilogb(max_h |a_ih|), beta_j, Cbar maxima clamped to >= 1
  r_const_exact    :74-81   constant part of R_b
  u_coef_exact     :84-87
  r_cheap_exact    :90-92
  eval_bound       :147-177 bound_ij = t (|A|v)_i 2^beta'_j + t 2^alpha'_i (v^T|B|)_j
                              + kpR_ij t^2 2^(alpha'_i + beta'_j)
  bound_tight      :182-195 kpR = k + r_const + u_coef |A'B'|_ij (exact |A'B'|)
  bound_cheap      :198-206 kpR = k + r_cheap
The reference evaluates in 128-bit MPFR with upward rounding; here every
quantity is exact (Fractions) except the two square roots and t, which mpmath
evaluates at 320 bits — so these values are the formula to ~2^-300 relative,
the yardstick a certificate must not fall below.
"""
from __future__ import annotations

import math
from fractions import Fraction

import mpmath
import numpy as np

from . import moduli as M


def r_const_exact(t: dict) -> Fraction:
    u32, u64 = Fraction(1, 1 << 24), Fraction(1, 1 << 53)
    rho_p = Fraction(t["rho"]) * t["P"]
    if t["mode"] == M.F32:
        return (1 + u32) * (t["n"] + 2) * u64 * rho_p
    clr = M.ceil_log2_long(t["rho"])
    return (1 + 3 * u64) * (1 << (1 + clr)) * (t["n"] + 2) * u64 * u64 * rho_p


def u_coef_exact(t: dict) -> Fraction:
    return Fraction(1, 1 << 24) if t["mode"] == M.F32 else Fraction(3, 1 << 53)


def bounds(A: np.ndarray, B: np.ndarray, n: int, cmax_row, cmax_col, aprime=None, bprime=None):
    """Return (cheap, tight) as lists of mpmath values (tight needs A', B')."""
    mode = M.F64 if A.dtype == np.float64 else M.F32
    t = M.build_table(n, mode)
    m, k = A.shape
    nn = B.shape[1]
    mpmath.mp.prec = 320
    P = t["P"]
    tt = 1 / mpmath.sqrt(mpmath.mpf(32 * (P - 1)))
    t2 = 1 / mpmath.mpf(32 * (P - 1))
    rc = r_const_exact(t)
    uc = u_coef_exact(t)
    alpha = [math.frexp(float(np.max(np.abs(A[i].astype(np.float64)))))[1] - 1 for i in range(m)]
    beta = [math.frexp(float(np.max(np.abs(B[:, j].astype(np.float64)))))[1] - 1 for j in range(nn)]
    rs = [sum(Fraction(abs(float(x))) for x in A[i]) for i in range(m)]
    cs = [sum(Fraction(abs(float(x))) for x in B[:, j]) for j in range(nn)]
    pa = [mpmath.sqrt(max(1, int(cmax_row[i]))) * mpmath.mpf(2) ** alpha[i] for i in range(m)]
    pb = [mpmath.sqrt(max(1, int(cmax_col[j]))) * mpmath.mpf(2) ** beta[j] for j in range(nn)]
    kpr_cheap = Fraction(k) + rc + uc * Fraction(P, 2)
    ab = None
    if aprime is not None:
        Ai = [[int(x) for x in row] for row in aprime]
        Bi = [[int(x) for x in row] for row in bprime]
        ab = [[abs(sum(Ai[i][h] * Bi[h][j] for h in range(k))) for j in range(nn)] for i in range(m)]

    def mpq(f: Fraction):
        return mpmath.mpf(f.numerator) / f.denominator

    cheap = [[None] * nn for _ in range(m)]
    tight = [[None] * nn for _ in range(m)]
    for i in range(m):
        for j in range(nn):
            base = tt * mpq(rs[i]) * pb[j] + tt * pa[i] * mpq(cs[j])
            cheap[i][j] = base + mpq(kpr_cheap) * t2 * pa[i] * pb[j]
            if ab is not None:
                kt = Fraction(k) + rc + uc * ab[i][j]
                tight[i][j] = base + mpq(kt) * t2 * pa[i] * pb[j]
    return cheap, tight


def exact_product(A: np.ndarray, B: np.ndarray):
    """Exact A B as Fractions (small sizes)."""
    m, k = A.shape
    nn = B.shape[1]
    Af = [[Fraction(float(x)) for x in row] for row in A]
    Bf = [[Fraction(float(x)) for x in row] for row in B]
    return [[sum(Af[i][h] * Bf[h][j] for h in range(k)) for j in range(nn)] for i in range(m)]


def suggest_n(A: np.ndarray, B: np.ndarray, target: float, cmax_row, cmax_col):
    """bounds.hpp:217-243 with the cheap bound restated above (mpmath); the
    clearance maxima do not depend on N (bounds.hpp:214-216)."""
    mode = M.F64 if A.dtype == np.float64 else M.F32
    n_max = M.fp32_safe_moduli_max() if mode == M.F32 else M.K_MAX_MODULI
    last = None
    for n in range(2, n_max + 1):
        cheap, _ = bounds(A, B, n, cmax_row, cmax_col)
        mx = max(max(row) for row in cheap)
        last = mx
        if mx <= target:
            return True, n, mx
    return False, 0, last


def abs_product(A: np.ndarray, B: np.ndarray):
    """(|A||B|)_ij exactly, as Fractions (small sizes)."""
    return exact_product(np.abs(A.astype(np.float64)), np.abs(B.astype(np.float64)))


def tight_max(A: np.ndarray, B: np.ndarray, n: int, relative: bool, ora):
    """max_ij of the reference's tight bound (bounds.hpp:182-195, exact |A'B'|
    from the oracle's A', B' at this N), absolute or over (|A||B|)_ij."""
    r = ora.os_ii(A, B, n, keep_intermediates=True)
    _, tight = bounds(A, B, n, r.inter["cmax_row"], r.inter["cmax_col"], r.inter["Aprime"], r.inter["Bprime"])
    if not relative:
        return max(max(row) for row in tight)
    ab = abs_product(A, B)
    return max(tight[i][j] / (mpmath.mpf(ab[i][j].numerator) / ab[i][j].denominator)
               for i in range(len(tight)) for j in range(len(tight[0])))


def suggest_n_tight(A: np.ndarray, B: np.ndarray, target: float, relative: bool, ora, n_hi: int = None):
    """Smallest N whose reference tight-bound maximum meets `target` (the
    criterion oz2g_suggest_n_tight certifies from above)."""
    mode = M.F64 if A.dtype == np.float64 else M.F32
    n_max = M.fp32_safe_moduli_max() if mode == M.F32 else M.K_MAX_MODULI
    for n in range(2, min(n_max, n_hi or n_max) + 1):
        if tight_max(A, B, n, relative, ora) <= target:
            return n
    return 0
