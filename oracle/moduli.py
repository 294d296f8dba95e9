"""Exact restatement of the reference's per-(N, mode) constant tables.

TEST INFRASTRUCTURE ONLY (the oracle): tests/, bench.py's cpu_baseline leg and
__graft_entry__.smoke() may import this; the product package never does.

Restates /root/reference/proj/include/oz2/moduli.hpp:93-142 (build_table) and
mp.hpp:59-93 (rational_to_fp64_nearest, p_prime_fp32, scaling_coeff_fp32) with
Python integers and fractions instead of GMP/MPFR:

* P, q, r, rho are exact integers (moduli.hpp:100-110);
* P1 = RN64(P), P2 = RN64(P - P1) (fp64 mode only) (moduli.hpp:112-116);
* P_inv = RN64(1/P) via correctly rounded integer true division (moduli.hpp:117);
* beta/s1/s2 by split_upper_bits (moduli.hpp:60-69, :122-138);
* P' = RD32(log2(P-1)/2 - 1/2) (mp.hpp:67-85) with mpmath *interval*
  arithmetic — the interval is refined until both ends round down to the same
  binary32, exactly the bracketing criterion the reference uses.
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction
from functools import lru_cache

import mpmath

# moduli.hpp:31-36
K_MODULI = (
    256, 255, 253, 251, 247, 241, 239, 233, 229, 227,
    223, 217, 211, 199, 197, 193, 191, 181, 179, 173,
    167, 163, 157, 151, 149, 139, 137, 131, 127, 113,
    109, 107, 103, 101, 97, 89, 83, 79, 73, 71,
    67, 61, 59, 53, 47, 43, 41, 37, 29)
K_MAX_MODULI = 49
F32, F64 = 0, 1


def _f32_bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def _is_f32(x: float) -> bool:
    return struct.unpack("<f", struct.pack("<f", x))[0] == x


def round_down_f32(x: Fraction) -> float:
    """Largest binary32 value <= x (normal range only, which is all we need)."""
    if x == 0:
        return 0.0
    neg = x < 0
    a = -x if neg else x
    # binade: 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    ulp = Fraction(2) ** (e - 23)
    units = a / ulp
    if neg:
        u = -(-units.numerator // units.denominator)  # ceil of magnitude
    else:
        u = units.numerator // units.denominator  # floor
    return float(u * ulp) * (-1.0 if neg else 1.0)


def mod_inverse(a: int, p: int) -> int:
    """moduli.hpp:41-55 (extended Euclid); Python's pow gives the same unique inverse."""
    return pow(a % p, -1, p)


def split_upper_bits(x: int, beta: int) -> tuple[float, float]:
    """moduli.hpp:60-69."""
    if beta <= 0 or beta > 53:
        raise ValueError("split_upper_bits: beta out of (0, 53]")
    if x <= 0:
        raise ValueError("split_upper_bits: x must be positive")
    ln = x.bit_length()
    shift = ln - beta
    if shift <= 0:
        return float(x), 0.0
    head = (x >> shift) << shift
    rem = x - head
    return float(head), float(rem)  # int -> float is correctly rounded (RN-even)


def ceil_log2_long(v: int) -> int:
    """moduli.hpp:71-76."""
    bits = 0
    while (1 << bits) < v:
        bits += 1
    return bits


def p_prime_fp32(P: int) -> float:
    """mp.hpp:67-85: RD32(log2(P-1)/2 - 0.5) by interval bracketing."""
    pm1 = P - 1
    for prec in (192, 384, 768, 1536):
        iv = mpmath.iv
        saved = iv.prec
        iv.prec = prec
        try:
            v = iv.log(iv.mpf(pm1)) / iv.log(iv.mpf(2)) / 2 - iv.mpf("0.5")
            lo, hi = _mpf_to_fraction(v.a), _mpf_to_fraction(v.b)
        finally:
            iv.prec = saved
        flo, fhi = round_down_f32(lo), round_down_f32(hi)
        if flo == fhi:
            return flo
    raise RuntimeError("p_prime_fp32: bracketing did not converge")


def _mpf_to_fraction(x) -> Fraction:
    m, e = mpmath.mpf(x).man_exp
    return Fraction(int(m)) * (Fraction(2) ** int(e))


def scaling_coeff_fp32() -> float:
    """mp.hpp:89-93: RD32(-2^21/(2^22-1)) == -0x1.000006p-1."""
    return round_down_f32(Fraction(-(1 << 21), (1 << 22) - 1))


@lru_cache(maxsize=None)
def build_table(n: int, mode: int) -> dict:
    """moduli.hpp:93-142 build_table(n, mode)."""
    if n < 2 or n > K_MAX_MODULI:
        raise ValueError("build_table: N out of [2, 49]")
    p = list(K_MODULI[:n])
    P = 1
    for pl in p:
        P *= pl
    rho = sum(pl // 2 for pl in p)
    q, r = [], []
    for pl in p:
        mq = P // pl
        ql = mod_inverse(mq, pl)
        q.append(ql)
        r.append(mq * ql)
    P1 = float(P)
    P2 = float(P - int(P1)) if mode == F64 else 0.0
    P_inv = 1 / P  # int/int true division is correctly rounded
    beta = [0] * n
    s1 = [0.0] * n
    s2 = [0.0] * n
    if mode == F64:
        max_log2r = max(x.bit_length() - 1 for x in r)
        clr = ceil_log2_long(rho)
        for l in range(n):
            log2r = r[l].bit_length() - 1
            b = 53 - clr + log2r - max_log2r
            beta[l] = b
            s1[l], s2[l] = split_upper_bits(r[l], b)
    else:
        s1 = [float(x) for x in r]
    return dict(n=n, mode=mode, p=p, q=q, P=P, r=r, rho=rho, P1=P1, P2=P2, P_inv=P_inv,
                beta=beta, s1=s1, s2=s2, P_prime=p_prime_fp32(P))


def fp32_safe_moduli_max() -> int:
    """moduli.hpp:157-170."""
    limit = ((1 << 24) - 1) << 105
    prod, cnt = 1, 0
    for pl in K_MODULI:
        prod *= pl
        if prod > limit:
            break
        cnt += 1
    return cnt
