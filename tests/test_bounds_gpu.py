"""Error bounds and measured error on the GPU.

* The device-evaluated cheap / tight bounds are certificates: never below the
  formula of bounds.hpp (evaluated here to ~2^-300 by oracle/bounds.py) and
  within a few ulps above it.
* The actual error |C - AB| (exact AB as Fractions) is below both bounds for
  every entry — the paper's Theorem 2 on our outputs (SPEC: zero tolerance).
* The double-double reference GEMM used at scale matches exact products.
"""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n,phi,N,dt", [
    (9, 40, 7, 0.0, 8, np.float64), (9, 40, 7, 2.0, 14, np.float64), (6, 64, 5, 8.0, 20, np.float64),
    (12, 33, 10, 0.5, 16, np.float64), (7, 20, 6, 1.0, 9, np.float32), (8, 50, 8, 0.0, 16, np.float32),
])
def test_bounds_are_certificates(cuda, oracle, m, k, n, phi, N, dt):
    from oracle import bounds as OB
    A = oracle.gen_matrix(m, k, phi, oracle.derive_seed(11, m, 0), dt)
    B = oracle.gen_matrix(k, n, phi, oracle.derive_seed(11, n, 1), dt)
    ref = oracle.os_ii(A, B, N, keep_intermediates=True)
    got = oz.os_ii(A, B, N, bounds="full")
    assert np.array_equal(got.C, ref.C)
    cheap_or, tight_or = OB.bounds(A, B, N, ref.inter["cmax_row"], ref.inter["cmax_col"],
                                   ref.inter["Aprime"], ref.inter["Bprime"])
    exact = OB.exact_product(A, B)
    bc, bt = got.bounds["cheap"], got.bounds["tight"]
    mpmath.mp.prec = 320
    for i in range(m):
        for j in range(n):
            c_or, t_or = cheap_or[i][j], tight_or[i][j]
            assert mpmath.mpf(bc[i, j]) >= c_or                      # sound
            assert mpmath.mpf(bc[i, j]) <= c_or * (1 + mpmath.mpf(2) ** -45)   # tight
            assert mpmath.mpf(bt[i, j]) >= t_or
            # the device replaces the exact |A'B'| by (|C''| + r_const)/(1 - u): at most ~u r_const looser
            assert mpmath.mpf(bt[i, j]) <= t_or * (1 + mpmath.mpf(2) ** -20)
            assert bt[i, j] <= bc[i, j]
            err = abs(Fraction(float(got.C[i, j])) - exact[i][j])
            assert mpmath.mpf(err.numerator) / err.denominator <= t_or   # Theorem 2 on our output
    assert got.bounds["cheap_max"] == bc.max() and got.bounds["tight_max"] == bt.max()


def test_dd_gemm_matches_exact(cuda, oracle):
    import torch
    from oracle import bounds as OB
    A = oracle.gen_matrix(37, 130, 3.0, 5)
    B = oracle.gen_matrix(130, 29, 3.0, 6)
    hi, lo = oz.dd_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    hi, lo = hi.cpu().numpy(), lo.cpu().numpy()
    exact = OB.exact_product(A, B)
    absab = np.abs(A) @ np.abs(B)
    for i in range(37):
        for j in range(29):
            err = abs(Fraction(hi[i, j]) + Fraction(lo[i, j]) - exact[i][j])
            assert err <= Fraction(absab[i, j]) * Fraction(1, 1 << 95)


def test_bounds_device_tensors(cuda, oracle):
    import torch
    A = oracle.gen_matrix(300, 257, 0.0, 1)
    B = oracle.gen_matrix(257, 200, 0.0, 2)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    r = oz.os_ii(dA, dB, 16, bounds="full")
    hi, lo = oz.dd_gemm(dA, dB)
    err = ((r.C - hi) - lo).abs()
    assert bool((err <= r.bounds["tight"]).all())
    assert bool((r.bounds["tight"] <= r.bounds["cheap"]).all())
    host = oz.os_ii(A, B, 16, bounds=True)
    assert host.bounds["tight_max"] == float(r.bounds["tight"].max())


@pytest.mark.parametrize("phi,target,dt", [(0.0, 1e-12, np.float64), (2.0, 1e-9, np.float64),
                                           (0.5, 1e-14, np.float64), (0.0, 1e-4, np.float32),
                                           (8.0, 1e-30, np.float64)])
def test_suggest_n_matches_oracle(cuda, oracle, phi, target, dt):
    """suggest_n (bounds.hpp:217-243): same N as the restated cheap bound; at
    that N the bound holds and one N less fails (minimality)."""
    from oracle import bounds as OB
    A = oracle.gen_matrix(10, 48, phi, 71, dt)
    B = oracle.gen_matrix(48, 9, phi, 72, dt)
    r = oracle.os_ii(A, B, 8, want_cmax=True)
    ok, n_or, mx_or = OB.suggest_n(A, B, target, r.inter["cmax_row"], r.inter["cmax_col"])
    got = oz.suggest_n(A, B, target)
    assert got.achievable == ok
    assert got.n == n_or
    if ok:
        assert got.bound_max <= target and mpmath.mpf(got.bound_max) >= mx_or


@pytest.mark.parametrize("phi,target,relative,dt", [(0.0, 1e-15, True, np.float64), (0.5, 3e-15, True, np.float64),
                                                    (2.0, 1e-13, True, np.float64), (0.0, 1e-13, False, np.float64),
                                                    (0.0, 1e-6, True, np.float32)])
def test_suggest_n_tight(cuda, oracle, phi, target, relative, dt):
    """suggest_n(bound="tight", relative=...): the device criterion is a
    certificate of the reference's tight bound (bounds.hpp:182-195 with the
    exact |A'B'|, exact |A||B|), so its N is >= the reference-exact one and
    at most one more (only when the exact maximum sits within a few percent
    of the target); every smaller N fails — below `excluded_below` by the
    lower estimate (checked here against the exact maximum), above it by its
    own emulation."""
    from oracle import bounds as OB
    A = oracle.gen_matrix(10, 48, phi, 81, dt)
    B = oracle.gen_matrix(48, 9, phi, 82, dt)
    got = oz.suggest_n(A, B, target, bound="tight", relative=relative)
    n_ref = OB.suggest_n_tight(A, B, target, relative, oracle)
    assert got.achievable == (n_ref > 0) or (n_ref > 0 and got.n == 0)
    if n_ref == 0:
        return
    assert n_ref <= got.n <= n_ref + 1, (got, n_ref)
    if got.n > n_ref:
        assert OB.tight_max(A, B, n_ref, relative, oracle) > 0.9 * target
    # certificate and tightness at the chosen N
    exact = OB.tight_max(A, B, got.n, relative, oracle)
    crit = got.tight_rel_max if relative else got.tight_max
    assert crit <= target and mpmath.mpf(crit) >= exact and crit <= 1.1 * float(exact)
    # minimality: the lower estimate only excludes N whose exact maximum exceeds the target
    for nn in range(2, got.excluded_below):
        assert OB.tight_max(A, B, nn, relative, oracle) > target, nn
    for nn in range(got.excluded_below, got.n):
        r = oz.os_ii(A, B, nn, bounds=True, relative=relative)
        assert (r.bounds["tight_rel_max"] if relative else r.bounds["tight_max"]) > target, nn
    # the same N through device tensors
    import torch
    got_d = oz.suggest_n(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), target, bound="tight",
                         relative=relative)
    assert got_d.n == got.n and got_d.bound_max == got.bound_max
