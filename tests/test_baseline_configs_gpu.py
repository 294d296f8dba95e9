"""Parity at the BASELINE.json configurations the oracle can reach.

cfg1 (the reference's own CPU case): emulated DGEMM 1024^3, N = 14, phi = 0,
on the reference generator's inputs (gen.hpp:15-31, seeds derive_seed(1, 0,
0/1) as experiment.hpp:83-88) — the full CPU oracle os_ii (emulate.hpp:54-88)
against the device, every intermediate bit for bit: mu', nu', Cbar, Dbar,
all clearance maxima, mu, nu, e, f, A', B', every residue plane, every
wrapped INT32 product, W, C1, C2, Q, C'' and C.  The same at 1024^3 in
fp32 mode (N = 8; moduli.hpp:113-138, crt.hpp:139-148).

cfg2: emulated SGEMM 4096^3, N = 6, 7, 8, phi = 0 — the oracle's sampled
pieces (tests/test_fullsize_gpu.py::check_sampled): mu' / nu' everywhere,
clearance maxima / mu / nu on >= 64 rows and columns from the oracle's own
Abar, Bbar, and C at sampled entries bit-exact (fp32 bits).
"""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

from test_fullsize_gpu import check_sampled

pytestmark = pytest.mark.gpu


def _eq(name, a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, name
    if a.dtype.kind == "f":
        bits = {2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
        bad = np.flatnonzero(a.view(bits).ravel() != b.view(bits).ravel())
    else:
        bad = np.flatnonzero(a.ravel() != b.ravel())
    assert bad.size == 0, f"{name}: {bad.size} mismatches, first flat index {bad[0]}"


@pytest.mark.parametrize("N,dt", [(14, np.float64), (8, np.float32)])
def test_cfg1_full_oracle_1024(cuda, oracle, N, dt):
    m = n = k = 1024
    A = oracle.gen_matrix(m, k, 0.0, oracle.derive_seed(1, 0, 0), dt)
    B = oracle.gen_matrix(k, n, 0.0, oracle.derive_seed(1, 0, 1), dt)
    oracle.set_threads(16)
    ref = oracle.os_ii(A, B, N, keep_intermediates=True, residues=True)
    got = oz.os_ii(A, B, N, keep_intermediates=True, evidence=True)
    s, c, ri = got.scaling, got.crt, ref.inter
    for name in ("mu_prime", "nu_prime", "Cbar", "Dbar", "cmax_row", "cmax_col", "mu", "nu", "e", "f",
                 "Aprime", "Bprime"):
        _eq(name, getattr(s, name), ri[name])
    for name in ("Ares", "Bres", "Cprod", "W", "C1", "C2", "Q", "Cpp64"):
        _eq(name, getattr(c, name), ri[name])
    if dt == np.float32:
        _eq("Cpp32", c.Cpp32, ri["Cpp32"])
    _eq("C", got.C, ref.C)
    assert got.subnormal == ref.subnormal
    # the device-pointer path and the plain call return the same C
    import torch
    dC = oz.os_ii(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), N).C.cpu().numpy()
    _eq("C (device pointers)", dC, ref.C)


@pytest.mark.parametrize("N", [6, 7, 8])
def test_cfg2_sgemm_4096_sampled(cuda, oracle, N):
    m = n = k = 4096
    A = oracle.gen_matrix(m, k, 0.0, oracle.derive_seed(2, 0, 0), np.float32)
    B = oracle.gen_matrix(k, n, 0.0, oracle.derive_seed(2, 0, 1), np.float32)
    res = oz.os_ii(A, B, N, vectors=True)
    check_sampled(oracle, A.astype(np.float64), B.astype(np.float64), res, N, 0,
                  np.random.default_rng(4096 + N))
