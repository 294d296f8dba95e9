"""GPU parity: the CUDA product path (through the C ABI) vs the CPU oracle.

Bit-exact on every integer/byte stage (mu', nu', clearance maxima, mu, nu,
residue planes, wrapped INT32 products, W) and on the final C (0 ulp: the
fp64 stages are the reference's own RN operation sequence).
"""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


def _eq(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    if a.dtype.kind == "f":
        ok = np.array_equal(a.view(np.uint8), b.view(np.uint8))  # bitwise: -0.0 != +0.0
    else:
        ok = np.array_equal(a, b)
    if not ok:
        bad = np.argwhere(a != b)
        raise AssertionError(f"{bad.shape[0]} mismatches, first at {bad[:5].tolist()}: "
                             f"{a[tuple(bad[0])]} vs {b[tuple(bad[0])]}")


def test_unit_product_trace(cuda, oracle):
    # test_emulate.cpp:13-20: mu = nu = 7, A' = B' = 128, W = (0, 64), C1 = 16384, Q = 0, C = 1
    for dt in (np.float64, np.float32):
        one = np.ones((1, 1), dtype=dt)
        r = oz.os_ii(one, one, 2, keep_intermediates=True)
        assert r.C[0, 0] == 1.0
        assert r.scaling.mu[0] == 7 and r.scaling.nu[0] == 7
        assert r.crt.W[:, 0, 0].tolist() == [0, 64]
        assert r.crt.C1[0, 0] == 16384.0 and r.crt.Q[0, 0] == 0.0 and r.crt.Cpp64[0, 0] == 16384.0
        for n in (10, 30, 49) if dt == np.float64 else (10, 16):
            c = oz.os_ii(one, one, n).C[0, 0]
            assert abs(float(c) - 1.0) <= (2.0 ** -40 if dt == np.float64 else 2.0 ** -18)


CASES = [
    # (m, k, n, phi, N, dtype)
    (7, 20, 6, 0.0, 2, np.float64),
    (7, 20, 6, 4.0, 16, np.float64),
    (7, 20, 6, 4.0, 49, np.float64),
    (33, 100, 65, 0.5, 14, np.float64),
    (130, 300, 260, 2.0, 14, np.float64),
    (64, 1024, 64, 0.0, 16, np.float64),
    (200, 129, 300, 8.0, 20, np.float64),
    (7, 20, 6, 0.0, 9, np.float32),
    (33, 100, 65, 0.5, 8, np.float32),
    (130, 300, 260, 2.0, 16, np.float32),
    # rows over 256 KB: the row scan held to one row per SM (scale.cu)
    (5, 40000, 3, 0.5, 12, np.float64),
    (4, 70000, 3, 2.0, 8, np.float32),
    # rows of 8192 < kp <= 65536: the row scan over a cluster of 2 / 4 / 8 CTAs
    (3, 12000, 5, 1.0, 14, np.float64),
    (6, 30000, 4, 0.5, 16, np.float64),
    (5, 50000, 3, 2.0, 8, np.float32),
]


@pytest.mark.parametrize("m,k,n,phi,N,dt", CASES)
def test_os_ii_bit_parity(cuda, oracle, m, k, n, phi, N, dt):
    seed = 1000 * m + 10 * k + n
    A = oracle.gen_matrix(m, k, phi, oracle.derive_seed(seed, 0, 0), dt)
    B = oracle.gen_matrix(k, n, phi, oracle.derive_seed(seed, 0, 1), dt)
    ref = oracle.os_ii(A, B, N, keep_intermediates=True, residues=True)
    got = oz.os_ii(A, B, N, keep_intermediates=True, evidence=True)
    s, c, ri = got.scaling, got.crt, ref.inter
    _eq(s.mu_prime, ri["mu_prime"])
    _eq(s.nu_prime, ri["nu_prime"])
    _eq(s.Cbar, ri["Cbar"])
    _eq(s.Dbar, ri["Dbar"])
    _eq(s.mu, ri["mu"])
    _eq(s.nu, ri["nu"])
    _eq(s.e, ri["e"])
    _eq(s.f, ri["f"])
    _eq(s.Aprime, ri["Aprime"])
    _eq(s.Bprime, ri["Bprime"])
    _eq(c.Ares, ri["Ares"])
    _eq(c.Bres, ri["Bres"])
    _eq(c.Cprod, ri["Cprod"])
    _eq(c.W, ri["W"])
    _eq(c.C1, ri["C1"])
    _eq(c.C2, ri["C2"])
    _eq(c.Q, ri["Q"])
    _eq(c.Cpp64, ri["Cpp64"])
    if dt == np.float32:
        _eq(c.Cpp32, ri["Cpp32"])
    _eq(got.C, ref.C)
    assert got.subnormal == ref.subnormal


@pytest.mark.parametrize("m,k,n", [(2560, 300, 700), (2049, 129, 257), (4096, 1024, 512)])
def test_pipelined_host_path_matches_device(cuda, oracle, m, k, n):
    """Host-pointer calls on large problems stream A in row chunks and download
    C per row block on copy streams; the result must equal the device path."""
    import torch
    A = oracle.gen_matrix(m, k, 1.0, 21)
    B = oracle.gen_matrix(k, n, 1.0, 22)
    host = oz.os_ii(A, B, 14)
    devc = oz.os_ii(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 14).C.cpu().numpy()
    assert np.array_equal(host.C.view(np.uint64), devc.view(np.uint64))
    # pinned host buffers (the DMA path the bench uses) and a second call reusing the workspace
    Ap = torch.from_numpy(A).pin_memory().numpy()
    Bp = torch.from_numpy(B).pin_memory().numpy()
    Cp = torch.empty((m, n), dtype=torch.float64).pin_memory().numpy()
    oz.os_ii(Ap, Bp, 14, out=Cp)
    assert np.array_equal(Cp.view(np.uint64), devc.view(np.uint64))


def test_pipelined_matches_oracle(cuda, oracle):
    A = oracle.gen_matrix(2304, 64, 2.0, 31)
    B = oracle.gen_matrix(64, 300, 2.0, 32)
    ref = oracle.os_ii(A, B, 16)
    got = oz.os_ii(A, B, 16)
    assert np.array_equal(got.C.view(np.uint64), ref.C.view(np.uint64))


def _mixed_exponent_pair(oracle, m, k, n, phi, seed, dt):
    """Reference-generator A and B where every third row of A holds only its
    column-0 entry, every third column of B only its row-1 entry, and A's
    column 1 and B's row 0 are scaled by 2^-10: those rows / columns get a tiny
    clearance maximum, hence a large shift and |A'| >= 2^62 (the
    exponent-bucket path of the residue split), the others the balanced-digit
    fast path."""
    A = oracle.gen_matrix(m, k, phi, oracle.derive_seed(seed, 0, 0), dt).copy()
    B = oracle.gen_matrix(k, n, phi, oracle.derive_seed(seed, 0, 1), dt).copy()
    A[:, 1] *= dt(2.0 ** -10)
    B[0, :] *= dt(2.0 ** -10)
    A[::3, 1:] = 0
    B[:1, ::3] = 0
    B[2:, ::3] = 0
    return A, B


@pytest.mark.parametrize("m,k,n,phi,N,dt", [
    (96, 520, 72, 0.0, 16, np.float64),
    (40, 300, 33, 8.0, 20, np.float64),
    (33, 100, 65, 0.5, 49, np.float64),
    (64, 260, 48, 1.0, 8, np.float32),
    (31, 77, 29, 2.0, 16, np.float32),
    # wide spread, few moduli: four-digit and eight-digit chunks in one matrix
    (64, 520, 48, 8.0, 8, np.float64),
])
@pytest.mark.parametrize("fast", [1, 0])
def test_residue_split_paths(cuda, oracle, m, k, n, phi, N, dt, fast):
    """Both residue-split paths (resid.cu: balanced digits for |A'| < 2^62,
    exponent buckets otherwise; option "resid_fast") give the reference's
    residue planes, also when both occur in one matrix."""
    seed = 77 * m + k
    A, B = _mixed_exponent_pair(oracle, m, k, n, phi, seed, dt)
    ref = oracle.os_ii(A, B, N, keep_intermediates=True, residues=True)
    with oz.options(resid_fast=fast):
        got = oz.os_ii(A, B, N, keep_intermediates=True, evidence=True)
    _eq(got.scaling.mu, ref.inter["mu"])
    _eq(got.scaling.nu, ref.inter["nu"])
    _eq(got.crt.Ares, ref.inter["Ares"])
    _eq(got.crt.Bres, ref.inter["Bres"])
    _eq(got.crt.W, ref.inter["W"])
    _eq(got.C, ref.C)


@pytest.mark.parametrize("N", [8, 16])
def test_residue_digit_boundaries(cuda, oracle, N):
    """A' placed on the edges of the residue split's paths (resid.cu): four
    balanced digits (|A'| up to 0x7F7F7F7F / down to -0x80808080) against
    eight, |A'| just below 2^62 against the exponent buckets (A' = 2^62 at the
    row maximum), zeros, +-1 and values that truncate to 0.  B has one nonzero
    row, so every clearance maximum is 32 * 32 and mu = shift(1024) is known
    from the oracle; the residue planes must equal the oracle's."""
    k, n = 64, 8
    B = np.zeros((k, n))
    B[0, :] = 32.0
    probe = np.zeros((1, k)); probe[0, 0] = 32.0
    mu = int(oracle.os_ii(probe, B, N, keep_intermediates=True, residues=True).inter["mu"][0])
    targets = [0x7F7F7F7F, 0x7F7F7F80, 0x80808080, 0x80808081, (1 << 31) - 1, 1 << 31, 1, 0,
               (1 << 62) - (1 << 9), (1 << 53) - 1, 0x7F7F7F7F7F7F7F, 255, 256, 0x8080]
    rows = []
    for sign in (1, -1):
        for start in range(0, len(targets), 3):
            r = np.zeros(k)
            r[0] = 32.0  # the row maximum: A' = 32 * 2^mu
            for j, t in enumerate(targets[start:start + 3] + targets[:5]):
                v = sign * t * 2.0 ** -mu
                if abs(v) <= 32.0:
                    r[8 + j] = v  # the second 8-element chunk mixes four- and eight-digit values
            for j, t in enumerate(targets[start:start + 8]):
                v = sign * t * 2.0 ** -mu
                if abs(v) <= 32.0:
                    r[16 + j] = v
            for j in range(8):  # a chunk of values that truncate to 0 or +-1
                r[24 + j] = sign * (0.5 + j) * 2.0 ** -mu
            rows.append(r)
    A = np.array(rows)
    ref = oracle.os_ii(A, B, N, keep_intermediates=True, residues=True)
    assert int(ref.inter["mu"][0]) == mu
    for fast in (1, 0):
        with oz.options(resid_fast=fast):
            got = oz.os_ii(A, B, N, keep_intermediates=True, evidence=True)
        _eq(got.scaling.Aprime, ref.inter["Aprime"])
        _eq(got.crt.Ares, ref.inter["Ares"])
        _eq(got.crt.W, ref.inter["W"])
        _eq(got.C, ref.C)
