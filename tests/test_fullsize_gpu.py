"""Parity at the BASELINE sizes through sampled, size-independent checks.

The CPU oracle cannot run a 16384^3, N = 16 emulation (~1.5e14 int8 ops), so
the device result is verified piecewise with the oracle's exact pieces
(oracle/oz2_oracle.c, "sampled full-size checks"):
  * mu' and nu' for EVERY row / column (scaling.hpp:86-107);
  * the clearance-product maxima on sampled rows and columns (O(nk) each,
    scaling.hpp:140-192) — the device computes them with fused atomics;
  * mu and nu for EVERY row / column from the maxima (scaling.hpp:159-194);
  * C at sampled entries, recomputed by the reference pipeline (residues, N
    wrapped dot products, CRT, inverse scaling) from the device's mu / nu:
    bit-exact.
"""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


def _gen(shape, phi, seed):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    u = 1.0 - torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
    v = u - 0.5
    if phi:
        v = v * torch.exp(torch.randn(shape, dtype=torch.float64, device="cuda", generator=g) * phi)
    v[v == 0] = 0.25
    return v


@pytest.mark.parametrize("m,k,n,N,phi", [
    (16384, 16384, 16384, 16, 0.0),      # BASELINE cfg4 (metric config)
    (2048, 65536, 2048, 16, 0.5),        # cfg5 tall-skinny / large k
    (8192, 8192, 8192, 20, 2.0),         # cfg3 wide exponent spread
])
def test_sampled_parity_full_size(cuda, oracle, m, k, n, N, phi):
    import torch
    dA, dB = _gen((m, k), phi, 1000 + m), _gen((k, n), phi, 2000 + n)
    res = oz.os_ii(dA, dB, N, vectors=True)
    torch.cuda.synchronize()
    A, B = dA.cpu().numpy(), dB.cpu().numpy()
    C = res.C.cpu().numpy()
    s = res.scaling
    oracle.set_threads(8)
    mup = oracle.pre_exponents(A, False)
    nup = oracle.pre_exponents(B, True)
    assert np.array_equal(mup, s.mu_prime) and np.array_equal(nup, s.nu_prime)
    rng = np.random.default_rng(m + n + N)
    abar = oracle.ceil_scale(A, mup, False)
    bbar = oracle.ceil_scale(B, nup, True)
    rows = np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, 3)]))
    cols = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, 3)]))
    assert np.array_equal(oracle.cbar_row_max(abar, bbar, rows), s.cmax_row[rows])
    assert np.array_equal(oracle.cbar_col_max(abar, bbar, cols), s.cmax_col[cols])
    del abar, bbar
    # mu / nu for every row / column from the (device) maxima
    sh_r = np.array([oracle.shift_of_cmax(int(c), N)[0] for c in s.cmax_row])
    sh_c = np.array([oracle.shift_of_cmax(int(c), N)[0] for c in s.cmax_col])
    assert np.array_equal(s.mu, (s.mu_prime + sh_r).astype(np.int16))
    assert np.array_equal(s.nu, (s.nu_prime + sh_c).astype(np.int16))
    # C at sampled entries, bit-exact
    ri = np.concatenate([rng.integers(0, m, 96), [0, m - 1, 0, m - 1]])
    cj = np.concatenate([rng.integers(0, n, 96), [0, n - 1, n - 1, 0]])
    ref = oracle.entries(A, B, N, s.mu, s.nu, ri, cj)
    got = C[ri, cj]
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
