"""Parity at the BASELINE sizes through sampled, size-independent checks.

The CPU oracle cannot run a 16384^3, N = 16 emulation (~1.5e14 int8 ops), so
the device result is verified piecewise with the oracle's exact pieces
(oracle/oz2_oracle.c, "sampled full-size checks"), none of which reads a
device intermediate:
  * mu' and nu' for EVERY row / column (scaling.hpp:86-107);
  * the clearance-product maxima of >= 64 rows (every 2048-row block edge of
    the residue GEMM + CRT, api.cu kWBlockRows, and both ends) and >= 64
    columns (every 256-column tile edge sampled), computed by the oracle from
    its own Abar / Bbar (scaling.hpp:111-192);
  * mu and nu of those rows / columns from the ORACLE's maxima
    (scaling.hpp:159-194), against the device's;
  * C at >= 128 entries on those rows x columns, recomputed by the reference
    pipeline (residues, N wrapped dot products, CRT, inverse scaling) with
    the oracle's mu / nu: bit-exact;
  * and, for every row / column, that the device's mu / nu are the step
    function of its own maxima (the exponents kernel).
"""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu

BLOCK_ROWS = 2048  # row block of the residue GEMMs + CRT (api.cu kWBlockRows)


def _gen(shape, phi, seed, dtype=None):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    u = 1.0 - torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
    v = u - 0.5
    if phi:
        v = v * torch.exp(torch.randn(shape, dtype=torch.float64, device="cuda", generator=g) * phi)
    if dtype is not None:
        v = v.to(dtype)
    v[v == 0] = 0.25
    return v.contiguous()


def sample_rows(m, rng, count=64):
    edges = {0, m - 1}
    for r in range(BLOCK_ROWS, m, BLOCK_ROWS):
        edges.update((r - 1, r))
    rest = [int(x) for x in rng.permutation(m) if int(x) not in edges]
    return np.array(sorted(edges | set(rest[:max(0, count - len(edges))])), dtype=np.int64)


def sample_cols(n, rng, count=64):
    edges = {0, n - 1}
    for c in range(256, n, 256 * max(1, n // 256 // 16)):
        edges.update((c - 1, c))
    rest = [int(x) for x in rng.permutation(n) if int(x) not in edges]
    return np.array(sorted(edges | set(rest[:max(0, count - len(edges))])), dtype=np.int64)


def check_sampled(oracle, A, B, res, N, prec, rng, n_entries=128):
    """The oracle-only checks above on host copies A, B (float64 values) of the inputs."""
    m, k = A.shape
    n = B.shape[1]
    s = res.scaling
    C = res.C.cpu().numpy() if hasattr(res.C, "cpu") else res.C
    oracle.set_threads(16)
    mup = oracle.pre_exponents(A, False)
    nup = oracle.pre_exponents(B, True)
    assert np.array_equal(mup, s.mu_prime) and np.array_equal(nup, s.nu_prime)
    abar = oracle.ceil_scale(A, mup, False)
    bbar = oracle.ceil_scale(B, nup, True)
    rows, cols = sample_rows(m, rng), sample_cols(n, rng)
    assert len(rows) >= min(64, m) and len(cols) >= min(64, n)
    cmr = oracle.cbar_row_max(abar, bbar, rows)
    cmc = oracle.cbar_col_max(abar, bbar, cols)
    del abar, bbar
    assert np.array_equal(cmr, s.cmax_row[rows]), "clearance row maxima"
    assert np.array_equal(cmc, s.cmax_col[cols]), "clearance column maxima"
    mu_o = np.array([mup[i] + oracle.shift_of_cmax(int(c), N)[0] for i, c in zip(rows, cmr)], dtype=np.int16)
    nu_o = np.array([nup[j] + oracle.shift_of_cmax(int(c), N)[0] for j, c in zip(cols, cmc)], dtype=np.int16)
    assert np.array_equal(mu_o, s.mu[rows]) and np.array_equal(nu_o, s.nu[cols])
    # every row / column: the device exponents are the step function of the device maxima
    sh_r = np.array([oracle.shift_of_cmax(int(c), N)[0] for c in s.cmax_row])
    sh_c = np.array([oracle.shift_of_cmax(int(c), N)[0] for c in s.cmax_col])
    assert np.array_equal(s.mu, (s.mu_prime + sh_r).astype(np.int16))
    assert np.array_equal(s.nu, (s.nu_prime + sh_c).astype(np.int16))
    # C on rows x cols with the oracle's mu / nu (every sampled row and column at least once)
    nr, nc = len(rows), len(cols)
    extra = max(0, n_entries - nr - nc)
    qi = np.concatenate([np.arange(nr), rng.integers(0, nr, nc), rng.integers(0, nr, extra)])
    qj = np.concatenate([rng.integers(0, nc, nr), np.arange(nc), rng.integers(0, nc, extra)])
    mu_full = np.zeros(m, dtype=np.int16)
    nu_full = np.zeros(n, dtype=np.int16)
    mu_full[rows] = mu_o
    nu_full[cols] = nu_o
    ri, cj = rows[qi], cols[qj]
    ref = oracle.entries(A, B, N, mu_full, nu_full, ri, cj, prec=prec)
    got = C[ri, cj]
    bits = np.uint64 if prec else np.uint32
    bad = np.flatnonzero(got.view(bits) != ref.view(bits))
    assert bad.size == 0, f"{bad.size} of {len(ri)} sampled C entries differ, first ({ri[bad[0]]}, {cj[bad[0]]})"


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
    del dA, dB
    check_sampled(oracle, A, B, res, N, 1, np.random.default_rng(m + n + N))


def test_auto_n_cfg4(cuda):
    """The metric config's N from the paper's bound: at
    16384^3, phi = 0, the smallest N whose tight bound certifies 1e-15
    relative to (|A||B|)_ij is 16 (N = 15 is shown to fail)."""
    import torch
    dA, dB = _gen((16384, 16384), 0.0, 1234), _gen((16384, 16384), 0.0, 5678)
    r = oz.suggest_n(dA, dB, 1e-15, bound="tight", relative=True)
    torch.cuda.synchronize()
    assert r.achievable and r.n == 16, r
    assert r.tight_rel_max <= 1e-15


@pytest.mark.parametrize("m,k,n,N", [(16384, 16384, 16384, 16), (2048, 65536, 2048, 16)])
def test_host_pipeline_full_size(cuda, m, k, n, N):
    """The pipelined, speculated host-pointer path (PCIe uploads in row /
    column chunks, exponents speculated from the chunks present, re-checked at
    every arrival) returns the device path's C bit for bit at the BASELINE
    sizes."""
    import torch
    dA, dB = _gen((m, k), 0.0, 77 + m), _gen((k, n), 0.0, 78 + n)
    dev_c = oz.os_ii(dA, dB, N).C
    Ah = torch.empty((m, k), dtype=torch.float64, pin_memory=True)
    Bh = torch.empty((k, n), dtype=torch.float64, pin_memory=True)
    Ch = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
    Ah.copy_(dA)
    Bh.copy_(dB)
    r = oz.os_ii(Ah.numpy(), Bh.numpy(), N, out=Ch.numpy())
    assert r.speculation in (1, 2, 3)
    assert torch.equal(Ch.view(torch.int64), dev_c.cpu().view(torch.int64))
