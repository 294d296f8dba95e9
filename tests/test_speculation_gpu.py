"""Speculated scaling exponents on the blocking pipelined host-pointer path
(api.cu run_gemm).  mu_i / nu_j (scaling.hpp:159-194) need the clearance
maxima of row i / column j over the whole of B / A, i.e. the whole upload.
Mode 1 (OZ2G_SPEC=1) uploads B first and speculates nu from the first A row
chunk; mode 2 (default) uploads A row chunks and B column chunks alternately
and speculates both mu and nu from the maxima present.  After every arrival
the exponents are re-derived and whatever was computed with a moved exponent
is redone, so C is the unspeculated C bit for bit:
  * confirmed (the first chunks already hold the final maxima): speculation 1;
  * moved: speculation 2 (moved tiles / column tiles recomputed);
  * mode 1 only: moved, and a block computed with the superseded exponents
    raised a status flag: speculation 3 (every stage after the upload redone).
    Mode 2 keeps status flags per tile and resets them on recomputation."""

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

MODES = ["1", "2"]


def _same(a, b):
    assert a.dtype == b.dtype and a.shape == b.shape
    assert np.array_equal(a.view(np.uint64 if a.dtype == np.float64 else np.uint32),
                          b.view(np.uint64 if b.dtype == np.float64 else np.uint32))


def _call(mode, A, B, nmod, **kw):
    with oz.options(spec=int(mode)):
        return oz.os_ii(A, B, nmod, **kw)


def _unspeculated(A, B, nmod, **kw):
    r = _call("0", A, B, nmod, **kw)
    assert r.speculation == 0
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_speculation_confirmed(cuda, oracle, mode, dtype):
    """Every row chunk of A holds the same rows and every column chunk of B the
    same columns, so the first chunks' maxima are the final ones."""
    m, k, n = 4096, 128, 512
    A = np.tile(oracle.gen_matrix(512, k, 0.0, 901), (m // 512, 1)).astype(dtype)
    B = np.tile(oracle.gen_matrix(k, 256, 0.0, 902), (1, n // 256)).astype(dtype)
    nmod = 14 if dtype == np.float64 else 7
    r = _call(mode, A, B, nmod, vectors=True)
    assert r.speculation == 1
    r0 = _unspeculated(A, B, nmod, vectors=True)
    _same(r.C, r0.C)
    _same(r.C, oracle.os_ii(A, B, nmod).C)
    # the returned scaling vectors are the final ones (e, f from the complete maxima)
    for nm in ("mu", "nu", "e", "f", "cmax_row", "cmax_col"):
        assert np.array_equal(getattr(r.scaling, nm), getattr(r0.scaling, nm)), nm


def _moved_case(oracle, m, k, n, dtype):
    """Rows of the first seven chunks have a single nonzero, so their clearance
    products are <= 64 * 64; the dense rows of the last chunk raise every
    column maximum past several step thresholds."""
    rng = np.random.default_rng(7)
    A = np.zeros((m, k), dtype=dtype)
    sparse = m - m // 8
    A[np.arange(sparse), np.arange(sparse) % k] = rng.uniform(0.1, 1.0, sparse)
    A[sparse:] = oracle.gen_matrix(m - sparse, k, 0.0, 903)
    B = oracle.gen_matrix(k, n, 0.0, 904).astype(dtype)
    return A, B


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_speculation_moved(cuda, oracle, mode, dtype):
    m, k, n = 4096, 128, 512
    A, B = _moved_case(oracle, m, k, n, dtype)
    nmod = 14 if dtype == np.float64 else 7
    r = _call(mode, A, B, nmod, vectors=True)
    assert r.speculation == 2
    r0 = _unspeculated(A, B, nmod)
    assert not r.subnormal and not r0.subnormal
    _same(r.C, r0.C)
    ref = oracle.os_ii(A, B, nmod, keep_intermediates=True)
    _same(r.C, ref.C)
    assert np.array_equal(r.scaling.nu, ref.inter["nu"]) and np.array_equal(r.scaling.mu, ref.inter["mu"])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
def test_speculation_moved_then_error(cuda, oracle, mode):
    """Exponents move and the last chunk holds a zero row: the call reports
    the error the unspeculated call reports."""
    m, k, n = 4096, 128, 512
    A, B = _moved_case(oracle, m, k, n, np.float64)
    A[m - 3, :] = 0.0
    with pytest.raises(oz.DomainError) as e1:
        _call(mode, A, B, 14)
    with pytest.raises(oz.DomainError) as e0:
        _unspeculated(A, B, 14)
    assert str(e1.value) == str(e0.value)
    # the workspace is usable afterwards
    A2, B2 = _moved_case(oracle, m, k, n, np.float64)
    assert _call(mode, A2, B2, 14).speculation == 2


@pytest.mark.gpu
@pytest.mark.parametrize("mode,expect", [("1", 3), ("2", 2)])
def test_speculation_moved_with_flag(cuda, oracle, mode, expect):
    """The first row chunk's C is subnormal, so its first CRT raises the
    subnormal flag with exponents that later move."""
    m, k, n = 4096, 128, 512
    A, B = _moved_case(oracle, m, k, n, np.float64)
    A[:64] *= 1e-300
    B *= 1e-12
    r = _call(mode, A, B, 14)
    assert r.speculation == expect and r.subnormal
    ref = oracle.os_ii(A, B, 14)
    _same(r.C, ref.C)
    assert ref.subnormal


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("phi,seed", [(0.0, 11), (1.0, 12), (4.0, 13)])
def test_speculation_random(cuda, oracle, mode, phi, seed):
    """Reference-generator inputs at a small k, where later chunks often move
    some exponents; ragged chunk edges (m, n not multiples of the chunk)."""
    m, k, n = 2304, 96, 1100
    A = oracle.gen_matrix(m, k, phi, seed)
    B = oracle.gen_matrix(k, n, phi, seed + 100)
    r = _call(mode, A, B, 12, vectors=True)
    assert r.speculation in (1, 2, 3)
    r0 = _unspeculated(A, B, 12, vectors=True)
    _same(r.C, r0.C)
    _same(r.C, oracle.os_ii(A, B, 12).C)
    for nm in ("mu", "nu", "e", "f"):
        assert np.array_equal(getattr(r.scaling, nm), getattr(r0.scaling, nm)), nm


@pytest.mark.gpu
@pytest.mark.parametrize("tail", [2, 3])
@pytest.mark.parametrize("case", ["moved", "random", "flag"])
def test_speculation_tail_halvings(cuda, oracle, tail, case):
    """Option "spec_tail": the last column chunks halve 2 or 3 times (chunks
    shorter than the default unit, so the per-unit statuses and moved flags
    use the finer unit); C, exponents and flags equal the unspeculated call."""
    if case == "random":
        m, k, n = 2304, 96, 4100
        A, B = oracle.gen_matrix(m, k, 1.0, 21), oracle.gen_matrix(k, n, 1.0, 22)
    else:
        m, k, n = 4096, 128, 4096
        A, B = _moved_case(oracle, m, k, n, np.float64)
        if case == "flag":
            A[:64] *= 1e-300
            B *= 1e-12
    with oz.options(spec_tail=tail):
        r = _call("2", A, B, 14, vectors=True)
    assert r.speculation in ((2,) if case != "random" else (1, 2))
    r0 = _unspeculated(A, B, 14, vectors=True)
    _same(r.C, r0.C)
    _same(r.C, oracle.os_ii(A, B, 14).C)
    assert r.subnormal == r0.subnormal == (case == "flag")
    for nm in ("mu", "nu", "e", "f"):
        assert np.array_equal(getattr(r.scaling, nm), getattr(r0.scaling, nm)), nm
