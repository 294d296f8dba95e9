"""Speculative column exponents on the pipelined host-pointer path (api.cu
run_gemm).  nu_j (scaling.hpp:159-194) needs the clearance maxima of column j
over every row of A; the pipelined call takes it from the first uploaded row
chunk, runs the B residues and every residue GEMM + CRT while the rest of A is
still uploading, and checks the final nu against the speculated one.  C must
be the unspeculated C bit for bit in both outcomes:
  * confirmed (typical inputs): speculation == 1;
  * moved (a later chunk raises column maxima across a step threshold):
    speculation == 2, the B residues and the moved 256-column tiles of the
    blocks already computed are redone;
  * moved, and a block computed with the superseded exponents raised a status
    flag (subnormal output): speculation == 3, every stage after the upload is
    redone unspeculated."""
import os

import numpy as np
import pytest

import paper_2602_02549_b200 as oz


def _same(a, b):
    assert a.dtype == b.dtype and a.shape == b.shape
    assert np.array_equal(a.view(np.uint64 if a.dtype == np.float64 else np.uint32),
                          b.view(np.uint64 if b.dtype == np.float64 else np.uint32))


def _unspeculated(A, B, nmod, **kw):
    os.environ["OZ2G_SPEC"] = "0"
    try:
        r = oz.os_ii(A, B, nmod, **kw)
    finally:
        del os.environ["OZ2G_SPEC"]
    assert r.speculation == 0
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_speculation_confirmed(cuda, oracle, dtype):
    """Every row chunk of A holds the same rows, so the first chunk's column
    maxima are the final ones."""
    m, k, n = 4096, 128, 512
    A = np.tile(oracle.gen_matrix(512, k, 0.0, 901), (m // 512, 1)).astype(dtype)
    B = oracle.gen_matrix(k, n, 0.0, 902).astype(dtype)
    nmod = 14 if dtype == np.float64 else 7
    r = oz.os_ii(A, B, nmod, vectors=True)
    assert r.speculation == 1
    r0 = _unspeculated(A, B, nmod, vectors=True)
    _same(r.C, r0.C)
    _same(r.C, oracle.os_ii(A, B, nmod).C)
    # the returned scaling vectors are the final ones (f from the complete maxima)
    for nm in ("mu", "nu", "e", "f", "cmax_col"):
        assert np.array_equal(getattr(r.scaling, nm), getattr(r0.scaling, nm)), nm


def _miss_case(oracle, m, k, n, dtype):
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
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_speculation_missed(cuda, oracle, dtype):
    m, k, n = 4096, 128, 512
    A, B = _miss_case(oracle, m, k, n, dtype)
    nmod = 14 if dtype == np.float64 else 7
    r = oz.os_ii(A, B, nmod, vectors=True)
    assert r.speculation == 2
    r0 = _unspeculated(A, B, nmod)
    assert not r.subnormal and not r0.subnormal
    _same(r.C, r0.C)
    _same(r.C, oracle.os_ii(A, B, nmod).C)
    assert np.array_equal(r.scaling.nu, oracle.os_ii(A, B, nmod, keep_intermediates=True).inter["nu"])


@pytest.mark.gpu
def test_speculation_missed_then_error(cuda, oracle):
    """A missed speculation whose redo raises: the redo reports the error the
    unspeculated call reports."""
    m, k, n = 4096, 128, 512
    A, B = _miss_case(oracle, m, k, n, np.float64)
    A[m - 3, :] = 0.0
    with pytest.raises(oz.DomainError) as e1:
        oz.os_ii(A, B, 14)
    os.environ["OZ2G_SPEC"] = "0"
    try:
        with pytest.raises(oz.DomainError) as e0:
            oz.os_ii(A, B, 14)
    finally:
        del os.environ["OZ2G_SPEC"]
    assert str(e1.value) == str(e0.value)
    # the workspace is usable afterwards
    A2, B2 = _miss_case(oracle, m, k, n, np.float64)
    assert oz.os_ii(A2, B2, 14).speculation == 2


@pytest.mark.gpu
def test_speculation_moved_with_flag_redone(cuda, oracle):
    m, k, n = 4096, 128, 512
    A, B = _miss_case(oracle, m, k, n, np.float64)
    A[:64] *= 1e-300   # first-chunk rows of C are subnormal: the first CRT of block 0 flags it
    B *= 1e-12
    r = oz.os_ii(A, B, 14)
    assert r.speculation == 3 and r.subnormal
    ref = oracle.os_ii(A, B, 14)
    _same(r.C, ref.C)
    assert ref.subnormal


@pytest.mark.gpu
@pytest.mark.parametrize("phi,seed", [(0.0, 11), (1.0, 12), (4.0, 13)])
def test_speculation_random(cuda, oracle, phi, seed):
    """Reference-generator inputs at a small k, where the maxima of later
    chunks often move some column exponents: whatever the outcome, C is the
    unspeculated C."""
    m, k, n = 2304, 96, 700
    A = oracle.gen_matrix(m, k, phi, seed)
    B = oracle.gen_matrix(k, n, phi, seed + 100)
    r = oz.os_ii(A, B, 12)
    assert r.speculation in (1, 2, 3)
    _same(r.C, _unspeculated(A, B, 12).C)
    _same(r.C, oracle.os_ii(A, B, 12).C)
