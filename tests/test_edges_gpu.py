"""Edge cases of the device path, bit for bit against the oracle:
strided operands (lda > k, ldb > n, ldc > n), subnormal outputs (the two
roundings of inverse_scale, emulate.hpp:37-42, and the subnormal flag), the
largest inner dimension k = 2^17 (int8gemm.hpp:12; INT32 wrap and the 2^29
clearance ceiling), vector shapes, sparse rows and extreme magnitudes."""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), np.argwhere(a != b)[:5]


def test_strided_device_operands(cuda, oracle):
    import torch
    m, k, n = 70, 150, 90
    A = oracle.gen_matrix(m, k, 1.0, 91)
    B = oracle.gen_matrix(k, n, 1.0, 92)
    ref = oracle.os_ii(A, B, 14)
    Abig = torch.zeros((m, k + 37), dtype=torch.float64, device="cuda")
    Bbig = torch.zeros((k, n + 11), dtype=torch.float64, device="cuda")
    Cbig = torch.full((m, n + 5), 7.0, dtype=torch.float64, device="cuda")
    Abig[:, :k] = torch.from_numpy(A).cuda()
    Bbig[:, :n] = torch.from_numpy(B).cuda()
    C = Cbig[:, :n]
    oz.os_ii(Abig[:, :k], Bbig[:, :n], 14, out=C)
    _same(C.cpu().numpy(), ref.C)
    assert bool((Cbig[:, n:] == 7.0).all())  # padding columns untouched


def test_strided_host_operands_via_c_abi(cuda, oracle):
    import ctypes as C
    from paper_2602_02549_b200 import _lib
    m, k, n = 40, 64, 50
    A = oracle.gen_matrix(m, k, 0.5, 93)
    B = oracle.gen_matrix(k, n, 0.5, 94)
    ref = oracle.os_ii(A, B, 12)
    Ap = np.zeros((m, k + 3)); Ap[:, :k] = A
    Bp = np.zeros((k, n + 9)); Bp[:, :n] = B
    Cp = np.full((m, n + 2), -1.0)
    rc = _lib.load().oz2g_dgemm(m, n, k, Ap.ctypes.data, k + 3, Bp.ctypes.data, n + 9, Cp.ctypes.data, n + 2,
                                12, 0, None, None)
    assert rc == 0, _lib.load().oz2g_last_error()
    _same(np.ascontiguousarray(Cp[:, :n]), ref.C)
    assert (Cp[:, n:] == -1.0).all()


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_strided_host_operands_pipelined(cuda, oracle, mode):
    """The pipelined host path (chunked uploads, per-block / per-tile
    downloads) with leading dimensions larger than the matrices, for every
    speculation mode (OZ2G_SPEC): C bit-exact, the padding never written."""
    import os
    from paper_2602_02549_b200 import _lib
    m, k, n = 2304, 96, 1100
    A = oracle.gen_matrix(m, k, 0.5, 95)
    B = oracle.gen_matrix(k, n, 0.5, 96)
    ref = oracle.os_ii(A, B, 12)
    Ap = np.zeros((m, k + 5)); Ap[:, :k] = A
    Bp = np.zeros((k, n + 13)); Bp[:, :n] = B
    Cp = np.full((m, n + 3), -1.0)
    with oz.options(spec=int(mode)):
        rc = _lib.load().oz2g_dgemm(m, n, k, Ap.ctypes.data, k + 5, Bp.ctypes.data, n + 13, Cp.ctypes.data, n + 3,
                                    12, 0, None, None)
    assert rc == 0, _lib.load().oz2g_last_error()
    _same(np.ascontiguousarray(Cp[:, :n]), ref.C)
    assert (Cp[:, n:] == -1.0).all()


@pytest.mark.parametrize("scale,dt", [(1e-160, np.float64), (1e-155, np.float64), (1e-21, np.float32)])
def test_subnormal_outputs(cuda, oracle, scale, dt):
    A = (oracle.gen_matrix(24, 40, 1.0, 95) * scale).astype(dt)
    B = (oracle.gen_matrix(40, 30, 1.0, 96) * scale).astype(dt)
    ref = oracle.os_ii(A, B, 14 if dt == np.float64 else 8)
    got = oz.os_ii(A, B, 14 if dt == np.float64 else 8)
    _same(got.C, ref.C)
    assert got.subnormal == ref.subnormal
    assert got.subnormal  # these scales do produce subnormal entries


def test_max_inner_dimension(cuda, oracle):
    k = 1 << 17
    A = oracle.gen_matrix(5, k, 0.0, 97)
    B = oracle.gen_matrix(k, 3, 0.0, 98)
    # entries just below a power of two scale to Abar = Bbar = 64, so C̄[0, 0]
    # reaches the clearance ceiling 64 * 64 * 2^17 = 2^29
    A[0, :] = 0.9999999
    B[:, 0] = -0.9999999
    ref = oracle.os_ii(A, B, 16, want_cmax=True)
    got = oz.os_ii(A, B, 16, vectors=True)
    _same(got.C, ref.C)
    assert int(got.scaling.cmax_row[0]) == int(ref.inter["cmax_row"][0]) == 1 << 29
    with pytest.raises(oz.DomainError):
        oz.os_ii(np.ones((2, k + 1)), np.ones((k + 1, 2)), 16)


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (1, 300, 1), (1, 64, 200), (200, 64, 1), (300, 1, 200)])
def test_vector_shapes(cuda, oracle, m, k, n):
    A = oracle.gen_matrix(m, k, 2.0, 99 + m)
    B = oracle.gen_matrix(k, n, 2.0, 199 + n)
    _same(oz.os_ii(A, B, 14).C, oracle.os_ii(A, B, 14).C)


def test_sparse_and_extreme_entries(cuda, oracle):
    rng = np.random.default_rng(5)
    A = oracle.gen_matrix(60, 90, 1.0, 301)
    B = oracle.gen_matrix(90, 45, 1.0, 302)
    A[rng.random(A.shape) < 0.7] = 0.0        # sparse rows (never fully zero: column 0 kept)
    A[:, 0] = 1.0
    B[rng.random(B.shape) < 0.5] = 0.0
    B[0, :] = -2.0
    A[3, 5] = 1e300; A[4, 6] = 5e-324        # largest magnitudes and a subnormal input
    B[7, 2] = 1e-300; B[8, 3] = -1.7e308
    for N in (8, 16, 30):
        try:
            ref = oracle.os_ii(A, B, N)
        except Exception as e:  # noqa: BLE001 - the device must raise the same
            with pytest.raises(Exception) as got:
                oz.os_ii(A, B, N)
            assert str(got.value) == str(e)
            continue
        _same(oz.os_ii(A, B, N).C, ref.C)
