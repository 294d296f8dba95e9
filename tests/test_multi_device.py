"""oz2g_gemm_multi: one emulated GEMM tiled over several devices of one
process.  On this one-GPU pool the device list repeats device 0:
every tile still has its own workspace, stream and host thread, and the
clearance maxima still cross tiles through the host exchange, so the tiling
and the exchange are exercised on real kernels (the tiles' kernels never wait
on one another, so sharing one GPU changes only the timing)."""
import ctypes as C

import numpy as np
import pytest

import paper_2602_02549_b200 as oz
from paper_2602_02549_b200 import _lib
from paper_2602_02549_b200 import dist as pdist


def test_grid_shape_matches_dist():
    L = _lib.load()
    for count in range(1, 17):
        r, c = C.c_int(), C.c_int()
        assert L.oz2g_grid_shape(count, C.byref(r), C.byref(c)) == 0
        assert (r.value, c.value) == pdist.grid_shape(count)


@pytest.mark.gpu
@pytest.mark.parametrize("count", [1, 2, 4, 8])
@pytest.mark.parametrize("m,k,n,phi,dt", [(96, 200, 80, 1.0, np.float64), (3, 64, 17, 0.0, np.float64),
                                          (257, 130, 300, 2.0, np.float64), (64, 96, 72, 0.5, np.float32)])
def test_tiled_equals_single(cuda, oracle, count, m, k, n, phi, dt):
    A = oracle.gen_matrix(m, k, phi, 81).astype(dt)
    B = oracle.gen_matrix(k, n, phi, 82).astype(dt)
    N = 12 if dt == np.float64 else 8
    single = oz.os_ii(A, B, N).C
    tiled = oz.os_ii(A, B, N, devices=[0] * count).C
    assert np.array_equal(tiled.view(np.uint8), single.view(np.uint8))
    if dt == np.float64:
        assert np.array_equal(tiled.view(np.uint64), oracle.os_ii(A, B, N).C.view(np.uint64))


@pytest.mark.gpu
def test_tiled_errors_match_single(cuda, oracle):
    m, k, n = 130, 40, 90
    A = oracle.gen_matrix(m, k, 1.0, 83)
    B = oracle.gen_matrix(k, n, 1.0, 84)
    cases = []
    a = A.copy(); a[100, :] = 0.0          # zero row in grid row 1
    b = B.copy(); b[:, 3] = 0.0            # zero column in grid column 0
    cases.append((a, b))                   # -> the row is reported (A is checked first)
    b = B.copy(); b[:, 80] = 0.0           # zero column in the last grid column (global index)
    cases.append((A, b))
    a = A.copy(); a[120, 7] = np.nan
    cases.append((a, B))
    cases.append((A * 1e200, B * 1e200))   # inverse-scaling overflow
    for a, b in cases:
        with pytest.raises(Exception) as ref:
            oz.os_ii(a, b, 14)
        for count in (2, 4, 8):
            with pytest.raises(type(ref.value)) as got:
                oz.os_ii(a, b, 14, devices=[0] * count)
            assert str(got.value) == str(ref.value)
    # still usable afterwards
    assert np.array_equal(oz.os_ii(A, B, 14, devices=[0, 0, 0, 0]).C, oz.os_ii(A, B, 14).C)


@pytest.mark.gpu
def test_multi_argument_checks(cuda):
    import torch
    A = np.ones((4, 4))
    with pytest.raises(oz.InvalidArgument):
        oz.os_ii(A, A, 8, devices=[])
    with pytest.raises(oz.InvalidArgument):
        oz.os_ii(A, A, 8, devices=[torch.cuda.device_count()])
    with pytest.raises(oz.InvalidArgument):
        oz.os_ii(torch.ones((4, 4), dtype=torch.float64, device="cuda"),
                 torch.ones((4, 4), dtype=torch.float64, device="cuda"), 8, devices=[0])
    with pytest.raises(oz.DomainError):
        oz.os_ii(A, A, 50, devices=[0, 0])
    L = _lib.load()
    ds = (C.c_int * 1)(0)
    assert L.oz2g_init(ds, 1) == 0
