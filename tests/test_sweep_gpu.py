"""oz2g_gemm_sweep / os_ii_sweep: the N sweep of the paper's experiments
("C̄ maxima reused across N").  The scaling scans and the
clearance product are computed once; every C must equal the per-N call bit
for bit (and the oracle's)."""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n,phi,dt,ns", [
    (130, 300, 97, 2.0, np.float64, [8, 12, 16, 20]),
    (2304, 64, 300, 0.5, np.float64, [14, 16]),
    (120, 200, 80, 1.0, np.float32, [6, 8, 16]),
])
def test_sweep_equals_per_n(cuda, oracle, m, k, n, phi, dt, ns):
    import torch
    A = oracle.gen_matrix(m, k, phi, 1100 + m).astype(dt)
    B = oracle.gen_matrix(k, n, phi, 1200 + n).astype(dt)
    host = oz.os_ii_sweep(A, B, ns)
    devc = oz.os_ii_sweep(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), ns)
    for N, h, d in zip(ns, host, devc):
        ref = oz.os_ii(A, B, N).C
        assert np.array_equal(h.view(np.uint8), ref.view(np.uint8)), N
        assert np.array_equal(d.cpu().numpy().view(np.uint8), ref.view(np.uint8)), N
        if dt == np.float64 and m * k < 100000:
            assert np.array_equal(h.view(np.uint64), oracle.os_ii(A, B, N).C.view(np.uint64))


def test_sweep_rejects_bad_n_before_work(cuda):
    A = np.ones((8, 8))
    with pytest.raises(oz.DomainError):
        oz.os_ii_sweep(A, A, [8, 50])
    with pytest.raises(oz.DomainError, match="zero row"):
        Z = A.copy(); Z[3] = 0.0
        oz.os_ii_sweep(Z, A, [8, 12])
