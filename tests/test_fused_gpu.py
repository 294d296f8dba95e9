"""The fused residue-GEMM + CRT kernel (csrc/fused.cu, OZ2G_FUSED=1): the N
residue GEMMs with accumulate / compute_q / final_reduce / inverse_scale
(crt.hpp:91-150, emulate.hpp:30-46) in their epilogue, no W in HBM.  C must
equal the oracle and the two-pass path bit for bit: ragged tile edges, fp32
mode, many N, error flags, subnormal outputs and the BASELINE 16384^3 size."""

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


@pytest.fixture
def fused():
    with oz.options(fused=1):
        yield


CASES = [
    (7, 20, 6, 0.0, 2, np.float64),
    (33, 100, 65, 0.5, 14, np.float64),
    (130, 300, 260, 2.0, 16, np.float64),
    (200, 129, 300, 8.0, 20, np.float64),
    (300, 1024, 520, 1.0, 49, np.float64),
    (7, 20, 6, 0.0, 9, np.float32),
    (130, 300, 260, 2.0, 16, np.float32),
    (2304, 512, 640, 1.0, 14, np.float64),
]


@pytest.mark.parametrize("m,k,n,phi,N,dt", CASES)
def test_fused_bit_parity(cuda, oracle, fused, m, k, n, phi, N, dt):
    import torch
    A = oracle.gen_matrix(m, k, phi, oracle.derive_seed(m + 7, k, 0), dt)
    B = oracle.gen_matrix(k, n, phi, oracle.derive_seed(m + 7, k, 1), dt)
    ref = oracle.os_ii(A, B, N)
    got = oz.os_ii(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), N)
    bits = np.uint64 if dt == np.float64 else np.uint32
    C = got.C.cpu().numpy()
    bad = np.flatnonzero(C.view(bits) != ref.C.view(bits))
    assert bad.size == 0, f"{bad.size} entries differ, first {np.unravel_index(bad[0], C.shape)}"
    assert got.subnormal == ref.subnormal


def test_fused_flags(cuda, oracle, fused):
    """Inverse-scaling overflow and the fp32 final_reduce guard are raised from
    the fused epilogue as from the CRT pass (crt.hpp:144, emulate.hpp:39);
    subnormal outputs set the flag (emulate.hpp:41-42)."""
    import torch
    A = oracle.gen_matrix(64, 48, 1.0, 11)
    B = oracle.gen_matrix(48, 40, 1.0, 12)
    with pytest.raises(oz.RangeError):
        oz.os_ii(torch.from_numpy(A * 1e200).cuda(), torch.from_numpy(B * 1e200).cuda(), 14)
    with pytest.raises(oz.RangeError):
        oz.os_ii(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(B.astype(np.float32)).cuda(), 20)
    tiny_a, tiny_b = A * 1e-160, B * 1e-160
    ref = oracle.os_ii(tiny_a, tiny_b, 14)
    got = oz.os_ii(torch.from_numpy(tiny_a).cuda(), torch.from_numpy(tiny_b).cuda(), 14)
    assert np.array_equal(got.C.cpu().numpy().view(np.uint64), ref.C.view(np.uint64))
    assert got.subnormal == ref.subnormal and ref.subnormal


def test_fused_equals_two_pass_full_size(cuda):
    """BASELINE cfg4: 16384^3, N = 16 — the fused C is the two-pass C bit for bit."""
    import torch
    from test_fullsize_gpu import _gen
    dA, dB = _gen((16384, 16384), 0.0, 1234), _gen((16384, 16384), 0.0, 5678)
    with oz.options(fused=0):
        two = oz.os_ii(dA, dB, 16).C
    with oz.options(fused=1):
        one = oz.os_ii(dA, dB, 16).C
    torch.cuda.synchronize()
    assert torch.equal(one.view(torch.int64), two.view(torch.int64))
