"""The alternative residue-GEMM kernels (gemm_tc.cu), selected per process by
OZ2G_GEMM: "pair" (CTA-pair cta_group::2, 256x256 tiles) and "mcast" (2-CTA
clusters sharing a TMA-multicast B tile), with and without the unit fence
(OZ2G_GEMM_FENCE), and the fused kernel's single-CTA / unfenced forms.  Each runs in a subprocess (the
variant is read once per process) and must reproduce the oracle bit for bit:
the wrapped INT32 products and W of every plane, and C — on shapes with
ragged tile edges, several 2048-row blocks, and fp32 mode."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2602_02549_b200 as oz
from oracle import oracle as O
O.set_threads(16)
cases = [(300, 1024, 520, 1.0, 14, np.float64), (129, 200, 257, 0.5, 8, np.float32),
         (2304, 256, 640, 2.0, 16, np.float64)]
for m, k, n, phi, N, dt in cases:
    A = O.gen_matrix(m, k, phi, O.derive_seed(m, 1, 0), dt)
    B = O.gen_matrix(k, n, phi, O.derive_seed(m, 1, 1), dt)
    ref = O.os_ii(A, B, N, keep_intermediates=True, residues=True)
    got = oz.os_ii(A, B, N, keep_intermediates=True, evidence=True)
    assert np.array_equal(got.crt.Cprod, ref.inter["Cprod"]), ("Cprod", m, k, n)
    assert np.array_equal(got.crt.W, ref.inter["W"]), ("W", m, k, n)
    bits = np.uint64 if dt == np.float64 else np.uint32
    assert np.array_equal(got.C.view(bits), ref.C.view(bits)), ("C", m, k, n)
    plain = oz.os_ii(A, B, N)  # the per-block W path without intermediates
    assert np.array_equal(plain.C.view(bits), ref.C.view(bits)), ("C plain", m, k, n)
    import torch
    for _ in range(3):  # device pointers: plain call, graph capture, replay
        dC = oz.os_ii(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), N).C.cpu().numpy()
        assert np.array_equal(dC.view(bits), ref.C.view(bits)), ("C device", m, k, n)
print("variant ok")
'''


VARIANTS = {
    "pair": {"OZ2G_GEMM": "pair"},
    "mcast": {"OZ2G_GEMM": "mcast"},
    "pair6-fence": {"OZ2G_GEMM": "pair", "OZ2G_PAIR_STAGES": "6", "OZ2G_GEMM_FENCE": "1"},
    "single-fence": {"OZ2G_GEMM_FENCE": "1"},
    # the fused residue-GEMM + CRT kernel without its B multicast / plane fence
    "fused-mc": {"OZ2G_FUSED": "1", "OZ2G_FUSED_MC": "1"},
    "fused-no-fence": {"OZ2G_FUSED": "1", "OZ2G_FUSED_FENCE": "0"},
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_gemm_variant_bit_exact(cuda, variant):
    env = dict(os.environ, **VARIANTS[variant])
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
