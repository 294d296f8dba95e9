"""Row-blocked residue GEMM + CRT (W held per 2048-row block): every output
that the CRT writes per entry, and the per-row bound vectors it reads, must be
addressed from the block's first row.  Blocking normally starts at 2 GB of W;
a subprocess lowers the threshold (OZ2G_WBLOCK_MIN_MB=0) so a 4500-row problem
runs as three blocks, and its outputs are compared with the unblocked call and
the oracle: C, the cheap / tight bound matrices, and C1, C2, Q, C'' and the
wrapped INT32 products requested without W through the C ABI."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_2602_02549_b200 as oz
from paper_2602_02549_b200 import _lib
A = np.load("A.npy"); B = np.load("B.npy")
m, k = A.shape; n = B.shape[1]
r = oz.os_ii(A, B, 14, bounds="full")
np.save("C.npy", r.C); np.save("cheap.npy", r.bounds["cheap"]); np.save("tight.npy", r.bounds["tight"])
L = _lib.load()
it = _lib.Intermediates()
arrs = {nm: np.zeros((m, n)) for nm in ("C1", "C2", "Q", "Cpp64")}
for nm, a in arrs.items():
    setattr(it, nm, a.ctypes.data)
cprod = np.zeros((14, m, n), dtype=np.int32)
it.Cprod = cprod.ctypes.data
Cc = np.zeros((m, n)); diag = _lib.Diag()
rc = L.oz2g_gemm(_lib.OZ2G_FP64, m, n, k, A.ctypes.data, k, B.ctypes.data, n, Cc.ctypes.data, n, 14,
                 _lib.OZ2G_HOST_PTRS, None, C.byref(it), C.byref(diag), _lib.REDUCE_FN(), None)
assert rc == 0, L.oz2g_last_error()
np.save("C_abi.npy", Cc)
for nm, a in arrs.items():
    np.save(nm + ".npy", a)
np.save("Cprod.npy", cprod)
""".replace("ROOT", repr(ROOT))


@pytest.mark.gpu
def test_row_blocked_crt_outputs(cuda, oracle, tmp_path):
    m, k, n = 4500, 64, 130
    A = oracle.gen_matrix(m, k, 1.0, 801)
    B = oracle.gen_matrix(k, n, 1.0, 802)
    np.save(tmp_path / "A.npy", A)
    np.save(tmp_path / "B.npy", B)
    env = dict(os.environ, OZ2G_WBLOCK_MIN_MB="0")
    subprocess.run([sys.executable, "-c", SCRIPT], env=env, check=True, cwd=tmp_path, timeout=600)

    ref = oz.os_ii(A, B, 14, bounds="full")          # this process: one block
    ora = oracle.os_ii(A, B, 14, keep_intermediates=True)

    def same(a, b):
        assert np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))

    same(np.load(tmp_path / "C.npy"), ora.C)
    same(np.load(tmp_path / "C_abi.npy"), ora.C)
    same(np.load(tmp_path / "cheap.npy"), ref.bounds["cheap"])
    same(np.load(tmp_path / "tight.npy"), ref.bounds["tight"])
    for nm in ("C1", "C2", "Q", "Cpp64"):  # intermediates: equal values (+0.0 == -0.0, as in test_parity_gpu)
        assert np.array_equal(np.load(tmp_path / f"{nm}.npy"), ora.inter[nm]), nm
    # wrapped INT32 residue products of every block, against the unblocked evidence export
    ev = oz.os_ii(A[:, :], B, 14, evidence=True)
    assert np.array_equal(np.load(tmp_path / "Cprod.npy"), ev.crt.Cprod)


@pytest.mark.gpu
@pytest.mark.parametrize("dt,nmod", [(np.float64, 14), (np.float32, 7)])
def test_streamed_a_residues(cuda, oracle, dt, nmod):
    """Option "resid_stream": the A residues of row block b + 1 are split on
    the side stream beside block b's residue GEMMs (device pointers, three
    2048-row blocks); C and the bounds equal the oracle / the default path."""
    import torch
    m, k, n = 4500, 300, 200
    A = oracle.gen_matrix(m, k, 1.0, 811).astype(dt)
    B = oracle.gen_matrix(k, n, 1.0, 812).astype(dt)
    ref = oracle.os_ii(A, B, nmod).C
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    base = oz.os_ii(dA, dB, nmod, bounds="full")
    with oz.options(resid_stream=1):
        for _ in range(3):  # plain, captured, replayed
            r = oz.os_ii(dA, dB, nmod, bounds="full")
            got = r.C.cpu().numpy()
            assert np.array_equal(got.view(np.uint64 if dt == np.float64 else np.uint32),
                                  ref.view(np.uint64 if dt == np.float64 else np.uint32))
        assert torch.equal(r.bounds["tight"], base.bounds["tight"])
        assert r.kernels_launched > base.kernels_launched  # three blocks, three A splits
