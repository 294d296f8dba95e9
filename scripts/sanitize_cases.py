"""Small os_ii calls covering the code paths, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02549_b200 as oz  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(1)
cases = [(7, 20, 6, 14, np.float64), (33, 129, 65, 16, np.float64), (130, 300, 257, 8, np.float32),
         (1, 1, 1, 2, np.float64), (3, 64, 17, 49, np.float64), (200, 64, 1, 12, np.float32)]
for m, k, n, N, dt in cases:
    A = O.gen_matrix(m, k, 1.0, 11 + m).astype(dt)
    B = O.gen_matrix(k, n, 1.0, 12 + n).astype(dt)
    ref = O.os_ii(A.astype(np.float64) if dt == np.float64 else A, B, N) if dt == np.float64 else None
    r = oz.os_ii(A, B, N, keep_intermediates=True, bounds="full")
    r2 = oz.os_ii(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), N, evidence=True)
    if ref is not None:
        assert np.array_equal(r.C.view(np.uint64), ref.C.view(np.uint64))
# strided device operands
Ab = torch.zeros((40, 77), dtype=torch.float64, device="cuda"); Ab[:, :64] = torch.rand(40, 64, dtype=torch.float64, device="cuda") - 0.5
Bb = torch.zeros((64, 50), dtype=torch.float64, device="cuda"); Bb[:, :33] = torch.rand(64, 33, dtype=torch.float64, device="cuda") - 0.5
oz.os_ii(Ab[:, :64], Bb[:, :33], 14)
# pipelined host path (m >= 2048, n >= 256) and the row-blocked CRT
A = O.gen_matrix(2304, 64, 0.5, 31); B = O.gen_matrix(64, 300, 0.5, 32)
oz.os_ii(A, B, 16)
oz.os_ii(A, B, 16, vectors=True)
# every speculation mode of the pipelined path, bit-identical to the device path
Ad = oz.os_ii(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 16).C
Ad = Ad.cpu().numpy() if hasattr(Ad, "cpu") else np.asarray(Ad)
for mode in (0, 1, 2):
    with oz.options(spec=mode):
        assert np.array_equal(oz.os_ii(A, B, 16).C.view(np.uint64), Ad.view(np.uint64)), mode
# asynchronous calls back to back
outs = [np.empty((A.shape[0], B.shape[1])) for _ in range(3)]
for c in outs:
    oz.os_ii(A, B, 16, out=c, blocking=False)
oz.synchronize()
for c in outs:
    assert np.array_equal(c.view(np.uint64), Ad.view(np.uint64))
# device-pointer graph replays (programmatic dependent launches at this size), blocking and asynchronous
dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
dC = torch.empty((A.shape[0], B.shape[1]), dtype=torch.float64, device="cuda")
for _ in range(3):
    oz.os_ii(dA, dB, 16, out=dC)
for _ in range(3):
    oz.os_ii(dA, dB, 16, out=dC, blocking=False)
oz.synchronize()
assert np.array_equal(dC.cpu().numpy().view(np.uint64), Ad.view(np.uint64))
# A residues streamed beside the residue GEMMs (three row blocks)
A3 = O.gen_matrix(4500, 64, 0.5, 41)
with oz.options(resid_stream=1):
    oz.os_ii(torch.from_numpy(A3).cuda(), torch.from_numpy(B).cuda(), 12)
# multi-device tiling (device listed twice)
oz.os_ii(A[:300], B, 12, devices=[0, 0])
# error paths
for bad in (np.zeros((5, 8)), np.full((5, 8), np.nan)):
    try:
        oz.os_ii(bad, np.ones((8, 4)), 8)
    except oz.DomainError:
        pass
print("sanitize cases done")
