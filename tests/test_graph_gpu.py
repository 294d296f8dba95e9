"""Device-pointer calls replayed as a CUDA graph (api.cu run_gemm_graph): the
first call runs plainly, the second captures the pipeline, later calls
replay it.  Every replay must equal the oracle bit for bit, read the inputs'
current contents, report errors from the status word like a plain call, and
be invalidated when a workspace buffer is reallocated."""

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


def test_graph_replays_bit_exact(cuda, oracle):
    import torch
    A = oracle.gen_matrix(300, 257, 1.0, 51)
    B = oracle.gen_matrix(257, 190, 1.0, 52)
    ref = oracle.os_ii(A, B, 14).C
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty((300, 190), dtype=torch.float64, device="cuda")
    for i in range(4):  # plain, capture + replay, replay, replay
        out.zero_()
        r = oz.os_ii(dA, dB, 14, out=out)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64)), i
        assert r.kernels_launched > 0
    # new contents at the same addresses: the replay reads them
    A2 = oracle.gen_matrix(300, 257, 2.0, 53)
    dA.copy_(torch.from_numpy(A2))
    oz.os_ii(dA, dB, 14, out=out)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle.os_ii(A2, B, 14).C.view(np.uint64))
    # an error raised by a replay, with the reference's message
    bad = A2.copy()
    bad[17, :] = 0.0
    dA.copy_(torch.from_numpy(bad))
    with pytest.raises(oz.DomainError, match="zero row 17"):
        oz.os_ii(dA, dB, 14, out=out)
    # a larger call reallocates the workspace; the graph is re-captured
    big = oracle.gen_matrix(700, 257, 1.0, 54)
    oz.os_ii(torch.from_numpy(big).cuda(), dB, 14)
    dA.copy_(torch.from_numpy(A))
    for _ in range(3):
        oz.os_ii(dA, dB, 14, out=out)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))


def test_graph_subnormal_flag_and_fp32(cuda, oracle):
    import torch
    A = oracle.gen_matrix(64, 48, 1.0, 61) * 1e-160
    B = oracle.gen_matrix(48, 40, 1.0, 62) * 1e-160
    ref = oracle.os_ii(A, B, 14)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty((64, 40), dtype=torch.float64, device="cuda")
    for _ in range(3):
        r = oz.os_ii(dA, dB, 14, out=out)
        assert r.subnormal == ref.subnormal and ref.subnormal
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.C.view(np.uint64))
    A32 = oracle.gen_matrix(96, 80, 0.5, 63, np.float32)
    B32 = oracle.gen_matrix(80, 72, 0.5, 64, np.float32)
    ref32 = oracle.os_ii(A32, B32, 8).C
    d32a, d32b = torch.from_numpy(A32).cuda(), torch.from_numpy(B32).cuda()
    for _ in range(3):
        c = oz.os_ii(d32a, d32b, 8).C  # fresh output each call: a new key, plain + capture paths
        assert np.array_equal(c.cpu().numpy().view(np.uint32), ref32.view(np.uint32))


def test_graph_disabled_matches(cuda, oracle):
    import torch
    A = oracle.gen_matrix(130, 70, 1.0, 71)
    B = oracle.gen_matrix(70, 90, 1.0, 72)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    with oz.options(graph=0):
        plain = oz.os_ii(dA, dB, 12).C.clone()
    out = torch.empty_like(plain)
    for _ in range(3):
        oz.os_ii(dA, dB, 12, out=out)
    assert torch.equal(out.view(torch.int64), plain.view(torch.int64))


def test_set_option_recaptures(cuda, oracle):
    """oz2g_set_option invalidates the captured graphs: a replayed call picks
    up the new choice (the fused kernel launches fewer kernels) with the same C."""
    import torch
    A = oracle.gen_matrix(200, 160, 1.0, 81)
    B = oracle.gen_matrix(160, 140, 1.0, 82)
    ref = oracle.os_ii(A, B, 14).C
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty((200, 140), dtype=torch.float64, device="cuda")
    with oz.options(fused=0):
        two = [oz.os_ii(dA, dB, 14, out=out).kernels_launched for _ in range(4)]
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))
    with oz.options(fused=1):
        one = [oz.os_ii(dA, dB, 14, out=out).kernels_launched for _ in range(4)]
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))
    assert len(set(two)) == 1 and len(set(one)) == 1 and one[0] < two[0], (two, one)
