"""OZ2G_ASYNC (os_ii(..., blocking=False) + synchronize()): calls are enqueued
and complete later; the next call's uploads overlap the previous call's
residue GEMMs.  Every result must still be bit-exact, the uploads of call
i + 1 must not overwrite inputs call i still reads, and failures surface at
synchronize() in call order."""
import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


@pytest.mark.parametrize("m,k,n", [(70, 90, 50), (2304, 96, 300)])  # small, and the pipelined host path
def test_async_calls_bit_exact(cuda, oracle, m, k, n):
    cases = [(oracle.gen_matrix(m, k, 1.0, 900 + i), oracle.gen_matrix(k, n, 1.0, 950 + i)) for i in range(4)]
    refs = [oracle.os_ii(a, b, 14).C for a, b in cases]
    ins = [(_pinned(a), _pinned(b)) for a, b in cases]
    outs = [_pinned(np.zeros((m, n))) for _ in cases]
    for (a, b), c in zip(ins, outs):
        oz.os_ii(a, b, 14, out=c, blocking=False)
    oz.synchronize()
    for c, ref in zip(outs, refs):
        assert np.array_equal(c.view(np.uint64), ref.view(np.uint64))


def test_async_device_pointers(cuda, oracle):
    import torch
    A = oracle.gen_matrix(300, 200, 2.0, 961)
    B = oracle.gen_matrix(200, 260, 2.0, 962)
    ref = oracle.os_ii(A, B, 16).C
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    outs = [torch.empty((300, 260), dtype=torch.float64, device="cuda") for _ in range(3)]
    for c in outs:
        oz.os_ii(dA, dB, 16, out=c, blocking=False)
    oz.synchronize()
    for c in outs:
        assert np.array_equal(c.cpu().numpy().view(np.uint64), ref.view(np.uint64))


def test_async_errors_in_call_order(cuda, oracle):
    good_a, good_b = oracle.gen_matrix(40, 30, 1.0, 971), oracle.gen_matrix(30, 20, 1.0, 972)
    bad1 = good_a.copy(); bad1[7, :] = 0.0                 # zero row 7
    bad2 = good_a.copy(); bad2[3, 3] = np.inf              # not finite
    ref = oracle.os_ii(good_a, good_b, 12).C
    outs = [_pinned(np.zeros((40, 20))) for _ in range(4)]
    ins = [(_pinned(good_a), _pinned(good_b)), (_pinned(bad1), _pinned(good_b)),
           (_pinned(bad2), _pinned(good_b)), (_pinned(good_a), _pinned(good_b))]
    for (a, b), c in zip(ins, outs):
        oz.os_ii(a, b, 12, out=c, blocking=False)
    with pytest.raises(oz.DomainError, match="zero row 7"):
        oz.synchronize()
    oz.synchronize()  # nothing pending any more
    for i in (0, 3):  # the good calls still produced their C
        assert np.array_equal(outs[i].view(np.uint64), ref.view(np.uint64))
    # a blocking call completes pending async calls first (and reports their failure)
    oz.os_ii(_pinned(bad2), _pinned(good_b), 12, out=outs[1], blocking=False)
    with pytest.raises(oz.DomainError, match="not finite"):
        oz.os_ii(good_a, good_b, 12)
    assert np.array_equal(oz.os_ii(good_a, good_b, 12).C.view(np.uint64), ref.view(np.uint64))


def test_async_rejects_intermediates(cuda):
    A = np.ones((4, 4))
    for kw in ({"keep_intermediates": True}, {"bounds": True}, {"timing": True}, {"devices": [0]}):
        with pytest.raises(oz.InvalidArgument):
            oz.os_ii(A, A, 8, blocking=False, **kw)


def test_async_device_graph_replays(cuda, oracle):
    """Asynchronous device-pointer calls replay the captured graph too (plain,
    capture, replays); each replay's status lands in its own ring slot, so
    a failing replay among good ones is reported at synchronize() in order,
    and contents changed between enqueued calls are read by each call."""
    import torch
    m, k, n = 256, 300, 180
    A1 = oracle.gen_matrix(m, k, 1.0, 981)
    A2 = oracle.gen_matrix(m, k, 2.0, 982)
    B = oracle.gen_matrix(k, n, 1.0, 983)
    bad = A1.copy()
    bad[9, :] = 0.0
    r1, r2 = oracle.os_ii(A1, B, 14).C, oracle.os_ii(A2, B, 14).C
    dA, dB = torch.empty((m, k), dtype=torch.float64, device="cuda"), torch.from_numpy(B).cuda()
    out = torch.empty((m, n), dtype=torch.float64, device="cuda")
    seq = [A1, A2, A1, A2, A1, bad, A2, A1]
    res = []
    for x in seq:  # same addresses every call: call 1 plain, 2 captures, 3+ replay
        dA.copy_(torch.from_numpy(x))
        oz.os_ii(dA, dB, 14, out=out, blocking=False)
        res.append(out.clone())  # stream-ordered after the call
    with pytest.raises(oz.DomainError, match="zero row 9"):
        oz.synchronize()
    torch.cuda.synchronize()
    for i, (x, c) in enumerate(zip(seq, res)):
        if x is bad:
            continue
        ref = r1 if x is A1 else r2
        assert np.array_equal(c.cpu().numpy().view(np.uint64), ref.view(np.uint64)), i
    # many replays: the status ring wraps (completes the oldest calls itself)
    dA.copy_(torch.from_numpy(A2))
    for _ in range(150):
        oz.os_ii(dA, dB, 14, out=out, blocking=False)
    oz.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), r2.view(np.uint64))
