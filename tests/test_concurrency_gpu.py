"""Calls from several host threads at once (the reference's os_ii is reentrant,
SPEC.md:434 per SURVEY §8b): device-pointer calls on private streams and
host-pointer calls, interleaved, on one device; every result bit-exact."""
import threading

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu


def test_concurrent_calls_one_device(cuda, oracle):
    import torch
    cases = [(oracle.gen_matrix(64 + 7 * i, 96, 1.0, 500 + i), oracle.gen_matrix(96, 48 + 5 * i, 1.0, 600 + i))
             for i in range(6)]
    refs = [oracle.os_ii(a, b, 12).C for a, b in cases]
    results = [None] * len(cases)
    errors = []

    def work(i):
        try:
            a, b = cases[i]
            if i % 2:
                for _ in range(3):
                    results[i] = oz.os_ii(a, b, 12).C
            else:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
                    for _ in range(3):
                        c = oz.os_ii(da, db, 12, stream=s.cuda_stream).C
                    s.synchronize()
                    results[i] = c.cpu().numpy()
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append((i, e))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for got, ref in zip(results, refs):
        assert np.array_equal(np.asarray(got).view(np.uint64), ref.view(np.uint64))


def test_concurrent_pipelined_calls(cuda, oracle):
    """Host-pointer calls large enough for the pipelined, speculated path
    (chunked uploads, exponent checks through mapped memory) from several
    threads at once, beside device-pointer calls."""
    import torch
    shapes = [(2304, 96, 1100), (2560, 64, 700), (2048, 128, 512)]
    cases = [(oracle.gen_matrix(m, k, 0.5, 700 + i), oracle.gen_matrix(k, n, 0.5, 800 + i))
             for i, (m, k, n) in enumerate(shapes)]
    refs = [oracle.os_ii(a, b, 12).C for a, b in cases]
    results = [[] for _ in range(4)]
    errors = []

    def work(t):
        try:
            for rep in range(2):
                i = (t + rep) % len(cases)
                a, b = cases[i]
                if t == 3:  # device pointers on a private stream
                    s = torch.cuda.Stream()
                    with torch.cuda.stream(s):
                        c = oz.os_ii(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 12,
                                     stream=s.cuda_stream).C
                        s.synchronize()
                    results[t].append((i, c.cpu().numpy()))
                else:
                    results[t].append((i, oz.os_ii(a, b, 12).C))
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append((t, e))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=600)
    assert not errors, errors
    for per_thread in results:
        assert len(per_thread) == 2
        for i, got in per_thread:
            assert np.array_equal(np.asarray(got).view(np.uint64), refs[i].view(np.uint64))


@pytest.mark.parametrize("explicit", [True, False])
def test_caller_stream_ordering(cuda, oracle, explicit):
    """Inputs produced on the caller's stream are consumed in order on it, and
    the result is ready on that stream when the call returns (the stream
    passed, or torch's current stream when none is)."""
    import torch
    A = oracle.gen_matrix(100, 80, 0.5, 701)
    B = oracle.gen_matrix(80, 60, 0.5, 702)
    ref = oracle.os_ii(A, B, 14).C
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        da = torch.empty((100, 80), dtype=torch.float64, device="cuda")
        db = torch.empty((80, 60), dtype=torch.float64, device="cuda")
        da.copy_(torch.from_numpy(A).pin_memory(), non_blocking=True)
        db.copy_(torch.from_numpy(B).pin_memory(), non_blocking=True)
        out = torch.empty((100, 60), dtype=torch.float64, device="cuda")
        oz.os_ii(da, db, 14, out=out, stream=s.cuda_stream if explicit else None)
        host = torch.empty((100, 60), dtype=torch.float64).pin_memory()
        host.copy_(out, non_blocking=True)
    s.synchronize()
    assert np.array_equal(host.numpy().view(np.uint64), ref.view(np.uint64))
