"""Interleaved A/B of a tuning option (oz2g_set_option) on device-resident
inputs: per shape, the values take turns (rounds x reps calls each, CUDA
events around each value's calls), and every value's C must equal the
first value's bit for bit.  One JSON line per shape.

    python scripts/option_ab.py resid_stream 0,1 16384x16384x16384x16 8192x16384x4096x16 [--rounds 3]
    python scripts/option_ab.py spec_tail 1,2,3 16384x16384x16384x16 --host   # end to end (pinned host
                                                                               # buffers, wall clock)
    python scripts/option_ab.py gemm+pair_stages+gemm_fence 0:4:0,1:6:1 16384x16384x16384x16   # option sets
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("option")
    ap.add_argument("values")
    ap.add_argument("shapes", nargs="+", help="m x k x n x N")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--host", action="store_true", help="pinned host buffers (copies inside), wall clock")
    a = ap.parse_args()
    import torch

    import paper_2602_02549_b200 as oz
    from bench import gen_device
    dev = torch.device("cuda", 0)
    names = a.option.split("+")
    values = a.values.split(",")  # one value per name, ':'-separated
    for shape in a.shapes:
        m, k, n, N = (int(x) for x in shape.split("x"))
        A = gen_device(m, k, 0.0, 1234, torch.float64, dev)
        B = gen_device(k, n, 0.0, 5678, torch.float64, dev)
        C = torch.empty((m, n), dtype=torch.float64, device=dev)
        if a.host:
            def pinned(t):
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t)
                return h
            A, B, C = pinned(A), pinned(B), pinned(C)
            args = (A.numpy(), B.numpy(), C.numpy())
        else:
            args = (A, B, C)
        ref, ms = None, {v: [] for v in values}
        for _ in range(a.rounds):
            for v in values:
                for nm, x in zip(names, v.split(":")):
                    oz.set_option(nm, int(x))
                for _ in range(2):
                    oz.os_ii(args[0], args[1], N, out=args[2])
                torch.cuda.synchronize()
                if a.host:
                    t0 = time.perf_counter()
                    for _ in range(a.reps):
                        oz.os_ii(args[0], args[1], N, out=args[2])
                    ms[v].append((time.perf_counter() - t0) / a.reps * 1e3)
                else:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.reps):
                        oz.os_ii(A, B, N, out=C)
                    e1.record()
                    torch.cuda.synchronize()
                    ms[v].append(e0.elapsed_time(e1) / a.reps)
                if ref is None:
                    ref = C.clone()
                elif not torch.equal(C.view(torch.int64), ref.view(torch.int64)):
                    raise SystemExit(f"{a.option}={v}: C differs at {shape}")
        flops = 2.0 * m * n * k
        print(json.dumps({"shape": shape, "option": a.option,
                          "ms": {v: [round(x, 3) for x in ms[v]] for v in values},
                          "tflops_best": {v: round(flops / min(ms[v]) / 1e9, 1) for v in values}}), flush=True)


if __name__ == "__main__":
    main()
