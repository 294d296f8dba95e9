"""Throughput of every BASELINE.json config on one GPU (one JSON line each).

    python scripts/configs.py [--out profiles/r01_configs.jsonl]

Per config: device-resident emulated TFLOP/s (CUDA events around back-to-back
os_ii calls, inputs in HBM; blocking calls, and asynchronous ones without a
host synchronisation per call), end-to-end TFLOP/s through the host-pointer API
(pinned buffers, copies inside), native cuBLAS GEMM of the same precision on
the same box, and for the phi sweep the max error against a double-double
product next to the device-evaluated tight bound.  cfg4 (2-D tiling over 2-8
GPUs) needs more than one GPU; its single-GPU tile is cfg "16384".
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_02549_b200 as oz  # noqa: E402
from bench import gen_device  # noqa: E402


def timed(fn, reps):
    for _ in range(3):  # plain call, graph capture, first replay (device-pointer calls replay a CUDA graph)
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(name, m, n, k, nmod, dtype, phi=0.0, reps=5, accuracy=False):
    dev = torch.device("cuda", 0)
    A = gen_device(m, k, phi, 11, dtype, dev)
    B = gen_device(k, n, phi, 12, dtype, dev)
    C = torch.empty((m, n), dtype=dtype, device=dev)
    flops = 2.0 * m * n * k
    ms = timed(lambda: oz.os_ii(A, B, nmod, out=C), reps)
    # asynchronous calls: no host synchronisation per call, timed like the native GEMM below
    ms_async = timed(lambda: oz.os_ii(A, B, nmod, out=C, blocking=False), reps)
    oz.synchronize()
    nat_ms = timed(lambda: torch.matmul(A, B), reps)
    Ah = torch.empty(A.shape, dtype=dtype, pin_memory=True)
    Bh = torch.empty(B.shape, dtype=dtype, pin_memory=True)
    Ch = torch.empty(C.shape, dtype=dtype, pin_memory=True)
    Ah.copy_(A)
    Bh.copy_(B)
    a, b, c = Ah.numpy(), Bh.numpy(), Ch.numpy()
    oz.os_ii(a, b, nmod, out=c)
    t0 = time.perf_counter()
    for _ in range(reps):
        oz.os_ii(a, b, nmod, out=c)
    e2e_ms = (time.perf_counter() - t0) / reps * 1e3
    st = oz.os_ii(A, B, nmod, out=C, timing=True).stage_ms
    row = {"config": name, "m": m, "n": n, "k": k, "moduli": nmod, "dtype": str(dtype).replace("torch.", ""),
           "phi": phi, "ms": ms, "tflops": flops / ms / 1e9, "async_tflops": flops / ms_async / 1e9,
           "e2e_tflops": flops / e2e_ms / 1e9,
           "native_tflops": flops / nat_ms / 1e9,
           "stages_ms": dict(zip(["h2d", "scale", "clearance_gemm", "exponents", "residues", "residue_gemms",
                                  "crt_unscale", "d2h"], [round(x, 4) for x in st]))}
    if accuracy:
        r = oz.os_ii(A, B, nmod, bounds="full")
        rows = torch.linspace(0, m - 1, min(128, m), device=dev).long().unique()
        As = A[rows].contiguous()
        hi, lo = oz.dd_gemm(As, B)
        err = ((r.C[rows] - hi) - lo).abs()
        absAB = torch.matmul(As.abs(), B.abs())
        row["max_rel_err"] = float((err / absAB).max())
        row["tight_bound_rel_max"] = float((r.bounds["tight"][rows] / absAB).max())
        row["err_le_tight_bound"] = bool((err <= r.bounds["tight"][rows]).all())
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = [
        run("cfg1 1024^3 N=14 (the reference's CPU case)", 1024, 1024, 1024, 14, torch.float64, reps=20),
        run("cfg2 SGEMM 4096^3 N=6", 4096, 4096, 4096, 6, torch.float32, reps=10),
        run("cfg2 SGEMM 4096^3 N=7", 4096, 4096, 4096, 7, torch.float32, reps=10),
        run("cfg2 SGEMM 4096^3 N=8", 4096, 4096, 4096, 8, torch.float32, reps=10),
    ]
    for phi in (0.0, 0.5, 2.0, 8.0):  # the reference's sweep {0.5, 2, 8}, plus phi = 0
        for nmod in (8, 12, 16, 20):
            rows.append(run(f"cfg3 8192^3 phi={phi} N={nmod}", 8192, 8192, 8192, nmod, torch.float64, phi=phi,
                            reps=3, accuracy=True))
    rows.append(run("cfg4 tile: 16384^3 N=16 (one GPU's share at 1 GPU)", 16384, 16384, 16384, 16, torch.float64,
                    reps=3))
    rows.append(run("cfg5 2048x65536x2048 N=16", 2048, 2048, 65536, 16, torch.float64, reps=5))
    out = open(args.out, "w") if args.out else sys.stdout
    for r in rows:
        print(json.dumps(r), file=out, flush=True)


if __name__ == "__main__":
    main()
