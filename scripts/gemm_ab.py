"""Device time per os_ii call at 16384^3 (or --m), N = 16, for the GEMM
variant selected by the environment (OZ2G_GEMM, OZ2G_PAIR_STAGES,
OZ2G_GEMM_FENCE are read once per process): one JSON line, with the
residue-GEMM stage time and whether C equals the default path's C (saved
once to /tmp)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--moduli", type=int, default=16)
    ap.add_argument("--reps", type=int, default=6)
    a = ap.parse_args()
    import torch

    import paper_2602_02549_b200 as oz
    from bench import gen_device
    dev = torch.device("cuda", 0)
    m = n = a.m
    k = a.k or m
    A = gen_device(m, k, 0.0, 1234, torch.float64, dev)
    B = gen_device(k, n, 0.0, 5678, torch.float64, dev)
    C = torch.empty((m, n), dtype=torch.float64, device=dev)
    for _ in range(3):
        oz.os_ii(A, B, a.moduli, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        oz.os_ii(A, B, a.moduli, out=C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    st = oz.os_ii(A, B, a.moduli, out=C, timing=True).stage_ms
    ref_path = f"/tmp/gemm_ab_ref_{m}_{k}_{a.moduli}.pt"
    if not os.path.exists(ref_path):
        torch.save(C.cpu(), ref_path)
        same = None
    else:
        same = bool(torch.equal(torch.load(ref_path).view(torch.int64), C.cpu().view(torch.int64)))
    env = {k2: os.environ.get(k2) for k2 in ("OZ2G_GEMM", "OZ2G_PAIR_STAGES", "OZ2G_GEMM_FENCE") if os.environ.get(k2)}
    print(json.dumps({"env": env, "m": m, "k": k, "N": a.moduli, "ms": round(ms, 3),
                      "tflops": round(2.0 * m * n * k / ms / 1e9, 1), "residue_gemms_ms": round(st[5], 3),
                      "bit_equal_default": same}), flush=True)


if __name__ == "__main__":
    main()
