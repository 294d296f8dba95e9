"""A/B of the fused residue-GEMM + CRT kernel (OZ2G_FUSED=1) against the
two-pass path (int8 W per plane, then crt.cu): device time per os_ii call
(CUDA events, inputs resident) and per-stage busy time, at the BASELINE
shapes.  Prints one JSON line per (config, mode)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2602_02549_b200 as oz
    from bench import gen_device
    dev = torch.device("cuda", 0)
    cfgs = [(16384, 16384, 16384, 16), (2048, 65536, 2048, 16), (8192, 8192, 8192, 16), (4096, 4096, 4096, 16)]
    if len(sys.argv) > 1:
        cfgs = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
    modes = os.environ.get("AB_MODES", "0,1,0,1").split(",")
    for m, k, n, N in cfgs:
        A = gen_device(m, k, 0.0, 1234, torch.float64, dev)
        B = gen_device(k, n, 0.0, 5678, torch.float64, dev)
        C = torch.empty((m, n), dtype=torch.float64, device=dev)
        ref = None
        for mode in modes:
            oz.set_option("fused", int(mode))
            for _ in range(2):
                oz.os_ii(A, B, N, out=C)
            torch.cuda.synchronize()
            if ref is None:
                ref = C.clone()
            same = bool(torch.equal(C.view(torch.int64), ref.view(torch.int64)))
            reps = 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                oz.os_ii(A, B, N, out=C)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            st = oz.os_ii(A, B, N, out=C, timing=True).stage_ms
            print(json.dumps({"m": m, "k": k, "n": n, "N": N, "fused": mode, "ms": ms,
                              "tflops": 2.0 * m * n * k / ms / 1e9, "bit_equal_two_pass": same,
                              "stages_ms": [round(x, 3) for x in st]}), flush=True)
        del A, B, C, ref
        torch.cuda.empty_cache()
    oz.set_option("fused", 0)


if __name__ == "__main__":
    main()
