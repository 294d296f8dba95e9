"""Strong-scaling projection from one GPU: time one rank's tile of the
bench.py --gpus N decomposition (dist.tile_of, rank 0) on a single B200.

Each rank of `bench.py --gpus N` runs os_ii on its A row block and B column
block (full k) plus an NCCL MAX all-reduce of m/R + n/C int32 clearance
maxima; this times everything but that all-reduce.  Projected whole-job
TFLOP/s = N x (tile flops / tile time), i.e. perfect NVLink and equal ranks.

    python scripts/experiments/tile_projection.py [--m 16384] [--moduli 16]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import torch  # noqa: E402

import paper_2602_02549_b200 as oz  # noqa: E402
from bench import gen_device  # noqa: E402
from paper_2602_02549_b200 import dist as pdist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--moduli", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=3, help="interleaved passes over the worlds (median per world)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    m = n = k = args.m
    A_full = gen_device(m, k, 0.0, 1234, torch.float64, dev)
    B_full = gen_device(k, n, 0.0, 5678, torch.float64, dev)
    worlds = (1, 2, 4, 8)
    tiles = {}
    for world in worlds:
        tile = pdist.tile_of(0, world, m, n)
        A = A_full[tile.rows].contiguous()
        B = B_full[:, tile.cols].contiguous()
        C = torch.empty((A.shape[0], B.shape[1]), dtype=torch.float64, device=dev)
        tiles[world] = (tile, A, B, C)
    del A_full, B_full
    # The worlds take turns, so none of them is timed only on a GPU that the
    # previous (larger) tiles left hot; the median of the rounds is reported.
    times = {w: [] for w in worlds}
    for _ in range(args.rounds):
        for world in worlds:
            _, A, B, C = tiles[world]
            for _ in range(args.warmup):
                oz.os_ii(A, B, args.moduli, out=C)
            torch.cuda.synchronize()
            s = torch.cuda.current_stream(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(args.steps):
                oz.os_ii(A, B, args.moduli, out=C)
            e1.record(s)
            torch.cuda.synchronize()
            times[world].append(e0.elapsed_time(e1) / args.steps)
    base = None
    for world in worlds:
        tile, A, B, C = tiles[world]
        t = sorted(times[world])[len(times[world]) // 2]
        stages = oz.os_ii(A, B, args.moduli, out=C, timing=True).stage_ms
        tf = 2.0 * A.shape[0] * B.shape[1] * k / (t * 1e-3) / 1e12
        proj = world * tf
        base = base or proj
        print(json.dumps({"world": world, "grid": [tile.R, tile.C], "tile": [A.shape[0], B.shape[1], k],
                          "ms_per_step": round(t, 3), "ms_rounds": [round(x, 3) for x in times[world]],
                          "tile_tflops": round(tf, 1), "projected_job_tflops": round(proj, 1),
                          "projected_speedup": round(proj / base, 2),
                          "stages_ms": [round(x, 3) for x in stages]}), flush=True)


if __name__ == "__main__":
    main()
