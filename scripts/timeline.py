"""GPU timeline of os_ii calls (CUPTI kernel records via torch.profiler):
per-kernel start / end on the device, the idle gaps between consecutive
kernels, and the host-side time of each call — where a step's time goes
beyond the kernels' own durations.

    python scripts/timeline.py [--m 16384] [--k K] [--moduli 16] [--calls 3] [--out gpurun_out/timeline.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--moduli", type=int, default=16)
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2602_02549_b200 as oz
    from bench import gen_device
    m = a.m
    n = a.n or m
    k = a.k or m
    dt = torch.float32 if a.fp32 else torch.float64
    dev = torch.device("cuda", 0)
    A = gen_device(m, k, 0.0, 1234, dt, dev)
    B = gen_device(k, n, 0.0, 5678, dt, dev)
    out = torch.empty((m, n), dtype=dt, device=dev)
    for _ in range(3):
        oz.os_ii(A, B, a.moduli, out=out)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(a.calls):
        oz.os_ii(A, B, a.moduli, out=out)
    ev1.record()
    torch.cuda.synchronize()
    per_call_ms = ev0.elapsed_time(ev1) / a.calls
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.calls):
            oz.os_ii(A, B, a.moduli, out=out)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() >= 0]
    kern = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    # split into calls at the largest gaps
    gaps = [(kern[i + 1][0] - kern[i][1], i) for i in range(len(kern) - 1)]
    big = sorted(sorted(gaps, reverse=True)[: a.calls - 1], key=lambda g: g[1])
    bounds = [0] + [g[1] + 1 for g in big] + [len(kern)]
    calls = []
    for c in range(len(bounds) - 1):
        ks = kern[bounds[c]:bounds[c + 1]]
        if not ks:
            continue
        span = ks[-1][1] - ks[0][0]
        busy = sum(e - s for s, e, _ in ks)
        inner = [(ks[i + 1][0] - ks[i][1], ks[i][2][:40], ks[i + 1][2][:40]) for i in range(len(ks) - 1)]
        calls.append({"kernels": len(ks), "span_us": span, "busy_us": busy, "idle_us": span - busy,
                      "largest_gaps_us": sorted(inner, reverse=True)[:6],
                      "per_kernel": [(nm[:60], round(e - s, 1)) for s, e, nm in ks]})
    between = [g[0] for g in big]
    res = {"m": m, "n": n, "k": k, "moduli": a.moduli, "dtype": str(dt), "event_ms_per_call": per_call_ms,
           "gap_between_calls_us": between, "calls": calls}
    txt = json.dumps(res, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        open(a.out, "w").write(txt)
    c0 = calls[-1]
    print(json.dumps({"event_ms_per_call": per_call_ms, "span_us": c0["span_us"], "busy_us": c0["busy_us"],
                      "idle_us": c0["idle_us"], "gap_between_calls_us": between,
                      "largest_gaps_us": c0["largest_gaps_us"]}))


if __name__ == "__main__":
    main()
