"""Timeline of one end-to-end os_ii call with pinned host buffers (16384^3,
N = 16): when the last upload ends, when the last kernel ends and when the
last download ends (CUPTI records via torch.profiler), and how busy the
copy engines and the SMs are before and after the last upload — where the
e2e time goes beyond the PCIe floor."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2602_02549_b200 as oz
    from bench import gen_device
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    N = 16
    dev = torch.device("cuda", 0)
    A = gen_device(m, m, 0.0, 1234, torch.float64, dev).cpu().pin_memory()
    B = gen_device(m, m, 0.0, 5678, torch.float64, dev).cpu().pin_memory()
    C = torch.empty((m, m), dtype=torch.float64).pin_memory()
    a, b, c = A.numpy(), B.numpy(), C.numpy()
    for _ in range(2):
        oz.os_ii(a, b, N, out=c)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        oz.os_ii(a, b, N, out=c)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in ev)
    h2d = [e for e in ev if "HtoD" in e.name]
    d2h = [e for e in ev if "DtoH" in e.name]
    ker = [e for e in ev if "Memcpy" not in e.name and "Memset" not in e.name]
    last_up = max(e.time_range.end for e in h2d) - t0
    last_k = max(e.time_range.end for e in ker) - t0
    end = max(e.time_range.end for e in ev) - t0

    def busy(evs, lo, hi):
        iv = sorted((max(e.time_range.start - t0, lo), min(e.time_range.end - t0, hi)) for e in evs)
        tot, cur = 0.0, None
        for s, t in iv:
            if t <= s:
                continue
            if cur is None or s > cur[1]:
                if cur:
                    tot += cur[1] - cur[0]
                cur = [s, t]
            else:
                cur[1] = max(cur[1], t)
        if cur:
            tot += cur[1] - cur[0]
        return tot / 1e3

    out = {"m": m, "call_ms": end / 1e3, "last_upload_ms": last_up / 1e3, "last_kernel_ms": last_k / 1e3,
           "h2d_bytes": sum(1 for _ in h2d), "sm_busy_before_last_upload_ms": busy(ker, 0, last_up),
           "sm_busy_after_last_upload_ms": busy(ker, last_up, end),
           "d2h_busy_after_last_upload_ms": busy(d2h, last_up, end),
           "h2d_busy_ms": busy(h2d, 0, end), "d2h_busy_ms": busy(d2h, 0, end)}
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
