"""Host->device bandwidth with one copy stream vs two or four concurrent copy
streams over the same bytes (does splitting the upload across copy engines help?)."""
import torch
n = 1 << 28  # 2 GiB of fp64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
def t(nst, reps=3):
    ss = [torch.cuda.Stream() for _ in range(nst)]
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in ss: s.wait_stream(torch.cuda.current_stream())
        part = n // nst
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in ss: torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 8 * n / best / 1e6
for k in (1, 2, 4):
    print(f"{k} stream(s): {t(k):.1f} GB/s")
