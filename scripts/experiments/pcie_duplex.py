"""PCIe bandwidth of pinned copies: H2D alone, D2H alone, and both at once
(the async e2e stream overlaps the next call's upload with this call's download)."""
import torch
n = 1 << 27  # 1 GiB of fp64
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); 
        for s in (s1, s2): torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
def up():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def down():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    up(); down()
for s in (s1, s2): s.wait_stream(torch.cuda.current_stream())
tu, td, tb = t(up), t(down), t(both)
g = 8 * n / 1e9
print(f"h2d {g/tu*1e3:.1f} GB/s  d2h {g/td*1e3:.1f} GB/s  both {tb:.1f} ms (h2d alone {tu:.1f}, d2h alone {td:.1f}) -> aggregate {2*g/tb*1e3:.1f} GB/s")
