"""cfg5 (2048 x 65536 x 2048, N=16): blocking device-pointer calls vs
back-to-back asynchronous calls vs the per-stage device busy time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02549_b200 as oz
from bench import gen_device
m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
k = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
dev = torch.device("cuda", 0)
A = gen_device(m, k, 0.0, 11, torch.float64, dev)
B = gen_device(k, n, 0.0, 12, torch.float64, dev)
C = torch.empty((m, n), dtype=torch.float64, device=dev)
def ev_time(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
tb = ev_time(lambda: oz.os_ii(A, B, 16, out=C))
def asy():
    oz.os_ii(A, B, 16, out=C, blocking=False)
ta = ev_time(lambda: (asy(), None))
oz.synchronize()
def asy_many(reps=10):
    oz.os_ii(A, B, 16, out=C, blocking=False); oz.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): oz.os_ii(A, B, 16, out=C, blocking=False)
    e1.record(); oz.synchronize()
    return e0.elapsed_time(e1) / reps
ta = asy_many()
st = oz.os_ii(A, B, 16, out=C, timing=True).stage_ms
t0 = time.perf_counter(); oz.os_ii(A, B, 16, out=C); th = (time.perf_counter() - t0) * 1e3
fl = 2.0 * m * n * k
print(f"blocking {tb:.3f} ms ({fl/tb/1e9:.1f} TF/s)  async back-to-back {ta:.3f} ms ({fl/ta/1e9:.1f} TF/s)  "
      f"stage sum {sum(st):.3f} ms {[round(x, 3) for x in st]}  one call wall {th:.3f} ms")
