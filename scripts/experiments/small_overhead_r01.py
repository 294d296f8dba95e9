"""Host overhead of a small blocking call (1024^3, N = 14, device pointers):
Python os_ii vs the C ABI called directly, against the device time."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02549_b200 as oz
from paper_2602_02549_b200 import _lib
from bench import gen_device
dev = torch.device("cuda", 0)
n = 1024
A = gen_device(n, n, 0.0, 1, torch.float64, dev); B = gen_device(n, n, 0.0, 2, torch.float64, dev)
Cm = torch.empty((n, n), dtype=torch.float64, device=dev)
L = _lib.load()
def py():
    oz.os_ii(A, B, 14, out=Cm)
def abi():
    rc = L.oz2g_gemm(_lib.OZ2G_FP64, n, n, n, C.c_void_p(A.data_ptr()), n, C.c_void_p(B.data_ptr()), n,
                     C.c_void_p(Cm.data_ptr()), n, 14, _lib.OZ2G_DEVICE_PTRS, None, None, None, _lib.REDUCE_FN(), None)
    assert rc == 0
for name, fn in (("python os_ii", py), ("C ABI", abi)):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 200 * 1e3:.3f} ms per call", flush=True)
st = oz.os_ii(A, B, 14, out=Cm, timing=True).stage_ms
print("device stage sum", round(sum(st), 3), [round(x, 3) for x in st])
