"""Pitched host->device copies (cudaMemcpy2DAsync): a column block of a pinned
row-major matrix, as the row + column speculated path uploads B, against a
contiguous row block of the same bytes."""
import ctypes, glob, torch
lib = ctypes.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
n = 16384
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
def cp2d(w, rows=n):
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.cudaMemcpy2DAsync(ctypes.c_void_p(d.data_ptr()), ctypes.c_size_t(8 * n), ctypes.c_void_p(h.data_ptr()),
                               ctypes.c_size_t(8 * n), ctypes.c_size_t(8 * w), ctypes.c_size_t(rows), 1,
                               ctypes.c_void_p(s))
    assert rc == 0, rc
for w in (16384, 8192, 4096, 2048, 1024, 512, 256):
    ms = t(lambda: cp2d(w))
    print(f"cudaMemcpy2DAsync column block {n}x{w}: {8*n*w/ms/1e6:.1f} GB/s ({ms:.2f} ms)")
# concurrent: column-block uploads on one stream, tile downloads (2048 x 2048 of a row-major C) on another
hc = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
dc = torch.empty((n, n), dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def up_cols():
    for j in range(8):
        rc = lib.cudaMemcpy2DAsync(ctypes.c_void_p(d.data_ptr() + 8 * 2048 * j), ctypes.c_size_t(8 * n),
                                   ctypes.c_void_p(h.data_ptr() + 8 * 2048 * j), ctypes.c_size_t(8 * n),
                                   ctypes.c_size_t(8 * 2048), ctypes.c_size_t(n), 1, ctypes.c_void_p(s1.cuda_stream))
        assert rc == 0
def down_tiles():
    for i in range(8):
        for j in range(8):
            off = 8 * (2048 * i * n + 2048 * j)
            rc = lib.cudaMemcpy2DAsync(ctypes.c_void_p(hc.data_ptr() + off), ctypes.c_size_t(8 * n),
                                       ctypes.c_void_p(dc.data_ptr() + off), ctypes.c_size_t(8 * n),
                                       ctypes.c_size_t(8 * 2048), ctypes.c_size_t(2048), 2,
                                       ctypes.c_void_p(s2.cuda_stream))
            assert rc == 0
def both():
    up_cols(); down_tiles()
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
for s in (s1, s2): s.wait_stream(torch.cuda.current_stream())
print(f"8 column-block uploads alone {t(lambda: (up_cols(), torch.cuda.current_stream().wait_stream(s1))):.1f} ms, "
      f"64 tile downloads alone {t(lambda: (down_tiles(), torch.cuda.current_stream().wait_stream(s2))):.1f} ms, "
      f"both {t(both):.1f} ms")
