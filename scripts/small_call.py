"""Per-call time of a small emulated DGEMM (default 1024^3, N = 14) through
the Python API and through the C ABI directly (ctypes, prebuilt arguments):
the difference is the Python wrapper's cost.  Blocking calls (host sync per
call, wall clock) and asynchronous ones (device-timed back to back, like the
native torch.matmul beside them)."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2602_02549_b200 as oz
    from bench import gen_device
    from paper_2602_02549_b200 import _lib
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 14
    dev = torch.device("cuda", 0)
    A = gen_device(m, m, 0.0, 11, torch.float64, dev)
    B = gen_device(m, m, 0.0, 12, torch.float64, dev)
    Cout = torch.empty((m, m), dtype=torch.float64, device=dev)
    reps = 200
    out = {"m": m, "N": N}
    for _ in range(5):
        oz.os_ii(A, B, N, out=Cout)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        oz.os_ii(A, B, N, out=Cout)
    torch.cuda.synchronize()
    out["python_us"] = (time.perf_counter() - t0) / reps * 1e6
    # native cuBLAS DGEMM the same way (a host synchronisation per call)
    for _ in range(5):
        torch.matmul(A, B, out=Cout)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        torch.matmul(A, B, out=Cout)
        torch.cuda.synchronize()
    out["native_blocking_us"] = (time.perf_counter() - t0) / reps * 1e6
    L = _lib.load()
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    diag = _lib.Diag()
    args = (_lib.OZ2G_FP64, m, m, m, A.data_ptr(), m, B.data_ptr(), m, Cout.data_ptr(), m, N, _lib.OZ2G_DEVICE_PTRS,
            stream, None, C.byref(diag), _lib.REDUCE_FN(), None)
    for _ in range(5):
        L.oz2g_gemm(*args)
    t0 = time.perf_counter()
    for _ in range(reps):
        L.oz2g_gemm(*args)
    out["c_abi_us"] = (time.perf_counter() - t0) / reps * 1e6
    # asynchronous calls (OZ2G_ASYNC: graph replays, no per-call host sync),
    # timed on the device like torch.matmul
    def dev_us(fn):
        for _ in range(5):
            fn()
        oz.synchronize()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        oz.synchronize()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    out["python_async_us"] = dev_us(lambda: oz.os_ii(A, B, N, out=Cout, blocking=False))
    aargs = args[:11] + (_lib.OZ2G_DEVICE_PTRS | _lib.OZ2G_ASYNC,) + args[12:]
    out["c_abi_async_us"] = dev_us(lambda: L.oz2g_gemm(*aargs))
    out["native_us"] = dev_us(lambda: torch.matmul(A, B, out=Cout))
    flops = 2.0 * m * m * m
    for key in ("python_async", "c_abi_async", "native"):
        out[key + "_tflops"] = flops / out[key + "_us"] / 1e6
    out["python_tflops"] = flops / out["python_us"] / 1e6
    out["native_blocking_tflops"] = flops / out["native_blocking_us"] / 1e6
    out["c_abi_tflops"] = flops / out["c_abi_us"] / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
