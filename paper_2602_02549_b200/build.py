"""In-tree build of the native library liboz2g.so (sm_100a only).

    python -m paper_2602_02549_b200.build      # or __graft_entry__.build()

nvcc compiles the CUDA stages and the host orchestration into one shared
library next to this file, so it travels with the repository snapshot to the
GPU box.  No JIT cache, no torch extension machinery.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liboz2g.so")
SOURCES = ["api.cu", "api_ext.cu", "gemm_tc.cu", "scale.cu", "resid.cu", "crt.cu", "bounds.cu", "tables.cpp", "harness.cpp",
           "comm.cpp", "fused.cu", "options.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "-fmad=false", "-cudart", "shared", "-I", os.path.join(HERE, "..", "include")]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "oz2g.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src: str) -> str:
        obj = os.path.join(CSRC, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", OUT, *objs,
           "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-L/usr/local/cuda/lib64", "-lcudart", "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
