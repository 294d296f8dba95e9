"""Dense INT8 tensor-core peak of this B200 (oz2g_i8_peak: tcgen05.mma
kind::i8 128x256x32 issued back to back from shared memory on every SM),
burst (one ~30 ms launch after warm-up) and sustained (back-to-back launches
for ~4 s, the state the residue GEMM runs in), with nvidia-smi clocks and
throttle reasons sampled during each.

    python scripts/int8_peak.py [--out profiles/r02_int8_peak.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(L, iters, launches, random):
    ms, ops = C.c_double(), C.c_double()
    rc = L.oz2g_i8_peak(iters, launches, random, C.byref(ms), C.byref(ops))
    if rc:
        raise RuntimeError(L.oz2g_last_error().decode())
    return ops.value / (ms.value * 1e-3) / 1e12, ms.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import paper_2602_02549_b200 as oz
    from bench import ClockSampler
    torch.cuda.set_device(0)
    L = oz.load_library()
    # iterations per launch for ~30 ms at ~3 POP/s: 148 SMs x 4 MMAs x 2^21 ops
    iters = 40000
    res = {"what": "dense INT8 tensor peak: tcgen05.mma.cta_group::1.kind::i8 128x256x32, operands in shared memory, "
                   "one CTA per SM, int8 ops = 2 x multiply-adds; 'ideal' = low-toggle operand bytes, 'random' = "
                   "pseudo-random operand bytes (power draw of real data)",
           "gpu": torch.cuda.get_device_name(0), "sms": torch.cuda.get_device_properties(0).multi_processor_count}
    for rnd, key in ((0, "ideal"), (1, "random")):
        measure(L, iters, 3, rnd)
        with ClockSampler(0) as cs_b:
            burst, ms_b = measure(L, iters, 1, rnd)
            time.sleep(0.2)
        with ClockSampler(0) as cs_s:
            sustained, ms_s = measure(L, iters, 130, rnd)
        res[key] = {"burst_tops": burst, "burst_ms": ms_b, "burst_clocks": cs_b.summary(),
                    "sustained_tops": sustained, "sustained_ms": ms_s, "sustained_clocks": cs_s.summary()}
        time.sleep(2.0)
    print(json.dumps(res))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
