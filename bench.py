#!/usr/bin/env python
"""Benchmark of the B200-native Ozaki-II emulated DGEMM (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3], the metric's own config): emulated DGEMM
m = n = k = 16384 with N = 16 moduli (the smallest N whose tight bound
certifies 1e-15 relative to |A||B| at phi = 0), uniform-exponent
synthetic inputs (phi = 0, entries (u - 1/2), the reference generator's
distribution, gen.hpp:15-31).  Inputs are 2 GiB each, larger than L2, so no
flush is needed between steps.

One step = one full os_ii call (scaling, clearance GEMM, residues, N residue
GEMMs, CRT, inverse scaling).  `value` is device-timed with inputs resident in
HBM; `e2e` is the same call through the public API with pinned HOST buffers
(host->device copies of A, B and the device->host copy of C inside the timed
region).  N > 1 GPUs: C is tiled 2-D over the ranks (strong scaling, SURVEY
§8e); the clearance maxima are max-reduced over the row / column groups with
NCCL through the library's reduce hook; time is the max over ranks.

`--impl reference` times the reference algorithm on the host cores instead
(the CPU oracle port, all threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "emulated DGEMM TFLOPS (m=n=k=16384) vs moduli N; max rel err vs bound"
UNIT = "TFLOP/s"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        ClockSampler._n = getattr(ClockSampler, "_n", 0) + 1  # one file per sampler
        self.path = os.path.join("/tmp", f"oz2g_clocks_{os.getpid()}_{ClockSampler._n}.csv")

    window = None  # (start, end) datetimes of the timed region; None: every sample

    def mark_start(self):
        import datetime
        self._t0 = datetime.datetime.now()

    def mark_end(self):
        import datetime
        self.window = (self._t0, datetime.datetime.now())

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        """Median SM clock, power and throttle reasons of the samples inside the
        marked window (nvidia-smi needs ~0.5 s to deliver its first sample, so
        the sampler starts before the warm-up); all samples when none fall in it."""
        import datetime
        rows, stamped = [], []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts[1:])
                    try:
                        stamped.append((datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f"), parts[1:]))
                    except ValueError:
                        pass
        except Exception:
            pass
        if self.window is not None and stamped:
            lo = self.window[0] - datetime.timedelta(milliseconds=60)
            hi = self.window[1] + datetime.timedelta(milliseconds=60)
            inside = [r for t, r in stamped if lo <= t <= hi]
            if inside:
                rows = inside
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, val in zip(names, r[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit()),
                "reasons": sorted(reasons)}


def _ncu_traffic(m: int, nmod: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of the residue GEMM launch
    from the committed `ncu --set full` capture of this configuration (one
    launch), or None when no capture matches."""
    import csv
    path = None
    for rnd in ("r02", "r01"):  # the newest committed capture
        p = os.path.join(ROOT, "profiles", f"{rnd}_ncu_full_residue_gemm_{m}.csv")
        if os.path.exists(p):
            path = p
            break
    if nmod != 16 or path is None:
        return None
    try:
        rows = list(csv.reader(open(path)))
        h, units = rows[0], rows[1]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        for r in rows[2:]:
            name = r[h.index("Kernel Name")]
            if "gemm_i8_tc_kernel<1>" in name or "gemm_i8_tc_kernel<1," in name:  # <EPI_RESID(, epilogue warps)>
                tot = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    i = h.index(key)
                    tot += float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
                return tot
    except Exception:
        return None
    return None


def gen_device(rows, cols, phi, seed, dtype, device):
    """The reference generator's distribution, (u - 1/2) * exp(g * phi) with
    u uniform on (0, 1] and g standard normal (gen.hpp:15-31), drawn on the GPU
    (torch Philox stream, not the reference's xoshiro stream — parity tests use
    the exact host stream; the benchmark only needs the distribution)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.rand((rows, cols), dtype=torch.float64, device=device, generator=g)
    u = 1.0 - u  # (0, 1]
    v = u - 0.5
    if phi:
        v = v * torch.exp(torch.randn((rows, cols), dtype=torch.float64, device=device, generator=g) * phi)
    v = v.to(dtype)
    v[v == 0] = 0.25  # the reference redraws zeros; any nonzero keeps rows/cols nonzero
    return v.contiguous()


def measure_int8_peak(oz):
    """Dense INT8 tensor peak of this GPU (oz2g_i8_peak, tcgen05 kind::i8 from
    shared memory on every SM): `ideal` on low-toggle operands (the clock-
    limited hardware peak), `random` on pseudo-random operand bytes (the power
    draw of real residue planes: under the board power cap the clock drops) —
    each sustained over ~1 s of back-to-back launches."""
    import ctypes as C
    L = oz.load_library()
    out = {}
    try:
        iters = 40000
        for rnd, key in ((0, "ideal"), (1, "random")):
            for launches, tag in ((3, None), (60, "sustained")):
                ms, ops = C.c_double(), C.c_double()
                if L.oz2g_i8_peak(iters, launches, rnd, C.byref(ms), C.byref(ops)) != 0:
                    return None
                if tag:
                    out[f"{key}_{tag}_tops"] = ops.value / (ms.value * 1e-3) / 1e12
                    out[f"{key}_{tag}_ms"] = ms.value
    except Exception:
        return None
    return out


def cpu_baseline(sample_m: int, sample_n: int, k: int, nmod: int, phi: float, threads: int):
    """The oracle port (oracle/oz2_oracle.c, restating os_ii) on host cores."""
    from oracle import oracle as O
    O.set_threads(threads)
    A = O.gen_matrix(sample_m, k, phi, O.derive_seed(1, 0, 0))
    B = O.gen_matrix(k, sample_n, phi, O.derive_seed(1, 0, 1))
    t0 = time.perf_counter()
    O.os_ii(A, B, nmod)
    dt = time.perf_counter() - t0
    return 2.0 * sample_m * sample_n * k / dt / 1e12, dt


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    m_s = args.cpu_sample
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(m_s, m_s, args.k, args.moduli, args.phi, threads)
    t_all = 0.0
    for _ in range(args.steps):
        v, dt = cpu_baseline(m_s, m_s, args.k, args.moduli, args.phi, threads)
        vals.append(v)
        t_all += dt
    value = float(np.median(vals))
    sample = f"os_ii on A {m_s}x{args.k} * B {args.k}x{m_s} (full k), N={args.moduli}, phi={args.phi}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator gen.hpp, xoshiro256** stream)",
        "config": {"workload": f"Ozaki-II emulated DGEMM m=n=k={args.m}, N={args.moduli} moduli, phi={args.phi}",
                   "m": args.m, "n": args.m, "k": args.k, "moduli": args.moduli, "phi": args.phi,
                   "timed_sample": {"m": m_s, "n": m_s, "k": args.k,
                                    "note": "each step times os_ii on this bounded sample of the workload "
                                            "(full k); value = its emulated TFLOP/s"}},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


_OPTION_DEFAULTS = {"gemm": 0, "fused": 0, "fused_mc": 0, "fused_fence": 1, "spec": -1, "graph": 1, "pdl": 1,
                    "group_m": 0, "group_n": 0, "l2hint": 0, "crt_overlap": 0, "crt_cv": 8, "wblock_min_mb": 2048,
                    "gemm_fence": 0, "epi_warps": 0, "pair_stages": 4, "rowscan_threads": 0, "resid_stream": 0,
                    "spec_tail": 1, "dist_pipeline": 1, "debug_sync": 0, "resid_fast": 1}


def non_default_options() -> dict:
    """The library's tuning options in effect that differ from the defaults
    (oz2g_get_option; set through the environment or set_option)."""
    import paper_2602_02549_b200 as oz
    out = {}
    for name in oz.option_names():
        v = oz.get_option(name)
        if _OPTION_DEFAULTS.get(name) != v:
            out[name] = v
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--moduli", type=int, default=None,
                    help="N; default: chosen by suggest_n(bound='tight', relative=True) for --target")
    ap.add_argument("--target", type=float, default=1e-15, help="relative accuracy target of the automatic N")
    ap.add_argument("--phi", type=float, default=0.0)
    ap.add_argument("--cpu-sample", type=int, default=512, help="rows/cols of the bounded CPU sample (~10 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-native", action="store_true")
    ap.add_argument("--no-int8-peak", action="store_true")
    ap.add_argument("--force-comm", action="store_true",
                    help="run the multi-rank path (library NCCL communicator, shards) even on one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.k is None:
        args.k = args.m
    if args.impl == "reference":
        if args.moduli is None:
            args.moduli = 16  # what the automatic rule picks for this workload (tests/test_fullsize_gpu.py)
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2602_02549_b200 as oz

    from paper_2602_02549_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_comm = world > 1 or args.force_comm
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    elif use_comm:  # one rank: a local process group only carries the NCCL id
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    m = n = args.m
    k = args.k
    tile = pdist.tile_of(rank, world, m, n)
    R, Cc = tile.R, tile.C
    rows, cols = tile.rows, tile.cols

    # global inputs from one seed; this rank's blocks (for the automatic N) and,
    # with several ranks, its 1-D shards — what each rank holds before a step:
    # the library all-gathers the row / column blocks over NVLink (comm.cpp)
    A_full = gen_device(m, k, args.phi, 1234, torch.float64, dev)
    B_full = gen_device(k, n, args.phi, 5678, torch.float64, dev)
    A = A_full[rows].contiguous()
    B = B_full[:, cols].contiguous()
    if use_comm:
        lay = pdist.layout(world, rank, m, n)
        A_sh = A_full[lay["a_shard"]].contiguous()
        B_sh = B_full[:, lay["b_shard"]].contiguous()
    del A_full, B_full
    Cout = torch.empty((A.shape[0], B.shape[1]), dtype=torch.float64, device=dev)

    # N from the paper's bound (north star): the smallest N whose
    # tight bound certifies args.target relative to (|A||B|)_ij, every smaller N
    # shown to fail; ranks take the maximum over their tiles
    auto_n = None
    if args.moduli is None:
        t0 = time.perf_counter()
        sug = oz.suggest_n(A, B, args.target, bound="tight", relative=True)
        if not sug.achievable:
            raise SystemExit(f"bench: no N in range certifies {args.target} relative on this workload")
        n_t = torch.tensor([sug.n], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(n_t, op=dist.ReduceOp.MAX)
        args.moduli = int(n_t.item())
        auto_n = {"rule": f"smallest N with max_ij tight_bound_ij / (|A||B|)_ij <= {args.target} "
                          "(suggest_n(bound='tight', relative=True), bounds.hpp:182-195)",
                  "n": args.moduli, "tight_rel_max": sug.tight_rel_max, "excluded_below": sug.excluded_below,
                  "emulations": sug.emulations, "seconds": round(time.perf_counter() - t0, 3)}

    reduce_cb = None
    comm = None
    if use_comm:
        # the library's own NCCL communicator (world + ncclCommSplit row / column comms)
        comm = pdist.NativeComm(dist, world, rank)
        if world > 1:
            del A, B

    stream = torch.cuda.current_stream(dev)

    class _Step:
        def __init__(self, d):
            self.stage_ms = tuple(d.stage_ms)
            self.kernels_launched = d.kernels_launched

    def step(timing=False):
        if comm is not None:  # shards in, tile out: all-gathers + pipeline + MAX all-reduce (oz2g_gemm_dist)
            return _Step(comm.gemm(A_sh, B_sh, args.moduli, m, n, Cout, timing=timing))
        return oz.os_ii(A, B, args.moduli, out=Cout, timing=timing, reduce_maxima=reduce_cb)

    sampler = ClockSampler(local)
    sampler.__enter__()  # running through the warm-up: samples exist when the timed region starts
    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()

    # per-stage CUDA-event times (one instrumented step, outside the timed loop)
    stage = step(timing=True).stage_ms
    launches_per_step = res.kernels_launched

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    # ---- device-timed region ----
    barrier()
    sampler.mark_start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    barrier()
    sampler.mark_end()
    sampler.__exit__(None, None, None)
    t_ms = ev0.elapsed_time(ev1)
    clocks_timed = sampler.summary()  # the timed region's samples (before any other sampler runs)
    # instrumented steps for the dominant kernel (residue GEMMs), same stream
    gemm_ms = []
    for _ in range(3):
        gemm_ms.append(step(timing=True).stage_ms[5])
    t_tensor = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    t_ms = float(t_tensor.item())
    ms_per_step = t_ms / args.steps
    flops = 2.0 * m * n * k
    value = flops / (ms_per_step * 1e-3) / 1e12

    # ---- end-to-end through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e and comm is not None:
        # each rank: its shards from pinned host memory, the library call, its C tile back
        A_h = torch.empty(A_sh.shape, dtype=torch.float64, pin_memory=True)
        B_h = torch.empty(B_sh.shape, dtype=torch.float64, pin_memory=True)
        C_h = torch.empty(Cout.shape, dtype=torch.float64, pin_memory=True)
        A_h.copy_(A_sh)
        B_h.copy_(B_sh)
        Ad, Bd = torch.empty_like(A_sh), torch.empty_like(B_sh)

        def e2e_step():
            Ad.copy_(A_h, non_blocking=True)
            Bd.copy_(B_h, non_blocking=True)
            comm.gemm(Ad, Bd, args.moduli, m, n, Cout)
            C_h.copy_(Cout, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()

        e2e_step()
        barrier()
        e_steps = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": flops / float(te.item()) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": int(8 * (A_sh.numel() + B_sh.numel()) * world),
               "d2h_bytes_per_step": int(8 * m * n),
               "timing": "wall clock, max over ranks: pinned host shards -> device, oz2g_gemm_dist "
                         "(NCCL all-gathers + pipeline + MAX all-reduce), C tile -> pinned host"}
    elif not args.no_e2e:
        A_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
        B_h = torch.empty(B.shape, dtype=torch.float64, pin_memory=True)
        C_h = torch.empty(Cout.shape, dtype=torch.float64, pin_memory=True)
        A_h.copy_(A)
        B_h.copy_(B)
        a_np, b_np, c_np = A_h.numpy(), B_h.numpy(), C_h.numpy()
        oz.os_ii(a_np, b_np, args.moduli, out=c_np, reduce_maxima=reduce_cb)  # warm
        barrier()
        e_steps = max(1, min(args.steps, 5))
        p_steps = max(1, min(args.steps, 10))  # a stream of calls: enough of them to amortise fill and drain
        t0 = time.perf_counter()
        for _ in range(e_steps):
            oz.os_ii(a_np, b_np, args.moduli, out=c_np, reduce_maxima=reduce_cb)
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        r_e2e = oz.os_ii(a_np, b_np, args.moduli, out=c_np, reduce_maxima=reduce_cb, timing=True)
        st_e2e = r_e2e.stage_ms
        e2e = {"value": flops / float(te.item()) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": int(8 * (A.numel() + B.numel()) * world),
               "d2h_bytes_per_step": int(8 * Cout.numel() * world),
               "timing": "wall clock around blocking os_ii calls (host pointers; copies inside)",
               # one call's per-stage device busy time (stages overlap in the pipelined host path)
               "stages_busy_ms": {nm: round(v, 3) for nm, v in zip(
                   ["h2d", "scale", "clearance_gemm", "exponents", "residues", "residue_gemms", "crt_unscale",
                    "d2h"], st_e2e)}}
        if not torch.equal(torch.from_numpy(c_np).to(dev), Cout):
            e2e["mismatch_vs_device_path"] = True
        # speculated exponents (pipelined host path): A row chunks and B column
        # chunks arrive alternately and the residue GEMMs of every tile start
        # as soon as both of its chunks are present
        e2e["speculation"] = {0: "none", 1: "confirmed", 2: "missed (call redone)"}[r_e2e.speculation]
        if r_e2e.speculation:
            # the same calls with column-only speculation (OZ2G_SPEC=1) and none (0), same box
            for mode, key in ((1, "columns_only_value"), (0, "unspeculated_value")):
                with oz.options(spec=mode):
                    oz.os_ii(a_np, b_np, args.moduli, out=c_np, reduce_maxima=reduce_cb)  # warm (buffer sizes differ)
                    barrier()
                    t0 = time.perf_counter()
                    for _ in range(2):
                        oz.os_ii(a_np, b_np, args.moduli, out=c_np, reduce_maxima=reduce_cb)
                    barrier()
                e2e[key] = flops / ((time.perf_counter() - t0) / 2) / 1e12
        # the same calls enqueued back to back through the asynchronous API
        # (blocking=False, one synchronize at the end): each step still uploads
        # its inputs and downloads its C, but the next upload overlaps the
        # previous residue GEMMs, so a stream of calls is PCIe-bound
        if world == 1:
            oz.os_ii(a_np, b_np, args.moduli, out=c_np, blocking=False)
            oz.synchronize()
            t0 = time.perf_counter()
            for _ in range(p_steps):
                oz.os_ii(a_np, b_np, args.moduli, out=c_np, blocking=False)
            oz.synchronize()
            tp = (time.perf_counter() - t0) / p_steps
            e2e["pipelined"] = {"value": flops / tp / 1e12, "unit": UNIT, "steps": p_steps,
                                "timing": "wall clock around back-to-back os_ii(..., blocking=False) calls and one "
                                          "synchronize(); same host->device / device->host bytes per step"}
            if not torch.equal(torch.from_numpy(c_np).to(dev), Cout):
                e2e["pipelined"]["mismatch_vs_device_path"] = True
        # PCIe reference: plain pinned copies of the same bytes (what bounds e2e from below
        # together with the work that must follow the last uploaded byte)
        ce0 = torch.cuda.Event(enable_timing=True)
        ce1 = torch.cuda.Event(enable_timing=True)
        ce2 = torch.cuda.Event(enable_timing=True)
        Ad = torch.empty_like(A)
        ce0.record(stream)
        Ad.copy_(A_h, non_blocking=True)
        ce1.record(stream)
        C_h.copy_(Cout, non_blocking=True)
        ce2.record(stream)
        torch.cuda.synchronize()
        e2e["pcie_h2d_gbs"] = 8 * A.numel() / (ce0.elapsed_time(ce1) * 1e-3) / 1e9
        e2e["pcie_d2h_gbs"] = 8 * Cout.numel() / (ce1.elapsed_time(ce2) * 1e-3) / 1e9
        del Ad

    # ---- native cuBLAS DGEMM on the same box (the bar to beat) ----
    native = None
    err = None
    by_moduli = None
    if not args.no_native and world == 1:
        Cn = torch.matmul(A, B)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            torch.matmul(A, B, out=Cn)
        e1.record(stream)
        torch.cuda.synchronize()
        native = flops / (e0.elapsed_time(e1) / 3 * 1e-3) / 1e12

        # ---- accuracy: error vs a double-double product, within the paper's bounds ----
        # bounds.hpp:182-206 evaluated on the device for every entry; the error is
        # measured on a row sample against oz2g_dd_gemm (exact products, dd sums).
        rb = oz.os_ii(A, B, args.moduli, bounds="full")
        sample = torch.linspace(0, A.shape[0] - 1, min(256, A.shape[0]), device=dev).long().unique()
        As = A[sample].contiguous()
        hi, lo = oz.dd_gemm(As, B)
        e_abs = ((rb.C[sample] - hi) - lo).abs()
        absAB = torch.matmul(As.abs(), B.abs())
        tight_s, cheap_s = rb.bounds["tight"][sample], rb.bounds["cheap"][sample]
        nat_err = ((Cn[sample] - hi) - lo).abs()
        err = {"reference": "double-double GEMM (oz2g_dd_gemm) on %d sampled rows" % sample.numel(),
               "max_rel_err": float((e_abs / absAB).max().item()),
               "native_dgemm_max_rel_err": float((nat_err / absAB).max().item()),
               "tight_bound_rel_max": float((tight_s / absAB).max().item()),
               "cheap_bound_rel_max": float((cheap_s / absAB).max().item()),
               "tight_bound_max_abs": rb.bounds["tight_max"], "cheap_bound_max_abs": rb.bounds["cheap_max"],
               "err_le_tight_bound_all": bool((e_abs <= tight_s).all().item()),
               "rel": "relative to (|A||B|)_ij"}
        del Cn, absAB, hi, lo, e_abs, rb, tight_s, cheap_s, nat_err

        # ---- throughput vs the number of moduli (device-resident, short) ----
        by_moduli = {}
        for nm in sorted({8, 12, args.moduli, 20}):
            for _ in range(2):
                oz.os_ii(A, B, nm, out=Cout)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(3):
                oz.os_ii(A, B, nm, out=Cout)
            s1.record(stream)
            torch.cuda.synchronize()
            by_moduli[str(nm)] = flops / (s0.elapsed_time(s1) / 3 * 1e-3) / 1e12

    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    peaks, peak_kind = _peaks()
    # dominant kernel: the N residue GEMMs (one launch); algorithmic int8 ops = 2*N*m_loc*n_loc*k
    ops = 2.0 * args.moduli * Cout.shape[0] * Cout.shape[1] * k
    gemm_avg = float(np.mean(gemm_ms))   # all residue-GEMM launches of one step
    achieved = ops / (gemm_avg * 1e-3) / 1e12
    # the residue GEMMs run per 2048-row block of C (W is held per block): equal launches
    n_gemm_launches = -(-Cout.shape[0] // 2048)
    # the residue GEMM is timed inside back-to-back steps: the sustained (power-capped) figure applies.
    # Denominator: the dense INT8 peak measured live on this GPU by a tcgen05 kind::i8 microbenchmark
    # (oz2g_i8_peak: MMAs from shared memory on every SM, no loads / epilogue), burst and sustained.
    i8 = None
    if not args.no_int8_peak:
        with ClockSampler(local) as i8_clk:
            i8 = measure_int8_peak(oz)
        if i8:
            i8["clocks"] = i8_clk.summary()
    if i8:
        int8_peak, int8_capped = i8["ideal_sustained_tops"], i8["random_sustained_tops"]
        peak_note = (f"dense INT8 measured live (oz2g_i8_peak, tcgen05 kind::i8 from shared memory on every SM): "
                     f"{int8_peak:.0f} TOP/s on low-toggle operands (the hardware peak), {int8_capped:.0f} on "
                     f"random operands (power-capped, the state the residue GEMM runs in)")
    else:
        int8_peak = 2.0 * peaks["bf16_tflops"]
        int8_capped = 2.0 * peaks["bf16_tflops_sustained"]
        peak_note = (f"of {peak_kind}: dense INT8 = 2 x bf16 ({peaks['bf16_tflops']} TF/s burst, "
                     f"{peaks['bf16_tflops_sustained']} sustained); int8 ops counted as FLOPs")
    traffic = _ncu_traffic(m, args.moduli) if world == 1 else None
    roof = {"bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s", "frac": achieved / int8_peak,
            "frac_of_power_capped_peak": achieved / int8_capped,
            "traffic": traffic, "traffic_unit": "bytes per launch (ncu --set full, profiles/)",
            "kernel": "gemm_i8_tc_kernel<EPI_RESID> (N residue GEMMs of one 2048-row block of C per launch)",
            "peak_note": peak_note, "int8_peak": i8,
            "algorithmic_ops_per_launch": ops / n_gemm_launches, "launch_ms": gemm_avg / n_gemm_launches,
            "launches_per_step": n_gemm_launches}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        v, dt = cpu_baseline(args.cpu_sample, args.cpu_sample, k, args.moduli, args.phi, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle os_ii on A {args.cpu_sample}x{k} * B {k}x{args.cpu_sample}, N={args.moduli} ({dt:.1f} s)"}

    names = ["h2d", "scale", "clearance_gemm", "exponents", "residues", "residue_gemms", "crt_unscale", "d2h"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator distribution, phi=0 uniform exponent; drawn on device)",
        "config": {"workload": f"Ozaki-II emulated DGEMM m=n=k={m}" + (f" (k={k})" if k != m else "")
                   + f", N={args.moduli} moduli, phi={args.phi}", "m": m, "n": n, "k": k,
                   "moduli": args.moduli, "moduli_choice": auto_n or "fixed (--moduli)",
                   "phi": args.phi, "parallelism": f"2d-tile {R}x{Cc}",
                   "l2": "inputs 2 GiB each > L2, no flush",
                   "library_options": non_default_options() or "defaults"},
        "clocks": clocks_timed,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roof,
        "cpu_baseline": cpu,
        "stages_ms": {nm: round(v, 4) for nm, v in zip(names, stage)},
        "native_dgemm_tflops": native,
        "accuracy": err,
        "tflops_by_moduli": by_moduli,
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
