"""PCIe bandwidth of pinned copies by host NUMA node: for every node with
CPUs, pin the process to that node's CPUs, allocate the pinned buffers there
(first touch) and time H2D, D2H and both at once.  Also prints the GPU's own
node (sysfs) so a bench can place its host buffers next to the GPU."""
import json
import os
import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out


def main():
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
    info = {"torch_pci": bus}
    import subprocess
    try:
        q = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True)
        pci = q.stdout.strip().splitlines()[0].lower()
        pci = pci[4:] if len(pci.split(":")[0]) == 8 else pci  # 00000000:xx:... -> 0000:xx:...
        dev = f"/sys/bus/pci/devices/{pci}"
        info["pci"] = pci
        info["gpu_numa_node"] = open(f"{dev}/numa_node").read().strip()
        info["gpu_local_cpus"] = open(f"{dev}/local_cpulist").read().strip()
    except Exception as e:  # noqa: BLE001
        info["err"] = repr(e)
    nodes = sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
    info["nodes"] = {n: open(f"/sys/devices/system/node/node{n}/cpulist").read().strip() for n in nodes}
    print(json.dumps(info), flush=True)
    n = 1 << 27
    d1 = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for node, cl in info["nodes"].items():
        cpus = cpulist(cl)
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h1.fill_(1.0)
        h2 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2.fill_(1.0)

        def t(fn, reps=3):
            best = 1e9
            for _ in range(reps):
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); fn()
                for s in (s1, s2):
                    torch.cuda.current_stream().wait_stream(s)
                e1.record(); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            return best

        def up():
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)

        def down():
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)

        for s in (s1, s2):
            s.wait_stream(torch.cuda.current_stream())
        tu, td = t(up), t(down)
        tb = t(lambda: (up(), down()))
        g = 8 * n / 1e9
        print(json.dumps({"node": node, "h2d_gbs": round(g / tu * 1e3, 1), "d2h_gbs": round(g / td * 1e3, 1),
                          "both_gbs": round(2 * g / tb * 1e3, 1)}), flush=True)
        del h1, h2


if __name__ == "__main__":
    main()
