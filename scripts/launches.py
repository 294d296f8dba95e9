"""Summarise an ncu --metrics CSV launch list (one or more metrics per launch).

Prints per kernel: launches, mean/min duration (ms) and, when captured, mean
DRAM read/write GB per launch."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = OrderedDict()  # launch id -> (name, {metric: value})
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("oz2g::<unnamed>::", "")
    launch.setdefault(r[ii], (name, {}))[1][r[mi]] = float(r[vi].replace(",", ""))
agg = OrderedDict()
for name, met in launch.values():
    agg.setdefault(name, []).append(met)


def col(v, key, scale):
    xs = [m[key] for m in v if key in m]
    return (sum(xs) / len(xs) / scale) if xs else float("nan")


print(f"{'kernel':56s} {'n':>3s} {'mean ms':>9s} {'min ms':>9s} {'rd GB':>8s} {'wr GB':>8s}")
for k, v in agg.items():
    ts = [m["gpu__time_duration.sum"] / 1e6 for m in v if "gpu__time_duration.sum" in m]
    print(f"{k[:56]:56s} {len(v):3d} {sum(ts)/len(ts):9.3f} {min(ts):9.3f} "
          f"{col(v, 'dram__bytes_read.sum', 1e9):8.2f} {col(v, 'dram__bytes_write.sum', 1e9):8.2f}")
