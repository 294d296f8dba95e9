"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        name = r[ki].split("(")[0].replace("void ", "").replace("oz2g::<unnamed>::", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1e6)
tot = sum(sum(v) for k, v in agg.items() if "oz2g" in k or "gemm_i8" in k or "kernel" in k)
print(f"{'kernel':60s} {'n':>3s} {'mean ms':>9s} {'min ms':>9s}")
for k, v in agg.items():
    print(f"{k[:60]:60s} {len(v):3d} {sum(v)/len(v):9.3f} {min(v):9.3f}")
