"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import csv
import sys
from collections import OrderedDict

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
            t = float(r[vi].replace(",", ""))
            c, s = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, s + t)
    tot = sum(s for _, s in agg.values())
    print(path, f"total {tot/1e6:.3f} ms")
    for k, (c, s) in agg.items():
        print(f"  {k:45s} x{c:<3d} {s/1e6:9.3f} ms  {100*s/tot:5.1f}%")
