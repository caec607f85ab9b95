"""Hot SASS regions of an ncu source page (--print-source sass --csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, ei, ni = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((r[ai], r[si], float(r[ei] or 0), float(r[ni] or 0)))
    except (ValueError, IndexError):
        pass
tot_e = sum(d[2] for d in data)
tot_s = sum(d[3] for d in data)
print(f"total executed {tot_e:.3e}, samples {tot_s:.0f}")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else None
if lo is not None:
    for a, s, e, n in data:
        if lo <= int(a, 16) <= hi:
            print(f"{a} {e:11.3e} {n:7.0f}  {s[:90]}")
else:
    for a, s, e, n in sorted(data, key=lambda d: -d[3])[:N]:
        print(f"{a} {e:11.3e} {n:7.0f}  {s[:90]}")
