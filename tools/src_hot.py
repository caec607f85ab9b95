"""Per-source-line stall samples / executed instructions from an ncu source
page exported with --print-source cuda,sass --csv.  Usage: src_hot.py CSV [N] [sort=s|i]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by = sys.argv[3] if len(sys.argv) > 3 else "s"
cur, hdr, agg, src = None, None, defaultdict(lambda: [0.0, 0.0]), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Kernel Name"):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip():
        continue
    key = (cur, int(r[0]))
    src[key] = r[1]
    try:
        agg[key][0] += float(r[4] or 0)
        agg[key][1] += float(r[7] or 0)
    except (ValueError, IndexError):
        pass
tn = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"samples {tn:.0f} inst {te:.3e}")
idx = 0 if by == "s" else 1
for k, (n, e) in sorted(agg.items(), key=lambda kv: -kv[1][idx])[:N]:
    print(f"{k[0]:12s}:{k[1]:<5d} s {100*n/tn:5.1f}% i {100*e/te:5.1f}%  {(src.get(k) or '').strip()[:85]}")
