"""Slab-join instruction mix from an ncu source page (ncu -i REP --page source --csv --print-source
cuda,sass -k regex:slab_kernel): executed warp instructions and stall samples per code region of
slab_kernel, found by source anchors in csrc/edges.cu.  Usage: slab_mix.py CSV"""
import csv
import json
import os
import sys
from collections import defaultdict

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1710_07565_b200", "csrc", "edges.cu")
lines = open(SRC).read().split("\n")


def find(s, start=0):
    for i in range(start, len(lines)):
        if s in lines[i]:
            return i + 1
    raise SystemExit(f"anchor not found: {s}")


k0 = find("__launch_bounds__(NT, MINB) slab_kernel(EdgeArgs A)")
own = find("// ---- own pass", k0)
grp = find("for (std::uint32_t gi = warp; gi < ngroups", own)
dirl = find("// narrow windows (every lane", grp)
flat = find("// flattened pair list over the warp", dirl)
floop = find("if (t < te) {", flat)
end = find("Acc acc;", floop)
regions = [("prologue (staging, records, runs)", k0, own - 1), ("own pass", own, grp - 1),
           ("group setup (window ends)", grp, dirl - 1), ("direct loop", dirl, flat - 1),
           ("flat setup (prefix, rows)", flat, floop - 1), ("flat loop", floop, end - 1)]
agg, cur, hdr = defaultdict(lambda: [0.0, 0.0]), None, None
for r in csv.reader(open(sys.argv[1])):
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
    try:
        agg[(cur, int(r[0]))][0] += float(r[4] or 0)
        agg[(cur, int(r[0]))][1] += float(r[7] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1.0
ti = sum(v[1] for v in agg.values()) or 1.0
out = {"warp_instructions": ti, "mix": {}}
for name, a, b in regions:
    s = sum(v[0] for k, v in agg.items() if k[0] == "edges.cu" and a <= k[1] <= b)
    i = sum(v[1] for k, v in agg.items() if k[0] == "edges.cu" and a <= k[1] <= b)
    out["mix"][name] = {"inst_share": round(i / ti, 4), "stall_sample_share": round(s / ts, 4)}
rest_i = 1.0 - sum(v["inst_share"] for v in out["mix"].values())
rest_s = 1.0 - sum(v["stall_sample_share"] for v in out["mix"].values())
out["mix"]["other (helpers: window search, libm, intrinsics)"] = {"inst_share": round(rest_i, 4),
                                                                  "stall_sample_share": round(rest_s, 4)}
print(json.dumps(out, indent=1))
