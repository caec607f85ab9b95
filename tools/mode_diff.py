"""Compare the counters-only (MODE 0) and degree (MODE 1) paths on golden grid cases."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg
from oracle.refbind import Oracle
orc = Oracle()
g = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "stats.json")))
bad = 0
for s in g:
    if s["name"] != "grid" or s["n"] > 2000:
        continue
    p = rhg.ModelParams(s["n"], s["alpha"], float.fromhex(s["C"]), s["seed"], s["P"])
    pts = orc.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    a = rhg.count_edges_from_points(p, pts)
    b = rhg.count_edges_from_points(p, pts, degrees=True)
    if (a.total.comps, a.total.edges) != (s["comps"], s["edges"]) or (b.total.comps, b.total.edges) != (s["comps"], s["edges"]):
        bad += 1
        if bad < 6:
            print(s["n"], s["alpha"], s["P"], "want", s["edges"], s["comps"], "m0", a.total.edges, a.total.comps,
                  (a.global_comps, a.stream_comps, a.dense_comps), "m1", b.total.edges, b.total.comps,
                  (b.global_comps, b.stream_comps, b.dense_comps))
print("bad", bad)
