"""Full-size parity in "same points" mode: the device edge kernels on the
reference's own point set (the oracle's points are bit-identical to the
reference's) must reproduce the reference's golden (edges, fingerprint,
comps) exactly.  Large configs run as engine shards (rank r of W) whose
partial results must sum to the golden.  Also reports the device-sampler
result next to the golden.  Writes one JSON line per config."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_07565_b200 as rhg  # noqa: E402
from oracle.refbind import Oracle  # noqa: E402

golden = {(s["name"], s["P"]): s for s in json.load(open(os.path.join(ROOT, "tests", "golden", "stats.json")))}
orc = Oracle()
which = sys.argv[1:] or ["cfg2", "cfg3", "cfg4_1gpu", "cfg5"]
P_OF = {"cfg1": 8, "cfg2": 64, "cfg3": 512, "cfg4_1gpu": 4096, "cfg4_2gpu": 8192, "cfg5": 2048}
SHARDS = {"cfg5": 8, "cfg4_2gpu": 2}
for name in which:
    g = golden[(name, P_OF[name])]
    p = rhg.ModelParams(g["n"], g["alpha"], float.fromhex(g["C"]), g["seed"], g["P"])
    t = time.time()
    pts = orc.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    t_pts = time.time() - t
    W = SHARDS.get(name, 1)
    acc = [0, 0, 0]
    dev_ms = []
    for r in range(W):
        st = rhg.count_edges_from_points(p, pts, rhg.GenOptions(rank=r, world=W))
        acc = [acc[0] + st.total.edges, (acc[1] + st.total.fingerprint) % 2**64, acc[2] + st.total.comps]
        dev_ms.append(st.device_ms)
    del pts
    want = [g["edges"], g["fingerprint"], g["comps"]]
    acc2 = [0, 0, 0]
    dev2 = []
    for r in range(W):
        st = rhg.generate_stats(p, rhg.GenOptions(rank=r, world=W))
        acc2 = [acc2[0] + st.total.edges, (acc2[1] + st.total.fingerprint) % 2**64, acc2[2] + st.total.comps]
        dev2.append(st.device_ms)
    print(json.dumps({"config": name, "n": p.n, "P": p.chunks, "shards": W, "same_points_exact": acc == want,
                      "same_points": acc, "golden": want, "device_ms_per_shard": dev_ms,
                      "device_sampler": acc2, "device_sampler_edges_rel_diff": (acc2[0] - want[0]) / want[0],
                      "device_sampler_comps_rel_diff": (acc2[2] - want[2]) / want[2],
                      "device_sampler_ms_per_shard": dev2, "host_points_s": t_pts}), flush=True)
