"""Quick device diagnostics: FP64 peak, per-config timing and sampler
mismatch rates vs the oracle (run on a GPU box)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1710_07565_b200 as rhg  # noqa: E402
from oracle.refbind import Oracle  # noqa: E402

orc = Oracle()
ops, lat, ms = rhg.fp64_peak(0)
print(json.dumps({"fp64_ops_per_s": ops, "dmul_latency_cycles": lat, "probe_ms": ms}), flush=True)
CFG = {"cfg1": (1 << 20, 16.0, 3.0, 1, 8), "cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512),
       "cfg4": (1 << 28, 4.0, 3.0, 13, 4096)}
which = sys.argv[1:] or ["cfg1", "cfg2"]
for name in which:
    n, d, g, seed, P = CFG[name]
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    for rep in range(3):
        t = time.time()
        st = rhg.generate_stats(p)
        wall = time.time() - t
    print(json.dumps({"cfg": name, "edges": st.total.edges, "fp": st.total.fingerprint, "comps": st.total.comps,
                      "device_ms": st.device_ms, "sample_ms": st.sample_ms, "edges_ms": st.edges_ms,
                      "host_ms": st.host_ms, "wall_s": wall, "global_edges": st.global_edges,
                      "global_comps": st.global_comps, "edges_per_s": st.total.edges / (st.device_ms * 1e-3)}),
          flush=True)
    if n <= 1 << 24:
        dev = rhg.sample_points(p)
        ref = orc.points(n, p.alpha, p.C, seed, P)
        rates = {f: float(np.mean(getattr(dev, f).view(np.uint64) != getattr(ref, f).view(np.uint64)))
                 for f in rhg.Points.FIELDS}
        print(json.dumps({"cfg": name, "mismatch_rate": rates}), flush=True)
