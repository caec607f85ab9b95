"""Materialised edge stream throughput: edges/s of
rhg_generate_edges (device generation + canonical sort + copy of every pair to
host memory, host wall clock per call) beside the reference's generate() with
an edge sink that stores the pairs (oracle/_ref, all host threads), on the
same graph.  One JSON line.

    python tools/bench_edges.py [cfg1|cfg2] [steps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_07565_b200 as rhg  # noqa: E402

CFG = {"cfg1": (1 << 20, 16.0, 3.0, 1, 8), "cfg2": (1 << 24, 64.0, 2.2, 7, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n, d, g, seed, P = CFG[name]
p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
rhg.generate_edges(p)  # warm-up (allocations)
t = time.perf_counter()
for _ in range(steps):
    e, st = rhg.generate_edges(p)
gpu_s = (time.perf_counter() - t) / steps
line = {"metric": "materialised edges/s (generate_edges: device + sort + host copy)", "config": name, "n": n,
        "edges": int(len(e)), "gpu_edges_per_s": len(e) / gpu_s, "gpu_ms_per_call": gpu_s * 1e3,
        "device_ms": st.device_ms, "d2h_bytes": int(len(e)) * 16}
try:
    from oracle.refbind import Ref
    ref = Ref()
    t = time.perf_counter()
    re = ref.generate_edges(p.n, p.alpha, p.C, p.seed, p.chunks)
    cpu_s = time.perf_counter() - t
    line.update({"cpu_reference_edges_per_s": len(re) / cpu_s, "cpu_reference_s": cpu_s,
                 "cpu_cores": os.cpu_count(), "same_count": int(len(re)) == int(len(e))})
except Exception as ex:  # noqa: BLE001
    line["cpu_reference"] = f"unavailable: {ex}"
print(json.dumps(line))
