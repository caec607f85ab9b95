"""One warm-up + one timed generate_stats on cuda:0 (for ncu launch lists)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg  # noqa: E402

CFG = {"cfg1": (1 << 20, 16.0, 3.0, 1, 8), "cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512),
       "cfg4": (1 << 28, 4.0, 3.0, 13, 4096), "cfg5": (1 << 30, 16.0, 2.6, 17, 2048)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if name in CFG:
    n, d, g, seed, P = CFG[name]
else:  # n:avg_degree:gamma:seed:chunks
    f = name.split(":")
    n, d, g, seed, P = int(f[0]), float(f[1]), float(f[2]), int(f[3]), int(f[4])
p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for _ in range(reps):
    st = rhg.generate_stats(p)
print(json.dumps({"edges": st.total.edges, "fp": st.total.fingerprint, "comps": st.total.comps,
                  "device_ms": st.device_ms, "sample_ms": st.sample_ms, "edges_ms": st.edges_ms,
                  "pairs_ms": st.pairs_ms, "stream_comps": st.stream_comps, "launches": st.kernel_launches}))
