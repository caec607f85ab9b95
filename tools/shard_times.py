"""Strong / weak scaling prediction from one GPU: every engine shard of an N-GPU run is run
alone on this GPU (exactly the work one rank of the N-GPU run does; the only cross-GPU step
is the 72-byte counter all-reduce) and the slowest shard's median device time is the
predicted N-GPU step time.

    python tools/shard_times.py [config] [N ...]     (default: cfg3 1 2 4 8)

cfg4 is weak scaling (n = 2^28 N, P = 4096 N).  Prints one JSON line per N with the
predicted step time, edges/s and strong-scaling efficiency against N = 1.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg  # noqa: E402

CFG = {"cfg2": (1 << 24, 64.0, 2.2, 7, 64, False), "cfg3": (1 << 26, 256.0, 3.0, 11, 512, False),
       "cfg4": (1 << 28, 4.0, 3.0, 13, 4096, True), "cfg5": (1 << 30, 16.0, 2.6, 17, 2048, False)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
Ns = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
n0, d, g, seed, P0, weak = CFG[name]
base = None
for W in Ns:
    n, P = (n0 * W, P0 * W) if weak else (n0, P0)
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    times, edges, fp, comps = [], 0, 0, 0
    for r in range(W):
        o = rhg.GenOptions(rank=r, world=W)
        rhg.generate_stats(p, o)  # warm-up
        runs = [rhg.generate_stats(p, o) for _ in range(3)]
        times.append(sorted(s.device_ms for s in runs)[1])
        st = runs[0].total
        edges, fp, comps = edges + st.edges, (fp + st.fingerprint) % 2**64, comps + st.comps
    step = max(times)
    v = edges / (step * 1e-3)
    if base is None:
        base = v
    print(json.dumps({"config": name, "n_gpus": W, "n": n, "chunks": P, "predicted_step_ms": step,
                      "shard_ms": [round(t, 3) for t in times], "edges": edges, "fingerprint": fp, "comps": comps,
                      "predicted_edges_per_s": v,
                      "efficiency_vs_1": None if weak else v / (base * W)}), flush=True)
