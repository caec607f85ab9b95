"""RHG_TIMELINE of one engine shard (what one rank of an N-GPU run does), for scaling analysis.
Usage: RHG_TIMELINE=1 python tools/shard_timeline.py CONFIG RANK WORLD"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg  # noqa: E402

CFG = {"cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512),
       "cfg4": (1 << 28, 4.0, 3.0, 13, 4096), "cfg5": (1 << 30, 16.0, 2.6, 17, 2048)}
n, d, g, seed, P = CFG[sys.argv[1]]
r, w = int(sys.argv[2]), int(sys.argv[3])
p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
o = rhg.GenOptions(rank=r, world=w)
for _ in range(3):
    st = rhg.generate_stats(p, o)
print(json.dumps({"device_ms": st.device_ms, "sample_ms": st.sample_ms, "edges_ms": st.edges_ms,
                  "pairs_ms": st.pairs_ms, "host_ms": st.host_ms, "stream_comps": st.stream_comps,
                  "dense_comps": st.dense_comps, "global_comps": st.global_comps}))
