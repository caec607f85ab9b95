"""Device time of each engine shard of cfg2 run alone on one GPU (what one GPU of an
N-GPU strong-scaling run computes), RHG_TIMELINE-free.  Usage: shard_times.py N [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = rhg.ModelParams.from_avg_degree(1 << 24, rhg.alpha_from_gamma(2.2), 64.0, 7, 64)
for r in range(W):
    o = rhg.GenOptions(rank=r, world=W)
    rhg.generate_stats(p, o)
    ts = sorted(rhg.generate_stats(p, o).device_ms for _ in range(5))
    print(f"world {W} rank {r}: device {ts[2]:.3f} ms")
