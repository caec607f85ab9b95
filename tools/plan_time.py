"""Host plan-head time (layout, stream jobs, chain bins) per config, 25 repetitions: python tools/plan_time.py cfg2 cfg4"""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg
CFG = {"cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512),
       "cfg4": (1 << 28, 4.0, 3.0, 13, 4096), "cfg5": (1 << 30, 16.0, 2.6, 17, 2048)}
for c in sys.argv[1:]:
    n, d, g, seed, P = CFG[c]
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    ts = []
    for _ in range(25):
        t = time.perf_counter(); rhg.shard_extent(p, 0, 1); ts.append((time.perf_counter() - t) * 1e3)
    print(c, "plan head median %.3f ms (min %.3f)" % (statistics.median(ts), min(ts)))
