"""`rhg bench` grid on the GPU (proj/tools/rhg.cpp:166-185):
gamma in {2.2, 3.0} x target average degree in {4, 16, 64, 256} at one n,
one CSV row per point in the reference's column layout
  n,avg_degree_target,gamma,chunks,workers,seconds,edges_per_sec,overestimation_ratio
(`seconds` = RunStats.seconds of one generate_stats call through the public
API, median of --reps; `workers` = GPUs), plus device_ms and — with
--reference — the reference CPU generator's edges/s on the same graph
(oracle/_ref, all host threads).

    python tools/bench_grid.py [--n 16777216] [--chunks 64] [--seed 1] [--reps 5] [--reference]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_07565_b200 as rhg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--chunks", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--reference", action="store_true")
    a = ap.parse_args()
    ref = None
    if a.reference:
        from oracle.refbind import Ref
        ref = Ref()
    cols = "n,avg_degree_target,gamma,chunks,workers,seconds,edges_per_sec,overestimation_ratio,device_ms"
    print(cols + (",reference_seconds,reference_edges_per_sec" if ref else ""), flush=True)
    for gamma in (2.2, 3.0):
        for dbar in (4.0, 16.0, 64.0, 256.0):
            p = rhg.ModelParams.from_avg_degree(a.n, rhg.alpha_from_gamma(gamma), dbar, a.seed, a.chunks)
            rhg.generate_stats(p)  # warm-up
            runs = [rhg.generate_stats(p) for _ in range(a.reps)]
            secs = statistics.median(st.seconds for st in runs)
            st = runs[0]
            row = [a.n, f"{dbar:g}", f"{gamma:g}", a.chunks, 1, f"{secs:.6g}", f"{st.total.edges / secs:.6g}",
                   f"{st.overestimation_ratio():.6g}", f"{statistics.median(r.device_ms for r in runs):.4f}"]
            if ref:
                rs = ref.generate_stats(p.n, p.alpha, p.C, p.seed, p.chunks)
                row += [f"{rs['seconds']:.6g}", f"{rs['edges'] / rs['seconds']:.6g}"]
            print(",".join(map(str, row)), flush=True)


if __name__ == "__main__":
    main()
