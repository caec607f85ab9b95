"""Generate tests/golden/*.json by running the REFERENCE itself.

    python tests/golden/make_golden.py [--big]

Uses oracle/_ref/librhg_ref.so (the unmodified reference headers compiled in
place by oracle/Makefile; needs /root/reference at build time).  The output is
committed; the GPU box never reads /root/reference.

* known_answers.json — rng.hpp seed hashing, std::mt19937_64 outputs,
  sorted-uniform streams, binomial draws, geometry constants.
* layouts.json       — make_layout tables (sha256 of every array) for the
  BASELINE configs at their recommended chunk counts.
* points.json        — sha256 of every point attribute (bitwise) for small
  parameter corners, plus a few literal values.
* stats.json         — generate_stats (edges, fingerprint, comps, n_G, r_G)
  for the acceptance-style grid, the reference's tiny cases, cfg1 at
  P in {1, 8, 64}, cfg2 at P=64 and (with --big) cfg3-cfg5 at the
  recommended P.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.refbind import Ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# BASELINE.json configs: (name, n, d_bar, gamma, seed, recommended P)
CONFIGS = [
    ("cfg1", 1 << 20, 16.0, 3.0, 1, 8),
    ("cfg2", 1 << 24, 64.0, 2.2, 7, 64),
    ("cfg3", 1 << 26, 256.0, 3.0, 11, 512),
    ("cfg4_1gpu", 1 << 28, 4.0, 3.0, 13, 4096),
    ("cfg4_2gpu", 1 << 29, 4.0, 3.0, 13, 8192),
    ("cfg5", 1 << 30, 16.0, 2.6, 17, 2048),
    ("cfg4_4gpu", 1 << 30, 4.0, 3.0, 13, 16384),
    ("cfg4_8gpu", 1 << 31, 4.0, 3.0, 13, 32768),
]
BIG = ("cfg3", "cfg4_1gpu", "cfg4_2gpu", "cfg5", "cfg4_4gpu", "cfg4_8gpu")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def known_answers(r: Ref) -> dict:
    ka = {}
    ka["derive_seed"] = [{"root": root, "comps": comps, "seed": r.derive_seed(root, comps)}
                         for root, comps in [(0, []), (1, [1]), (42, [3, 0, 0]), (7, [4, 15, 63]),
                                             (2**64 - 1, [2, 5, 1023]), (13, [2, 28, 1])]]
    mt = r.mt_outputs(5489, 10000)
    ka["mt19937_64_seed5489_first5"] = [int(x) for x in mt[:5]]
    ka["mt19937_64_seed5489_10000th"] = int(mt[-1])
    ka["mt19937_64_seed_12345_sha_1000"] = sha(r.mt_outputs(12345, 1000))
    su = r.sorted_uniforms(1000, 0.5, 1.25, 99, [3, 4, 5])
    ka["sorted_uniforms"] = {"count": 1000, "a": 0.5, "b": 1.25, "root": 99, "comps": [3, 4, 5],
                             "first3": [float(x).hex() for x in su[:3]], "sha": sha(su)}
    ka["binomial"] = [{"trials": t, "p": p, "seed": s, "value": r.binomial(t, p, s)}
                      for t, p, s in [(10, 0.3, 1), (1000, 0.5, 2), (10**6, 0.25, 3), (10**9, 0.001, 4),
                                      (10**12, 0.7, 5), (5, 1.0, 6), (0, 0.5, 7), (123456789, 0.5, 8)]]
    ka["alpha_from_gamma"] = {str(g): r.alpha_from_gamma(g) for g in (2.2, 2.6, 3.0)}
    ka["radial_const"] = {f"{d}_{a}": r.radial_const_from_avg_degree(d, a).hex()
                          for d, a in [(16.0, 1.0), (64.0, 0.6), (256.0, 1.0), (4.0, 1.0), (16.0, 0.8)]}
    return ka


def layout_record(r: Ref, n, d, g, seed, P) -> dict:
    a = r.alpha_from_gamma(g)
    C = r.radial_const_from_avg_degree(d, a)
    L = r.layout(n, a, C, seed, P)
    rec = {"n": n, "d": d, "gamma": g, "seed": seed, "P": P, "count": L.count, "R": L.R.hex(),
           "cosh_R": L.cosh_R.hex(), "r_G": L.r_G.hex(), "first_streaming": L.first_streaming,
           "counts": [int(x) for x in L.counts]}
    for f in ["lower", "upper", "probs", "cosh_alpha_lower", "cosh_alpha_upper", "coth_lower",
              "coshR_inv_sinh_lower", "chunk_counts", "id_base", "classes"]:
        rec["sha_" + f] = sha(getattr(L, f))
    return rec


POINT_CASES = [(2000, 16.0, 2.5, 3, 4), (1500, 12.0, 3.0, 1, 1), (500, 4.0, 2.1, 9, 8), (50, 6.0, 2.6, 13, 32),
               (20000, 16.0, 2.6, 5, 4), (3, 4.0, 2.2, 0, 1)]


def point_record(r: Ref, n, d, g, seed, P) -> dict:
    a = r.alpha_from_gamma(g)
    C = r.radial_const_from_avg_degree(d, a)
    pts = r.points(n, a, C, seed, P)
    rec = {"n": n, "d": d, "gamma": g, "seed": seed, "P": P}
    for f in ["beta", "r", "theta", "half_width", "coth_r", "inv_sinh_r", "cos_theta", "sin_theta", "annulus"]:
        arr = getattr(pts, f)
        rec["sha_" + f] = sha(arr)
        if arr.dtype == np.float64:
            rec["last_" + f] = float(arr[-1]).hex()
    return rec


def stats_record(r: Ref, name, n, alpha, C, seed, P, extra=None) -> dict:
    t = time.time()
    s = r.generate_stats(n, alpha, C, seed, P, 0)
    rec = {"name": name, "n": n, "alpha": alpha, "C": C.hex(), "seed": seed, "P": P, "edges": s["edges"],
           "fingerprint": s["fingerprint"], "comps": s["comps"], "global_vertices": s["global_vertices"],
           "r_G": s["r_G"].hex(), "annuli": s["annuli"], "first_streaming": s["first_streaming"],
           "ref_seconds_here": round(time.time() - t, 3)}
    if extra:
        rec.update(extra)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also cfg3..cfg5 and cfg4 at 2^30/2^31 (tens of minutes of CPU)")
    ap.add_argument("--only", nargs="+", choices=BIG,
                    help="(re)compute just these big stats rows and merge them into stats.json")
    args = ap.parse_args()
    r = Ref()
    path = os.path.join(OUT, "stats.json")
    if args.only:
        rows = [s for s in json.load(open(path)) if s["name"] not in args.only]
        for name, n, d, g, seed, P in CONFIGS:
            if name in args.only:
                alpha = r.alpha_from_gamma(g)
                C = r.radial_const_from_avg_degree(d, alpha)
                print("stats", name, P, flush=True)
                rows.append(stats_record(r, name, n, alpha, C, seed, P, {"d": d, "gamma": g}))
        with open(path, "w") as f:
            json.dump(rows, f, indent=1)
        print("wrote", path)
        return
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(known_answers(r), f, indent=1)
    with open(os.path.join(OUT, "layouts.json"), "w") as f:
        json.dump([layout_record(r, n, d, g, s, P) for _, n, d, g, s, P in CONFIGS], f, indent=1)
    with open(os.path.join(OUT, "points.json"), "w") as f:
        json.dump([point_record(r, *c) for c in POINT_CASES], f, indent=1)
    stats = []
    # acceptance.cpp:32-61 grid (seeds 1..2), generated by the reference
    for n in (100, 500, 2000):
        for alpha in (0.55, 0.75, 1.0):
            for d in (4.0, 16.0):
                for P in (1, 2, 4, 8):
                    for seed in (1, 2):
                        C = r.radial_const_from_avg_degree(d, alpha)
                        stats.append(stats_record(r, "grid", n, alpha, C, seed, P, {"d": d}))
    # test_sweep.cpp:138-162 tiny instances
    stats.append(stats_record(r, "n1", 1, 1.0, 5.0, 9, 1))
    for seed in range(10):
        stats.append(stats_record(r, "n2", 2, 2.0, 20.0, seed, 1))
    C = r.radial_const_from_avg_degree(6.0, 0.8)
    stats.append(stats_record(r, "more_chunks_than_points", 50, 0.8, C, 13, 32, {"d": 6.0}))
    for P in (3, 5, 7, 16):
        C = r.radial_const_from_avg_degree(12.0, 0.75)
        stats.append(stats_record(r, "odd_P", 20000, 0.75, C, 77, P, {"d": 12.0}))
    C = r.radial_const_from_avg_degree(16.0, 0.8)
    stats.append(stats_record(r, "smoke", 20000, 0.8, C, 5, 4, {"d": 16.0}))
    big = {"cfg1", "cfg2"} | (set(BIG) if args.big else set())
    for name, n, d, g, seed, P in CONFIGS:
        if name not in big:
            continue
        alpha = r.alpha_from_gamma(g)
        C = r.radial_const_from_avg_degree(d, alpha)
        Ps = (1, 8, 64) if name == "cfg1" else (P,)
        for PP in Ps:
            print("stats", name, PP, flush=True)
            stats.append(stats_record(r, name, n, alpha, C, seed, PP, {"d": d, "gamma": g}))
    if not args.big and os.path.exists(path):  # keep previously generated big rows
        old = [s for s in json.load(open(path)) if s["name"] in BIG]
        stats.extend(old)
    with open(path, "w") as f:
        json.dump(stats, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
