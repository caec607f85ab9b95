"""Borderline-pair report (north_star: "threshold-borderline pairs ... listed explicitly";
SURVEY 8(c)).  TEST / REPORTING TOOL -- not the product path.

  python tools/borderline_report.py --device   # on a GPU box: (i)+(ii) for every config
  python tools/borderline_report.py --host     # host cores:  (iii) for every config

(i)+(ii) device: rhg.audit_predicate on the full graph -- every pair the slab join's FP32
      pre-filter decided is re-evaluated with the reference predicate (sweep.hpp:531-533):
      disagreements must be 0, max |D32 - D64| / tau < 1 is the pre-filter's margin; the
      other engines evaluate the reference predicate itself.  The counters must equal the
      reference goldens.
(iii) host, informational: the oracle's sweep of one engine shard re-decides every tested
      pair within the rounding band |lhs - rhs| <= 1e-13 x (term magnitude) with the exact
      distance test d < R (geometry.hpp:117-123) in binary128 from (r, theta): how often the
      reference's FP64 predicate differs from the exact geometry (its own rounding), and the
      pairs with |d - R| < 1e-12 listed explicitly (<= 10^4).
Writes profiles/r02/borderline_{device,host}.json (merged by --merge into borderline.json).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# name: (n, d, gamma, seed, P, host shard world) -- the host audit runs shard 0 of `world`
CONFIGS = {
    "cfg1": (1 << 20, 16.0, 3.0, 1, 8, 1),
    "cfg2": (1 << 24, 64.0, 2.2, 7, 64, 1),
    "cfg3": (1 << 26, 256.0, 3.0, 11, 512, 8),
    "cfg4_1gpu": (1 << 28, 4.0, 3.0, 13, 4096, 64),
    "cfg5": (1 << 30, 16.0, 2.6, 17, 2048, 256),
    "cfg4_8gpu": (1 << 31, 4.0, 3.0, 13, 32768, 1024),
}
OUT = os.path.join(ROOT, "profiles", "r02")


def golden(name):
    for s in json.load(open(os.path.join(ROOT, "tests", "golden", "stats.json"))):
        if s["name"] == name and s["P"] == CONFIGS[name][4]:
            return s
    return None


def device(names):
    import paper_1710_07565_b200 as rhg
    rows = {}
    for name in names:
        n, d, g, seed, P, _ = CONFIGS[name]
        p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
        world = 8 if n > (1 << 30) else 1  # 2^31 points: 8 shards in sequence on one GPU
        acc = None
        for r in range(world):
            rep, st = rhg.audit_predicate(p, rhg.GenOptions(rank=r, world=world))
            rep = dict(rep, edges=st.total.edges, fingerprint=st.total.fingerprint, comps=st.total.comps)
            if acc is None:
                acc = rep
            else:
                for k, v in rep.items():
                    acc[k] = max(acc[k], v) if k == "max_err_over_tau" else (
                        (acc[k] + v) % 2**64 if k == "fingerprint" else acc[k] + v)
        gd = golden(name)
        acc["equals_reference_golden"] = bool(gd and (acc["edges"], acc["fingerprint"], acc["comps"]) ==
                                              (gd["edges"], gd["fingerprint"], gd["comps"]))
        acc["shards"] = world
        rows[name] = acc
        print(name, json.dumps(acc), flush=True)
    return rows


def host(names, threads):
    from oracle.refbind import Oracle
    o = Oracle()
    rows = {}
    for name in names:
        n, d, g, seed, P, world = CONFIGS[name]
        a = o.alpha_from_gamma(g)
        C = o.radial_const_from_avg_degree(d, a)
        t = time.time()
        r = o.borderline(n, a, C, seed, P, rank=0, world=world, band=1e-13, cap=10000, threads=threads)
        r["shard"] = f"0 of {world}" if world > 1 else "whole graph"
        r["wall_s"] = round(time.time() - t, 1)
        flips = r["flips_to_edge"] + r["flips_to_nonedge"]
        r["flip_rate_of_band"] = flips / r["band_pairs"] if r["band_pairs"] else 0.0
        r["flip_rate_of_edges"] = flips / r["edges"] if r["edges"] else 0.0
        r["pairs_listed"] = r.pop("pairs")
        rows[name] = r
        print(name, json.dumps({k: v for k, v in r.items() if k != "pairs_listed"}), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--device", action="store_true")
    ap.add_argument("--host", action="store_true")
    ap.add_argument("--merge", action="store_true")
    ap.add_argument("--configs", nargs="+", default=list(CONFIGS))
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out-dir", default=OUT, help="where the JSON goes (on a GPU box: gpurun_out)")
    a = ap.parse_args()
    out = a.out_dir
    os.makedirs(out, exist_ok=True)
    if a.device:
        json.dump(device(a.configs), open(os.path.join(out, "borderline_device.json"), "w"), indent=1)
    if a.host:
        path = os.path.join(out, "borderline_host.json")
        old = json.load(open(path)) if os.path.exists(path) else {}
        old.update(host(a.configs, a.threads))
        json.dump(old, open(path, "w"), indent=1)
    if a.merge:
        dev = json.load(open(os.path.join(out, "borderline_device.json")))
        hst = json.load(open(os.path.join(out, "borderline_host.json")))
        json.dump({k: {"device_predicate_audit": dev.get(k), "host_binary128_audit": hst.get(k)}
                   for k in CONFIGS}, open(os.path.join(out, "borderline.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
