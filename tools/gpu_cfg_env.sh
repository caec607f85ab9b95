# device ms (median of 5) at cfg1..cfg4 for env variants: ENVS="K=V[,K=V] ..." ("-" = none)
for e in ${ENVS}; do
  envs=""; [ "$e" != "-" ] && envs=${e//,/ }
  env $envs timeout 900 python - "$e" <<'P'
import sys, statistics
sys.path.insert(0, '.')
import paper_1710_07565_b200 as rhg
CFG = {"cfg1": (1 << 20, 16.0, 3.0, 1, 8), "cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512), "cfg4": (1 << 28, 4.0, 3.0, 13, 4096)}
out = []
for name, (n, d, g, seed, P) in CFG.items():
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    r0 = rhg.generate_stats(p)
    runs = [rhg.generate_stats(p) for _ in range(5)]
    assert all((r.total.edges, r.total.fingerprint, r.total.comps) == (r0.total.edges, r0.total.fingerprint, r0.total.comps) for r in runs)
    out.append(f"{name} {statistics.median(r.device_ms for r in runs):.3f} ({r0.total.edges})")
print(sys.argv[1], " | ".join(out))
P
done
