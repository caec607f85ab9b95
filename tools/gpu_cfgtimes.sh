# device ms (median of 7 calls) at cfg1/cfg2/cfg3 per library variant: VARIANTS="so[@K=V,...]"
for v in ${VARIANTS}; do
  so=${v%%@*}; envs=""; [[ "$v" == *@* ]] && envs=${v#*@}; envs=${envs//,/ }
  cp build/alt/$so.so paper_1710_07565_b200/librhg_b200.so
  env $envs timeout 600 python - "$v" <<'P'
import sys, statistics
sys.path.insert(0, '.')
import paper_1710_07565_b200 as rhg
CFG = {"cfg1": (1 << 20, 16.0, 3.0, 1, 8), "cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512)}
out = []
for name, (n, d, g, seed, P) in CFG.items():
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    rhg.generate_stats(p)
    runs = [rhg.generate_stats(p) for _ in range(7)]
    out.append(f"{name} dev {statistics.median(r.device_ms for r in runs):.3f} wall {1e3 * statistics.median(r.seconds for r in runs):.3f}")
print(sys.argv[1], " | ".join(out))
P
done
