# A/B of prebuilt library variants with per-variant env: VARIANTS="so[@K=V[,K=V]]" (timeline + bench)
for v in ${VARIANTS}; do
  so=${v%%@*}; envs=""; [[ "$v" == *@* ]] && envs=${v#*@}; envs=${envs//,/ }
  cp build/alt/$so.so paper_1710_07565_b200/librhg_b200.so; echo "== $v"
  env $envs RHG_TIMELINE=1 timeout 300 python tools/run_once.py cfg2 3 2>&1 | grep TIMELINE | tail -1
  env $envs timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms',d['ms_per_step'], 'e2e', d['e2e']['value'], 'edges', d['result']['edges'])"
done
