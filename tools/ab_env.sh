#!/usr/bin/env bash
# A/B of environment switches on the in-tree build (run under gpurun from the repo root):
#   tools/ab_env.sh "cfg2 cfg3" "RHG_DENSE_MIN=64" "RHG_DENSE_MIN=128" ...   ("-" = no switch)
set -u
CFGS=$1; shift
for c in $CFGS; do
  for rep in 1 2; do
    for ev in "$@"; do
      if [ "$ev" = "-" ]; then out=$(timeout 600 python bench.py --config "$c" --steps 10 --no-cpu-baseline 2>/dev/null | grep '^{')
      else out=$(env "$ev" timeout 600 python bench.py --config "$c" --steps 10 --no-cpu-baseline 2>/dev/null | grep '^{'); fi
      python -c "import json,sys; d=json.loads(sys.argv[1]); print('$c', '$ev', round(d['ms_per_step'],3), d['parity']['equal'])" "$out" 2>/dev/null || echo "$c $ev FAILED"
    done
  done
done
