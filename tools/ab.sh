#!/usr/bin/env bash
# A/B timing of library builds on one GPU (run under gpurun from the repo root):
#   tools/ab.sh "cfg2 cfg3 cfg4" LIB_A LIB_B ...   (LIB "-" = the in-tree build)
# Each config runs every library twice, interleaved; prints ms/step and the parity flag per run.
set -u
CFGS=$1; shift
for c in $CFGS; do
  for rep in 1 2; do
    for lib in "$@"; do
      if [ "$lib" = "-" ]; then unset RHG_LIB_PATH; else export RHG_LIB_PATH=$lib; fi
      out=$(timeout 600 python bench.py --config "$c" --steps 10 --no-cpu-baseline 2>/dev/null | grep '^{')
      python -c "import json,sys; d=json.loads(sys.argv[1]); print('$c', '$lib', round(d['ms_per_step'],3), d['parity']['equal'], round((d['roofline'].get('isolated') or {}).get('kernel_ms',0),3))" "$out" 2>/dev/null || echo "$c $lib FAILED"
    done
  done
done
