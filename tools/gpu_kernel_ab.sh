# per-variant ncu duration of one kernel family (KREGEX) over a cfg2 run_once, plus bench ms: VARIANTS="so ..."
for v in ${VARIANTS}; do cp build/alt/$v.so paper_1710_07565_b200/librhg_b200.so; echo "== $v"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX}" --csv python tools/run_once.py cfg2 2 2>/dev/null | grep -E "gpu__time_duration" | awk -F'","' '{print $5, $NF}' | tail -4
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms',d['ms_per_step'], 'e2e', d['e2e']['value'], 'edges', d['result']['edges'])"
done
