timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print("cfg2 ms",d["ms_per_step"], "e2e",d["e2e"]["value"], "slab_ms",d["roofline"]["kernel_ms"])'
for c in ${MCFGS:-cfg3 cfg4}; do timeout 300 python tools/run_once.py $c 3 2>&1 | tail -1 | sed "s/^/$c /"; done
RHG_DEBUG_STATS=1 timeout 300 python tools/run_once.py cfg2 1 2>&1 | grep DEBUG
RHG_DEBUG_STATS=1 timeout 300 python tools/run_once.py cfg4 1 2>&1 | grep DEBUG
