timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in "" 1; do echo "serial=$v"; RHG_SERIAL_ENGINES=$v RHG_TIMELINE=1 timeout 300 python tools/run_once.py cfg2 3 2>&1 | grep TIMELINE | tail -1; done
for v in "" 1; do RHG_SERIAL_ENGINES=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print("cfg2 ms",d["ms_per_step"], "e2e",d["e2e"]["value"], "slab_ms",d["roofline"]["kernel_ms"])'; done
