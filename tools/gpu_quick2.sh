mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
RHG_DEBUG_STATS=1 timeout 300 python tools/run_once.py cfg2 1 2>&1 | tail -2
RHG_TIMELINE=1 timeout 300 python tools/run_once.py cfg2 3 2>&1 | grep TIMELINE | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print("ms",d["ms_per_step"], "val",d["value"], "e2e",d["e2e"]["value"], "slab_ms",d["roofline"]["kernel_ms"], "frac", d["roofline"]["frac"])'
