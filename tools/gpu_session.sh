timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 120 python tools/run_once.py cfg2 2 > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/run_once.py cfg2 2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches.csv | grep -E "total|slab|tiles|rows|glob_pairs"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c180-260
