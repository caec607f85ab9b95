timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms',d['ms_per_step'], 'e2e', d['e2e']['value'], 'slab_ms',d['roofline']['kernel_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_q.csv python tools/run_once.py cfg2 2 > /dev/null 2>&1; python tools/launches.py gpurun_out/launches_q.csv | grep -E "${KGREP:-rank|beta_cells|lambda_cells|scatter|total}"
