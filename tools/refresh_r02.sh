#!/usr/bin/env bash
# Round-2 profile refresh on one GPU (run under gpurun from the repo root); outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tools/profile_round.sh cfg2
for c in cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; grep '^{' gpurun_out/bench_$c.log > gpurun_out/bench_$c.json
  RHG_TIMELINE=1 timeout 300 python tools/run_once.py $c 3 2>&1 | grep -E "RHG_TIMELINE|RHG_HOST" | tail -2 > gpurun_out/timeline_$c.txt
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_cfg2.log 2>&1; grep '^{' gpurun_out/bench_ref_cfg2.log > gpurun_out/bench_ref_cfg2.json
for c in cfg3 cfg4 cfg5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python tools/launches.py gpurun_out/launches_$c.csv > gpurun_out/launches_$c.txt 2>&1
done
(timeout 900 python tools/shard_times.py cfg3 1 2 4 8; timeout 600 python tools/shard_times.py cfg5 8) > gpurun_out/shard_times.jsonl 2> gpurun_out/shard_times.err
echo refresh done
