# Round profile refresh: bench line (+CPU baseline), reference arm, ncu launch list, ncu --set full of the dominant kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
RHG_TIMELINE=1 timeout 300 python tools/run_once.py cfg2 3 2>&1 | grep -E "RHG_TIMELINE|RHG_HOST" | tail -2 > gpurun_out/timeline.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
python tools/launches.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slab_kernel|glob_tiles|mt_uniforms|glob_pairs|rank_kernel" -s 8 -c 8 -o gpurun_out/kernels python tools/run_once.py cfg2 2 > gpurun_out/ncu_kernels.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/kernels.ncu-rep > gpurun_out/kernels_summary.json 2>&1
