#!/usr/bin/env bash
# Round profile refresh on a GPU box (run under gpurun from the repo root):
#   tools/profile_round.sh CONFIG [KERNEL_REGEX]
# bench line (clocks, roofline, cpu_baseline), RHG_TIMELINE, the ncu launch list of the
# bench command (gpu__time_duration, --clock-control none) and one ncu --set full capture
# of the dominant kernels; everything lands in gpurun_out/ (copy summaries to profiles/rNN/).
set -u
CFG=${1:-cfg2}
KRX=${2:-"slab_kernel|glob_tiles|angle_side|glob_pairs|rank_kernel|point_radial"}
mkdir -p gpurun_out
timeout 900 python bench.py --config "$CFG" --steps 10 > "gpurun_out/bench_$CFG.log" 2>&1; echo "bench rc=$?"
grep '^{' "gpurun_out/bench_$CFG.log" > "gpurun_out/bench_$CFG.json"
RHG_TIMELINE=1 timeout 300 python tools/run_once.py "$CFG" 3 2>&1 | grep -E "RHG_TIMELINE|RHG_HOST" | tail -2 > "gpurun_out/timeline_$CFG.txt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file "gpurun_out/launches_$CFG.csv" \
    python bench.py --config "$CFG" --steps 5 --warmup 3 --no-cpu-baseline > "gpurun_out/ncu_launch_$CFG.log" 2>&1; echo "ncu list rc=$?"
python tools/launches.py "gpurun_out/launches_$CFG.csv" > "gpurun_out/launches_$CFG.txt" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KRX" -s 12 -c 12 \
    -o "gpurun_out/kernels_$CFG" python tools/run_once.py "$CFG" 2 > "gpurun_out/ncu_kernels_$CFG.log" 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py "gpurun_out/kernels_$CFG.ncu-rep" > "gpurun_out/kernels_$CFG.json" 2>&1
