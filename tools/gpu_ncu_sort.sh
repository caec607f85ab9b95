timeout 900 ncu --set full --clock-control none -k regex:"rank_kernel|beta_cells|lambda_cells|angular_scatter" -s 8 -c 4 -o gpurun_out/sortprof python tools/run_once.py cfg2 2 > gpurun_out/ncu_sort.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py gpurun_out/sortprof.ncu-rep > gpurun_out/sortprof.txt 2>&1
