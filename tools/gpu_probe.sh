mkdir -p gpurun_out
RHG_DEBUG_STATS=1 timeout 300 python tools/run_once.py cfg2 1 > gpurun_out/dbg.log 2>&1; tail -3 gpurun_out/dbg.log
RHG_TIMELINE=1 timeout 300 python tools/run_once.py cfg2 3 > gpurun_out/timeline.log 2>&1; tail -4 gpurun_out/timeline.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -s 2 -c 1 -o gpurun_out/slab python tools/run_once.py cfg2 2 > gpurun_out/ncu_slab.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/slab.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/slab_src.csv 2>/dev/null; echo done
