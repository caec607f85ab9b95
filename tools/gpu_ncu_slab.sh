mkdir -p gpurun_out
K=${KREGEX:-slab_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c 1 -o gpurun_out/prof python tools/run_once.py cfg2 2 > gpurun_out/ncu_prof.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_src.csv 2>/dev/null
ncu -i gpurun_out/prof.ncu-rep --page details --csv > gpurun_out/prof_details.csv 2>/dev/null; echo done
