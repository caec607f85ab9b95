# ncu --set full of the radius-side MT kernel (second call of run_once = warm)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mt_uniforms|point_radial" -s 2 -c 2 -o gpurun_out/mt python tools/run_once.py cfg2 2 > gpurun_out/ncu_mt.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/mt.ncu-rep > gpurun_out/mt_summary.json 2>&1
ncu -i gpurun_out/mt.ncu-rep --page details --csv > gpurun_out/mt_details.csv 2>/dev/null
