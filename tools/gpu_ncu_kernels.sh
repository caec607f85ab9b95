timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slab_kernel|glob_tiles|sorted_chain|glob_pairs|angular_scatter|rank_kernel" -s 11 -c 11 -o gpurun_out/kernels python tools/run_once.py cfg2 2 > gpurun_out/ncu_kernels.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/kernels.ncu-rep > gpurun_out/kernels_summary.json 2>&1
ncu -i gpurun_out/kernels.ncu-rep --page details --csv > gpurun_out/kernels_details.csv 2>/dev/null
