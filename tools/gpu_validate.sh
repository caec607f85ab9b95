timeout 1500 python tools/validate_scale.py cfg2 cfg3 cfg4_1gpu cfg5 > gpurun_out/validate_scale.jsonl 2> gpurun_out/validate_scale.err; echo "validate rc=$?"; tail -3 gpurun_out/validate_scale.err
