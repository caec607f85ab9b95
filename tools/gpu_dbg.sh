RHG_DEBUG_STATS=1 timeout 120 python tools/run_once.py cfg2 1 2>&1 | tail -2
