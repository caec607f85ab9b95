for s in 0 1 2; do RHG_SCHED=$s RHG_TIMELINE=1 timeout 300 python tools/run_once.py cfg2 3 2>&1 | grep TIMELINE | tail -1 | sed "s/^/sched=$s /"; done
