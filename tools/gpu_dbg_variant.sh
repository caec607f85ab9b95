# RHG_DEBUG_STATS counters of one cfg2 call per library variant: VARIANTS="so ..."
for v in ${VARIANTS}; do cp build/alt/$v.so paper_1710_07565_b200/librhg_b200.so; echo "== $v"; RHG_DEBUG_STATS=1 timeout 300 python tools/run_once.py cfg2 1 2>&1 | grep DEBUG; done
