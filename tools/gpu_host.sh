#!/bin/bash
# Host-side overhead of one generate_stats call on the GPU box: layout alone
# (tools/layout_time.cpp), the RHG_HOST plan breakdown, and wall vs device time.
cd "$(dirname "$0")/.."
nproc; python -c 'import os; print(len(os.sched_getaffinity(0)), os.cpu_count())'
g++ -O2 -std=c++17 -Ipaper_1710_07565_b200/csrc tools/layout_time.cpp build/csrc/layout.o -pthread -o /tmp/layout_time && /tmp/layout_time
RHG_TIMELINE=1 python tools/run_once.py cfg2 6 2>&1 | grep -v "^ *\[" | tail -30
python - <<'P'
import time, sys
sys.path.insert(0, '.')
import paper_1710_07565_b200 as rhg
p = rhg.ModelParams.from_avg_degree(1 << 24, rhg.alpha_from_gamma(2.2), 64.0, 7, 64)
for _ in range(3): rhg.generate_stats(p)
w = []; d = []
for _ in range(20):
    t = time.perf_counter(); st = rhg.generate_stats(p); w.append(time.perf_counter() - t); d.append(st.device_ms)
w.sort(); d.sort()
print("wall ms median", w[10] * 1e3, "device ms median", d[10], "seconds", st.seconds * 1e3)
P
