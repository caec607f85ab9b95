"""Host-side cost of one generate_stats call (layout + plan + upload vs device)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07565_b200 as rhg  # noqa: E402

CFG = {"cfg2": (1 << 24, 64.0, 2.2, 7, 64), "cfg3": (1 << 26, 256.0, 3.0, 11, 512)}
n, d, g, seed, P = CFG[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
for i in range(6):
    t = time.perf_counter()
    st = rhg.generate_stats(p)
    wall = time.perf_counter() - t
    print(f"wall {wall*1e3:.3f} ms  host(layout+plan+upload) {st.host_ms:.3f} ms  device {st.device_ms:.3f} ms  "
          f"seconds {st.seconds*1e3:.3f} ms")
