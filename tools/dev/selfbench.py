"""Self-join / long AB-join throughput probe (development tool).
usage: python tools/selfbench.py [n ...]   (m = 256)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
m = int(os.environ.get("M", "256"))
for n in [int(x) for x in (sys.argv[1:] or ["262144", "1048576"])]:
    x = synth.walk(7, n)
    t.self_join(x, m)  # warm
    t0 = time.perf_counter(); P = t.self_join(x, m); dt = time.perf_counter() - t0
    cnt = n - m + 1
    full = cnt * cnt  # cells the full-matrix kernel sweeps
    ref = (cnt - m // 2 - 1) * (cnt - m // 2) / 2  # upper-triangle cells the reference computes
    print(f"self n={n} m={m}: {dt*1e3:.1f} ms (host API) -> {full/dt/1e12:.3f} TCell/s swept, "
          f"{ref/dt/1e12:.3f} TCell/s reference-cells", flush=True)
    y = synth.walk(8, n)
    t.ab_join(x[: n // 4], y, m)
    t0 = time.perf_counter(); t.ab_join(x[: n // 4], y, m); dt = time.perf_counter() - t0
    cells = (n // 4 - m + 1) * cnt
    print(f"ab   {n//4}x{n} m={m}: {dt*1e3:.1f} ms -> {cells/dt/1e12:.3f} TCell/s", flush=True)
