"""Self-join time vs data and shape around BASELINE C2 (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth


def run(name, x, m, excl):
    t.self_join(x, m, excl=excl)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); t.self_join(x, m, excl=excl); ts.append(time.perf_counter() - t0)
    dt = sorted(ts)[2]
    cnt = x.size - m + 1
    print(f"{name:28s} n={x.size} m={m} excl={excl}: {dt*1e3:7.2f} ms  {cnt*cnt/dt/1e12:.2f} TCell/s full  "
          f"{(cnt-excl-1)*(cnt-excl)/2/dt/1e12:.2f} TPair/s", flush=True)


n = 131072
run("ecg", synth.ecg(2, n)[0], 250, 62)
run("walk", synth.walk(2, n), 250, 62)
run("noise", np.random.default_rng(2).standard_normal(n), 250, 62)
run("ecg+walk", synth.ecg(2, n)[0] + 0.3 * synth.walk(3, n), 250, 62)
run("ecg 4x", synth.ecg(2, 4 * n)[0], 250, 62)
run("walk 4x", synth.walk(2, 4 * n), 250, 62)
