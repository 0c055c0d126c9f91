"""Self-join probe (development tool): bench shapes (2^21 prefix of the C4
query walk, m=512; BASELINE C2 ECG, m=250, excl=62), host API timing.
usage: [TSD_LIB=...] [TSD_SYM=0|1] [TSD_VERBOSE=1] python tools/symprobe.py [reps]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cases = [("C2", synth.ecg(2, 131072)[0], 250, 62), ("w21", synth.walk(4, 1 << 21), 512, None)]
if os.environ.get("REV"):
    cases = cases[::-1]
if os.environ.get("ONLY"):
    cases = [c for c in cases if c[0] == os.environ["ONLY"]]
for name, x, m, excl in cases:
    P = t.self_join(x, m, excl=excl)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); P = t.self_join(x, m, excl=excl); ts.append(time.perf_counter() - t0)
    e = m // 2 if excl is None else excl
    cnt = x.size - m + 1
    pairs = (cnt - e - 1) * (cnt - e) / 2
    dt = min(ts) if ts else float("nan")
    print(f"{name}: n={x.size} m={m} excl={e}: {dt*1e3:.2f} ms  {pairs/dt/1e9:.0f} GPair/s  "
          f"frac={pairs*6/dt/34.19e12:.3f}  chk={np.sum(P.values):.12e} {np.sum(P.indices)}", flush=True)
