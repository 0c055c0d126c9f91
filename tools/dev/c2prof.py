"""BASELINE C2 self-join once (development tool): ECG n=131072, m=250, excl=62."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
x = synth.ecg(2, 131072)[0]
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    t0 = time.perf_counter(); P = t.self_join(x, 250, excl=62); print(f"{(time.perf_counter()-t0)*1e3:.2f} ms")
