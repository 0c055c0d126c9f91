"""exact-path frequency probe with the TSD_COUNT_EXACT build (development tool)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
n = 131072
for name, x in (("ecg", synth.ecg(2, n)[0]), ("walk", synth.walk(2, n)), ("noise", np.random.default_rng(2).standard_normal(n))):
    print(name, flush=True); t.self_join(x, 250, excl=62)
print("ab walk 1M x 262144 m=512", flush=True)
t.ab_join(synth.walk(4, 1 << 20), synth.walk(5, 1 << 18), 512)
