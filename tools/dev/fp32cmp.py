"""FP32 sweep A/B check (development tool): TSD_LIB_B vs the default library,
bitwise, on several shapes. usage: TSD_LIB_B=... python tools/fp32cmp.py"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
cases = []
q = synth.walk(4, 300000); segs = synth.walks(5, 16, 1024)
cases.append(("dict", lambda: t.join_dictionary(q, t.Dictionary([t.Segment(1024 * s, segs[s]) for s in range(16)], m=512, source_length=16 * 1024), 512, precision="fp32")))
x = synth.walk(7, 70000)
cases.append(("self", lambda: t.self_join(x, 128, precision="fp32")))
a = synth.walk(8, 50000); b = synth.walk(9, 40000)
cases.append(("ab", lambda: t.ab_join(a, b, 100, precision="fp32")))
e = synth.ecg(2, 131072)[0]
cases.append(("ecg", lambda: t.self_join(e, 250, excl=62, precision="fp32")))
res = {k: f() for k, f in cases}
lib_b = os.environ["TSD_LIB_B"]
t._lib = None; t.LIB_PATH = lib_b
res_b = {k: f() for k, f in cases}
for k in res:
    A, B = res[k], res_b[k]
    print(k, "idx equal" if np.array_equal(A.indices, B.indices) else f"idx diff {np.sum(A.indices != B.indices)}",
          "vals equal" if np.array_equal(A.values, B.values) else f"max |dv| {np.max(np.abs(A.values - B.values)):.3g}", flush=True)
