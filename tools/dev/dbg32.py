import sys, numpy as np
import os; R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, R)
import paper_2112_12965_b200 as tsd
from paper_2112_12965_b200 import synth
from oracle import py_oracle as O
m = 32
t = np.arange(6000)
q = np.sin(2 * np.pi * t / 97.0) + 0.01 * synth.Rng(41).noise(6000)
anti = -np.sin(2 * np.pi * np.arange(700) / 97.0)
flat_head = np.concatenate([np.full(40, 3.0), anti[:300]])
single = anti[5:5 + m]
rep = np.tile(q[100:100 + 97], 5)
segs = [anti, flat_head, single, rep]
starts = [0, 1000, 2000, 3000]
for sub in ([3], [0], [1], [2], [0, 3], [0,1,2], [0,1,2,3]):
    ss = [segs[k] for k in sub]; st = [starts[k] for k in sub]
    D = tsd.Dictionary([tsd.Segment(a, s) for s, a in zip(ss, st)], m=m, source_length=max(a + len(s) for s, a in zip(ss, st)))
    P = tsd.join_dictionary(q, D, m, precision="fp32")
    P64 = tsd.join_dictionary(q, D, m, precision="fp64")
    rv, ri = O.dict_join(q, ss, st, m)
    e = np.abs(P.values - rv); i = int(np.argmax(e))
    print(sub, f"fp32 maxerr {e.max():.3g} at row {i}: got {P.values[i]:.6f} idx {P.indices[i]} oracle {rv[i]:.6f} idx {ri[i]}; fp64 err {np.max(np.abs(P64.values-rv)):.3g}")
