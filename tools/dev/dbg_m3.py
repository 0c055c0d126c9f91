"""debug tiny-window AB-join mismatches (development tool)"""
import sys, os
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, R); sys.path.insert(0, R + "/tests")
import numpy as np
import paper_2112_12965_b200 as tsd
from paper_2112_12965_b200 import synth
from oracle import py_oracle as O
a, b = synth.walk(81, 700), synth.walk(82, 500)
for m in (3, 2):
    P = tsd.ab_join(a, b, m)
    rv, ri = O.ab_join(a, b, m)
    bv, bi = O.ab_join_brute(a, b, m)
    d = np.abs(P.values - rv)
    bad = np.argsort(-d)[:4]
    for i in bad:
        print(f"m={m} row {i}: gpu ({P.values[i]:.3e}, {P.indices[i]}) oracle ({rv[i]:.3e}, {ri[i]}) brute ({bv[i]:.3e}, {bi[i]}) "
              f"pair(gpu idx)={O.pair_dist(a, i, b, P.indices[i], m):.3e} pair(oracle idx)={O.pair_dist(a, i, b, ri[i], m):.3e}")
    print("max |gpu-brute|", np.max(np.abs(P.values - bv)), "max |oracle-brute|", np.max(np.abs(rv - bv)))
