import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
from oracle import py_oracle as O
for (nq, nseg, L, m) in [(20000, 8, 512, 100), (60000, 16, 1024, 512), (50000, 4, 4096, 64)]:
    q = synth.walk(4, nq); segs = synth.walks(5, nseg, L)
    D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
    P = t.join_dictionary(q, D, m, precision="fp32")
    P64 = t.join_dictionary(q, D, m)
    d = np.abs(P.values - P64.values)
    mism = np.nonzero(P.indices != P64.indices)[0]
    print(f"fp32 {nq}x{nseg}x{L} m{m}: max|dd| vs fp64 {d.max():.3g}, idx mismatches {len(mism)}", flush=True)
a = synth.walk(7, 30000); b = synth.walk(8, 20000)
P = t.ab_join(a, b, 128, precision="fp32"); P64 = t.ab_join(a, b, 128)
print("ab fp32 long B:", np.abs(P.values - P64.values).max(), (P.indices != P64.indices).sum())
T = synth.walk(9, 20000)
P = t.self_join(T, 100, precision="fp32"); P64 = t.self_join(T, 100)
print("self fp32:", np.abs(P.values - P64.values).max(), (P.indices != P64.indices).sum())
