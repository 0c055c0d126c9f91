"""Development: symmetric self-join against the oracle over exclusion widths (sentinel / value mismatches)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
os.environ["TSD_SYM"] = "1"
rng = np.random.default_rng(1)
for n, m in ((715, 130), (1500, 64), (3000, 32), (6000, 100)):
    t = np.cumsum(rng.standard_normal(n)); cnt = n - m + 1
    res = []
    for excl in sorted(set([m // 2, m, 2 * m, 200, 230, 250, 256, 260, 300, 384, 500, 511, 512, 513, 700, 1000, 2000, cnt - 40])):
        if excl >= cnt - 1: continue
        P = tsd.self_join(t, m, excl=excl); rv, ri = O.self_join(t, m, excl)
        s = int(np.sum(np.isfinite(P.values) != np.isfinite(rv)))
        f = np.isfinite(rv) & np.isfinite(P.values)
        v = int(np.sum(np.abs(P.values[f] - rv[f]) > 1e-6 * np.maximum(rv[f], 1e-9)))
        res.append((excl, s, v))
    print(f"n={n} m={m} cnt={cnt}: (excl, sentinel mismatches, value mismatches):", res, flush=True)
