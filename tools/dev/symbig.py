"""Development: a large symmetric self-join (auto-selected sweep, coarse seeds) with wide exclusion zones
against oracle row blocks."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
from parity import check_profile, ab_dist
rng = np.random.default_rng(9)
n, m = 300000, 256
t = np.cumsum(rng.standard_normal(n)); cnt = n - m + 1
for excl in (128, 5000, 100000, 280000):
    t0 = time.perf_counter(); P = tsd.self_join(t, m, excl=excl); dt = time.perf_counter() - t0
    tot = 0
    for r0 in (0, 40000, 70000 - 128, cnt - 256):
        rv, ri = O.self_join_rows(t, m, r0, 256, excl)
        st = check_profile(P.values[r0:r0 + 256], P.indices[r0:r0 + 256], rv, ri, m, lambda i, j, r0=r0: ab_dist(t, t, m)(i + r0, j),
                           label=f"big sym excl={excl} rows {r0}", truth=True)
        tot += st["rows"]
    print(f"excl={excl}: {dt*1e3:.1f} ms, {tot} rows checked, sentinel rows {int(np.sum(~np.isfinite(P.values)))}", flush=True)
