"""Development: window statistics of one randomized case (SEED) against the reference and a long-double two-pass."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
import test_parity_gpu as T
seed = int(sys.argv[1])
rng = np.random.default_rng(4000 + seed)
kind = int(rng.integers(0, 3)); m = int(rng.choice([2, 3, 7, 16, 50, 128, 300])); n = int(m + rng.integers(1, 6000))
x = T._random_series(rng, n, kind)
st = tsd.compute_stats(x, m); mu, sd, iv, fl = O.ref_compute_stats(x, m)
w = np.lib.stride_tricks.sliding_window_view(x.astype(np.longdouble), m)
mean = w.mean(axis=1); sdx = np.sqrt(((w - mean[:, None]) ** 2).mean(axis=1))
nz = iv > 0
rg = np.abs(st.stds[nz] - sdx[nz]) / sdx[nz]; rr = np.abs(sd[nz] - sdx[nz]) / sdx[nz]
print(f"n={n} m={m} kind={kind}: std relative error vs long double: GPU max {float(rg.max()):.2e}, reference max {float(rr.max()):.2e}; "
      f"invn GPU-vs-ref max rel {np.max(np.abs(st.invn[nz]-iv[nz])/iv[nz]):.2e}")
