"""Development: FP32-mode distance error over the randomized shapes of
tests/test_parity_gpu.py::test_randomized_shapes_vs_oracle (no assertion)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
import test_parity_gpu as T
for seed in range(8):
    rng = np.random.default_rng(1000 + seed)
    for case in range(5):
        m = int(rng.choice([2, 3, 5, 8, 16, 31, 64, 100, 257]))
        nseg = int(rng.integers(1, 9))
        lens = [int(m + rng.integers(0, 600)) for _ in range(nseg)]
        gaps = [int(rng.integers(0, 50)) for _ in range(nseg)]
        starts, pos = [], 0
        for L, g in zip(lens, gaps):
            pos += g; starts.append(pos); pos += L
        kind = int(rng.integers(0, 3))
        segs = [T._random_series(rng, L, kind) for L in lens]
        nq = int(m + rng.integers(0, 1500))
        q = T._random_series(rng, nq, kind)
        rv, ri = O.dict_join(q, segs, starts, m)
        P32 = tsd.join_dictionary(q, T._dict(segs, starts, m), m, precision="fp32")
        P64 = tsd.join_dictionary(q, T._dict(segs, starts, m), m)
        e32 = np.abs(P32.values - rv); e64 = np.abs(P64.values - rv) / np.maximum(rv, 1e-300)
        st = tsd.compute_stats(q, m)
        rng_q = float(np.max(st.stds[st.stds > 0]) / np.min(st.stds[st.stds > 0])) if np.any(st.stds > 0) else 0
        print(f"seed {seed}.{case} m={m:3d} kind={kind} nq={nq:5d} nseg={nseg}  fp32 max abs {e32.max():.2e} (rows>1e-3: {(e32>1e-3).sum()})  fp64 max rel {e64.max():.1e}  query std range {rng_q:.1e}", flush=True)
        # consume the same random numbers as the test (ab / self draw excl)
        if nq >= 2 * m:
            rng.choice([m // 2, m // 4, 0])
