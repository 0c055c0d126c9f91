"""Development: FP32 dictionary-join rows outside tolerance in a case of test_randomized_shapes_vs_oracle (SEED CASE)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
import test_parity_gpu as T
from parity import dict_dist
seed, want = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1000 + seed)
for case in range(5):
    big = 8 if case == 4 else 1
    m = int(rng.choice([2, 3, 5, 8, 16, 31, 64, 100, 257])); nseg = int(rng.integers(1, 9))
    lens = [int(m + rng.integers(0, 600 * big)) for _ in range(nseg)]
    gaps = [int(rng.integers(0, 50)) for _ in range(nseg)]
    starts, pos = [], 0
    for L, g in zip(lens, gaps):
        pos += g; starts.append(pos); pos += L
    kind = int(rng.integers(0, 3))
    segs = [T._random_series(rng, L, kind) for L in lens]
    nq = int(m + rng.integers(0, 1500 * big)); q = T._random_series(rng, nq, kind)
    if nq >= 2 * m: rng.choice([m // 2, m // 4, 0])
    if case != want: continue
    os.environ["TSD_VERBOSE"] = "1"
    rv, ri = O.dict_join(q, segs, starts, m); P = tsd.join_dictionary(q, T._dict(segs, starts, m), m, precision="fp32")
    dist = dict_dist(q, segs, starts, m); st = tsd.compute_stats(q, m)
    bad = np.nonzero(np.abs(P.values - rv) > 1e-3)[0]
    print("m", m, "nq", nq, "kind", kind, "lens", lens, "q span", T._norm_span(q, m), "seg spans", [round(T._norm_span(s, m), 1) for s in segs], "bad rows", bad)
    for i in bad[:4]:
        print(f" row {i}: fp32 idx {P.indices[i]} d {P.values[i]:.6f} (exact {dist(int(i), int(P.indices[i])):.6f}); oracle idx {ri[i]} d {rv[i]:.6f}; row std {st.stds[i]:.3g}")
