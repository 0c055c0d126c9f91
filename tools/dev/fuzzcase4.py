"""Development: replay the batched join of a test_randomized_batched_symmetric_and_sharded case (SEED CASE)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
import test_parity_gpu as T
from parity import dict_dist
seed, want = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(2000 + seed)
for case in range(3):
    m = int(rng.choice([4, 9, 16, 33, 64, 130])); kind = int(rng.integers(0, 3)); nseg = int(rng.integers(1, 6))
    lens = [int(m + rng.integers(0, 400)) for _ in range(nseg)]
    starts, pos = [], 0
    for L in lens:
        pos += int(rng.integers(0, 30)); starts.append(pos); pos += L
    segs = [T._random_series(rng, L, kind) for L in lens]
    series = [T._random_series(rng, int(m + rng.integers(0, 900)), kind) for _ in range(int(rng.integers(1, 8)))]
    t = T._random_series(rng, int(2 * m + rng.integers(300, 6000)), kind); rng.choice([m // 2, m // 4, 0, 3 * m])
    if case != want: continue
    D = T._dict(segs, starts, m)
    outs = tsd.join_dictionary_batched(series, D, m)
    print("m", m, "kind", kind, "series lengths", [len(s) for s in series], "max|x| per series", [float(np.max(np.abs(s))) for s in series])
    for k, q in enumerate(series):
        rv, ri = O.dict_join(q, segs, starts, m); single = tsd.join_dictionary(q, D, m)
        dist = dict_dist(q, segs, starts, m)
        eb = np.abs(outs[k].values - rv); es = np.abs(single.values - rv)
        i = int(np.argmax(eb))
        print(f" series {k}: batched max |dd| {eb.max():.2e} at row {i} (d_ref {rv[i]:.4g}, exact {dist(i, int(ri[i])):.6g}, batched {outs[k].values[i]:.6g}); alone max |dd| {es.max():.2e}; norm span {T._norm_span(q, m):.3g}")
