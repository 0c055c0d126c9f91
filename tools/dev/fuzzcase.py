"""Development: one case of test_randomized_shapes_vs_oracle (SEED CASE): the self-join's rows where GPU and
oracle differ, both against the long-double brute-force distance."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
import test_parity_gpu as T
from parity import ab_dist
seed, want = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1000 + seed)
for case in range(5):
    m = int(rng.choice([2, 3, 5, 8, 16, 31, 64, 100, 257]))
    nseg = int(rng.integers(1, 9))
    lens = [int(m + rng.integers(0, 600)) for _ in range(nseg)]
    gaps = [int(rng.integers(0, 50)) for _ in range(nseg)]
    kind = int(rng.integers(0, 3))
    segs = [T._random_series(rng, L, kind) for L in lens]
    nq = int(m + rng.integers(0, 1500))
    q = T._random_series(rng, nq, kind)
    excl = int(rng.choice([m // 2, m // 4, 0])) if nq >= 2 * m else None
    if case != want:
        continue
    print("m", m, "nq", nq, "kind", kind, "excl", excl, "span", T._norm_span(q, m))
    rv, ri = O.self_join(q, m, excl)
    for env in ({}, {"TSD_FFT_HEADS": "0", "TSD_FFT_TOP": "0"}):
        os.environ.update(env)
        P = tsd.self_join(q, m, excl=excl)
        dist = ab_dist(q, q, m)
        bad = np.nonzero(np.abs(P.values - rv) > 1e-8 * rv)[0]
        print(env, "rows with rel diff > 1e-8:", len(bad))
        for i in bad[:12]:
            tg, tr = dist(int(i), int(P.indices[i])), dist(int(i), int(ri[i]))
            print(f"  row {i}: gpu d={P.values[i]:.12e} idx {P.indices[i]} (true {tg:.12e}, err {P.values[i]-tg:+.2e}) | "
                  f"oracle d={rv[i]:.12e} idx {ri[i]} (true {tr:.12e}, err {rv[i]-tr:+.2e})")
