"""Development: replay cases of the randomized batched/symmetric and learning tests (MODE SEED CASE)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2112_12965_b200 as tsd
from oracle import py_oracle as O
import test_parity_gpu as T
mode, seed, want = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if mode == "sym":
    rng = np.random.default_rng(2000 + seed)
    for case in range(3):
        m = int(rng.choice([4, 9, 16, 33, 64, 130])); kind = int(rng.integers(0, 3)); nseg = int(rng.integers(1, 6))
        lens = [int(m + rng.integers(0, 400)) for _ in range(nseg)]
        for L in lens: rng.integers(0, 30)
        segs = [T._random_series(rng, L, kind) for L in lens]
        series = [T._random_series(rng, int(m + rng.integers(0, 900)), kind) for _ in range(int(rng.integers(1, 8)))]
        t = T._random_series(rng, int(2 * m + rng.integers(300, 6000)), kind)
        excl = int(rng.choice([m // 2, m // 4, 0, 3 * m]))
        if len(t) - m + 1 <= excl + 1: excl = m // 2
        if case != want: continue
        cnt = len(t) - m + 1
        print("m", m, "n", len(t), "cnt", cnt, "excl", excl, "kind", kind)
        rv, ri = O.self_join(t, m, excl)
        for sym in ("1", "0"):
            os.environ["TSD_SYM"] = sym
            P = tsd.self_join(t, m, excl=excl)
            bad = np.nonzero(np.isfinite(P.values) != np.isfinite(rv))[0]
            print("TSD_SYM", sym, "sentinel mismatches:", len(bad), bad[:10], "oracle inf rows", np.nonzero(~np.isfinite(rv))[0][[0, -1]] if (~np.isfinite(rv)).any() else None)
            for i in bad[:5]:
                print("  row", i, "gpu", P.values[i], P.indices[i], "oracle", rv[i], ri[i], "flat?", tsd.compute_stats(t, m).constant_mask[i])
else:
    rng = np.random.default_rng(3000 + seed)
    for case in range(3):
        n = int(rng.integers(1500, 9000)); m = int(rng.choice([16, 40, 64, 100])); k = float(rng.choice([1.0, 1.5, 2.5]))
        t = np.cumsum(rng.standard_normal(n)); rule = int(rng.integers(0, 3))
        value = [float(rng.choice([0.5, 0.8, 0.95])), float(rng.integers(4 * m, n // 2)), float(rng.choice([0.5, 2.0]))][rule]
        if case != want: continue
        cfg = tsd.LearnConfig(m=m, k=k)
        if rule == 0: cfg.space_saving_target = value
        elif rule == 1: cfg.sample_budget = int(value)
        else: cfg.error_target = value
        R = O.ref_learn_dictionary_full(t, m, k, rule, value); D = tsd.learn_dictionary(t, cfg)
        rc, gc = [int(x) for x in R["cores"]], D.core_starts
        print("n", n, "m", m, "k", k, "rule", rule, "value", value, "| ref picks", len(rc), "gpu picks", len(gc))
        d = next((i for i, (a, b) in enumerate(zip(rc, gc)) if a != b), min(len(rc), len(gc)))
        print("first difference at pick", d, "ref", rc[d:d + 3], "gpu", gc[d:d + 3], "e_max ref", R["e_max"], "gpu", D.e_max)
if mode == "sym":
    os.environ.pop("TSD_SYM", None)
    c, j = tsd.self_join_partial(t, m, excl, 0, 1)
    print("partials: rows without a candidate:", np.nonzero(j < 0)[0][[0, -1]], "count", int((j < 0).sum()),
          "| rows 110..120 cols", j[110:120], "| rows 190..198", j[190:198])
    for e2 in (389, 390, 391, 392, 400, 383, 384, 352):
        os.environ["TSD_SYM"] = "1"
        P = tsd.self_join(t, m, excl=e2); rv2, _ = O.self_join(t, m, e2)
        bad = np.nonzero(np.isfinite(P.values) != np.isfinite(rv2))[0]
        print("excl", e2, "sentinel mismatches", len(bad), (bad[0], bad[-1]) if len(bad) else "")
if mode == "sym":
    os.environ["TSD_SYM"] = "1"; os.environ["TSD_SELF_SEEDS"] = "0"
    c, j = tsd.self_join_partial(t, m, excl, 0, 1)
    rv, ri = O.self_join(t, m, excl)
    print("rows 0..194: partial col == oracle idx:", int(np.sum(j[:195] == ri[:195])), "of 195; oracle idx range of rows 100..194:", ri[100:195].min(), ri[100:195].max())
    print("partial cols rows 0..20:", j[:20], "oracle:", ri[:20])
    print("rows 391..585 (lower triangle side) partial ok:", int(np.sum(j[391:] == ri[391:])), "of", cnt - 391, "; missing:", int(np.sum(j[391:] < 0)))
