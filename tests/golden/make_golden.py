"""Generate tests/golden/reference_cases.npz from the UNMODIFIED reference.

Runs in the build container only (needs /root/reference, compiled into
oracle/_ref/libtsdict_ref.so by oracle/Makefile). Inputs are drawn with the
reference's own tests/synth.hpp generators (replaying the seeds and draw
order of the reference tests cited per case); outputs come from the
reference's own functions. The fixture is committed; tests read it on any box.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import py_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_cases.npz")


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libtsdict_ref.so missing: run `make -C oracle` with /root/reference present")
    d = {}
    cases = []

    def stats_case(name, x, m):
        mu, sd, iv, fl = O.ref_compute_stats(x, m)
        d[f"{name}__x"], d[f"{name}__m"] = x, np.int64(m)
        d[f"{name}__means"], d[f"{name}__stds"], d[f"{name}__invn"], d[f"{name}__flat"] = mu, sd, iv, fl
        cases.append(("stats", name))

    def ab_case(name, a, b, m):
        v, i = O.ref_ab_join(a, b, m, threads=3)
        d[f"{name}__a"], d[f"{name}__b"], d[f"{name}__m"] = a, b, np.int64(m)
        d[f"{name}__val"], d[f"{name}__idx"] = v, i
        cases.append(("ab", name))

    def self_case(name, t, m):
        v, i = O.ref_self_join(t, m, threads=3)
        d[f"{name}__t"], d[f"{name}__m"] = t, np.int64(m)
        d[f"{name}__val"], d[f"{name}__idx"] = v, i
        cases.append(("self", name))

    def dict_case(name, q, segs, starts, m):
        v, i = O.ref_join_dictionary(q, segs, starts, m, threads=3)
        d[f"{name}__q"], d[f"{name}__m"] = q, np.int64(m)
        d[f"{name}__seg_vals"] = np.concatenate(segs)
        d[f"{name}__seg_len"] = np.asarray([len(s) for s in segs], dtype=np.int64)
        d[f"{name}__seg_start"] = np.asarray(starts, dtype=np.int64)
        d[f"{name}__val"], d[f"{name}__idx"] = v, i
        cases.append(("dict", name))

    def learn_case(name, t, m, k, rule, value, max_iterations=1000000):
        r = O.ref_learn_dictionary_full(t, m, k, rule, value, max_iterations, threads=3)
        d[f"{name}__t"], d[f"{name}__m"], d[f"{name}__k"] = t, np.int64(m), np.float64(k)
        d[f"{name}__rule"], d[f"{name}__value"] = np.int64(rule), np.float64(value)
        for key, v in r.items():
            d[f"{name}__{key}"] = np.asarray(v)
        cases.append(("learn", name))

    # stats (test_series.cpp:42-69, :94-105)
    r = O.RefRng(101)
    stats_case("stats_noise2048_m64", r.noise(2048), 64)
    r = O.RefRng(102)
    stats_case("stats_walk3000_m200", r.walk(3000), 200)
    stats_case("stats_scale_relative", np.array([5.0, 5.0, 5.0 + 1e-9, 5.0, 1.0, 9.0]), 4)
    stats_case("stats_constant", np.ones(4), 2)
    # ab-join (test_profiles.cpp:231-250, :293-301, :215-229, :252-264)
    r = O.RefRng(35)
    a = r.noise(300)
    ab_case("ab_noise_35", a, r.noise(200), 20)
    r = O.RefRng(36)
    for t in range(8):
        A = r.walk(220 + t * 17) if t % 2 == 0 else r.noise(180 + t * 23)
        B = r.noise(150 + t * 11) if t % 3 == 0 else r.walk(240 - t * 9)
        ab_case(f"ab_shapes_36_{t}", A, B, 8 + t * 5)
    r = O.RefRng(40)
    ab_case("ab_walk_40", r.walk(1500), r.walk(900), 40)
    r = O.RefRng(34)
    w = r.walk(300)
    ab_case("ab_same_content_34", w, w.copy(), 20)
    A = O.ref_sine(500, 50.0)
    A[230:250] += 6.0
    ab_case("ab_planted_spike_37", A, O.ref_sine(600, 50.0), 25)
    # self-join (test_profiles.cpp:137-193, :206-213)
    r = O.RefRng(28)
    self_case("self_noise_28", r.noise(256), 16)
    r = O.RefRng(29)
    for t in range(8):
        n, m = 64 + t * 48, 8 + t * 3
        T = r.walk(n) if t % 2 == 0 else r.noise(n)
        if t == 5:
            T[20:60] = 1.25  # flat stretch (:162)
        self_case(f"self_shapes_29_{t}", T, m)
    r = O.RefRng(31)
    self_case("self_min_length_31", r.noise(16), 8)
    r = O.RefRng(33)
    self_case("self_walk_33", r.walk(2048), 50)
    r = O.RefRng(27)
    half = r.walk(512)
    self_case("self_repeated_27", np.concatenate([half, half]), 64)
    # dictionary joins (test_dict_join.cpp:48-81)
    r = O.RefRng(70)
    B = r.walk(600)
    A = r.walk(400)
    dict_case("dict_single_full_segment_70", A, [B], [0], 50)
    r = O.RefRng(71)
    B = r.walk(800)
    A = r.walk(300)
    segs, starts, _ = O.ref_learn_dictionary(B, 40, 0.6)
    dict_case("dict_learned_71", A, segs, starts, 40)
    r = O.RefRng(75)
    B = r.walk(900)
    A = r.walk(500)
    segs, starts, _ = O.ref_learn_dictionary(B, 60, 0.0)
    dict_case("dict_zero_saving_75", A, segs, starts, 60)
    # BASELINE configs[0] (C1): walk seed 0 (16384) vs 8 walks of 512 (seed 1), m = 100
    q = O.RefRng(0).walk(16384)
    rs = O.RefRng(1)
    segs = [rs.walk(512) for _ in range(8)]
    dict_case("dict_C1", q, segs, [512 * s for s in range(8)], 100)
    # greedy learning, every stop rule (test_dictionary.cpp:250-400 shapes):
    # space saving, sample budget, error target, k = 0, no progress
    learn_case("learn_saving_walk_80", O.RefRng(80).walk(3000), 50, 1.5, 0, 0.5)
    learn_case("learn_budget_walk_81", O.RefRng(81).walk(2500), 60, 1.5, 1, 700)
    learn_case("learn_error_walk_82", O.RefRng(82).walk(2000), 60, 1.5, 2, 3.0)
    r = O.RefRng(83)
    per = np.sin(2 * np.pi * np.arange(4000) / 97.0) + 0.05 * r.noise(4000)
    learn_case("learn_saving_periodic_83", per, 100, 1.5, 0, 0.7)
    learn_case("learn_k0_budget_walk_84", O.RefRng(84).walk(1800), 40, 0.0, 1, 400)
    learn_case("learn_no_progress_85", O.RefRng(85).walk(1500), 100, 1.5, 1, 100000)
    learn_case("learn_zero_saving_86", O.RefRng(86).walk(900), 60, 1.5, 0, 0.0)
    # discords / labels / AUC (dict_join.hpp:54-165; test_dict_join.cpp shapes):
    # the C3-like reduced join profile with planted anomalies, a profile with
    # sentinel (+inf) rows and exact ties, a flat profile (vacuous runner-up)
    def discord_case(name, values, m, e_max, top_k):
        st, sc, ce = O.ref_find_discords(values, m, e_max, top_k)
        d[f"{name}__values"], d[f"{name}__m"] = np.asarray(values, dtype=np.float64), np.int64(m)
        d[f"{name}__e_max"], d[f"{name}__top_k"] = np.float64(e_max), np.int64(top_k)
        d[f"{name}__starts"], d[f"{name}__scores"], d[f"{name}__certified"] = st, sc, ce.astype(np.uint8)
        cases.append(("discords", name))

    rq = O.RefRng(120)
    q = rq.walk(6000)
    q[2000:2100] += 8.0 * np.sin(np.linspace(0, 3 * np.pi, 100))
    q[4500:4560] = q[4500]
    segs = [O.RefRng(121 + s).walk(700) for s in range(6)]
    v, _ = O.ref_join_dictionary(q, segs, [1000 * s for s in range(6)], 80, threads=3)
    discord_case("discords_planted_120", v, 80, 0.5, 20)
    discord_case("discords_planted_certify_120", v, 80, 1e-3, 5)
    w = np.abs(O.RefRng(122).noise(500))
    w[[10, 11, 300]] = np.inf
    w[[100, 400]] = 7.0
    discord_case("discords_inf_ties_122", w, 16, 0.1, 6)
    discord_case("discords_single_123", np.ones(30), 40, 0.0, 3)
    rl = O.RefRng(124)
    regions = [(100, 180), (170, 260), (900, 950), (1990, 2000)]
    lab = O.ref_window_labels(regions, 2000, 64)
    d["labels_124__lo"] = np.asarray([a for a, _ in regions], dtype=np.int64)
    d["labels_124__hi"] = np.asarray([b for _, b in regions], dtype=np.int64)
    d["labels_124__n"], d["labels_124__m"], d["labels_124__labels"] = np.int64(2000), np.int64(64), lab
    sc = np.round(rl.noise(lab.size), 1)  # coarse scores: many ties
    d["labels_124__scores"], d["labels_124__auc"] = sc, np.float64(O.ref_auc_score(sc, lab))
    cases.append(("labels", "labels_124"))
    d["__cases__"] = np.asarray([f"{k}:{n}" for k, n in cases])
    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}: {len(cases)} cases, {os.path.getsize(OUT) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
