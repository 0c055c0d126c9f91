"""Parity under every number bench.py prints: the BASELINE configs at their
full sizes, checked against the oracle on >= 1000 sampled rows (contiguous
blocks and single rows at random positions, plus a prefix), and the
symmetric self-join's flat-window rule (profiles.hpp:289-296).

Oracle row sampling (SURVEY 8(c) flavour 4): a block of B query rows starting
at i0 is exactly the dictionary join of q[i0 : i0+B+m-1] (dictionary.hpp:
149-193 restated by oracle/tsd_oracle.c); a block of self-join rows is
tsdo_self_join_rows (profiles.hpp:266-301 restricted to those rows). Oracle
calls run on host threads (ctypes releases the GIL).
"""
import os

import numpy as np
import pytest

import paper_2112_12965_b200 as tsd
import workloads as W
from oracle import py_oracle as O
from parity import check_blocks, check_profile, dict_dist, ab_dist, report

pytestmark = pytest.mark.gpu


def _dict_blocks(q, segs, starts, m, P_val, P_idx, blocks):
    """oracle dictionary join of each (i0, B) row block -> check_blocks input"""
    segs = list(segs)

    def one(i0, B):
        rv, ri = O.dict_join(q[i0:i0 + B + m - 1], segs, starts, m)
        return (np.arange(i0, i0 + B), P_val[i0:i0 + B], P_idx[i0:i0 + B], rv, ri)
    return O.parallel(one, blocks)


def _sample_blocks(n, rng, nblocks, B, nsingle, prefix=0):
    out = [(0, prefix)] if prefix else []
    out += [(int(i), B) for i in rng.choice(n - B, nblocks, replace=False)]
    out += [(int(i), 1) for i in rng.choice(n, nsingle, replace=False)]
    out += [(n - 1, 1)]
    return out


def _c4_check(precision):
    cfg = W.c4()
    q, segs, starts, m = cfg["q"], cfg["segs"], cfg["starts"], cfg["m"]
    P = tsd.join_dictionary(q, W.dictionary(cfg), m, precision=precision)
    n = q.size - m + 1
    assert P.values.shape == (n,) and np.all(np.isfinite(P.values))
    assert np.all(P.indices % 1024 <= 1024 - m), "an index points at a straddling window"
    rng = np.random.default_rng(11 if precision == "fp64" else 12)
    # 16384-row prefix (the reference's first query block) + 16 x 48 rows + 256 single rows
    blocks = [(b, 1024) for b in range(0, 16384, 1024)]
    blocks += _sample_blocks(n, rng, 16, 48, 256)
    res = _dict_blocks(q, segs, starts, m, P.values, P.indices, blocks)
    st = check_blocks(f"C4 {precision} full size", res, m, dict_dist(q, list(segs), starts, m),
                      fp32=precision == "fp32")
    assert st["rows"] >= 16384 + 1000
    return st


def test_C4_fp64_full_size_sampled_rows_and_prefix():
    """BASELINE C4 (the bench's headline line), FP64: the first 16384 rows and
    >= 1000 random rows against the oracle at 1e-8 relative"""
    _c4_check("fp64")


def test_C4_fp32_full_size_sampled_rows_and_prefix():
    """BASELINE C4 in the FP32 mode (the bench's fp32 line): the same rows at
    1e-3 absolute on distance, indices by the FP32 rule"""
    _c4_check("fp32")


def test_self_join_2p21_m512_sampled_row_blocks():
    """the bench's self_2^21_m512 line: the 2^21 prefix of the C4 query, m = 512,
    excl = m/2, through the default path (symmetric upper-triangle sweep with
    coarse-search seeds); 16 blocks x 64 rows plus the first and last rows
    against the oracle"""
    m = 512
    x = np.ascontiguousarray(W.c4()["q"][: 1 << 21])
    P = tsd.self_join(x, m)
    cnt = x.size - m + 1
    rng = np.random.default_rng(21)
    blocks = [(0, 64), (cnt - 64, 64)] + [(int(i), 64) for i in rng.choice(cnt - 64, 16, replace=False)]

    def one(i0, B):
        rv, ri = O.self_join_rows(x, m, i0, B)
        return (np.arange(i0, i0 + B), P.values[i0:i0 + B], P.indices[i0:i0 + B], rv, ri)
    res = O.parallel(one, blocks)
    st = check_blocks("self 2^21 m512", res, m, ab_dist(x, x, m))
    assert st["rows"] >= 1000 + 128


def test_C2_full_size_against_oracle():
    """BASELINE C2 at full size (ECG-like, n = 131072, m = 250, excl = m/4 = 62):
    every row against the oracle (the reference's self_join with the one
    exclusion constant changed, run on all host cores)"""
    cfg = W.c2()
    t, m, excl = cfg["t"], cfg["m"], cfg["excl"]
    P = tsd.self_join(t, m, excl=excl)
    rv, ri = O.self_join_mt(t, m, excl)
    check_profile(P.values, P.indices, rv, ri, m, ab_dist(t, t, m), label="C2 full")


def test_C5_full_batch_sampled_series_and_rows():
    """BASELINE C5 at full size (4096 series x 8192, one device pass): 4 whole
    series plus 40 blocks of 32 rows from random series against the oracle"""
    cfg = W.c5()
    series, segs, starts, m = cfg["series"], cfg["segs"], cfg["starts"], cfg["m"]
    outs = tsd.join_dictionary_batched(list(series), W.dictionary(cfg), m)
    assert len(outs) == series.shape[0]
    rng = np.random.default_rng(5)
    whole = [0, 4095] + [int(k) for k in rng.choice(4094, 2, replace=False) + 1]
    cnt = 8192 - m + 1
    picks = [(int(k), int(i)) for k, i in zip(rng.choice(4096, 40), rng.choice(cnt - 32, 40))]

    def one(k, i0, B):
        rv, ri = O.dict_join(series[k][i0:i0 + B + m - 1], segs, starts, m)
        return (np.arange(i0, i0 + B), outs[k].values[i0:i0 + B], outs[k].indices[i0:i0 + B], rv, ri)
    res = O.parallel(one, [(k, 0, cnt) for k in whole] + [(k, i, 32) for k, i in picks])
    for (k, _, _), r in zip([(k, 0, cnt) for k in whole], res[:len(whole)]):
        check_profile(r[1], r[2], r[3], r[4], m, dict_dist(series[k], segs, starts, m), label=f"C5 series {k}")
    rows = 0
    for (k, i0), r in zip(picks, res[len(whole):]):
        rows += check_profile(r[1], r[2], r[3], r[4], m, lambda a, j, k=k, i0=i0: dict_dist(
            series[k], segs, starts, m)(i0 + a, j), label=f"C5 series {k} rows {i0}+32")["rows"]
    assert rows + len(whole) * cnt >= 1000


def test_C3_pipeline_learn_join_discords():
    """BASELINE C3 end to end: learn the dictionary from the C2 series (m = 200,
    2048-sample contexts, sample budget 65536) on the device, join the 2^20-
    sample anomalous ECG query against it, report the top-20 discords.
    Learning against the reference's own learn_dictionary (identical picks,
    segments, space saving; e_max by the join rule), the join against the
    oracle on >= 1000 rows, the discords against the reference's
    find_discords on the same profile."""
    cfg = W.c3()
    q, train, m = cfg["q"], cfg["train"], cfg["m"]
    D = tsd.learn_dictionary(train, W.c3_learn_config())
    assert D.stored_samples() >= cfg["budget"] and not D.no_progress
    if O.ref_available():
        r = O.ref_learn_dictionary_full(train, m, k=cfg["k"], rule=1, value=cfg["budget"])
        assert D.core_starts == [int(c) for c in r["cores"]], "C3: greedy picks differ from the reference"
        assert [s.start for s in D.segments] == [int(s) for s in r["starts"]]
        assert [s.length() for s in D.segments] == [int(s) for s in r["lengths"]]
        assert abs(D.space_saving - r["space_saving"]) <= 1e-12
        assert abs(D.e_max - r["e_max"]) <= max(1e-8 * r["e_max"], 2e-5)
    P = tsd.join_dictionary(q, D, m)
    segs = [s.values for s in D.segments]
    starts = [s.start for s in D.segments]
    n = q.size - m + 1
    rng = np.random.default_rng(3)
    blocks = _sample_blocks(n, rng, 12, 64, 200, prefix=2048)
    res = _dict_blocks(q, segs, starts, m, P.values, P.indices, blocks)
    st = check_blocks("C3 join", res, m, dict_dist(q, segs, starts, m))
    assert st["rows"] >= 1000
    disc = tsd.find_discords(P, D.e_max, cfg["top_k"])
    assert len(disc) == cfg["top_k"]
    if O.ref_available():
        rs, rsc, rc = O.ref_find_discords(P.values, m, D.e_max, cfg["top_k"])
        assert [d.start for d in disc] == [int(s) for s in rs]
        assert [d.score for d in disc] == [float(s) for s in rsc]
        assert [d.certified for d in disc] == [bool(c) for c in rc]
    # detection quality (reported, not a parity criterion): discords within a
    # beat of an injected anomaly
    an = np.asarray(cfg["anomalies"])
    hits = sum(bool(np.any(np.abs(an - d.start) <= 300)) for d in disc)
    report({"label": "C3 discords", "top_k": len(disc), "near_injected_anomaly": int(hits),
            "segments": len(D.segments), "stored": D.stored_samples(), "e_max": D.e_max})


# ------------------------------------------------------------- flat windows, symmetric sweep
def _flat_cases():
    rng = np.random.default_rng(77)
    out = []
    m = 16
    # n = 2m, T[0:3m/2) constant: the last row's only admissible neighbours
    # (windows 0 .. m/2-1) are flat -> c = 0 at window 0, d = sqrt(2m)
    t = rng.standard_normal(2 * m)
    t[: 3 * m // 2] = 1.25
    out.append((t, m))
    # long flat runs between short noise stretches: non-flat rows whose
    # admissible non-flat neighbours are few (and often all anti-correlated)
    for s in range(6):
        t = rng.standard_normal(400)
        t[40:200] = -0.5
        t[260 + 10 * s: 330 + 10 * s] = 2.0
        out.append((t, 24))
    return out


@pytest.mark.parametrize("sym", ["1", "0"])
def test_self_join_flat_lower_neighbours(monkeypatch, sym):
    """a non-flat row's flat neighbours below its exclusion zone give c = 0
    (profiles.hpp:289-296): the symmetric sweep (TSD_SYM=1), whose column
    side skips flat rows, and the full-matrix sweep against the oracle"""
    monkeypatch.setenv("TSD_SYM", sym)
    hit = 0
    for t, m in _flat_cases():
        P = tsd.self_join(t, m)
        rv, ri = O.self_join(t, m)
        check_profile(P.values, P.indices, rv, ri, m, ab_dist(t, t, m), label=f"flat self sym={sym}")
        _, _, _, fl = O.compute_stats(t, m)
        cnt = t.size - m + 1
        # rows whose answer is a flat window below them at c = 0
        hit += int(np.sum([(not fl[i]) and ri[i] >= 0 and ri[i] < i - m // 2 and fl[ri[i]] for i in range(cnt)]))
    assert hit > 0, "no row exercised the flat-lower-neighbour rule"


def test_learn_dictionary_flat_series_vs_reference():
    """learn_dictionary (which always runs the symmetric sweep) on series with
    long flat runs: identical picks to the reference's own learn_dictionary"""
    if not O.ref_available():
        pytest.skip("reference build absent")
    # one flat run per series: two runs would make the single-outlier windows
    # at their edges identical after z-normalisation (exact ties of P that
    # rounding orders either way)
    rng = np.random.default_rng(78)
    cases = []
    for s in range(5):
        t = rng.standard_normal(400 + 20 * s)
        t[60 + 15 * s: 230 + 15 * s] = 0.75
        cases.append((t, 24))
    for t, m in cases:
        for rule, value in ((0, 0.5), (1, 120)):
            cfg = tsd.LearnConfig(m=m, k=1.5)
            if rule == 0:
                cfg.space_saving_target = value
            else:
                cfg.sample_budget = value
            D = tsd.learn_dictionary(t, cfg)
            r = O.ref_learn_dictionary_full(t, m, k=1.5, rule=rule, value=value)
            assert D.core_starts == [int(c) for c in r["cores"]]
            assert [s.start for s in D.segments] == [int(s) for s in r["starts"]]
            assert abs(D.e_max - r["e_max"]) <= max(1e-8 * r["e_max"], 2e-5)
