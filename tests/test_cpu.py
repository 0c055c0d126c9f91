"""CPU tests (no GPU): the oracle pinned to the reference's own outputs, the
C ABI library's exported surface and host-side validation, the generators,
and the multi-rank sharding logic (gloo, world_size 2)."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import paper_2112_12965_b200 as tsd
from paper_2112_12965_b200 import synth
from oracle import py_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- oracle pin
def test_oracle_restatement_is_bit_identical_to_reference(golden):
    """oracle/tsd_oracle.c vs the reference outputs in tests/golden (bit-exact)."""
    n = 0
    for name, (kind, c) in golden.items():
        m = int(c["m"])
        if kind == "stats":
            mu, sd, iv, fl = O.compute_stats(c["x"], m)
            assert np.array_equal(mu, c["means"]) and np.array_equal(sd, c["stds"]), name
            assert np.array_equal(iv, c["invn"]) and np.array_equal(fl, c["flat"]), name
        elif kind == "ab":
            v, i = O.ab_join(c["a"], c["b"], m)
            assert np.array_equal(v, c["val"]) and np.array_equal(i, c["idx"]), name
        elif kind == "self":
            v, i = O.self_join(c["t"], m)
            assert np.array_equal(v, c["val"]) and np.array_equal(i, c["idx"]), name
        elif kind == "dict":
            segs = np.split(c["seg_vals"], np.cumsum(c["seg_len"])[:-1])
            v, i = O.dict_join(c["q"], segs, c["seg_start"], m)
            assert np.array_equal(v, c["val"]) and np.array_equal(i, c["idx"]), name
        n += 1
    assert n >= 30


def test_oracle_matches_long_double_brute_force():
    """the restatement's streaming join vs tests/oracles.hpp-style brute force (1e-5, test_profiles.cpp:42)"""
    a, b = synth.Rng(35).noise(300), synth.Rng(36).noise(200)
    v, i = O.ab_join(a, b, 20)
    bv, bi = O.ab_join_brute(a, b, 20)
    assert np.max(np.abs(v - bv)) < 1e-5
    t = synth.Rng(28).noise(256)
    for excl in (None, 4):
        v, i = O.self_join(t, 16, excl)
        bv, bi = O.self_join_brute(t, 16, excl)
        assert np.max(np.abs(v - bv)) < 1e-5


def test_oracle_self_join_excl_parameter_reduces_to_reference():
    """excl = m/2 restatement == the reference's hard-coded self_join (profiles.hpp:273)"""
    if not O.ref_available():
        pytest.skip("reference build absent")
    t = synth.Rng(3).walk(1500)
    v, i = O.self_join(t, 50, 25)
    rv, ri = O.ref_self_join(t, 50)
    assert np.array_equal(v, rv) and np.array_equal(i, ri)


def test_oracle_threaded_and_row_block_self_joins():
    """the checker's two large-shape helpers: the thread-split self-join
    (run_diagonals, profiles.hpp:118-140) is bit-identical to the sequential
    one; row blocks started mid-series agree to rounding, flat stretches and
    both exclusion conventions included"""
    t = synth.ecg(5, 6000)[0]
    t[1000:1400] = 0.5  # flat rows and columns
    for excl in (None, 62, 0):
        v, i = O.self_join(t, 100, excl)
        mv, mi = O.self_join_mt(t, 100, excl, threads=5)
        assert np.array_equal(v, mv) and np.array_equal(i, mi)
        for r0, nr in ((0, 50), (900, 700), (5850, 100), (3000, 1)):
            bv, bi = O.self_join_rows(t, 100, r0, nr, excl)
            rv, ri = v[r0:r0 + bv.size], i[r0:r0 + bv.size]
            assert bv.size == min(nr, v.size - r0)
            assert np.allclose(bv, rv, rtol=1e-9, atol=1e-9)
            assert np.mean(bi == ri) > 0.99


@pytest.mark.skipif(not O.ref_available(), reason="reference build absent")
def test_generators_replay_reference_synth():
    """paper_2112_12965_b200.synth draws exactly what the reference's synth.hpp draws"""
    r1, r2 = synth.Rng(7), O.RefRng(7)
    assert np.array_equal(r1.walk(1000), r2.walk(1000))
    assert np.array_equal(r1.noise(777), r2.noise(777))
    assert np.array_equal(synth.sine(300, 50.0), O.ref_sine(300, 50.0))


def test_generators_are_seeded():
    assert np.array_equal(synth.walk(4, 1000), synth.walk(4, 1000))
    e1, a1 = synth.ecg(3, 20000, 5)
    e2, a2 = synth.ecg(3, 20000, 5)
    assert np.array_equal(e1, e2) and np.array_equal(a1, a2) and len(a1) == 5
    tr = synth.traffic(6, 3, 1000)
    assert tr.shape == (3, 1000) and np.isfinite(tr).all()
    w = synth.walks(5, 4, 100)
    assert np.array_equal(w[0], synth.Rng(5).walk(100))


# ---------------------------------------------------------------- C ABI surface
def _header_symbols():
    text = open(os.path.join(ROOT, "include", "tsdict_cuda.h")).read()
    return set(re.findall(r"\b(tsd_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = tsd.load_library()
    declared = _header_symbols()
    assert declared == set(tsd.C_SYMBOLS), declared ^ set(tsd.C_SYMBOLS)
    for name in declared:
        assert getattr(lib, name) is not None
    out = subprocess.run(["nm", "-D", "--defined-only", tsd.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tsd_\w+)", out))
    assert declared <= exported, declared - exported


def test_status_names_match_reference_errc():
    names = [tsd.load_library().tsd_status_name(k + 1).decode() for k in range(16)]
    assert names[:5] == ["WindowTooSmall", "WindowTooLarge", "NonFiniteInput", "LengthMismatch", "SeriesTooShort"]
    assert names[7:9] == ["WindowMismatch", "EmptyDictionary"] and names[15] == "InvalidArgument"


@pytest.mark.parametrize("call,code", [
    (lambda: tsd.ab_join(np.zeros(10), np.zeros(100), 20), tsd.errc.series_too_short),   # profiles.hpp:307-309
    (lambda: tsd.ab_join(np.zeros(10), np.zeros(10), 1), tsd.errc.window_too_small),     # series.hpp:85
    (lambda: tsd.self_join(np.zeros(15), 8), tsd.errc.series_too_short),                 # profiles.hpp:268-270
    (lambda: tsd.self_join(np.zeros(15), 0), tsd.errc.window_too_small),
    (lambda: tsd.compute_stats([1, 2, 3], 4), tsd.errc.window_too_large),                # series.hpp:86
    (lambda: tsd.compute_stats([1, 2, 3], 1), tsd.errc.window_too_small),
    (lambda: tsd.join_dictionary(np.zeros(50), tsd.Dictionary([], m=10), 10), tsd.errc.empty_dictionary),
    (lambda: tsd.join_dictionary(np.zeros(50), tsd.Dictionary([tsd.Segment(0, np.zeros(5))], m=10), 10),
     tsd.errc.window_mismatch),                                                            # dictionary.hpp:152-156
    (lambda: tsd.join_dictionary(np.zeros(5), tsd.Dictionary([tsd.Segment(0, np.zeros(50))], m=10), 10),
     tsd.errc.window_too_large),                                                           # dictionary.hpp:158
    (lambda: tsd.join_dictionary(np.zeros(50), tsd.Dictionary([tsd.Segment(0, np.zeros(50))], m=10), 11),
     tsd.errc.window_mismatch),                                                            # dict_join.hpp:44-46
    (lambda: tsd.compute_e_max(tsd.Dictionary([tsd.Segment(0, np.zeros(50))], m=10, source_length=60),
                               np.zeros(50)), tsd.errc.source_mismatch),                   # dictionary.hpp:248-250
    (lambda: tsd.distance_profile_naive(np.zeros(50), np.zeros(9), tsd.SubseqStats(10, *(np.zeros(41),) * 4)),
     tsd.errc.length_mismatch),                                                            # profiles.hpp:167-169
    (lambda: tsd.distance_profile_mass(np.zeros(50), np.zeros(10), tsd.SubseqStats(10, *(np.zeros(40),) * 4)),
     tsd.errc.length_mismatch),                                                            # profiles.hpp:192-194
])
def test_host_validation_matches_reference_error_codes(call, code):
    with pytest.raises(tsd.TsdictError) as ei:
        call()
    assert ei.value.code() == code
    assert str(ei.value).split(":")[0] in {"WindowTooSmall", "WindowTooLarge", "SeriesTooShort", "EmptyDictionary",
                                           "WindowMismatch", "SourceMismatch", "LengthMismatch"}


def test_column_index_range_is_checked_before_any_device_work():
    """the sweeps keep column indices in 32 bits: a target of 2^31 samples is
    rejected with invalid_argument (no pointer is touched, no GPU needed)"""
    lib = tsd.load_library()
    a = np.zeros(1000)
    huge = (1 << 31)
    f64p = ctypes.POINTER(ctypes.c_double)
    v, i = np.empty(901), np.empty(901, dtype=np.int64)
    rc = lib.tsd_ab_join(a.ctypes.data_as(f64p), a.size, a.ctypes.data_as(f64p), huge, 100, 0,
                         v.ctypes.data_as(f64p), i.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    assert rc == 1 + int(tsd.errc.invalid_argument), rc
    rc = lib.tsd_self_join(a.ctypes.data_as(f64p), huge, 100, ctypes.c_size_t(-1).value, 0,
                           v.ctypes.data_as(f64p), i.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    assert rc == 1 + int(tsd.errc.invalid_argument), rc


def test_no_cpu_fallback_without_gpu():
    """a compute call fails loudly when no CUDA device is present"""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tsd.TsdictError) as ei:
        tsd.ab_join(np.random.rand(100), np.random.rand(100), 10)
    assert ei.value.code() == tsd.errc.cuda_error
    assert "no CPU fallback" in str(ei.value)


# ---------------------------------------------------------------- multi-rank logic
@pytest.mark.parametrize("world", [2, 3])
def test_row_sharding_gloo(world):
    """join_dictionary_sharded over world_size 2 and 3 gloo groups: block-aligned
    row shards (tsd_dict_shard_rows), one all-gather, bit-identical to the
    unsharded join. Per-shard compute uses the oracle (CPU test)."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + world + os.getpid() % 1000))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_shard_worker.py"), str(world)], env=env,
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHARD_OK" in r.stdout


def test_learning_replay_matches_reference_golden(golden):
    """the oracle's restatement of the greedy learning loop reproduces the
    reference's learn_dictionary picks and merged segments on the
    well-conditioned golden cases (the periodic one ties to ~1e-12)"""
    n = 0
    for name, (kind, c) in golden.items():
        if kind != "learn" or "periodic" in name:
            continue
        n += 1
        cores, merged, stall = O.learn_dictionary_replay(c["t"], int(c["m"]), float(c["k"]), int(c["rule"]),
                                                         float(c["value"]))
        assert cores == [int(x) for x in c["cores"]], name
        assert [lo for lo, _ in merged] == [int(x) for x in c["starts"]], name
        assert [hi - lo for lo, hi in merged] == [int(x) for x in c["lengths"]], name
        assert stall == bool(int(c["no_progress"])), name
    assert n == 6


def test_window_labels_and_auc_match_reference(golden):
    """window_labels / auc_score (dict_join.hpp:102-162, host) against the
    reference's outputs, incl. overlapping / touching regions and many ties"""
    import paper_2112_12965_b200 as tsd
    c = golden["labels_124"][1]
    regions = list(zip(c["lo"].tolist(), c["hi"].tolist()))
    lab = tsd.window_labels(regions, int(c["n"]), int(c["m"]))
    assert np.array_equal(lab, c["labels"])
    assert tsd.auc_score(c["scores"], c["labels"]) == float(c["auc"])


def test_sharded_self_join_exchange_two_ranks_gloo():
    """the sharded self-join's exchange step (all-gather of per-row partials +
    acc_merge through the C ABI's tsd_profile_merge) over a world_size-2 gloo
    group reproduces the single-rank result; partials from a numpy brute force"""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(30500 + os.getpid() % 1000))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_selfshard_worker.py")], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SELFSHARD_OK" in r.stdout


def test_file_formats_match_reference(tmp_path):
    """include/tsdict/io.hpp: the reference-written files of
    tests/golden/io parse to the fixed objects, every golden document
    (valid and corrupted) gets the reference parser's outcome, our files
    round-trip (tests/cpp/test_io.cpp); and when the reference I/O driver was
    built here (oracle/_ref/ref_io, unmodified reference io.hpp), it reads our
    files back to the same objects."""
    exe = os.path.join(ROOT, "tests", "cpp", "build", "test_io")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe, str(tmp_path), os.path.join(ROOT, "tests", "golden", "io")], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_io")
    if os.path.exists(ref):
        r = subprocess.run([ref, "read", str(tmp_path)], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
