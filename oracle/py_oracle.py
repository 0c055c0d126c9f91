"""ctypes bindings of the CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this module. It loads
  oracle/build/libtsd_oracle.so  -- plain-C restatement (tsd_oracle.c)
  oracle/_ref/libtsdict_ref.so   -- the unmodified reference headers (ref_shim.cpp)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libtsd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtsdict_ref.so")

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_szp = ctypes.POINTER(ctypes.c_size_t)
_sz = ctypes.c_size_t
_int = ctypes.c_int


def _p(a, t):
    return a.ctypes.data_as(t)


def _f(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle status {rc}")
        self.rc = rc


def _chk(rc):
    if rc != 0:
        raise OracleError(rc)


_o = None
_r = None


def lib():
    global _o
    if _o is None:
        _o = ctypes.CDLL(ORACLE_SO)
        _o.tsdo_compute_stats.argtypes = [_f64p, _sz, _sz, _f64p, _f64p, _f64p, _u8p]
        _o.tsdo_ab_join.argtypes = [_f64p, _sz, _f64p, _sz, _sz, _f64p, _i64p]
        _o.tsdo_self_join.argtypes = [_f64p, _sz, _sz, _sz, _f64p, _i64p]
        _o.tsdo_self_join_mt.argtypes = [_f64p, _sz, _sz, _sz, ctypes.c_uint, _f64p, _i64p]
        _o.tsdo_self_join_rows.argtypes = [_f64p, _sz, _sz, _sz, _sz, _sz, _f64p, _i64p]
        _o.tsdo_dict_join.argtypes = [_f64p, _sz, _f64p, _szp, _szp, _sz, _sz, _f64p, _i64p]
        _o.tsdo_corr_to_dist.restype = ctypes.c_double
        _o.tsdo_corr_to_dist.argtypes = [ctypes.c_double, _sz]
        _o.tsdo_pair_dist.restype = ctypes.c_double
        _o.tsdo_pair_dist.argtypes = [_f64p, _sz, _sz, _f64p, _sz, _sz, _sz]
        _o.tsdo_ab_join_brute.argtypes = [_f64p, _sz, _f64p, _sz, _sz, _f64p, _i64p]
        _o.tsdo_self_join_brute.argtypes = [_f64p, _sz, _sz, _sz, _f64p, _i64p]
    return _o


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _r
    if _r is None:
        _r = ctypes.CDLL(REF_SO)
        _r.tsdr_compute_stats.argtypes = [_f64p, _sz, _sz, _f64p, _f64p, _f64p, _u8p]
        _r.tsdr_ab_join.argtypes = [_f64p, _sz, _f64p, _sz, _sz, ctypes.c_uint, _f64p, _i64p]
        _r.tsdr_self_join.argtypes = [_f64p, _sz, _sz, ctypes.c_uint, _f64p, _i64p]
        _r.tsdr_join_dictionary.argtypes = [_f64p, _sz, _f64p, _szp, _szp, _sz, _sz, _sz, ctypes.c_uint, _f64p, _i64p]
        _r.tsdr_compute_e_max.argtypes = [_f64p, _sz, _f64p, _szp, _szp, _sz, _sz, ctypes.c_uint, _f64p]
        _r.tsdr_ab_join_brute.argtypes = [_f64p, _sz, _f64p, _sz, _sz, _f64p, _i64p]
        _r.tsdr_self_join_brute.argtypes = [_f64p, _sz, _sz, _f64p, _i64p]
        _r.tsdr_rng_new.restype = ctypes.c_void_p
        _r.tsdr_rng_new.argtypes = [ctypes.c_uint64]
        _r.tsdr_rng_free.argtypes = [ctypes.c_void_p]
        _r.tsdr_noise.argtypes = [ctypes.c_void_p, _sz, _f64p]
        _r.tsdr_walk.argtypes = [ctypes.c_void_p, _sz, _f64p]
        _r.tsdr_sine.argtypes = [_sz, ctypes.c_double, ctypes.c_double, _f64p]
    return _r


# ---------------------------------------------------------------- restatement
def compute_stats(x, m):
    x = _f(x)
    cnt = x.size - m + 1
    mu, sd, iv = np.empty(cnt), np.empty(cnt), np.empty(cnt)
    fl = np.empty(cnt, dtype=np.uint8)
    _chk(lib().tsdo_compute_stats(_p(x, _f64p), x.size, m, _p(mu, _f64p), _p(sd, _f64p), _p(iv, _f64p), _p(fl, _u8p)))
    return mu, sd, iv, fl


def ab_join(a, b, m):
    a, b = _f(a), _f(b)
    cnt = max(1, a.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(lib().tsdo_ab_join(_p(a, _f64p), a.size, _p(b, _f64p), b.size, m, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def self_join(t, m, excl=None):
    t = _f(t)
    cnt = max(1, t.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(lib().tsdo_self_join(_p(t, _f64p), t.size, m, m // 2 if excl is None else excl, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def self_join_mt(t, m, excl=None, threads=None):
    """self_join with the reference's diagonal thread split (bit-identical to
    self_join); threads defaults to every host core"""
    t = _f(t)
    cnt = max(1, t.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(lib().tsdo_self_join_mt(_p(t, _f64p), t.size, m, m // 2 if excl is None else excl,
                                 threads or os.cpu_count() or 1, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def self_join_rows(t, m, r0, nr, excl=None):
    """rows [r0, r0 + nr) of self_join's profile (diagonals started at r0)"""
    t = _f(t)
    nr = min(nr, t.size - m + 1 - r0)
    v, i = np.empty(nr), np.empty(nr, dtype=np.int64)
    _chk(lib().tsdo_self_join_rows(_p(t, _f64p), t.size, m, m // 2 if excl is None else excl, r0, nr,
                                   _p(v, _f64p), _p(i, _i64p)))
    return v, i


def parallel(fn, args, workers=None):
    """run fn(*a) for every a in args on host threads (ctypes releases the
    GIL during the oracle calls); results in order"""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=workers or os.cpu_count() or 1) as ex:
        return list(ex.map(lambda a: fn(*a), args))


def dict_join(q, segments, starts, m):
    """segments: list of 1-D arrays; starts: source coordinates."""
    q = _f(q)
    lens = np.asarray([len(s) for s in segments], dtype=np.uintp)
    st = np.asarray(starts, dtype=np.uintp)
    vals = _f(np.concatenate(segments))
    cnt = max(1, q.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(lib().tsdo_dict_join(_p(q, _f64p), q.size, _p(vals, _f64p), _p(lens, _szp), _p(st, _szp), len(segments), m,
                              _p(v, _f64p), _p(i, _i64p)))
    return v, i


def pair_dist(a, i, b, j, m):
    a, b = _f(a), _f(b)
    return lib().tsdo_pair_dist(_p(a, _f64p), a.size, i, _p(b, _f64p), b.size, j, m)


def _kahan_mean_sd(q):
    """MASS's query statistics: Kahan mean, Kahan two-pass std (profiles.hpp:203-213)"""
    s = c = 0.0
    for x in q:
        y = x - c
        t = s + y
        c = (t - s) - y
        s = t
    mu = s / q.size
    s = c = 0.0
    for x in q:
        y = (x - mu) * (x - mu) - c
        t = s + y
        c = (t - s) - y
        s = t
    return mu, np.sqrt(max(0.0, s / q.size))


def learn_dictionary_replay(t, m, k=1.5, rule=0, value=0.5, max_iterations=1000000):
    """ORACLE restatement of the greedy learning loop (dictionary.hpp:259-321,
    replayed the way test_dictionary.cpp:94-158 does): argmin of P - S over
    unmasked windows (first minimum), select_state masking / context
    intervals / merging, distance profiles of the picks folded into S, stop
    rules. P is this oracle's self_join (bit-identical to the reference);
    distance profiles are exact dot products (MASS without its FFT round-off,
    with its constant-window rules). Returns (cores, merged intervals,
    no_progress)."""
    t = _f(t)
    n, cnt, excl = t.size, t.size - m + 1, m // 2
    P, _ = self_join(t, m)
    mu, _, invn, flat = compute_stats(t, m)
    W = np.lib.stride_tricks.sliding_window_view(t, m) - mu[:, None]
    far = np.sqrt(2.0 * m)
    total = int(k * m + 1e-9)
    before = total // 2
    masked = np.zeros(cnt, dtype=bool)
    S = np.zeros(cnt)
    s_init, cores, ivs, stall = False, [], [], False
    need = value if rule == 1 else (1.0 - value) * n - 1e-6
    for it in range(max_iterations + 1):
        if it >= max_iterations:
            raise RuntimeError("iteration cap")
        cand = np.where(~masked)[0]
        if cand.size == 0:
            stall = True
            break
        j = int(cand[np.argmin(P[cand] - S[cand])])  # argmin returns the first minimum
        cores.append(j)
        masked[max(0, j - excl): min(cnt, j + excl + 1)] = True
        ivs.append((max(0, j - before), min(n, j + m + (total - before))))
        merged = []
        for lo, hi in sorted(ivs):
            if merged and lo <= merged[-1][1]:
                merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
            else:
                merged.append((lo, hi))
        if rule != 2 and sum(hi - lo for lo, hi in merged) >= need:
            break
        q = t[j:j + m]
        mq, sq = _kahan_mean_sd(q)
        if sq < 1e-8 * max(1.0, float(np.max(np.abs(q)))):
            dp = np.where(flat & 2 > 0, 0.0, far)
        else:
            rho = (W @ (q - mq)) * invn / (sq * np.sqrt(m))
            dp = np.sqrt(np.clip(2.0 * m * (1.0 - np.clip(rho, -1.0, 1.0)), 0.0, 4.0 * m))
            dp[flat & 2 > 0] = far
            if not flat[j] & 2:
                dp[j] = pair_dist(t, j, t, j, m)
        S = dp if not s_init else np.minimum(S, dp)
        s_init = True
        if rule == 2 and S.max() <= value:
            break
    merged = []
    for lo, hi in sorted(ivs):
        if merged and lo <= merged[-1][1]:
            merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
        else:
            merged.append((lo, hi))
    return cores, merged, stall


def ab_join_brute(a, b, m):
    a, b = _f(a), _f(b)
    cnt = a.size - m + 1
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(lib().tsdo_ab_join_brute(_p(a, _f64p), a.size, _p(b, _f64p), b.size, m, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def self_join_brute(t, m, excl=None):
    t = _f(t)
    cnt = t.size - m + 1
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(lib().tsdo_self_join_brute(_p(t, _f64p), t.size, m, m // 2 if excl is None else excl, _p(v, _f64p),
                                    _p(i, _i64p)))
    return v, i


# ---------------------------------------------------------------- reference
def ref_ab_join(a, b, m, threads=1):
    a, b = _f(a), _f(b)
    cnt = max(1, a.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(ref().tsdr_ab_join(_p(a, _f64p), a.size, _p(b, _f64p), b.size, m, threads, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def ref_self_join(t, m, threads=1):
    t = _f(t)
    cnt = max(1, t.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(ref().tsdr_self_join(_p(t, _f64p), t.size, m, threads, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def ref_join_dictionary(q, segments, starts, m, threads=1):
    q = _f(q)
    lens = np.asarray([len(s) for s in segments], dtype=np.uintp)
    st = np.asarray(starts, dtype=np.uintp)
    vals = _f(np.concatenate(segments))
    cnt = max(1, q.size - m + 1)
    v, i = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _chk(ref().tsdr_join_dictionary(_p(q, _f64p), q.size, _p(vals, _f64p), _p(lens, _szp), _p(st, _szp),
                                    len(segments), m, m, threads, _p(v, _f64p), _p(i, _i64p)))
    return v, i


def ref_distance_profile(t, q, m, mass=False, origin=None):
    """the reference's distance_profile_naive / distance_profile_mass
    (profiles.hpp:164-260; MASS with the oracle/standin FFT) over its own stats"""
    t, q = _f(t), _f(q)
    out = np.empty(t.size - m + 1)
    r = ref()
    r.tsdr_distance_profile.argtypes = [_f64p, _sz, _f64p, _sz, _int, _sz, _f64p]
    _chk(r.tsdr_distance_profile(_p(t, _f64p), t.size, _p(q, _f64p), m, 1 if mass else 0,
                                 ctypes.c_size_t(-1).value if origin is None else origin, _p(out, _f64p)))
    return out


def ref_compute_stats(x, m):
    x = _f(x)
    cnt = x.size - m + 1
    mu, sd, iv = np.empty(cnt), np.empty(cnt), np.empty(cnt)
    fl = np.empty(cnt, dtype=np.uint8)
    _chk(ref().tsdr_compute_stats(_p(x, _f64p), x.size, m, _p(mu, _f64p), _p(sd, _f64p), _p(iv, _f64p), _p(fl, _u8p)))
    return mu, sd, iv, fl


class RefRng:
    """the reference's own synth.hpp generators on a std::mt19937_64 stream"""

    def __init__(self, seed):
        self.h = ctypes.c_void_p(ref().tsdr_rng_new(seed))

    def noise(self, n):
        o = np.empty(n)
        ref().tsdr_noise(self.h, n, _p(o, _f64p))
        return o

    def walk(self, n):
        o = np.empty(n)
        ref().tsdr_walk(self.h, n, _p(o, _f64p))
        return o

    def __del__(self):
        try:
            ref().tsdr_rng_free(self.h)
        except Exception:
            pass


def ref_sine(n, period, amp=1.0):
    o = np.empty(n)
    ref().tsdr_sine(n, period, amp, _p(o, _f64p))
    return o


def ref_learn_dictionary_full(t, m, k=1.5, rule=0, value=0.5, max_iterations=1000000, threads=0):
    """the reference's learn_dictionary with any stop rule (0 space saving,
    1 sample budget, 2 error target); returns a dict with starts, lengths,
    cores, e_max, space_saving, no_progress"""
    t = _f(t)
    n = t.size
    st = np.zeros(n, dtype=np.uintp)
    ln = np.zeros(n, dtype=np.uintp)
    vals = np.zeros(n)
    cores = np.zeros(n, dtype=np.uintp)
    ns, nc = ctypes.c_size_t(), ctypes.c_size_t()
    em, ss, npg = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    r = ref()
    r.tsdr_learn_dictionary2.argtypes = [_f64p, _sz, _sz, ctypes.c_double, ctypes.c_int, ctypes.c_double, _sz,
                                         ctypes.c_uint, _szp, _szp, _f64p, ctypes.POINTER(ctypes.c_size_t), _szp,
                                         ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    _chk(r.tsdr_learn_dictionary2(_p(t, _f64p), n, m, k, rule, value, max_iterations, threads, _p(st, _szp),
                                  _p(ln, _szp), _p(vals, _f64p), ctypes.byref(ns), _p(cores, _szp), ctypes.byref(nc),
                                  ctypes.byref(em), ctypes.byref(ss), ctypes.byref(npg)))
    return {"starts": st[:ns.value].astype(np.int64), "lengths": ln[:ns.value].astype(np.int64),
            "cores": cores[:nc.value].astype(np.int64), "e_max": em.value, "space_saving": ss.value,
            "no_progress": int(npg.value)}


def ref_find_discords(values, m, e_max, top_k):
    """the reference's find_discords (dict_join.hpp:54-93) -> (starts, scores, certified)"""
    v = _f(values)
    cap = max(top_k, 1)
    st, sc, ce = np.zeros(cap, dtype=np.uintp), np.zeros(cap), np.zeros(cap, dtype=np.int32)
    cnt = ctypes.c_size_t()
    r = ref()
    r.tsdr_find_discords.argtypes = [_f64p, _sz, _sz, ctypes.c_double, _sz, _szp, _f64p,
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_size_t)]
    _chk(r.tsdr_find_discords(_p(v, _f64p), v.size, m, e_max, top_k, _p(st, _szp), _p(sc, _f64p),
                              ce.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), ctypes.byref(cnt)))
    k = cnt.value
    return st[:k].astype(np.int64), sc[:k].copy(), ce[:k].astype(bool)


def ref_window_labels(regions, n, m):
    lo = np.asarray([a for a, _ in regions], dtype=np.uintp)
    hi = np.asarray([b for _, b in regions], dtype=np.uintp)
    out = np.zeros(n - m + 1, dtype=np.uint8)
    r = ref()
    r.tsdr_window_labels.argtypes = [_szp, _szp, _sz, _sz, _sz, _u8p]
    _chk(r.tsdr_window_labels(_p(lo, _szp), _p(hi, _szp), len(regions), n, m, _p(out, _u8p)))
    return out


def ref_auc_score(scores, labels):
    s, l = _f(scores), np.ascontiguousarray(labels, dtype=np.uint8)
    out = ctypes.c_double()
    r = ref()
    r.tsdr_auc_score.argtypes = [_f64p, _u8p, _sz, ctypes.POINTER(ctypes.c_double)]
    _chk(r.tsdr_auc_score(_p(s, _f64p), _p(l, _u8p), s.size, ctypes.byref(out)))
    return out.value


def ref_learn_dictionary(t, m, space_saving, threads=0):
    """the reference's greedy learn_dictionary (dictionary.hpp:259-328);
    returns (segments, starts, e_max)"""
    t = _f(t)
    n = t.size
    st = np.zeros(n, dtype=np.uintp)
    ln = np.zeros(n, dtype=np.uintp)
    vals = np.zeros(n)
    ns = ctypes.c_size_t()
    em = ctypes.c_double()
    r = ref()
    r.tsdr_learn_dictionary.argtypes = [_f64p, _sz, _sz, ctypes.c_double, ctypes.c_uint, _szp, _szp, _f64p,
                                        ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_double)]
    _chk(r.tsdr_learn_dictionary(_p(t, _f64p), n, m, space_saving, threads, _p(st, _szp), _p(ln, _szp),
                                 _p(vals, _f64p), ctypes.byref(ns), ctypes.byref(em)))
    segs, starts, off = [], [], 0
    for s in range(ns.value):
        segs.append(vals[off:off + ln[s]].copy())
        starts.append(int(st[s]))
        off += int(ln[s])
    return segs, starts, em.value
