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
