"""Seeded synthetic inputs for the BASELINE configurations (ctypes over
libtsd_synth.so, host C++ with std::mt19937_64; see csrc/synth.cpp)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtsd_synth.so")
_lib = None
_f64p = ctypes.POINTER(ctypes.c_double)
_szp = ctypes.POINTER(ctypes.c_size_t)


def _l():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(_LIB)
        _lib.tsd_rng_new.restype = ctypes.c_void_p
        _lib.tsd_rng_new.argtypes = [ctypes.c_uint64]
        _lib.tsd_rng_free.argtypes = [ctypes.c_void_p]
        for f in ("tsd_rng_walk", "tsd_rng_noise"):
            getattr(_lib, f).argtypes = [ctypes.c_void_p, ctypes.c_size_t, _f64p]
        _lib.tsd_synth_walk.argtypes = [ctypes.c_uint64, ctypes.c_size_t, _f64p]
        _lib.tsd_synth_walks.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, _f64p]
        _lib.tsd_synth_sine.argtypes = [ctypes.c_size_t, ctypes.c_double, ctypes.c_double, _f64p]
        _lib.tsd_synth_ecg.restype = ctypes.c_size_t
        _lib.tsd_synth_ecg.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, _f64p, _szp]
        _lib.tsd_synth_traffic.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, _f64p]
    return _lib


class Rng:
    """A std::mt19937_64 stream; walk()/noise() draw like the reference synth.hpp:23-39."""

    def __init__(self, seed: int):
        self._h = ctypes.c_void_p(_l().tsd_rng_new(seed))

    def walk(self, n: int) -> np.ndarray:
        out = np.empty(n)
        _l().tsd_rng_walk(self._h, n, out.ctypes.data_as(_f64p))
        return out

    def noise(self, n: int) -> np.ndarray:
        out = np.empty(n)
        _l().tsd_rng_noise(self._h, n, out.ctypes.data_as(_f64p))
        return out

    def __del__(self):
        try:
            _l().tsd_rng_free(self._h)
        except Exception:
            pass


def walk(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    _l().tsd_synth_walk(seed, n, out.ctypes.data_as(_f64p))
    return out


def walks(seed: int, count: int, length: int) -> np.ndarray:
    out = np.empty(count * length)
    _l().tsd_synth_walks(seed, count, length, out.ctypes.data_as(_f64p))
    return out.reshape(count, length)


def sine(n: int, period: float, amp: float = 1.0) -> np.ndarray:
    out = np.empty(n)
    _l().tsd_synth_sine(n, period, amp, out.ctypes.data_as(_f64p))
    return out


def ecg(seed: int, n: int, n_anom: int = 0):
    out = np.empty(n)
    starts = np.zeros(max(1, n_anom), dtype=np.uintp)
    _l().tsd_synth_ecg(seed, n, n_anom, out.ctypes.data_as(_f64p), starts.ctypes.data_as(_szp))
    return out, starts[:n_anom].astype(np.int64)


def traffic(seed: int, nseries: int, length: int) -> np.ndarray:
    out = np.empty(nseries * length)
    _l().tsd_synth_traffic(seed, nseries, length, out.ctypes.data_as(_f64p))
    return out.reshape(nseries, length)
