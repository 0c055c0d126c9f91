"""tsdict-b200: the reference `tsdict` hot path on B200 (sm_100a).

Python mirror of the reference C++ API (namespace ``tsdict``, reference
proj/include/tsdict/*.hpp) over the C ABI in ``include/tsdict_cuda.h``
(built in-tree as ``libtsdict_cuda.so``). Same function names, argument
meaning and error behaviour: failures raise :class:`TsdictError` whose
``code`` is the reference ``tsdict::errc`` (errors.hpp:13-35) and whose
message is prefixed by the code name (errors.hpp:59-62).

There is no CPU fallback: every compute call runs the CUDA library and
raises if it is missing or no GPU is present.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSD_LIB") or os.path.join(_HERE, "libtsdict_cuda.so")

__all__ = [
    "errc", "TsdictError", "TimeSeries", "SubseqStats", "MatrixProfile", "Segment", "Dictionary",
    "compute_stats", "ab_join", "self_join", "join_dictionary", "dict_min_profile", "compute_e_max",
    "join_dictionary_batched", "corr_to_dist", "DictPlan", "load_library", "measure_peak", "build_info",
    "C_SYMBOLS",
    "LearnConfig",
    "learn_dictionary",
    "Discord",
    "find_discords",
    "self_join_partial",
    "merge_partials",
    "self_join_finish",
    "exchange_partials",
    "self_join_sharded",
    "dict_shard_rows",
    "join_dictionary_sharded",
    "window_labels",
    "auc_score",
    "DistanceProfile",
    "distance_profile_naive",
    "distance_profile_mass",
]


class errc(enum.IntEnum):
    """reference errors.hpp:13-35 (ordinal order preserved)."""
    window_too_small = 0
    window_too_large = 1
    non_finite_input = 2
    length_mismatch = 3
    series_too_short = 4
    iteration_cap_exceeded = 5
    source_mismatch = 6
    window_mismatch = 7
    empty_dictionary = 8
    empty_profile = 9
    degenerate_labels = 10
    parse_error = 11
    version_error = 12
    schema_error = 13
    io_error = 14
    invalid_argument = 15
    cuda_error = 99  # device failure; no reference counterpart


_ERRC_NAME = {
    errc.window_too_small: "WindowTooSmall", errc.window_too_large: "WindowTooLarge",
    errc.non_finite_input: "NonFiniteInput", errc.length_mismatch: "LengthMismatch",
    errc.series_too_short: "SeriesTooShort", errc.iteration_cap_exceeded: "IterationCapExceeded",
    errc.source_mismatch: "SourceMismatch", errc.window_mismatch: "WindowMismatch",
    errc.empty_dictionary: "EmptyDictionary", errc.empty_profile: "EmptyProfile",
    errc.degenerate_labels: "DegenerateLabels", errc.parse_error: "ParseError",
    errc.version_error: "VersionError", errc.schema_error: "SchemaError", errc.io_error: "IoError",
    errc.invalid_argument: "InvalidArgument", errc.cuda_error: "CudaError",
}


class TsdictError(RuntimeError):
    """reference tsdict::error (errors.hpp:59-68): what() = '<CodeName>: message'."""

    def __init__(self, code: errc, message: str):
        self._code = errc(code)
        text = message if message.startswith(_ERRC_NAME[self._code] + ":") else f"{_ERRC_NAME[self._code]}: {message}"
        super().__init__(text)

    def code(self) -> errc:
        return self._code


# ---------------------------------------------------------------------------
# library loading
# ---------------------------------------------------------------------------
_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_szp = ctypes.POINTER(ctypes.c_size_t)
_sz = ctypes.c_size_t
_int = ctypes.c_int
_vp = ctypes.c_void_p

# name -> (restype, argtypes); every symbol include/tsdict_cuda.h declares
C_SYMBOLS = {
    "tsd_compute_stats": (_int, [_f64p, _sz, _sz, _f64p, _f64p, _f64p, _u8p]),
    "tsd_ab_join": (_int, [_f64p, _sz, _f64p, _sz, _sz, _int, _f64p, _i64p]),
    "tsd_self_join": (_int, [_f64p, _sz, _sz, _sz, _int, _f64p, _i64p]),
    "tsd_dict_join": (_int, [_f64p, _sz, _f64p, _szp, _szp, _sz, _sz, _int, _f64p, _i64p]),
    "tsd_dict_join_batched": (_int, [_f64p, _szp, _sz, _f64p, _szp, _szp, _sz, _sz, _int, _f64p, _i64p]),
    "tsd_compute_e_max": (_int, [_f64p, _sz, _sz, _f64p, _szp, _szp, _sz, _sz, _f64p]),
    "tsd_find_discords": (_int, [_f64p, _sz, _sz, ctypes.c_double, _sz, _szp, _f64p, ctypes.POINTER(_int), _szp]),
    "tsd_find_discords_device": (_int, [_vp, _sz, _sz, ctypes.c_double, _sz, _szp, _f64p, ctypes.POINTER(_int), _szp,
                                        _vp]),
    "tsd_self_join_partial": (_int, [_f64p, _sz, _sz, _sz, _sz, _sz, _f64p, _i64p]),
    "tsd_profile_merge": (_int, [_f64p, _i64p, _sz, _sz, _f64p, _i64p]),
    "tsd_self_join_finish": (_int, [_f64p, _sz, _sz, _sz, _f64p, _i64p, _f64p, _i64p]),
    "tsd_self_join_partial_device": (_int, [_vp, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _vp]),
    "tsd_profile_merge_device": (_int, [_vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "tsd_self_join_finish_device": (_int, [_vp, _sz, _sz, _sz, _vp, _vp, _vp]),
    "tsd_dict_shard_rows": (_int, [_sz, _sz, _sz, _sz, _szp, _szp]),
    "tsd_learn_dictionary": (_int, [_f64p, _sz, _sz, ctypes.c_double, _int, ctypes.c_double, _sz, _f64p, _szp, _szp,
                                    _f64p, _szp, _szp, _szp, _f64p, _f64p, ctypes.POINTER(_int)]),
    "tsd_dict_plan_create": (_int, [_f64p, _szp, _szp, _sz, _sz, _int, ctypes.POINTER(_vp)]),
    "tsd_dict_plan_join_device": (_int, [_vp, _vp, _szp, _sz, _vp, _vp, _vp]),
    "tsd_dict_plan_join": (_int, [_vp, _f64p, _szp, _sz, _f64p, _i64p]),
    "tsd_dict_plan_destroy": (_int, [_vp]),
    "tsd_dict_plan_last_timing": (_int, [_vp, _f64p, _f64p, ctypes.POINTER(_int)]),
    "tsd_dict_plan_last_kernel_timing": (_int, [_vp, _f64p, _f64p]),
    "tsd_distance_profile_naive": (_int, [_f64p, _sz, _f64p, _sz, _f64p]),
    "tsd_distance_profile_mass": (_int, [_f64p, _sz, _f64p, _sz, _f64p, _f64p, _u8p, _sz, _f64p]),
    "tsd_last_error": (ctypes.c_char_p, []),
    "tsd_last_join_timing": (_int, [_f64p, _f64p, ctypes.POINTER(_int)]),
    "tsd_status_name": (ctypes.c_char_p, [_int]),
    "tsd_build_info": (ctypes.c_char_p, []),
    "tsd_measure_peak": (_int, [_int, ctypes.c_double, _f64p]),
    "tsd_measure_peak_clock": (_int, [_int, ctypes.c_double, _f64p, _f64p]),
}

_lib = None


def load_library() -> ctypes.CDLL:
    """Load libtsdict_cuda.so (built by __graft_entry__.build()). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TsdictError(errc.cuda_error, f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in C_SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = load_library().tsd_last_error().decode(errors="replace")
        code = errc.cuda_error if rc == 100 else errc(rc - 1)
        raise TsdictError(code, msg)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


_PREC = {"fp64": 0, "fp32": 1, 0: 0, 1: 1}


# ---------------------------------------------------------------------------
# types (series.hpp:27-45, profiles.hpp:44-51, dictionary.hpp:46-68)
# ---------------------------------------------------------------------------
@dataclass
class TimeSeries:
    values: np.ndarray

    def __post_init__(self):
        self.values = _f64(self.values)

    def n(self) -> int:
        return int(self.values.size)


def _vals(T) -> np.ndarray:
    return T.values if isinstance(T, TimeSeries) else _f64(T)


@dataclass
class SubseqStats:
    m: int
    means: np.ndarray
    stds: np.ndarray
    invn: np.ndarray
    constant_mask: np.ndarray

    def count(self) -> int:
        return int(self.means.size)


@dataclass
class MatrixProfile:
    no_neighbor = -1
    values: np.ndarray
    indices: np.ndarray
    kind: str = "self"
    m: int = 0


@dataclass
class Segment:
    start: int
    values: np.ndarray

    def __post_init__(self):
        self.values = _f64(self.values)

    def length(self) -> int:
        return int(self.values.size)


@dataclass
class Dictionary:
    segments: List[Segment] = field(default_factory=list)
    m: int = 0
    k: float = 1.5
    source_length: int = 0
    core_starts: List[int] = field(default_factory=list)
    e_max: Optional[float] = None
    space_saving: float = 0.0
    no_progress: bool = False

    def stored_samples(self) -> int:
        return sum(s.length() for s in self.segments)


def _pack_dict(D: Dictionary):
    lens = np.asarray([s.length() for s in D.segments], dtype=np.uintp)
    starts = np.asarray([s.start for s in D.segments], dtype=np.uintp)
    vals = _f64(np.concatenate([s.values for s in D.segments])) if D.segments else np.zeros(1)
    return vals, lens, starts


# ---------------------------------------------------------------------------
# hot-path API
# ---------------------------------------------------------------------------
def corr_to_dist(rho: float, m: int) -> float:
    """series.hpp:153-161 (host helper)."""
    rho = min(1.0, max(-1.0, rho))
    d = float(np.sqrt(2.0 * m * (1.0 - rho)))
    return min(max(d, 0.0), 2.0 * float(np.sqrt(m)))


def compute_stats(T, m: int) -> SubseqStats:
    """series.hpp:83-150."""
    x = _vals(T)
    lib = load_library()
    cnt = max(0, x.size - m + 1)
    means, stds, invn = (np.empty(max(cnt, 1)) for _ in range(3))
    flat = np.empty(max(cnt, 1), dtype=np.uint8)
    _check(lib.tsd_compute_stats(_ptr(x, _f64p), x.size, m, _ptr(means, _f64p), _ptr(stds, _f64p),
                                 _ptr(invn, _f64p), _ptr(flat, _u8p)))
    return SubseqStats(m, means[:cnt], stds[:cnt], invn[:cnt], flat[:cnt])


@dataclass
class DistanceProfile:
    """profiles.hpp:36-40"""
    values: np.ndarray
    query_origin: Optional[int] = None
    m: int = 0


def _dprof_check(x, Q, stats):
    """profiles.hpp:167-172 / :189-194"""
    if Q.size != stats.m:
        raise TsdictError(errc.length_mismatch, "query length does not match stats window length")
    if stats.count() != x.size - stats.m + 1:
        raise TsdictError(errc.length_mismatch, "stats were computed for a different series length")


def distance_profile_naive(T, Q, stats: SubseqStats, query_origin: Optional[int] = None) -> DistanceProfile:
    """profiles.hpp:164-181: znorm_distance (series.hpp:166-204) per window, on the device."""
    x, q = _vals(T), _f64(Q)
    _dprof_check(x, q, stats)
    out = np.empty(max(1, stats.count()))
    if stats.count() > 0:
        _check(load_library().tsd_distance_profile_naive(_ptr(x, _f64p), x.size, _ptr(q, _f64p), q.size,
                                                         _ptr(out, _f64p)))
    return DistanceProfile(out[:stats.count()], query_origin, stats.m)


def distance_profile_mass(T, Q, stats: SubseqStats, query_origin: Optional[int] = None) -> DistanceProfile:
    """profiles.hpp:186-260 (MASS's conventions; exact FP64 dot products on the
    device instead of the FFT convolution)."""
    x, q = _vals(T), _f64(Q)
    _dprof_check(x, q, stats)
    mu = _f64(stats.means)
    iv = _f64(stats.invn)
    cm = np.ascontiguousarray(stats.constant_mask, dtype=np.uint8)
    out = np.empty(max(1, stats.count()))
    org = ctypes.c_size_t(-1).value if query_origin is None else int(query_origin)
    _check(load_library().tsd_distance_profile_mass(_ptr(x, _f64p), x.size, _ptr(q, _f64p), q.size, _ptr(mu, _f64p),
                                                    _ptr(iv, _f64p), _ptr(cm, _u8p), org, _ptr(out, _f64p)))
    return DistanceProfile(out[:stats.count()], query_origin, stats.m)


def ab_join(A, B, m: int, threads: int = 0, precision="fp64") -> MatrixProfile:
    """profiles.hpp:306-342. `threads` is accepted for API parity and ignored."""
    a, b = _vals(A), _vals(B)
    lib = load_library()
    cnt = max(1, a.size - m + 1)
    val, idx = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _check(lib.tsd_ab_join(_ptr(a, _f64p), a.size, _ptr(b, _f64p), b.size, m, _PREC[precision],
                           _ptr(val, _f64p), _ptr(idx, _i64p)))
    return MatrixProfile(val, idx, "ab", m)


def self_join(T, m: int, threads: int = 0, excl: Optional[int] = None, precision="fp64") -> MatrixProfile:
    """profiles.hpp:266-301; `excl` defaults to the reference's m // 2 (:273)."""
    x = _vals(T)
    lib = load_library()
    cnt = max(1, x.size - m + 1)
    val, idx = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    e = ctypes.c_size_t(-1).value if excl is None else int(excl)
    _check(lib.tsd_self_join(_ptr(x, _f64p), x.size, m, e, _PREC[precision], _ptr(val, _f64p), _ptr(idx, _i64p)))
    return MatrixProfile(val, idx, "self", m)


def dict_min_profile(T, D: Dictionary, m: int, threads: int = 0, precision="fp64") -> MatrixProfile:
    """dictionary.hpp:149-193 (detail::dict_min_profile)."""
    q = _vals(T)
    vals, lens, starts = _pack_dict(D)
    lib = load_library()
    cnt = max(1, q.size - m + 1)
    val, idx = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _check(lib.tsd_dict_join(_ptr(q, _f64p), q.size, _ptr(vals, _f64p), _ptr(lens, _szp), _ptr(starts, _szp),
                             len(D.segments), m, _PREC[precision], _ptr(val, _f64p), _ptr(idx, _i64p)))
    return MatrixProfile(val, idx, "ab", m)


def join_dictionary(A, D: Dictionary, m: int, threads: int = 0, precision="fp64") -> MatrixProfile:
    """dict_join.hpp:42-48."""
    if m != D.m:
        raise TsdictError(errc.window_mismatch, "requested window length differs from the dictionary's")
    return dict_min_profile(A, D, m, threads, precision)


def join_dictionary_batched(series: Sequence, D: Dictionary, m: int, precision="fp64") -> List[MatrixProfile]:
    """join_dictionary over many query series in one device pass (BASELINE C5)."""
    if m != D.m:
        raise TsdictError(errc.window_mismatch, "requested window length differs from the dictionary's")
    qs = [_vals(s) for s in series]
    qlen = np.asarray([q.size for q in qs], dtype=np.uintp)
    q = _f64(np.concatenate(qs))
    vals, lens, starts = _pack_dict(D)
    lib = load_library()
    cnts = [max(0, int(n) - m + 1) for n in qlen]
    tot = max(1, sum(cnts))
    val, idx = np.empty(tot), np.empty(tot, dtype=np.int64)
    _check(lib.tsd_dict_join_batched(_ptr(q, _f64p), _ptr(qlen, _szp), len(qs), _ptr(vals, _f64p),
                                     _ptr(lens, _szp), _ptr(starts, _szp), len(D.segments), m, _PREC[precision],
                                     _ptr(val, _f64p), _ptr(idx, _i64p)))
    out, o = [], 0
    for c in cnts:
        out.append(MatrixProfile(val[o:o + c], idx[o:o + c], "ab", m))
        o += c
    return out


def compute_e_max(D: Dictionary, T_B, threads: int = 0) -> float:
    """dictionary.hpp:247-255."""
    x = _vals(T_B)
    vals, lens, starts = _pack_dict(D)
    lib = load_library()
    out = ctypes.c_double(0.0)
    _check(lib.tsd_compute_e_max(_ptr(x, _f64p), x.size, D.source_length, _ptr(vals, _f64p), _ptr(lens, _szp),
                                 _ptr(starts, _szp), len(D.segments), D.m, ctypes.byref(out)))
    return out.value


@dataclass
class LearnConfig:
    """dictionary.hpp:57-64 (exactly one stop rule)."""
    m: int = 0
    k: float = 1.5
    space_saving_target: Optional[float] = None
    sample_budget: Optional[int] = None
    error_target: Optional[float] = None
    max_iterations: int = 1000000


def learn_dictionary(T_B, cfg: LearnConfig, P_B: Optional[MatrixProfile] = None, threads: int = 0) -> Dictionary:
    """dictionary.hpp:259-328: greedy selection on the device, then compute_e_max.
    P_B: the exact self-join profile of T_B (learn_dictionary(T_B, cfg, P_B))."""
    x = _vals(T_B)
    n, m = x.size, cfg.m
    rules = [r for r in (cfg.space_saving_target, cfg.sample_budget, cfg.error_target) if r is not None]
    if len(rules) != 1:
        raise TsdictError(errc.invalid_argument, "exactly one stop rule must be set")
    if cfg.space_saving_target is not None:
        rule, val = 0, float(cfg.space_saving_target)
    elif cfg.sample_budget is not None:
        rule, val = 1, float(cfg.sample_budget)
    else:
        rule, val = 2, float(cfg.error_target)
    prof = None
    if P_B is not None:  # :267-271
        if n >= 2 * m and (P_B.m != m or P_B.kind != "self" or P_B.values.size != n - m + 1):
            raise TsdictError(errc.invalid_argument, "precomputed profile does not match the series and window")
        prof = _f64(P_B.values)
    cap = max(n, 1)
    starts = np.zeros(cap, dtype=np.uintp)
    lens = np.zeros(cap, dtype=np.uintp)
    vals = np.zeros(cap)
    cores = np.zeros(cap, dtype=np.uintp)
    nseg, ncores = ctypes.c_size_t(0), ctypes.c_size_t(0)
    e, ss, npg = ctypes.c_double(0.0), ctypes.c_double(0.0), ctypes.c_int(0)
    lib = load_library()
    _check(lib.tsd_learn_dictionary(_ptr(x, _f64p), n, m, cfg.k, rule, val, cfg.max_iterations,
                                    _ptr(prof, _f64p) if prof is not None else None, _ptr(starts, _szp),
                                    _ptr(lens, _szp), _ptr(vals, _f64p), ctypes.byref(nseg), _ptr(cores, _szp),
                                    ctypes.byref(ncores), ctypes.byref(e), ctypes.byref(ss), ctypes.byref(npg)))
    segs, off = [], 0
    for s in range(nseg.value):
        L = int(lens[s])
        segs.append(Segment(int(starts[s]), vals[off:off + L].copy()))
        off += L
    return Dictionary(segments=segs, m=m, k=cfg.k, source_length=n, core_starts=[int(c) for c in cores[:ncores.value]],
                      e_max=e.value, space_saving=ss.value, no_progress=bool(npg.value))


# --------------------------------------------------------------------------- sharded self-join
def _excl_arg(m, excl):
    return ctypes.c_size_t(-1).value if excl is None else int(excl)


def self_join_partial(T, m: int, excl: Optional[int] = None, shard: int = 0, nshards: int = 1):
    """One shard of the symmetric self-join: per-row (corr, window) partials over
    ALL rows (corr -2 / window -1 = none) for every nshards-th task."""
    x = _vals(T)
    cnt = max(1, x.size - m + 1)
    corr, col = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _check(load_library().tsd_self_join_partial(_ptr(x, _f64p), x.size, m, _excl_arg(m, excl), shard, nshards,
                                                _ptr(corr, _f64p), _ptr(col, _i64p)))
    return corr, col


def merge_partials(corrs, cols):
    """acc_merge's rule over shards (profiles.hpp:79-85): larger corr, then lower index."""
    C = np.ascontiguousarray(np.stack([np.asarray(c, dtype=np.float64) for c in corrs]))
    J = np.ascontiguousarray(np.stack([np.asarray(j, dtype=np.int64) for j in cols]))
    cnt = C.shape[1]
    corr, col = np.empty(cnt), np.empty(cnt, dtype=np.int64)
    _check(load_library().tsd_profile_merge(_ptr(C, _f64p), _ptr(J, _i64p), C.shape[0], cnt, _ptr(corr, _f64p),
                                            _ptr(col, _i64p)))
    return corr, col


def self_join_finish(T, m: int, excl: Optional[int], corr, col) -> MatrixProfile:
    """Merged partials -> the self-join profile (distances, flat rows, sentinel)."""
    x = _vals(T)
    c, j = _f64(corr), np.ascontiguousarray(col, dtype=np.int64)
    val, idx = np.empty(c.size), np.empty(c.size, dtype=np.int64)
    _check(load_library().tsd_self_join_finish(_ptr(x, _f64p), x.size, m, _excl_arg(m, excl), _ptr(c, _f64p),
                                               _ptr(j, _i64p), _ptr(val, _f64p), _ptr(idx, _i64p)))
    return MatrixProfile(values=val, indices=idx, kind="self", m=m)


def exchange_partials(corr, col, group=None):
    """The one exchange step of the sharded self-join: all-gather
    every rank's partials (NCCL has no (max, argmax) reduction) and merge."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    c = torch.from_numpy(np.ascontiguousarray(corr, dtype=np.float64)).to(dev)
    j = torch.from_numpy(np.ascontiguousarray(col, dtype=np.int64)).to(dev)
    cs = [torch.empty_like(c) for _ in range(world)]
    js = [torch.empty_like(j) for _ in range(world)]
    dist.all_gather(cs, c, group=group)
    dist.all_gather(js, j, group=group)
    return merge_partials([x.cpu().numpy() for x in cs], [x.cpu().numpy() for x in js])


def self_join_sharded(T, m: int, excl: Optional[int] = None, group=None) -> MatrixProfile:
    """Self-join over the ranks of a torch.distributed group (one GPU each):
    shard of the symmetric sweep, one all-gather, merge, finish.
    NCCL groups keep everything on the device -- partials, the all-gather,
    acc_merge (tsd_profile_merge_device) and the epilogue -- and copy only the
    final profile to the host; other backends exchange host partials."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if dist.get_backend(group) != "nccl":
        corr, col = self_join_partial(T, m, excl, rank, world)
        corr, col = exchange_partials(corr, col, group)
        return self_join_finish(T, m, excl, corr, col)
    x = _vals(T)
    lib = load_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    cnt = max(1, x.size - m + 1)
    d_t = torch.from_numpy(x).to(dev)
    pc = torch.empty(cnt, dtype=torch.float64, device=dev)
    pj = torch.empty(cnt, dtype=torch.int64, device=dev)
    e = _excl_arg(m, excl)
    _check(lib.tsd_self_join_partial_device(d_t.data_ptr(), x.size, m, e, rank, world, pc.data_ptr(), pj.data_ptr(),
                                            stream.cuda_stream))
    allc = torch.empty(world * cnt, dtype=torch.float64, device=dev)
    allj = torch.empty(world * cnt, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, pc, group=group)
    dist.all_gather_into_tensor(allj, pj, group=group)
    _check(lib.tsd_profile_merge_device(allc.data_ptr(), allj.data_ptr(), world, cnt, pc.data_ptr(), pj.data_ptr(),
                                        stream.cuda_stream))
    _check(lib.tsd_self_join_finish_device(d_t.data_ptr(), x.size, m, e, pc.data_ptr(), pj.data_ptr(),
                                           stream.cuda_stream))
    stream.synchronize()
    return MatrixProfile(values=pc.cpu().numpy(), indices=pj.cpu().numpy(), kind="self", m=m)


def dict_shard_rows(nq: int, m: int, shard: int, nshards: int):
    """[lo, hi) query windows of a row shard: whole 16384-window reference
    blocks (dictionary.hpp:175-180), so the shard's statistics match the
    unsharded join's (tsd_dict_shard_rows; host only)."""
    lo, hi = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(load_library().tsd_dict_shard_rows(nq, m, shard, nshards, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def join_dictionary_sharded(A, D: Dictionary, m: int, group=None, precision="fp64", _shard_join=None) -> MatrixProfile:
    """join_dictionary with the query windows sharded over the ranks of a
    torch.distributed group (one GPU each): each rank joins its
    block-aligned row range on its device, one all-gather (NCCL, device
    buffers) assembles the whole profile on every rank. Rows are independent:
    no other exchange. (_shard_join(q_slice) -> (values, indices) replaces the
    per-shard device join on non-NCCL groups; the gloo tests pass the oracle.)"""
    import torch
    import torch.distributed as dist
    if m != D.m:
        raise TsdictError(errc.window_mismatch, "requested window length differs from the dictionary's")
    q = _vals(A)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cnt = q.size - m + 1
    if m < 2 or cnt < 1:
        return join_dictionary(A, D, m, precision=precision)  # the reference's errors
    ranges = [dict_shard_rows(q.size, m, s, world) for s in range(world)]
    per = max(1, max(hi - lo for lo, hi in ranges))
    lo, hi = ranges[rank]
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    v = torch.full((per,), float("inf"), dtype=torch.float64, device=dev)
    j = torch.full((per,), -1, dtype=torch.int64, device=dev)
    if hi > lo:
        if nccl:
            plan = DictPlan(D, m, precision)
            d_q = torch.from_numpy(np.ascontiguousarray(q[lo:hi + m - 1])).to(dev)
            plan.join_device(d_q.data_ptr(), [hi + m - 1 - lo], v.data_ptr(), j.data_ptr(),
                             torch.cuda.current_stream(dev).cuda_stream)
            plan.close()
        else:
            if _shard_join is not None:
                pv, pi = _shard_join(q[lo:hi + m - 1])
            else:
                P = dict_min_profile(q[lo:hi + m - 1], D, m, precision=precision)
                pv, pi = P.values, P.indices
            v[: hi - lo] = torch.from_numpy(np.ascontiguousarray(pv, dtype=np.float64))
            j[: hi - lo] = torch.from_numpy(np.ascontiguousarray(pi, dtype=np.int64))
    av = torch.empty(world * per, dtype=torch.float64, device=dev)
    aj = torch.empty(world * per, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(av, v, group=group)
    dist.all_gather_into_tensor(aj, j, group=group)
    av, aj = av.cpu().numpy(), aj.cpu().numpy()
    vals = np.concatenate([av[s * per: s * per + (h - l)] for s, (l, h) in enumerate(ranges)])
    idx = np.concatenate([aj[s * per: s * per + (h - l)] for s, (l, h) in enumerate(ranges)])
    return MatrixProfile(vals, idx, "ab", m)


@dataclass
class Discord:
    """dict_join.hpp:28-32"""
    start: int
    score: float
    certified: bool = False


def find_discords(P, e_max: float, top_k: int) -> List[Discord]:
    """dict_join.hpp:54-93 on the device: greedy top-k peaks with +-floor(m/2)
    suppression; rank 1 certified when it leads the runner-up by > e_max.
    P: a MatrixProfile, or (d_values_ptr, count, m) of a device-resident profile."""
    lib = load_library()
    cap = max(int(top_k), 1)
    st = np.zeros(cap, dtype=np.uintp)
    sc = np.zeros(cap)
    ce = np.zeros(cap, dtype=np.int32)
    cnt = ctypes.c_size_t(0)
    cep = ce.ctypes.data_as(ctypes.POINTER(_int))
    if isinstance(P, tuple):
        ptr, n, m = P
        _check(lib.tsd_find_discords_device(ctypes.c_void_p(ptr), n, m, e_max, top_k, _ptr(st, _szp), _ptr(sc, _f64p),
                                            cep, ctypes.byref(cnt), None))
    else:
        v = _f64(P.values)
        _check(lib.tsd_find_discords(_ptr(v, _f64p), v.size, P.m, e_max, top_k, _ptr(st, _szp), _ptr(sc, _f64p), cep,
                                     ctypes.byref(cnt)))
    return [Discord(int(st[i]), float(sc[i]), bool(ce[i])) for i in range(cnt.value)]


def window_labels(regions, n: int, m: int) -> np.ndarray:
    """dict_join.hpp:102-127 (host): a window is positive when it overlaps a
    merged region by at least half its length"""
    if m < 2 or m > n:
        raise TsdictError(errc.invalid_argument, "window length out of range")
    for lo, hi in regions:
        if lo >= hi or hi > n:
            raise TsdictError(errc.invalid_argument, "label region out of range")
    merged = []
    for lo, hi in sorted(regions):
        if merged and lo <= merged[-1][1]:
            merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
        else:
            merged.append((lo, hi))
    cnt = n - m + 1
    out = np.zeros(cnt, dtype=np.uint8)
    for lo, hi in merged:  # windows overlapping [lo, hi) by >= m/2 samples
        for i in range(max(0, lo - m + 1), min(cnt, hi)):
            if 2 * (min(i + m, hi) - max(i, lo)) >= m:
                out[i] = 1
    return out


def auc_score(scores, labels) -> float:
    """dict_join.hpp:130-162 (host): exact Mann-Whitney AUC, ties count 1/2"""
    s = np.asarray(scores, dtype=np.float64)
    l = np.asarray(labels).astype(bool)
    if s.size != l.size:
        raise TsdictError(errc.length_mismatch, "scores and labels differ in length")
    if np.isnan(s).any():
        raise TsdictError(errc.invalid_argument, "scores must not contain NaN")
    pos, neg = int(l.sum()), int((~l).sum())
    if pos == 0 or neg == 0:
        raise TsdictError(errc.degenerate_labels, "AUC needs at least one positive and one negative label")
    u, inv = np.unique(s, return_inverse=True)  # ascending distinct scores
    gp = np.bincount(inv, weights=l, minlength=u.size)
    gn = np.bincount(inv, weights=~l, minlength=u.size)
    below = np.concatenate([[0.0], np.cumsum(gn)[:-1]])
    return float(np.sum(gp * (below + 0.5 * gn)) / (pos * neg))


class DictPlan:
    """Dictionary resident in HBM; joins device-resident queries (bench path)."""

    def __init__(self, D: Dictionary, m: int, precision="fp64"):
        vals, lens, starts = _pack_dict(D)
        self._lib = load_library()
        self._h = ctypes.c_void_p()
        self.m = m
        _check(self._lib.tsd_dict_plan_create(_ptr(vals, _f64p), _ptr(lens, _szp), _ptr(starts, _szp),
                                              len(D.segments), m, _PREC[precision], ctypes.byref(self._h)))

    def join_device(self, d_q: int, q_len: Sequence[int], d_val: int, d_idx: int, stream: int = 0) -> None:
        ql = np.asarray(q_len, dtype=np.uintp)
        _check(self._lib.tsd_dict_plan_join_device(self._h, ctypes.c_void_p(d_q), _ptr(ql, _szp), len(ql),
                                                   ctypes.c_void_p(d_val), ctypes.c_void_p(d_idx),
                                                   ctypes.c_void_p(stream)))

    def join_host(self, q: np.ndarray, q_len: Sequence[int], val: np.ndarray, idx: np.ndarray) -> None:
        ql = np.asarray(q_len, dtype=np.uintp)
        _check(self._lib.tsd_dict_plan_join(self._h, _ptr(q, _f64p), _ptr(ql, _szp), len(ql), _ptr(val, _f64p),
                                            _ptr(idx, _i64p)))

    def last_timing(self):
        s, j, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        _check(self._lib.tsd_dict_plan_last_timing(self._h, ctypes.byref(s), ctypes.byref(j), ctypes.byref(n)))
        return s.value, j.value, n.value

    def last_kernel_timing(self):
        """(join kernel ms, FFT heads pre-pass ms) of the last join call (CUDA events)."""
        k, h = ctypes.c_double(), ctypes.c_double()
        _check(self._lib.tsd_dict_plan_last_kernel_timing(self._h, ctypes.byref(k), ctypes.byref(h)))
        return k.value, h.value

    def close(self):
        if self._h:
            self._lib.tsd_dict_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def measure_peak(precision="fp64", seconds: float = 1.0) -> float:
    out = ctypes.c_double()
    _check(load_library().tsd_measure_peak(_PREC[precision], seconds, ctypes.byref(out)))
    return out.value


def measure_peak_clock(precision="fp64", seconds: float = 1.0):
    """(FLOP/s, SM MHz during the FP64 loop)"""
    out, mhz = ctypes.c_double(), ctypes.c_double()
    _check(load_library().tsd_measure_peak_clock(_PREC[precision], seconds, ctypes.byref(out), ctypes.byref(mhz)))
    return out.value, mhz.value


def last_join_timing():
    """(device_ms, kernel_ms, launches) of the last ab_join / self_join on this thread"""
    d, k, n = ctypes.c_double(0.0), ctypes.c_double(0.0), ctypes.c_int(0)
    load_library().tsd_last_join_timing(ctypes.byref(d), ctypes.byref(k), ctypes.byref(n))
    return d.value, k.value, n.value


def build_info() -> str:
    return load_library().tsd_build_info().decode()
