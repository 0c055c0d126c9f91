"""The five BASELINE.json configs as seeded synthetic inputs, shared by
bench.py and the parity tests so both see the same arrays.

No public dataset is used (BASELINE.json names none; the paper's MIT-BIH and
Melbourne data are not in the image): every input is drawn host-side by the
package's std::mt19937_64 generators (paper_2112_12965_b200/synth.py), with
the shapes, seeds and value distributions the configs state.

  C1  exact AB-join, m = 100: walk(seed 0, 16384) vs 8 walks x 512 (seed 1)
  C2  self-join, m = 250, excl = m/4 = 62: ECG-like, n = 131072 (seed 2)
  C3  streaming anomaly scoring, m = 200: ECG-like query of 2^20 samples with
      20 inverted/widened beats (seed 3) vs a dictionary LEARNED from the C2
      series (learn_dictionary, dictionary.hpp:259-328: k = 9.24 so each pick
      stores a 2048-sample context, sample budget 65536 = 32 x 2048), then the
      top-20 discords (find_discords, dict_join.hpp:54-92)
  C4  large AB-join, m = 512: walk(seed 4, 2^24) vs 256 walks x 1024 (seed 5)
  C5  batched joins, m = 128: 4096 traffic-like series x 8192 (seed 6) vs one
      shared dictionary of 64 segments x 1024 samples taken every 2048
      samples of a traffic-like source (seed 7)
"""
from __future__ import annotations

import functools

import numpy as np


def cells(nq_rows, seg_windows):
    """valid (query window, dictionary window) pairs"""
    return int(nq_rows) * int(seg_windows)


@functools.lru_cache(maxsize=None)
def c1():
    from paper_2112_12965_b200 import synth
    m = 100
    q = synth.walk(0, 16384)
    segs = [s.copy() for s in synth.walks(1, 8, 512)]
    starts = [512 * s for s in range(8)]
    return {"name": "C1", "m": m, "q": q, "segs": segs, "starts": starts, "source_length": 4096,
            "cells": cells(q.size - m + 1, sum(len(s) - m + 1 for s in segs))}


@functools.lru_cache(maxsize=None)
def c2():
    from paper_2112_12965_b200 import synth
    m, excl = 250, 62
    t = synth.ecg(2, 131072)[0]
    cnt = t.size - m + 1
    pairs = (cnt - excl - 1) * (cnt - excl) // 2
    return {"name": "C2", "m": m, "excl": excl, "t": t, "pairs": pairs}


C3_M = 200
C3_K = 2048 / C3_M - 1.0  # context k*m + window m = 2048 samples per pick (dictionary.hpp:78-84)
C3_BUDGET = 65536
C3_TOPK = 20


@functools.lru_cache(maxsize=None)
def c3():
    from paper_2112_12965_b200 import synth
    q, anom = synth.ecg(3, 1 << 20, 20)
    train = c2()["t"]
    return {"name": "C3", "m": C3_M, "q": q, "anomalies": anom, "train": train, "k": C3_K,
            "budget": C3_BUDGET, "top_k": C3_TOPK}


@functools.lru_cache(maxsize=None)
def c4():
    from paper_2112_12965_b200 import synth
    m = 512
    q = synth.walk(4, 1 << 24)
    segs = synth.walks(5, 256, 1024)
    starts = [1024 * s for s in range(256)]
    return {"name": "C4", "m": m, "q": q, "segs": segs, "starts": starts, "source_length": 256 * 1024,
            "cells": cells(q.size - m + 1, 256 * (1024 - m + 1))}


@functools.lru_cache(maxsize=None)
def c5():
    from paper_2112_12965_b200 import synth
    m = 128
    series = synth.traffic(6, 4096, 8192)
    src = synth.traffic(7, 1, 131072)[0]
    segs = [src[2048 * k: 2048 * k + 1024].copy() for k in range(64)]
    starts = [2048 * k for k in range(64)]
    return {"name": "C5", "m": m, "series": series, "segs": segs, "starts": starts, "source_length": src.size,
            "cells": cells(4096 * (8192 - m + 1), 64 * (1024 - m + 1))}


def dictionary(cfg):
    import paper_2112_12965_b200 as tsd
    return tsd.Dictionary([tsd.Segment(st, s) for st, s in zip(cfg["starts"], cfg["segs"])], m=cfg["m"],
                          source_length=cfg["source_length"])


def c3_learn_config():
    import paper_2112_12965_b200 as tsd
    return tsd.LearnConfig(m=C3_M, k=C3_K, sample_budget=C3_BUDGET)
