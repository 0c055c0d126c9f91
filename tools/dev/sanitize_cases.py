"""Small cases of every device path for compute-sanitizer (memcheck /
racecheck / synccheck): AB join, dictionary join with FFT heads and FFT top
edges, full-matrix and symmetric (seeded) self-joins, the FP32 mode, the
sharded self-join device steps, distance profiles, learning, discords.
usage: [compute-sanitizer --tool X] python tools/dev/sanitize_cases.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2112_12965_b200 as tsd
from paper_2112_12965_b200 import synth


def main():
    a, b = synth.walk(1, 3000), synth.walk(2, 2500)
    tsd.ab_join(a, b, 100)
    tsd.ab_join(a, b, 64, precision="fp32")
    q = synth.walk(3, 20000)
    segs = synth.walks(4, 6, 1024)
    D = tsd.Dictionary([tsd.Segment(2048 * s, segs[s]) for s in range(6)], m=256, source_length=12288)
    tsd.join_dictionary(q, D, 256)                      # FFT heads + FFT top edges
    tsd.join_dictionary(q, D, 256, precision="fp32")
    tsd.join_dictionary_batched([q[:5000], q[5000:9000]], D, 256)
    t = synth.ecg(5, 12000)[0]
    t[3000:3400] = 0.5
    os.environ["TSD_SYM"] = "0"
    tsd.self_join(t, 128)
    os.environ["TSD_SYM"] = "1"
    tsd.self_join(t, 128, excl=32)
    w = synth.walk(6, 40000)
    tsd.self_join(w, 128)                               # symmetric + coarse seeds
    corr, col = tsd.self_join_partial(w, 128, None, 0, 2)
    st = tsd.compute_stats(w, 128)
    tsd.distance_profile_naive(w, w[100:228], st, 100)
    tsd.distance_profile_mass(w, w[100:228], st, 100)
    P = tsd.join_dictionary(q, D, 256)
    tsd.find_discords(P, 0.5, 5)
    tsd.learn_dictionary(t, tsd.LearnConfig(m=100, space_saving_target=0.7))
    print("SANITIZE_CASES_OK", flush=True)


if __name__ == "__main__":
    main()
