"""Development: window-norm ranges the FP32 mode sees on the BASELINE shapes (TSD_VERBOSE line)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["TSD_VERBOSE"] = "1"
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
import workloads as W
def run(name, q, segs, starts, m):
    D = t.Dictionary([t.Segment(st, s) for s, st in zip(segs, starts)], m=m, source_length=max(st + len(s) for s, st in zip(segs, starts)))
    print("==", name, flush=True); t.join_dictionary(q, D, m, precision="fp32")
q = synth.walk(4, 1 << 24); segs = synth.walks(5, 256, 1024)
run("C4", q, list(segs), [1024 * s for s in range(256)], 512)
q = synth.walk(0, 16384); segs = synth.walks(1, 8, 512)
run("C1", q, list(segs), [512 * s for s in range(8)], 100)
q, _ = synth.ecg(3, 1 << 20, 20); train, _ = synth.ecg(13, 32 * 2048 * 4)
run("C3-like", q, [train[k * 8192: k * 8192 + 2048] for k in range(32)], [k * 8192 for k in range(32)], 200)
q = synth.traffic(6, 64, 8192).reshape(-1); segs = synth.traffic(7, 64, 1024)
run("C5-like (64 series concatenated as one)", q, list(segs), [1024 * s for s in range(64)], 128)
