"""Timing probe: device-resident dictionary joins (development tool).
usage: python tools/timing.py [configs...]  config = NQ:NSEG:L:M"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
cfgs = sys.argv[1:] or ["1048576:32:2048:200", "4194304:256:1024:512"]
tag = os.environ.get("TAG", "")
for c in cfgs:
    nq, nseg, L, m = (int(x) for x in c.split(":"))
    q = synth.walk(4, nq); segs = synth.walks(5, nseg, L)
    D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
    plan = t.DictPlan(D, m, os.environ.get("PREC", "fp64"))
    dq = torch.from_numpy(q).cuda(); cnt = nq - m + 1
    dv = torch.empty(cnt, dtype=torch.float64, device="cuda"); di = torch.empty(cnt, dtype=torch.int64, device="cuda")
    best = 1e9
    for rep in range(3):
        plan.join_device(dq.data_ptr(), [nq], dv.data_ptr(), di.data_ptr())
        best = min(best, plan.last_timing()[1])
    cells = cnt * nseg * (L - m + 1)
    print(f"{tag} {c}: join {best:.2f} ms -> {cells/best/1e9:.3f} TCell/s", flush=True)
