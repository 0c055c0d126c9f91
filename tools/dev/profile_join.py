"""One dictionary join on device-resident inputs, for ncu (development tool).
usage: python tools/profile_join.py NQ NSEG L M [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth

nq, nseg, L, m = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
q = synth.walk(4, nq); segs = synth.walks(5, nseg, L)
D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
plan = t.DictPlan(D, m, os.environ.get("PREC", "fp64"))
dq = torch.from_numpy(q).cuda(); cnt = nq - m + 1
dv = torch.empty(cnt, dtype=torch.float64, device="cuda"); di = torch.empty(cnt, dtype=torch.int64, device="cuda")
for _ in range(reps):
    plan.join_device(dq.data_ptr(), [nq], dv.data_ptr(), di.data_ptr())
    s, j, n = plan.last_timing()
    print(f"step {s:.3f} ms join {j:.3f} ms cells/s {cnt*nseg*(L-m+1)/(j*1e-3):.4g}")
