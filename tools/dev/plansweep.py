"""Forced decomposition plans on C4 (development tool): kernel and step ms
for G in 4..32 and several bands per task. usage: python tools/dev/plansweep.py fp32|fp64"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2112_12965_b200 as tsd
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
D, segs = bench.make_dictionary()
q = bench.make_query(4)
nrows = q.size - bench.M + 1
dq = torch.from_numpy(q).cuda()
dv = torch.empty(nrows, dtype=torch.float64, device="cuda"); di = torch.empty(nrows, dtype=torch.int64, device="cuda")
plan = tsd.DictPlan(D, bench.M, prec)
plan.join_device(dq.data_ptr(), [bench.Q_LEN], dv.data_ptr(), di.data_ptr())
res = []
for G in (4, 8, 16, 32):
    for bpt in ((2, 4, 7, 8) if prec == "fp32" else (7, 14, 28, 56)):
        os.environ["TSD_FORCE_G"] = str(G); os.environ["TSD_FORCE_BPT"] = str(bpt)
        ks = []
        for r in range(2):
            plan.join_device(dq.data_ptr(), [bench.Q_LEN], dv.data_ptr(), di.data_ptr())
            s, j, n = plan.last_timing(); k, h = plan.last_kernel_timing(); ks.append((k, s))
        k = min(x[0] for x in ks); s = min(x[1] for x in ks)
        print(f"G={G} bpt={bpt}: kernel {k:.1f} step {s:.1f}", flush=True)
