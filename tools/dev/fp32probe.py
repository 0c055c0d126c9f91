"""C4 FP32-mode probe (development tool): device-resident plan joins, kernel
timing, FP32 FFMA peak. usage: python tools/fp32probe.py [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench
import paper_2112_12965_b200 as tsd
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
D, segs = bench.make_dictionary()
q = bench.make_query(4)
nrows = q.size - bench.M + 1
dq = torch.from_numpy(q).cuda()
dv = torch.empty(nrows, dtype=torch.float64, device="cuda"); di = torch.empty(nrows, dtype=torch.int64, device="cuda")
for prec in ("fp32", "fp64"):
    plan = tsd.DictPlan(D, bench.M, prec)
    for r in range(reps + 1):
        plan.join_device(dq.data_ptr(), [bench.Q_LEN], dv.data_ptr(), di.data_ptr())
        s, j, n = plan.last_timing(); k, h = plan.last_kernel_timing()
        print(f"{prec}: step {s:.1f} ms join {j:.1f} kernel {k:.1f} heads {h:.1f} -> {bench.cells_per_step()/(s*1e-3)/1e9:.0f} GCell/s", flush=True)
    del plan
pk32 = tsd.measure_peak("fp32", 1.0); pk64 = tsd.measure_peak("fp64", 1.0)
print(f"peaks: fp32 {pk32/1e12:.1f} TFLOP/s, fp64 {pk64/1e12:.1f} TFLOP/s")
