"""Development tool: host-time phases of one device-resident join per BASELINE
config (TSD_VERBOSE=1 TSD_VMARKS=1 print them from the library).
usage: TSD_VERBOSE=1 TSD_VMARKS=1 python tools/dev/phases.py [C1 C3 C5]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2112_12965_b200 as tsd
import workloads as W

for name in sys.argv[1:] or ["C1", "C3", "C5"]:
    if name == "C3":
        c = W.c3()
        D = tsd.learn_dictionary(c["train"], W.c3_learn_config())
        series, m = [c["q"]], c["m"]
    else:
        c = {"C1": W.c1, "C5": W.c5, "C4": W.c4}[name]()
        D, m = W.dictionary(c), c["m"]
        series = [c["q"]] if "q" in c else list(c["series"])
    plan = tsd.DictPlan(D, m)
    lens = [len(x) for x in series]
    d_q = torch.from_numpy(np.ascontiguousarray(np.concatenate(series))).cuda()
    rows = sum(n - m + 1 for n in lens)
    dv = torch.empty(rows, dtype=torch.float64, device="cuda")
    di = torch.empty(rows, dtype=torch.int64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.join_device(d_q.data_ptr(), lens, dv.data_ptr(), di.data_ptr())
        t1 = time.perf_counter()
        s, j, nl = plan.last_timing()
        k, h = plan.last_kernel_timing()
        print(f"[{name}] rep {rep}: host {1e3*(t1-t0):.3f} ms, step {s:.3f} ms, join {j:.3f} ms, kernel {k:.3f} ms, "
              f"heads {h:.3f} ms, launches {nl}", file=sys.stderr, flush=True)
    plan.close()
