"""Development: window-statistics time and outputs of the fused tile kernel against the scan kernels
(TSD_STATS_TILE=0), through tsd_compute_stats_device-less public calls: a child process per setting."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import sys, time
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
import workloads as W
out = {}
for name, x, m in (("walk 2^24 m=512", synth.walk(4, 1 << 24), 512), ("ecg 2^20 m=200", synth.ecg(3, 1 << 20)[0], 200),
                   ("walk 70001 m=3000", synth.walk(9, 70001), 3000), ("noise 5000 m=2", synth.Rng(3).noise(5000), 2)):
    st = t.compute_stats(x, m)
    np.savez(%r + "/" + name.replace(" ", "_").replace("^", "") + ".npz", a=st.means, b=st.stds, c=st.invn, d=st.constant_mask)
# device time of the statistics inside a C4 dictionary join
c = W.c4(); D = W.dictionary(c); plan = t.DictPlan(D, c["m"])
dq = torch.from_numpy(c["q"]).cuda(); rows = len(c["q"]) - c["m"] + 1
dv = torch.empty(rows, dtype=torch.float64, device="cuda"); di = torch.empty(rows, dtype=torch.int64, device="cuda")
for rep in range(3):
    plan.join_device(dq.data_ptr(), [len(c["q"])], dv.data_ptr(), di.data_ptr())
print("C4 plan timing (stats ms, join ms, launches):", plan.last_timing(), flush=True)
np.savez(%r + "/c4join.npz", a=dv.cpu().numpy(), b=di.cpu().numpy())
'''
dirs = []
for tile in ("0", "1"):
    d = "/tmp/statstime_" + tile
    os.makedirs(d, exist_ok=True)
    dirs.append(d)
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, d, d)], env=dict(os.environ, TSD_STATS_TILE=tile),
                       capture_output=True, text=True)
    print("TSD_STATS_TILE=" + tile, r.stdout.strip()[-300:], r.stderr.strip()[-800:])
import numpy as np
for f in sorted(os.listdir(dirs[0])):
    a, b = np.load(os.path.join(dirs[0], f)), np.load(os.path.join(dirs[1], f))
    print(f, {k: bool(np.array_equal(a[k], b[k])) for k in a.files},
          {k: float(np.max(np.abs(a[k].astype(float) - b[k].astype(float)))) for k in a.files})
