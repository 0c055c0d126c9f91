"""Development tool: time library variants (tools/dev/abl_build.sh) on the
same inputs and check that their profiles are bit-identical to the first.
usage: python tools/dev/variants.py LIB1.so[@ENV=VAL,...] LIB2.so ... -- CFG ...
CFG = dict:NQ:NSEG:L:M[:PREC] | self:N:M[:EXCL]  (walk inputs, seeds 4 / 5)"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

CHILD = r'''
import sys, os, json, time
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
out = {}
for c in %r:
    f = c.split(":")
    if f[0] == "dict":
        nq, nseg, L, m = map(int, f[1:5]); prec = f[5] if len(f) > 5 else "fp64"
        if os.environ.get("DICTKIND") == "traffic":  # C5-like near-periodic query and dictionary
            q = synth.traffic(6, 1, nq)[0]; segs = synth.traffic(7, nseg, L)
        else:
            q = synth.walk(4, nq); segs = synth.walks(5, nseg, L)
        D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
        plan = t.DictPlan(D, m, prec)
        dq = torch.from_numpy(q).cuda(); cnt = nq - m + 1
        dv = torch.empty(cnt, dtype=torch.float64, device="cuda"); di = torch.empty(cnt, dtype=torch.int64, device="cuda")
        ks = []
        for rep in range(4):
            plan.join_device(dq.data_ptr(), [nq], dv.data_ptr(), di.data_ptr())
            ks.append(plan.last_kernel_timing()[0])
        cells = cnt * nseg * (L - m + 1)
        v, i = dv.cpu().numpy(), di.cpu().numpy()
        plan.close()
    else:
        n, m = int(f[1]), int(f[2]); excl = int(f[3]) if len(f) > 3 else None
        x = synth.walk(4, n) if os.environ.get("SELFKIND") != "ecg" else synth.ecg(2, n)[0]
        ks = []
        for rep in range(4):
            P = t.self_join(x, m, excl=excl)
            ks.append(t.last_join_timing()[1])
        cnt = n - m + 1; e = m // 2 if excl is None else excl
        cells = (cnt - e - 1) * (cnt - e) // 2
        v, i = P.values, P.indices
    k = sorted(ks[1:])[len(ks[1:]) // 2]
    np.savez(os.path.join(%r, c.replace(":", "_") + ".npz"), v=v, i=i)
    out[c] = {"kernel_ms": k, "all": ks, "frac_nominal": 6 * cells / (k * 1e-3) / 37.21e12}
print("RESULT " + json.dumps(out), flush=True)
'''

def main():
    a = sys.argv[1:]
    libs, cfgs = a[:a.index("--")], a[a.index("--") + 1:]
    res = {}
    base = None
    for spec in libs:
        lib, _, evs = spec.partition("@")
        d = os.path.join("/tmp", "tsd_variants", os.path.basename(spec).replace(".so", "").replace("=", "_").replace(",", "_"))
        os.makedirs(d, exist_ok=True)
        env = dict(os.environ, TSD_LIB=os.path.abspath(lib))
        for kv in filter(None, evs.split(",")):
            env[kv.split("=")[0]] = kv.split("=")[1]
        lib = spec
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfgs, d)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(lib, "FAILED", r.stdout[-2000:], r.stderr[-3000:], flush=True)
            continue
        res[lib] = json.loads(line[0][7:])
        import numpy as np
        same = {}
        if base is None:
            base = d
        else:
            for c in cfgs:
                fn = c.replace(":", "_") + ".npz"
                x, y = np.load(os.path.join(base, fn)), np.load(os.path.join(d, fn))
                same[c] = bool(np.array_equal(x["v"], y["v"]) and np.array_equal(x["i"], y["i"]))
                if not same[c]:  # different plans restart the recurrence at other rows: report the distance
                    fin = np.isfinite(x["v"]) & np.isfinite(y["v"])
                    rel = float(np.max(np.abs(x["v"][fin] - y["v"][fin]) / np.maximum(x["v"][fin], 1e-300))) if fin.any() else 0.0
                    same[c] = {"max_rel": rel, "index_mismatches": int(np.sum(x["i"] != y["i"])),
                               "nonfinite_mismatch": int(np.sum(np.isfinite(x["v"]) != np.isfinite(y["v"])))}
        print(json.dumps({"lib": lib, "res": res[lib], "bitwise_equal_to_first": same}), flush=True)

main()
