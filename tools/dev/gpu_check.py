"""Quick GPU parity + timing probe (development tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
from oracle import py_oracle as O

def cmp(name, gv, gi, ov, oi, a=None, b=None, m=None):
    fin = np.isfinite(ov)
    rel = np.abs(gv[fin] - ov[fin]) / np.maximum(ov[fin], 1e-300)
    mism = np.nonzero(gi != oi)[0]
    print(f"{name}: rows={len(gv)} max_rel={rel.max() if rel.size else 0:.3g} max_abs={np.abs(gv[fin]-ov[fin]).max() if fin.any() else 0:.3g} idx_mismatch={len(mism)} inf_match={np.array_equal(np.isinf(gv), np.isinf(ov))}", flush=True)
    if len(mism):
        for r in mism[:5]:
            print("   row", r, "gpu", gi[r], gv[r], "oracle", oi[r], ov[r])

rng = synth.Rng(35)
A = rng.noise(300); B = rng.noise(200)
v, i = t.ab_join(A, B, 20).values, t.ab_join(A, B, 20).indices
ov, oi = O.ab_join(A, B, 20)
cmp("ab noise 300x200 m20", v, i, ov, oi)

for (na, nb, m) in [(1000, 700, 16), (5000, 3000, 100), (20000, 4096, 100), (3000, 2500, 7)]:
    A = synth.walk(1, na); B = synth.walk(2, nb)
    P = t.ab_join(A, B, m)
    ov, oi = O.ab_join(A, B, m)
    cmp(f"ab walk {na}x{nb} m{m}", P.values, P.indices, ov, oi)

for (n, m, e) in [(2000, 50, None), (5000, 64, 16), (16, 8, None), (3000, 250, 62)]:
    T = synth.walk(3, n)
    P = t.self_join(T, m, excl=e)
    ov, oi = O.self_join(T, m, e)
    cmp(f"self walk n{n} m{m} excl{e}", P.values, P.indices, ov, oi)

# C1 config
q = synth.walk(0, 16384); segs = synth.walks(1, 8, 512)
D = t.Dictionary([t.Segment(512 * s, segs[s]) for s in range(8)], m=100, source_length=4096)
P = t.join_dictionary(q, D, 100)
ov, oi = O.dict_join(q, list(segs), [512 * s for s in range(8)], 100)
cmp("C1 dict join", P.values, P.indices, ov, oi)

# timing: C3-sized-ish (2^20 x 32 x 2048, m=200) and C4 prefix
for (nq, nseg, L, m) in [(1 << 20, 32, 2048, 200), (1 << 22, 256, 1024, 512)][:int(os.environ.get('NTIME','2'))]:
    q = synth.walk(4, nq); segs = synth.walks(5, nseg, L)
    D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
    plan = t.DictPlan(D, m)
    import torch
    dq = torch.from_numpy(q).cuda(); cnt = nq - m + 1
    dv = torch.empty(cnt, dtype=torch.float64, device="cuda"); di = torch.empty(cnt, dtype=torch.int64, device="cuda")
    for rep in range(3):
        plan.join_device(dq.data_ptr(), [nq], dv.data_ptr(), di.data_ptr())
        step, jms, nl = plan.last_timing()
        cells = cnt * nseg * (L - m + 1)
        print(f"timing nq={nq} nseg={nseg} L={L} m={m}: step {step:.2f} ms join {jms:.2f} ms -> {cells/jms/1e9:.1f} GCell/s (join), launches {nl}", flush=True)
    # spot-check a few rows against the oracle on the single-window slice
    gv = dv.cpu().numpy(); gi = di.cpu().numpy()
    rows = np.random.default_rng(0).choice(cnt, 8, replace=False)
    bad = 0
    for r in rows:
        ov, oi = O.dict_join(q[r:r + m], list(segs), [L * s for s in range(nseg)], m)
        if oi[0] != gi[r] or abs(ov[0] - gv[r]) > 1e-8 * ov[0]:
            bad += 1; print("  row", r, gi[r], gv[r], oi[0], ov[0])
    print("  sampled rows bad:", bad)
