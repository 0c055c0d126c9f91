# development: ncu --set full of the FP64 AB sweep on a C5-like (near-periodic) shape
cat > /tmp/c5one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
nq, nseg, L, m = 1048576, 64, 1024, 128
q = synth.traffic(6, 1, nq)[0]; segs = synth.traffic(7, nseg, L)
D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
t.join_dictionary(q, D, m)
PY
ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/c5like -f python /tmp/c5one.py > gpurun_out/ncu_c5.log 2>&1
tail -2 gpurun_out/ncu_c5.log
