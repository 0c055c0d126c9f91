"""Development: one dictionary join through a TSD_COUNT_EXACT build (TSD_LIB), counters on stderr.
usage: [DICTKIND=traffic] python tools/dev/cntdict.py NQ NSEG L M"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
nq, nseg, L, m = map(int, sys.argv[1:5])
if os.environ.get("DICTKIND") == "traffic":
    q = synth.traffic(6, 1, nq)[0]; segs = synth.traffic(7, nseg, L)
else:
    q = synth.walk(4, nq); segs = synth.walks(5, nseg, L)
D = t.Dictionary([t.Segment(L * s, segs[s]) for s in range(nseg)], m=m, source_length=nseg * L)
t.join_dictionary(q, D, m)
