"""One self-join for ncu (development tool). usage: python tools/selfprof.py n m"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2112_12965_b200 as t
from paper_2112_12965_b200 import synth
n, m = int(sys.argv[1]), int(sys.argv[2])
x = synth.walk(7, n)
P = t.self_join(x, m)
print("ok", P.values[:3])
