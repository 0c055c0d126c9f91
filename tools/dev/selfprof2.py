"""One symmetric self-join on the 2^21 prefix of the C4 query, m=512 (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2112_12965_b200 as t
import bench
q = bench.make_query(bench.Q_SEED)[: 1 << 21].copy()
P = t.self_join(q, 512)
print("ok")
