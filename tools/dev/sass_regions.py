"""Summarise an ncu source-page CSV (SASS view) by contiguous execution-count
regions (development tool).  usage: python tools/sass_regions.py sass.csv [min_frac]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))[1:]
h = rows[0]; rows = rows[1:]
isrc = h.index("Source"); ie = h.index("Instructions Executed"); ist = h.index("Warp Stall Sampling (All Samples)")
minf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
ex = [float(r[ie] or 0) for r in rows]; st = [float(r[ist] or 0) for r in rows]
mx = max(ex); tot = sum(ex); stot = sum(st)
print(f"total warp-inst {tot:.4g}  samples {stot:.0f}  max-count {mx:.4g}")
start = 0
def flush(a, b):
    acc = sum(ex[a:b + 1]); sacc = sum(st[a:b + 1])
    if acc / tot > minf or sacc / stot > minf:
        print(f"{a:5d}-{b:5d} n={b-a+1:4d} ratio~{ex[a]/mx:6.3f} inst {acc/tot*100:5.2f}% samples {sacc/stot*100:5.2f}%  {rows[a][isrc][:50]}")
for i in range(1, len(rows) + 1):
    if i == len(rows) or abs(ex[i] - ex[start]) > 0.002 * mx:
        flush(start, i - 1); start = i
