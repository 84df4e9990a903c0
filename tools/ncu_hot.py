"""Top SASS instructions by warp-stall samples from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))[1:]
hdr = rows[0]
i = hdr.index("Warp Stall Sampling (All Samples)")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
data = []
for k, r in enumerate(rows[1:]):
    try:
        data.append((float(r[i] or 0), k, r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for s, k, src in sorted(data, reverse=True)[:n]:
    print(f"{s / tot * 100:5.1f}%  #{k:5d}  {src[:100]}")
