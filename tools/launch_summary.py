"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) to
one step: the launches from occurrence k-1 of `first` up to occurrence k
(default k = -1: the last complete step; use -2 when extra launches follow
the timed steps).
usage: launch_summary.py launches.csv first_kernel_substring what [k] > summary.json"""
import csv
import json
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
launches = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
    name = name.replace("svt::", "").replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
    launches.append((name, us))
first = sys.argv[2]
idx = [i for i, (n, _) in enumerate(launches) if first in n]
k = int(sys.argv[4]) if len(sys.argv) > 4 else -1
a, b = idx[k - 1], idx[k]
step = launches[a:b]
tot = sum(u for _, u in step)
print(json.dumps({"what": sys.argv[3],
                  "step_kernels": [{"kernel": n, "us": u, "share": u / tot} for n, u in step],
                  "step_total_us": tot}, indent=1))
