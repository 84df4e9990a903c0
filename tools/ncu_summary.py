"""Summarise an ncu report's raw page (ncu -i X.ncu-rep --page raw --csv) to
JSON: per launch, time, DRAM bytes, throughputs, occupancy, launch shape and
the top warp-stall reasons (per issued instruction).
usage: ncu_summary.py raw.csv "command" "note" > summary.json"""
import csv
import json
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fma.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
STALL = "smsp__average_warps_issue_stalled_"
SUFFIX = "_per_issue_active.ratio"

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
out = []
for r in data:
    d = {"Kernel Name": r[col["Kernel Name"]]}
    for k in KEYS:
        if k in col and r[col[k]] not in ("", "n/a"):
            d[k] = f"{r[col[k]]} {units[col[k]]}".strip()
    stalls = {}
    for h, i in col.items():
        if h.startswith(STALL) and h.endswith(SUFFIX):
            try:
                stalls[h[len(STALL):-len(SUFFIX)]] = float(r[i].replace(",", ""))
            except ValueError:
                pass
    d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    out.append(d)
print(json.dumps({"command": sys.argv[2], "note": sys.argv[3] if len(sys.argv) > 3 else "",
                  "launches": out}, indent=1))
