"""Per-launch time of svt_greedy_certified_rows variants at cfg1 (events over
back-to-back launches, warm), for latency breakdown. SVT_ROWS_VARIANT is read
per launch: 0 full, 1 empty, 2 loads only, 3 no tail."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG1, 1, 64, 0, torch, th, synth)
res = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for var in ["1", "2", "3", "0"]:
    os.environ["SVT_ROWS_VARIANT"] = var
    for k in range(10):
        job.rdec.greedy(job.hidden[k][0], job.out[k])
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    job.rdec.stream = s
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for k in range(64):
            job.rdec.greedy(job.hidden[k][0], job.out[k])
    job.rdec.stream = None
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    warm = a.elapsed_time(b) / 640 * 1e3
    cold = []
    for k in range(20):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        job.rdec.greedy(job.hidden[k][0], job.out[k])
        e1.record()
        torch.cuda.synchronize()
        cold.append(e0.elapsed_time(e1) * 1e3)
    res[var] = {"warm_us": warm, "cold_us_med": sorted(cold)[10]}
# empty torch kernel for the event/launch floor
z = torch.zeros(1, device="cuda")
cold = []
for k in range(20):
    flush.fill_(k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    z.add_(1)
    e1.record()
    torch.cuda.synchronize()
    cold.append(e0.elapsed_time(e1) * 1e3)
res["torch_add_cold_us"] = sorted(cold)[10]
print(json.dumps(res, indent=1))
