import os, sys, json, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2508_15229_b200 import synth
from paper_2508_15229_b200 import tailored_head as th
job = bench.Job(bench.CFG2, 64, 64, 0, torch, th, synth)
res = {}
for w, st in [(0, 0), (4, 3), (8, 3), (6, 2), (6, 4), (12, 2), (16, 2)]:
    th._lib.lib.svt_set_tuning(w, st)
    s, prep, decode = bench.capture_job(job, "split", torch)
    with torch.cuda.stream(s):
        for _ in range(3):
            prep.replay(); decode.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        prep.replay(); a.record(s)
        for _ in range(5):
            decode.replay()
        b.record(s)
    torch.cuda.synchronize()
    res[f"{w},{st}"] = a.elapsed_time(b) / 5 / 64 * 1e3
print(json.dumps(res))
