"""cfg2 decode per step: split (shared static rows) vs interleaved (every
plan row per request), CUDA-graph replay of 64 steps; ids compared."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG2, 64, 64, 0, torch, th, synth)
res = {}
outs = {}
for mode in ("interleaved", "split"):
    s, prep, decode = bench.capture_job(job, mode, torch)
    with torch.cuda.stream(s):
        for _ in range(3):
            prep.replay()
            decode.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        prep.replay()
        a.record(s)
        for _ in range(5):
            decode.replay()
        b.record(s)
    torch.cuda.synchronize()
    res[mode + "_us_per_decode_step"] = a.elapsed_time(b) / 5 / 64 * 1e3
    outs[mode] = job.out.clone()
res["split_stats"] = list(job.sdec.stats())
res["ids_equal"] = bool(torch.equal(outs["interleaved"], outs["split"]))
res["split_bytes_per_step"] = job.decode_bytes("split")
res["interleaved_bytes_per_step"] = job.decode_bytes("interleaved")
print(json.dumps(res, indent=1))
