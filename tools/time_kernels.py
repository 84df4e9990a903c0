"""Time the non-decode kernels of one cfg2 job step (select, layout, gather)
with CUDA events over repeated launches."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402


def ev_time(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


job = bench.Job(bench.CFG2, 64, 2, 0, torch, th, synth)
tb = job.tb
n = int(tb.n_active.sum().item())
gbytes = 2 * n * 896 * 2
out = {"select_plus_layout_us": ev_time(tb.run_select),
       "gather_us": ev_time(lambda: tb.gather(job.head)),
       "gather_algorithmic_bytes": gbytes}
out["gather_gbs"] = gbytes / out["gather_us"] / 1e3
print(json.dumps(out))
