"""cfg2 split decode: the static half alone (SVT_SPLIT_STATIC_ONLY=1, measurement
knob) vs the whole step, CUDA-graph replay of 64 steps, warm; run with
SVT_SPLIT_EXACT=0/1 to compare the certified and the exact-chain halves."""
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
res = {"exact": os.environ.get("SVT_SPLIT_EXACT", "0"),
       "serial": os.environ.get("SVT_SPLIT_SERIAL", "0")}
for only in ("0", "1"):
    if only == "1":
        os.environ["SVT_SPLIT_STATIC_ONLY"] = "1"
    else:
        os.environ.pop("SVT_SPLIT_STATIC_ONLY", None)
    s, prep, decode = bench.capture_job(job, "split", torch)
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
    res["static_only_us" if only == "1" else "step_us"] = a.elapsed_time(b) / 5 / 64 * 1e3
res["cert_stats"] = job.sdec.stats()
print(json.dumps(res))
