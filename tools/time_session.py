"""Host-buffer session (svt_session_*) at cfg2: wall time of prepare and of
one greedy step (pinned buffers -> step graph), to split the e2e overhead."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import session, synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG2, 64, 64, 0, torch, th, synth)
d = job.cfg["d"]
hid_h = job.hidden[:, :, :d].cpu().pin_memory()
ids_h = torch.empty((64, 64), dtype=torch.int32).pin_memory()
res = {}
with session.Session(job.head, max_batch=64) as s:
    for _ in range(3):
        s.prepare(job.words_h, job.cfg["V"], job.flat_h, job.off_h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        s.prepare(job.words_h, job.cfg["V"], job.flat_h, job.off_h)
    torch.cuda.synchronize()
    res["prepare_us"] = (time.perf_counter() - t0) / 10 * 1e6
    for t in range(64):
        s.greedy(hid_h[t], ids_h[t])
    t0 = time.perf_counter()
    for k in range(5):
        for t in range(64):
            s.greedy(hid_h[t], ids_h[t])
    res["greedy_step_us"] = (time.perf_counter() - t0) / 320 * 1e6
    t0 = time.perf_counter()
    for k in range(320):
        s.greedy(hid_h[0], ids_h[0])
    res["greedy_same_buffers_us"] = (time.perf_counter() - t0) / 320 * 1e6
print(json.dumps(res))
