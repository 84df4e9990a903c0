"""cfg2 e2e per step through the session C-ABI (svt_session_prepare_host of
the 64-request batch + svt_session_decode_host of its 64 steps): host time
of each part, median over 30 steps (measurement)."""
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
B, steps, d = job.B, job.steps, job.cfg["d"]
hid_h = job.hidden[:, :, :d].contiguous().cpu().pin_memory()
ids_h = torch.empty((steps, B), dtype=torch.int32).pin_memory()
tp, td = [], []
with session.Session(job.head, max_batch=B) as s:
    for it in range(40):
        t0 = time.perf_counter()
        s.prepare(job.words_h, job.cfg["V"], job.flat_h, job.off_h)
        t1 = time.perf_counter()
        session.decode_host([s], hid_h, steps, ids_h)
        t2 = time.perf_counter()
        if it >= 10:
            tp.append(t1 - t0)
            td.append(t2 - t1)
print(json.dumps({"prepare_us": float(np.median(tp) * 1e6),
                  "decode_host_us": float(np.median(td) * 1e6),
                  "tokens_per_s": B * steps / (float(np.median(tp)) + float(np.median(td)))}))
