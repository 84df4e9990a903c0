"""cfg1 e2e per step through the host-buffer C-ABI (prepare_many over the 8
sessions + decode_host of their 64 tokens), median over 40 steps, host
clock (measurement; bench.py's e2e leg is the reported number)."""
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

jobs = bench.Cfg1Jobs(8, 64, 0, torch, th, synth)
V = bench.CFG1["V"]
st = torch.cuda.Stream()
sess = [session.Session(jobs.head, max_batch=1, stream=st) for _ in range(8)]
offs = [np.array([0, len(p)], np.int64) for p in jobs.prompts_h]
hid_h = jobs.hidden.cpu().pin_memory()
ids_h = torch.zeros((64, 8), dtype=torch.int32).pin_memory()
tp, td, tt = [], [], []
for it in range(50):
    t0 = time.perf_counter()
    session.prepare_many(sess, jobs.words_h, V, jobs.prompts_h, offs)
    t1 = time.perf_counter()
    session.decode_host(sess, hid_h, 64, ids_h)
    t2 = time.perf_counter()
    if it >= 10:
        tp.append(t1 - t0)
        td.append(t2 - t1)
        tt.append(t2 - t0)
print(json.dumps({"prepare_us": float(np.median(tp) * 1e6), "decode_host_us": float(np.median(td) * 1e6),
                  "step_us": float(np.median(tt) * 1e6),
                  "tokens_per_s": 512 / float(np.median(tt))}))
