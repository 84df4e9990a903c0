"""Host time of svt_session_prepare_host_many for the cfg1 sessions (R=8
batch-1 sessions on one stream), per call, with the device drained before
each call (what the e2e loop sees after decode_host's synchronisation)."""
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

jobs = bench.Cfg1Jobs(8, 4, 0, torch, th, synth)
V = bench.CFG1["V"]
st = torch.cuda.Stream()
res = {}
for R in (1, 8):
    sess = [session.Session(jobs.head, max_batch=1, stream=st) for _ in range(R)]
    offs = [np.array([0, len(p)], np.int64) for p in jobs.prompts_h[:R]]
    ts, tw = [], []
    for it in range(60):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        session.prepare_many(sess, jobs.words_h, V, jobs.prompts_h[:R], offs)
        t1 = time.perf_counter()
        st.synchronize()
        t2 = time.perf_counter()
        if it >= 10:
            ts.append(t1 - t0)
            tw.append(t2 - t0)
    res[f"R{R}_call_us"] = float(np.median(ts) * 1e6)
    res[f"R{R}_call_plus_drain_us"] = float(np.median(tw) * 1e6)
    for s_ in sess:
        s_.close()
print(json.dumps(res))
