"""Steady-state timeline of the certified rows decode with R token-interleaved
cfg1 jobs (cold sub-heads, tools/time_cfg1_rot.py): per-launch %globaltimer
stamp regions (svt_rows_set_debug), medians over CTAs, in ns from the first
stamped CTA start."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = sys.argv[:1] + ["0"]
import time_cfg1_rot as rot  # noqa: E402

th = rot.th
R = int(os.environ.get("R", "8"))
jobs, hid, out = rot.make(R)
K = 16
dbg = torch.zeros((K, 256 * 128), dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()
for _, rd, _ in jobs:
    rd.stream = s


def decode(stamp):
    k = 0
    for t in range(4):
        for j, (_, rd, _) in enumerate(jobs):
            if stamp and k < K:
                th._lib.lib.svt_rows_set_debug(dbg[k].data_ptr())
            elif stamp:
                th._lib.lib.svt_rows_set_debug(None)
            rd.greedy(hid[t, j], out[t, j], hidden_stable=rot.HS)
            k += 1
    th._lib.lib.svt_rows_set_debug(None)


with torch.cuda.stream(s):
    decode(False)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    decode(True)
with torch.cuda.stream(s):
    for _ in range(3):
        g.replay()
torch.cuda.synchronize()
dbg.zero_()
with torch.cuda.stream(s):
    g.replay()
torch.cuda.synchronize()
d = dbg.view(K, 256, 128).cpu().numpy().astype(np.int64)
G = 148 if os.environ.get("SVT_ROWS_FAST", "1") == "0" else 147
t0 = d[0, :G, 0][d[0, :G, 0] > 0].min()
for k in range(K):
    x = d[k, :G, :8] - t0
    sm = d[k, :G, 8]
    print(json.dumps({"k": k, "start_min": int(x[:, 0].min()), "start_med": int(np.median(x[:, 0])), "start_max": int(x[:, 0].max()),
                      "distinct_sms": int(len(set(sm.tolist()))),
                      "depwait_med": int(np.median(x[:, 1])), "rows_in_med": int(np.median(x[:, 7])),
                      "rows_in_max": int(x[:, 7].max()), "h_med": int(np.median(x[:, 2])),
                      "reduced_med": int(np.median(x[:, 3])), "ctl_L_med": int(np.median(x[:, 5])),
                      "ctl_ids_med": int(np.median(x[:, 6])), "record_med": int(np.median(x[:, 4])),
                      "record_max": int(x[:, 4].max()),
                      "fin_start": int(d[k, 0, 123] - t0), "fin_seen": int(d[k, 0, 124] - t0), "fin_done": int(d[k, 0, 126] - t0)}))
