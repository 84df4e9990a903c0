"""Steady-state timeline of svt_greedy_certified_rows inside a CUDA graph
(cfg1): every launch gets its own %globaltimer stamp region, so the overlap
between step t's finalize and step t+1's rows grid is visible."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG1, 1, 64, 0, torch, th, synth)
dec = job.rdec
K = 8
dbg = torch.zeros((K, 256 * 128), dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()
dec.stream = s
with torch.cuda.stream(s):
    for k in range(K):
        dec.greedy(job.hidden[k][0], job.out[k])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for k in range(K):
        th._lib.lib.svt_rows_set_debug(dbg[k].data_ptr())
        dec.greedy(job.hidden[k][0], job.out[k])
th._lib.lib.svt_rows_set_debug(None)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
dbg.zero_()
g.replay()
torch.cuda.synchronize()
d = dbg.view(K, 256, 128).cpu().numpy().astype(np.int64)
G = 148
ghz = 1.965
t0 = d[0, :G, 0][d[0, :G, 0] > 0].min()
for k in range(K):
    st = d[k, :G, 0] - t0
    ns = lambda slot: d[k, :G, slot] / ghz  # noqa: E731  (cycles since the CTA's start -> ns)
    row = {"k": k, "start_min": int(st.min()), "start_max": int(st.max()),
           "depwait_med": int(np.median(st + ns(1))), "h_med": int(np.median(st + ns(2))),
           "rows_done_med": int(np.median(st + ns(3))), "record_med": int(np.median(st + ns(4))),
           "record_max": int((st + ns(4)).max()),
           "fin_L": int(d[k, 0, 125] - t0), "fin_done": int(d[k, 0, 126] - t0)}
    print(json.dumps(row))
k = 4
st = d[k, :G, 0] - t0
w = d[k, :G, 8:8 + 90].reshape(G, 15, 3, 2) / ghz + st[:, None, None, None]
for r in range(2):
    for j, nm in enumerate(("arrive", "computed")):
        col = w[:, :, r, j].reshape(-1)
        col = col[col > st.min()]
        if col.size:
            print(f"launch {k} row{r}_{nm}", [int(x) for x in np.percentile(col, [0, 50, 90, 100])])
print("phase medians (ns from CTA start):", {n: int(np.median(d[k, :G, sl] / ghz)) for n, sl in
                                              (("depwait", 1), ("h", 2), ("rows_done", 3),
                                               ("record", 4))})
