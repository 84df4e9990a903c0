"""Per-CTA globaltimer timeline of svt_greedy_certified_rows at cfg1 (one
launch after warm-up; ns relative to the earliest CTA start)."""
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
dbg = torch.zeros(256 * 128, dtype=torch.int64, device="cuda")
out = {}
for label, flush in (("warm", False), ("cold", True)):
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for k in range(5):
        job.rdec.greedy(job.hidden[k][0], job.out[k])
    if flush:
        fl.fill_(1)
        s = fl.sum()  # read-back: leaves clean lines
    runs = []
    for t in range(12):
        if flush:
            fl.fill_(1)
            s = fl.sum()
        th._lib.lib.svt_rows_set_debug(dbg.data_ptr())
        dbg.zero_()
        st0 = job.rdec.stats()
        job.rdec.greedy(job.hidden[t][0], job.out[t])
        torch.cuda.synchronize()
        th._lib.lib.svt_rows_set_debug(None)
        st1 = job.rdec.stats()
        full = dbg.view(-1, 128)[:148].cpu().numpy().astype("int64")
        d = full[:, :8]
        t0 = d[:, 0].min()
        names = ["start", "dep_wait", "h_staged", "rows_done", "record", "ticket", "tail_done",
                 "tail_L"]
        rel = {"recomputed": int(st1[1] - st0[1])}
        for i, nm in enumerate(names):
            col = d[:, i]
            col = col[col > 0] - t0
            if col.size:
                rel[nm] = int(sorted(col)[col.size // 2]) if col.size > 1 else int(col[0])
        w = full[:, 8:8 + 96].reshape(148, 16, 3, 2)
        for k in range(2):
            for j, nm in enumerate(("arrive", "computed")):
                col = w[:, :, k, j].reshape(-1)
                col = col[col > 0] - t0
                if col.size:
                    rel[f"row{k}_{nm}"] = [int(x) for x in np.percentile(col, [0, 50, 90, 100])]
        runs.append(rel)
    out[label] = runs
print(json.dumps(out, indent=1))
