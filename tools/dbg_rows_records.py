"""Dump svt_greedy_certified_rows per-CTA records for one identity-plan token."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

V, d, n = 128256, 2048, 16384
head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
hid = torch.empty(4 * d, dtype=torch.float32, device="cuda")
th._lib.call("svt_head_random", hid.data_ptr(), th.SVT_F32, th.SVT_BF16, 0, 4 * d, synth.SEED_H, None)
hid = hid.view(4, d)
out = torch.empty(4, dtype=torch.int32, device="cuda")
for ids_kind in ("identity", "random"):
    if ids_kind == "identity":
        ids_h = np.arange(n, dtype=np.uint32)
    else:
        ids_h = np.sort(np.random.default_rng(1).choice(V, n, replace=False)).astype(np.uint32)
    ids = torch.from_numpy(ids_h.view(np.int32)).cuda()
    dec = th.RowDecoder(head, ids, n)
    for t in range(4):
        dec.greedy(hid[t], out[t:t + 1])
        torch.cuda.synchronize()
        rec = dec.ws[256:256 + 148 * 32].view(torch.int32).view(148, 8).cpu().numpy()
        L = rec[:, 0].view(np.float32)
        cnt = rec[:, 1].view(np.uint32)
        hi0 = rec[:, 3].view(np.float32)
        Lg = L.max()
        print(ids_kind, t, "stats", dec.stats(), "cnt hist", np.unique(cnt, return_counts=True),
              "L", Lg, "cands(hi0>=L)", int((hi0 >= Lg).sum()), "top L gap",
              float(np.sort(L)[-1] - np.sort(L)[-2]))
