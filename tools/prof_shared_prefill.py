"""Shared-subset decode batch scored on tcgen05 (S=1 sequence, P=256
positions) at |S| = 1024 and 128256: for ncu launch lists."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_15229_b200 import prefill, synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

V, d, P = 128256, 2048, 256
head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
hid = torch.empty(P * d, dtype=torch.bfloat16, device="cuda")
th._lib.call("svt_head_random", hid.data_ptr(), th.SVT_BF16, th.SVT_BF16, 0, P * d, synth.SEED_H,
             None)
hid = hid.view(P, d)
out = torch.empty(P, dtype=torch.int32, device="cuda")
for k in (1024, 128256):
    ids = np.arange(V, dtype=np.uint32) if k == V else np.sort(
        np.random.default_rng(1).choice(V, k, replace=False)).astype(np.uint32)
    sc = prefill.PrefillScorer(head, torch.from_numpy(ids.view(np.int32)).cuda(),
                               np.array([0, k], np.int64), P)
    for _ in range(3):
        sc.score(hid, out)
    torch.cuda.synchronize()
    print(k, sc.stats())
