"""Small cfg3-shaped prefill run for ncu captures (SEQS sequences, pair on/off)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_15229_b200 import prefill, synth, _lib  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

S = int(os.environ.get("SEQS", 8))
prefill.PrefillScorer.set_tuning(int(os.environ.get("PAIR", 1)), int(os.environ.get("NSPLIT", 2)))
P, d, V = 2048, 3072, 128256
head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
rng = np.random.default_rng(0)
plans = [np.sort(rng.choice(V, 4050, replace=False)).astype(np.uint32) for _ in range(S)]
off = np.zeros(S + 1, np.int64)
off[1:] = np.cumsum([len(p) for p in plans])
ids = torch.from_numpy(np.concatenate(plans).view(np.int32)).cuda()
sc = prefill.PrefillScorer(head, ids, off, P)
hid = torch.empty(S * P * d, dtype=torch.bfloat16, device="cuda")
th._lib.call("svt_head_random", hid.data_ptr(), th.SVT_BF16, th.SVT_BF16, 0, S * P * d,
             synth.SEED_H, None)
out = torch.empty(S * P, dtype=torch.int32, device="cuda")
for _ in range(2):
    sc.score(hid.view(S * P, d), out)
torch.cuda.synchronize()
print("ok", sc.stats())
if int(os.environ.get("SVT_PREFILL_MODE", 0)) & 8:
    d = sc.profile_counters()
    names = ["prod_wait_empty", "mma_wait_acc_empty", "mma_wait_full", "mma_total",
             "epi_wait_full", "epi_work", "epi_tiles"]
    print({n: v for n, v in zip(names, d)})
    tiles = d[6] / 4
    print("per tile (cycles): mma_total/tile", d[3] / (tiles / 2 if sc.tuning()[0] else tiles),
          "epi_work/tile/warp", d[5] / d[6], "epi_wait/tile/warp", d[4] / d[6])
