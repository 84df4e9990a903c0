"""Per-role cycle counters (SVT_PREFILL_MODE=8) of the prefill GEMM for a
shared-subset decode batch (S=1, P=256) at |S| = 1024: where a small GEMM's
time goes (producer waits, MMA waits on full stages / free accumulators,
epilogue waits / work)."""
import json
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
res = {}
for small in ("1", "0"):
    os.environ["SVT_PREFILL_SMALL_N"] = small
    k = 1024
    ids = np.sort(np.random.default_rng(1).choice(V, k, replace=False)).astype(np.uint32)
    sc = prefill.PrefillScorer(head, torch.from_numpy(ids.view(np.int32)).cuda(),
                               np.array([0, k], np.int64), P)
    os.environ["SVT_PREFILL_MODE"] = "8"
    for _ in range(3):
        sc.score(hid, out)
    torch.cuda.synchronize()
    c = sc.profile_counters()
    os.environ["SVT_PREFILL_MODE"] = "24"  # GEMM alone, timed
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sc.score(hid, out)
    a.record()
    for _ in range(20):
        sc.score(hid, out)
    b.record()
    torch.cuda.synchronize()
    os.environ.pop("SVT_PREFILL_MODE")
    res["small_n" if small == "1" else "bn256"] = {
        "gemm_us": a.elapsed_time(b) / 20 * 1e3,
        "producer_wait_cyc": c[0], "mma_wait_acc_cyc": c[1], "mma_wait_full_cyc": c[2],
        "mma_total_cyc": c[3], "epi_wait_cyc": c[4], "epi_work_cyc": c[5], "tiles": c[6]}
print(json.dumps(res, indent=1))
