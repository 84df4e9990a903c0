"""cfg3 timing: 256 sequences x 2048 positions, d=3072 (Llama-3.2-3B shape),
per-sequence plans T(2048) ∪ prompt(2048) over V=128256, bf16.
Times the gather, the tensor-core scoring (norms + tcgen05 GEMM + certify)
and reports TFLOP/s on the algorithmic 2*P*d*|S| flops."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_15229_b200 import prefill, synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

S = int(os.environ.get("SEQS", 256))
prefill.PrefillScorer.set_tuning(int(os.environ.get("PAIR", 1)), int(os.environ.get("NSPLIT", 2)))
P, d, V = 2048, 3072, 128256
head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
t_ids = synth.static_ids(V, 2048)
words = synth.words_of(t_ids, V)
prompts = [synth.prompt_ids(V, 2048, r) for r in range(S)]
off = np.zeros(S + 1, np.int64)
off[1:] = np.cumsum([len(p) for p in prompts])
tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 2048, V,
                            torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(), off)
plans_n = tb.n_active.cpu().numpy()
ids = torch.cat([tb.active[int(tb.act_off_h[b]): int(tb.act_off_h[b]) + int(plans_n[b])]
                 for b in range(S)])
poff = np.zeros(S + 1, np.int64)
poff[1:] = np.cumsum(plans_n)
torch.cuda.synchronize()
t0 = time.perf_counter()
sc = prefill.PrefillScorer(head, ids, poff, P)
torch.cuda.synchronize()
gather_s = time.perf_counter() - t0
hid = torch.empty(S * P * d, dtype=torch.bfloat16, device="cuda")
th._lib.call("svt_head_random", hid.data_ptr(), th.SVT_BF16, th.SVT_BF16, 0, S * P * d,
             synth.SEED_H, None)
hid = hid.view(S * P, d)
out = torch.empty(S * P, dtype=torch.int32, device="cuda")
for _ in range(2):
    sc.score(hid, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(os.environ.get("REPS", 10))
a.record()
for _ in range(reps):
    sc.score(hid, out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps


def _allpath_sample(sc):
    v, _ = sc.top8()
    v = v.float().sort(dim=1, descending=True).values
    gap = (v[:, 0] - v[:, 7])
    return {"min_gap_top1_top8": float(gap.min()), "n_gap_lt_2": int((gap < 2).sum())}


flops = 2.0 * P * d * float(plans_n.sum())
print(json.dumps({"seqs": S, "mean_plan_rows": float(plans_n.mean()), "score_ms": ms,
                  "tflops": flops / ms / 1e9, "gather_s_wall": gather_s,
                  "stats": list(sc.stats()), "tuning": sc.tuning(), "top8_sample": _allpath_sample(sc), "tokens_per_s": S * P / (ms / 1e3)}))
