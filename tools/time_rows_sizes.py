"""svt_greedy_certified_rows over identity plans of growing size (bf16 and
f32, d=2048): warm graph time per token and the certification counters."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

V, d = 128256, 2048
res = []
for st in (th.SVT_BF16, th.SVT_F32):
    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=st)
    hid = torch.empty(16 * d, dtype=torch.float32, device="cuda")
    th._lib.call("svt_head_random", hid.data_ptr(), th.SVT_F32, st, 0, 16 * d, synth.SEED_H, None)
    hid = hid.view(16, d)
    out = torch.empty(16, dtype=torch.int32, device="cuda")
    for n in (16384, 65536, 100000, 120000, 128256):
        ids = torch.arange(n, dtype=torch.int32, device="cuda")
        dec = th.RowDecoder(head, ids, n)
        s = torch.cuda.Stream()
        dec.stream = s
        with torch.cuda.stream(s):
            dec.greedy(hid[0], out[0:1])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for k in range(16):
                dec.greedy(hid[k], out[k:k + 1])
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 80 * 1e3
        res.append({"dtype": st, "n": n, "us": us, "stats": dec.stats(),
                    "gbs": n * d * (4 if st == th.SVT_F32 else 2) / us / 1e3})
        print(json.dumps(res[-1]), flush=True)
        del dec, g
        torch.cuda.empty_cache()
