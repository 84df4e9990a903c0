"""cfg1 per-token time with the sub-head cold in L2 WITHOUT a flush kernel
between tokens: R independent cfg1 jobs (own prompt -> own plan -> own
row-major sub-head, 20.9 MB each) decoded token-interleaved, so consecutive
launches touch different sub-heads and the R x 20.9 MB working set exceeds
the 126 MB L2. R=1 is the warm (L2-resident) figure."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

V, d, STEPS = 128256, 2048, 64
HS = os.environ.get("SVT_HS", "0") == "1"  # SVT_ROWS_HIDDEN_STABLE
head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_F32)
t_ids = synth.static_ids(V, 2048)
words = torch.from_numpy(synth.words_of(t_ids, V).view(np.int64)).cuda()


def make(R):
    jobs = []
    for j in range(R):
        p = synth.prompt_ids(V, 512, j)
        off = np.array([0, len(p)], np.int64)
        tb = th.TailoredBatch.build(words, 2048, V, torch.from_numpy(p.view(np.int32)).cuda(), off)
        n = int(tb.n_active[0].item())
        jobs.append((tb, th.RowDecoder(head, tb.active[:n], n,
                                        materialize=os.environ.get("SVT_FUSED", "0") != "1"), n))
    n = STEPS * R * d
    hid = torch.empty(n, dtype=torch.float32, device="cuda")
    th._lib.call("svt_head_random", hid.data_ptr(), th.SVT_F32, th.SVT_F32, 0, n, synth.SEED_H,
                 None)
    hid = hid.view(STEPS, R, d)
    out = torch.zeros((STEPS, R), dtype=torch.int32, device="cuda")
    return jobs, hid, out


def run(R, reps=10):
    jobs, hid, out = make(R)
    s = torch.cuda.Stream()
    for _, rd, _ in jobs:
        rd.stream = s

    def decode():
        for t in range(STEPS):
            for j, (_, rd, _) in enumerate(jobs):
                rd.greedy(hid[t, j], out[t, j], hidden_stable=HS)

    with torch.cuda.stream(s):
        decode()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        decode()
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / (STEPS * R))
    nbytes = sum(n for _, _, n in jobs) / R * d * 4
    med = float(np.median(ts))
    stats = [rd.stats() for _, rd, _ in jobs]
    return {"R": R, "hs": HS, "nb": os.environ.get("SVT_ROWS_HS_NB"), "us_per_token": med, "min": min(ts), "gbs": nbytes / med / 1e3,
            "frac": nbytes / med / 1e3 / 6551.7, "rows": nbytes / d / 4,
            "recomputed": sum(s[1] for s in stats), "certified": sum(s[0] for s in stats)}


if __name__ == "__main__":
    res = [run(R) for R in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16").split(",")]]
    print(json.dumps(res, indent=1))
