"""cfg2 split decode, dynamic half alone: the exact-order GEMV (SVT_CERT_SKIP=3
static skipped, whole split step) vs svt_greedy_certified over the same
D_b \\ T sub-heads (split-K FFMA pass at HBM speed + per-request certify /
exact recompute), CUDA-graph replay, warm. Measurement for DESIGN 9."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG2, 64, 64, 0, torch, th, synth)
job.run("split")
torch.cuda.synchronize()
dec = job.sdec
h = job.head
cws = torch.zeros(max(1, th._lib.lib.svt_certified_workspace_bytes(64, dec.max_groups)),
                  dtype=torch.uint8, device="cuda")
out = torch.zeros((64, 64), dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()


def dyn(t):
    th.call("svt_greedy_certified", dec.sub.data_ptr(), h.storage, h.dim(), dec.gb.data_ptr(),
            dec.gm.data_ptr(), dec.dyn_ids.data_ptr(), 64, dec.max_groups,
            job.hidden[t].data_ptr(), job.hidden[t].stride(0), out[t].data_ptr(), None,
            cws.data_ptr(), s.cuda_stream)


def steps():
    for t in range(64):
        dyn(t)


with torch.cuda.stream(s):
    steps()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    steps()
with torch.cuda.stream(s):
    for _ in range(3):
        g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    a.record(s)
    for _ in range(5):
        g.replay()
    b.record(s)
torch.cuda.synchronize()
st = cws[-256:].view(torch.int32)[:2].cpu().tolist()
print(json.dumps({"dyn_certified_us": a.elapsed_time(b) / 5 / 64 * 1e3, "stats": st}))
