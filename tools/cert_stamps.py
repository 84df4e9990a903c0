"""Per-phase timeline of the certified static half's GEMM (measurement:
SVT_CERT_SKIP=18 -> stamps on, select skipped): medians over CTAs of
%globaltimer stamps relative to each CTA's start, ns."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

os.environ["SVT_CERT_SKIP"] = os.environ.get("SVT_CERT_SKIP", "16")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG2, 64, 4, 0, torch, th, synth)
job.run("split")
torch.cuda.synchronize()
# warm: back-to-back steps in a CUDA graph (stamps of the last one kept)
st = torch.cuda.Stream()
job.sdec.stream = st
with torch.cuda.stream(st):
    job.sdec.greedy(job.hidden[0], job.out[0])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for t in range(16):
        job.sdec.greedy(job.hidden[t % job.steps], job.out[0])
with torch.cuda.stream(st):
    for _ in range(4):
        g.replay()
torch.cuda.synchronize()
buf = np.zeros(512 * 8 + 256 * 8, np.uint64)
th._lib.lib.svt_cert_stamps_read.argtypes = [ctypes.c_void_p]
th._lib.lib.svt_cert_stamps_read(buf.ctypes.data)
allst = buf.astype(np.int64)
st = allst[:512 * 8].reshape(512, 8)[:64]
sel = allst[512 * 8:].reshape(256, 8)[:64]
t0 = st[:, 0]
names = ["start", "data_ready", "a_copies_issued", "h_split_written", "mmas_issued", "mma_done", "stored", "exit"]
res = {n: int(np.median(st[:, k] - t0)) for k, n in enumerate(names)}
res["start_spread"] = int(t0.max() - t0.min())
res["total_first_to_last"] = int(st[:, 7].max() - t0.min())
g0 = st[:, 0].min()
res["sel"] = {n: int(np.median(sel[:, k] - g0)) for k, n in enumerate(
    ["start", "after_wait", "hn_and_loads", "L", "candidates", "chains_done"])}
res["sel_max_chains_done"] = int((sel[:, 5] - g0).max())
res["gemm_last_exit"] = int((st[:, 7] - g0).max())
print(json.dumps(res))
