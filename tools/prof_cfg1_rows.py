"""Launch the cfg1 certified-rows decode 32 times (for ncu captures)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG1, 1, 64, 0, torch, th, synth)
torch.cuda.synchronize()
for k in range(32):
    job.rdec.greedy(job.hidden[k][0], job.out[k])
torch.cuda.synchronize()
print("stats", job.rdec.stats())
