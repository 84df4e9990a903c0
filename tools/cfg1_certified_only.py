import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2508_15229_b200 import synth
from paper_2508_15229_b200 import tailored_head as th
job = bench.Job(bench.CFG1, 1, 8, 0, torch, th, synth)
for t in range(8):
    job.tb.greedy_certified(job.hidden[t], job.out[t])
for t in range(8):
    job.tb.greedy(job.hidden[t], job.out[t])
torch.cuda.synchronize()
