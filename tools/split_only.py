import os, sys, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2508_15229_b200 import synth
from paper_2508_15229_b200 import tailored_head as th
job = bench.Job(bench.CFG2, 64, 4, 0, torch, th, synth)
job.run("split")
torch.cuda.synchronize()
job.run("split")
torch.cuda.synchronize()
print("ok")
