"""cfg2 decode step, L2 flushed (256 MB read) before every step and the flush
subtracted (bench._graph_ms): split vs interleaved. The split step's working
set (61.6 MB) fits the 126 MB L2, so this checks it is not flattered by
L2 residency across decode steps."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG2, 64, 4, 0, torch, th, synth)
job.run("split")
job.tb.gather(job.head)
torch.cuda.synchronize()
flush = torch.ones((256 << 20) // 4 // 1024, 1024, dtype=torch.float32, device="cuda")
sink = torch.empty(1024, dtype=torch.float32, device="cuda")
res = {}


def split_fn(s):
    job.sdec.stream = s
    job.sdec.greedy(job.hidden[0], job.out[0])


def inter_fn(s):
    job.tb.stream = s
    job.tb.greedy(job.hidden[0], job.out[1])


res["split_cold_us"] = bench._graph_ms(torch, split_fn, 8, flush, sink) * 1e3
res["interleaved_cold_us"] = bench._graph_ms(torch, inter_fn, 8, flush, sink) * 1e3
res["ids_equal"] = bool(torch.equal(job.out[0], job.out[1]))
print(json.dumps(res, indent=1))
