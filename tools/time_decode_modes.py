"""Decode-step latency per mode (exact interleaved / certified / fused) for
cfg1 (batch 1, f32) and cfg2 (batch 64, bf16): CUDA events over back-to-back
launches, and a CUDA graph of 64 steps (launch overhead removed)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402


def run_mode(job, mode, t):
    if mode == "certified":
        job.tb.greedy_certified(job.hidden[t], job.out[t])
    else:
        job.tb.greedy(job.hidden[t], job.out[t], fused=(mode == "fused"))


def measure(job, mode, graph):
    steps = job.steps
    s = torch.cuda.Stream()
    job.tb.stream = s
    with torch.cuda.stream(s):
        for t in range(steps):
            run_mode(job, mode, t)
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for t in range(steps):
                run_mode(job, mode, t)
        def fn():
            with torch.cuda.stream(s):
                g.replay()
    else:
        def fn():
            with torch.cuda.stream(s):
                for t in range(steps):
                    run_mode(job, mode, t)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    job.tb.stream = None
    return a.elapsed_time(b) / (reps * steps) * 1e3


for name, cfg, B in (("cfg1", bench.CFG1, 1), ("cfg2", bench.CFG2, 64)):
    job = bench.Job(cfg, B, 64, 0, torch, th, synth)
    nbytes = job.decode_bytes()
    for mode in ("interleaved", "certified", "fused"):
        for graph in (False, True):
            us = measure(job, mode, graph)
            print(json.dumps({"cfg": name, "mode": mode, "graph": graph, "us_per_step": round(us, 2),
                              "gbs": round(nbytes / us / 1e3, 1),
                              "tokens_per_s": round(B * 1e6 / us)}), flush=True)
    if name == "cfg1":
        print(json.dumps({"certified_stats": job.tb.certified_stats()}))
    del job
    torch.cuda.empty_cache()
