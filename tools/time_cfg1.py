"""cfg1 (Llama-3.2-1B shape, batch 1, f32) decode: certified rows path vs the
exact-order interleaved path, warm (graph replay) and L2-cold per token."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402

job = bench.Job(bench.CFG1, 1, 64, 0, torch, th, synth)
out = {}
ref = None
for mode in ("rows", "interleaved"):
    ms, dec_ms, clk = bench.time_job(job, mode, 10, 3, torch, None, 1)
    avg = sum(dec_ms) / len(dec_ms)
    ids = job.out.cpu().numpy().copy()
    out[mode] = {"step_ms": ms / 10, "us_per_token": avg * 1e3,
                 "gbs": job.decode_bytes() / (avg / 1e3) / 1e9, "clocks": clk}
    if ref is None:
        ref = ids
    else:
        out[mode]["ids_match"] = bool((ids == ref).all())
out["rows_cold"] = bench.cfg1_cold(job, torch)
out["stats"] = job.rdec.stats()
print(json.dumps(out, indent=1))
