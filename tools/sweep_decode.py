"""Sweep the exact-order GEMV launch shape (warps per CTA x ring stages) on
the cfg2 / cfg1 decode step; prints one line per point (device time via CUDA
events, average over repeated launches)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import _lib, synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402


def time_decode(job, fused, reps=30):
    for _ in range(3):
        job.tb.greedy(job.hidden[0], job.out[0], fused=fused)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for r in range(reps):
        job.tb.greedy(job.hidden[r % job.steps], job.out[r % job.steps], fused=fused)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = bench.CFG2 if which == "cfg2" else bench.CFG1
    B = 64 if which == "cfg2" else 1
    job = bench.Job(cfg, B, 8, 0, torch, th, synth)
    nbytes = job.decode_bytes()
    pts = [(0, 0)] + [(w, s) for w in (1, 2, 4, 6, 8) for s in (2, 3, 4, 6, 8, 12, 24)]
    for fused in (False, True):
        for w, s in pts:
            if w and w * s * 9216 > 224 * 1024:
                continue
            _lib.lib.svt_set_tuning(w, s)
            us = time_decode(job, fused)
            print(json.dumps({"cfg": which, "fused": fused, "warps": w, "stages": s,
                              "us": round(us, 2), "gbs": round(nbytes / us / 1e3, 1)}),
                  flush=True)
    _lib.lib.svt_set_tuning(0, 0)




def debug_counters(which="cfg1"):
    """Producer/consumer cycle breakdown of one decode launch."""
    cfg = bench.CFG2 if which == "cfg2" else bench.CFG1
    B = 64 if which == "cfg2" else 1
    job = bench.Job(cfg, B, 4, 0, torch, th, synth)
    dbg = torch.zeros(148 * 8 * 6, dtype=torch.int64, device="cuda")
    for fused in (False, True):
        for rep in range(2):
            _lib.lib.svt_set_debug(dbg.data_ptr())
            dbg.zero_()
            job.tb.greedy(job.hidden[0], job.out[0], fused=fused)
            torch.cuda.synchronize()
            _lib.lib.svt_set_debug(None)
        d = dbg.view(-1, 6).cpu().numpy()
        d = d[d[:, 2] > 0]
        print(json.dumps({"cfg": which, "fused": fused, "pairs": int(len(d)),
                          "prod_total": float(d[:, 0].mean()), "prod_wait": float(d[:, 1].mean()),
                          "cons_total": float(d[:, 2].mean()), "cons_wait": float(d[:, 3].mean()),
                          "cons_epilogue": float(d[:, 5].mean()),
                          "cons_total_max": float(d[:, 2].max())}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "debug":
        debug_counters(sys.argv[1])
    else:
        main()
