"""Split the per-token e2e cost of the host-buffer session at cfg2: the full
host call (H2D + step + D2H + sync), the device step alone with a sync per
call, and a bare 229 KB pinned H2D + sync."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_15229_b200 import session, synth  # noqa: E402
from paper_2508_15229_b200 import tailored_head as th  # noqa: E402
from paper_2508_15229_b200 import _lib  # noqa: E402

job = bench.Job(bench.CFG2, 64, 64, 0, torch, th, synth)
d = job.cfg["d"]
hid_h = job.hidden[:, :, :d].cpu().pin_memory()
ids_h = torch.empty((64, 64), dtype=torch.int32).pin_memory()
hid_d = job.hidden[:, :, :d].contiguous()
ids_d = torch.empty(64, dtype=torch.int32, device="cuda")
res = {}
N = 400


def wall(fn):
    for _ in range(20):
        fn(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        fn(k)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / N * 1e6


with session.Session(job.head, max_batch=64) as s:
    s.prepare(job.words_h, job.cfg["V"], job.flat_h, job.off_h)
    res["host_call_us"] = wall(lambda k: s.greedy(hid_h[k % 64], ids_h[k % 64]))

    def dev(k):
        _lib.call("svt_session_greedy_device", s.h, hid_d[k % 64].data_ptr(), d,
                  ids_d.data_ptr(), None)
        torch.cuda.synchronize()
    res["device_step_sync_us"] = wall(dev)

    def dev_nosync(k):
        _lib.call("svt_session_greedy_device", s.h, hid_d[k % 64].data_ptr(), d,
                  ids_d.data_ptr(), None)
    res["device_step_back_to_back_us"] = wall(dev_nosync)

buf = torch.empty_like(hid_d[0])


def h2d(k):
    buf.copy_(hid_h[k % 64], non_blocking=True)
    torch.cuda.synchronize()
res["h2d_229KB_sync_us"] = wall(h2d)


def d2h(k):
    ids_h[0].copy_(ids_d, non_blocking=True)
    torch.cuda.synchronize()
res["d2h_256B_sync_us"] = wall(d2h)
res["empty_sync_us"] = wall(lambda k: torch.cuda.synchronize())
print(json.dumps(res))
