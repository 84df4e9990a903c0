"""Host time of svt_session_decode_host over the cfg1 sessions (8 x batch 1,
64 steps), after a prepare_many, printed per call (measurement)."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2508_15229_b200 import session, synth
from paper_2508_15229_b200 import tailored_head as th
jobs = bench.Cfg1Jobs(8, 64, 0, torch, th, synth)
V = bench.CFG1["V"]
st = torch.cuda.Stream()
sess = [session.Session(jobs.head, max_batch=1, stream=st) for _ in range(8)]
offs = [np.array([0, len(p)], np.int64) for p in jobs.prompts_h]
hid_h = jobs.hidden.cpu().pin_memory()
ids_h = torch.zeros((64, 8), dtype=torch.int32).pin_memory()
for it in range(6):
    session.prepare_many(sess, jobs.words_h, V, jobs.prompts_h, offs)
    t0 = time.perf_counter()
    session.decode_host(sess, hid_h, 64, ids_h)
    print("decode_host us", (time.perf_counter() - t0) * 1e6, file=sys.stderr)
