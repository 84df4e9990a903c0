"""svt_session_decode_host over the cfg1 sessions (8 x batch 1, 64 steps)
after a prepare_many: host time, device time of the call (CUDA events on the
sessions' stream around it), and a bare H2D of the same hidden states, with
the decode_host graph on and off (measurement)."""
import os, sys, time, statistics, numpy as np, torch
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
dev = torch.empty_like(hid_h, device="cuda")
for mode in ["1", "0", "1", "0"]:
    os.environ["SVT_DECODE_GRAPH"] = mode
    host, gpu, h2d = [], [], []
    for it in range(12):
        session.prepare_many(sess, jobs.words_h, V, jobs.prompts_h, offs)
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        t0 = time.perf_counter()
        session.decode_host(sess, hid_h, 64, ids_h)
        t1 = time.perf_counter()
        b.record(st)
        b.synchronize()
        with torch.cuda.stream(st):
            c, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c.record(st)
            dev.copy_(hid_h, non_blocking=True)
            e.record(st)
        e.synchronize()
        if it >= 3:
            host.append((t1 - t0) * 1e6)
            gpu.append(a.elapsed_time(b) * 1e3)
            h2d.append(c.elapsed_time(e) * 1e3)
    print(f"graph={mode} host_us {statistics.median(host):.1f} gpu_us {statistics.median(gpu):.1f} "
          f"h2d_us {statistics.median(h2d):.1f} ({hid_h.numel()*4/1e6:.2f} MB)", flush=True)
