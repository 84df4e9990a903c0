"""Debug: the test_hs_cfg1_64_steps_three_jobs_graph sequence with per-phase
mismatch counts and the finalizer's timeout counter (ctrl[6])."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_parity import _build_workload, _rows_decoder
from oracle.oracle import c_oracle
from paper_2508_15229_b200 import tailored_head as th
orc = c_oracle()
torch.cuda.set_device(0)
V, d, steps, R = 128256, 2048, 64, 3
head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, R, 512, 2048, steps)
W = head.to_host()
plans = [orc.select(prompts[j], words, V, V).active_ids for j in range(R)]
want = np.array([[orc.greedy_step(W[plans[j]], hid[t][j], plans[j])[0] for j in range(R)] for t in range(steps)], np.uint32)
decs = [_rows_decoder(th, head, plans[j]) for j in range(R)]
hd = torch.from_numpy(np.ascontiguousarray(hid, np.float32)).cuda()
out = torch.full((steps, R), -1, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
for dcd in decs: dcd.stream = st
def run(jobs):
    for t in range(steps):
        for j in jobs:
            decs[j].greedy(hd[t, j], out[t, j], hidden_stable=True)
def report(tag, jobs, t0):
    got = out.cpu().numpy().view(np.uint32)
    bad = got[:, jobs] != want[:, jobs]
    print(tag, jobs, round(time.time() - t0, 3), "bad", int(bad.sum()), np.argwhere(bad)[:6].tolist(),
          "ctrl1", decs[1].ws[:64].view(torch.int32)[4:14].tolist())
for jobs in (list(range(R)), [1]):
    out.fill_(-1); t0 = time.time()
    with torch.cuda.stream(st): run(jobs)
    torch.cuda.synchronize(); report("eager", jobs, t0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st): run(jobs)
    for _ in range(3):
        out.fill_(-1); t0 = time.time()
        with torch.cuda.stream(st): g.replay()
        torch.cuda.synchronize(); report("graph", jobs, t0)
