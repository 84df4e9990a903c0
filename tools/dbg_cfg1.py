import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2508_15229_b200 import synth, tailored_head as th, session as session_mod
from oracle import oracle as O
R, steps = int(sys.argv[1]), int(sys.argv[2])
jobs = bench.Cfg1Jobs(R, steps, 0, torch, th, synth)
jobs.prep(); jobs.decode(); torch.cuda.synchronize()
eager = jobs.out.cpu().numpy().copy()
ms, dec_ms, warm, gen, clk = bench.time_cfg1(jobs, 5, 3, torch, None, 1)
graph = jobs.out.cpu().numpy().copy()
v, h2d, d2h, ok, sec = bench.cfg1_e2e(jobs, 2, 1, torch, th, session_mod)
orc = O.c_oracle()
V, d = 128256, 2048
W = orc.head_random(V, d, synth.SEED_W)
hid = synth.head_random(steps * R, d, synth.SEED_H).reshape(steps, R, d)
want = np.zeros((steps, 2), np.int64)
for j in range(2):
    plan = orc.select(jobs.prompts_h[j], jobs.words_h, V, V).active_ids
    sub = orc.gather(W, plan)
    for t in range(steps):
        want[t, j] = orc.greedy_step(sub, hid[t, j], plan)[0]
print("e2e ok", ok)
print("eager==graph", np.array_equal(eager, graph), "eager==oracle", np.array_equal(eager[:, :2], want), "graph==oracle", np.array_equal(graph[:, :2], want))
bad = np.argwhere(graph[:, :2] != want)
print("mismatch positions", bad[:10].tolist(), [(graph[t, j], want[t, j], eager[t, j]) for t, j in bad[:10]])
