"""GPU parity of the stable-hidden batch-1 decode (SVT_ROWS_HIDDEN_STABLE,
svt_decode_small.cu rows_hs_kernel): the same certified rows path with h read
and every row consumed before the programmatic-dependency wait, consecutive
launches overlapping on each SM. Ids (and exact winning logits) must equal
the reference greedy_step (head.cpp:203-217) exactly as the other paths do,
including back-to-back launches from several jobs in one CUDA graph, the
reference's NaN / tie / signed-zero rules, and a workspace shared with the
epoch-tagged kernel (rows_fast)."""
import numpy as np
import pytest
import torch

from oracle.oracle import c_oracle

from test_gpu_parity import _build_workload, _rows_decoder, bits

pytestmark = pytest.mark.gpu

orc = c_oracle()


@pytest.fixture(scope="module")
def th():
    from paper_2508_15229_b200 import tailored_head

    torch.cuda.set_device(0)
    return tailored_head


def _greedy_hs(dec, h, want_max=False):
    """One call with SVT_ROWS_HIDDEN_STABLE (and the weights marked stable:
    the decoder's rows were gathered by an earlier, completed kernel)."""
    dec._stable = 1
    hd = torch.from_numpy(np.ascontiguousarray(h, np.float32)).cuda()
    torch.cuda.synchronize()
    out = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    mx = torch.full((1,), -7.0, dtype=torch.float32, device="cuda") if want_max else None
    dec.greedy(hd, out, mx, hidden_stable=True)
    got = int(out.item()) & 0xFFFFFFFF
    return (got, float(mx.item())) if want_max else got


def test_hs_cfg1_64_steps_three_jobs_graph(th):
    """cfg1 at full shape (V=128256, d=2048, f32, 512-token prompts + 2048
    static), all 64 steps of three jobs token-interleaved in one CUDA graph
    with SVT_ROWS_HIDDEN_STABLE (launch t+1 overlaps launch t), replayed
    three times, then one job alone: ids equal the reference."""
    V, d, steps, R = 128256, 2048, 64, 3
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, R, 512, 2048, steps)
    W = head.to_host()
    plans = [orc.select(prompts[j], words, V, V).active_ids for j in range(R)]
    subs = [orc.gather(W, p) for p in plans]
    want = np.array([[orc.greedy_step(subs[j], hid[t][j], plans[j])[0] for j in range(R)]
                     for t in range(steps)], np.uint32)
    decs = [_rows_decoder(th, head, plans[j]) for j in range(R)]
    hd = torch.from_numpy(np.ascontiguousarray(hid, np.float32)).cuda()
    out = torch.full((steps, R), -1, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    for dcd in decs:
        dcd.stream = st

    def run(jobs):
        for t in range(steps):
            for j in jobs:
                decs[j].greedy(hd[t, j], out[t, j], hidden_stable=True)

    for jobs in (list(range(R)), [1]):
        with torch.cuda.stream(st):
            run(jobs)  # the first call per decoder takes the epoch-tagged kernel
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32)[:, jobs], want[:, jobs])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run(jobs)
        for _ in range(3):
            out.fill_(-1)
            with torch.cuda.stream(st):
                g.replay()
            torch.cuda.synchronize()
            got = out.cpu().numpy().view(np.uint32)
            assert np.array_equal(got[:, jobs], want[:, jobs]), jobs
    for dcd in decs:
        dcd.stream = None
    # exact logits through the stable-hidden path (every step recomputes the winner)
    for t in range(0, steps, 7):
        gid, gmax = _greedy_hs(decs[0], hid[t][0], want_max=True)
        w, wm = orc.greedy_step(subs[0], hid[t][0], plans[0])
        assert gid == w and bits([gmax])[0] == bits([wm])[0], t


def test_hs_alternating_with_epoch_kernel(th):
    """One workspace used by both record protocols in turn (stable-hidden
    records are cleared, epoch-tagged records are not): every id is right."""
    V, d = 128256, 2048
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, 1, 512, 2048, 10)
    W = head.to_host()
    plan = orc.select(prompts[0], words, V, V).active_ids
    sub = orc.gather(W, plan)
    dec = _rows_decoder(th, head, plan)
    hd = torch.from_numpy(np.ascontiguousarray(hid, np.float32)).cuda()
    out = torch.full((10,), -1, dtype=torch.int32, device="cuda")
    for rep in range(3):
        for t in range(10):
            dec.greedy(hd[t, 0], out[t], hidden_stable=bool((t + rep) % 2))
        torch.cuda.synchronize()
        want = [orc.greedy_step(sub, hid[t][0], plan)[0] for t in range(10)]
        assert out.cpu().numpy().view(np.uint32).tolist() == want, rep


@pytest.mark.parametrize("V,d,storage,n", [(151936, 896, "bf16", 2600), (256000, 2304, "bf16", 4000),
                                           (5000, 256, "f16", 700), (3000, 64, "f32", 300),
                                           (128256, 2048, "f32", 4700), (40000, 1024, "bf16", 4000),
                                           (50000, 4096, "bf16", 3000)])
def test_hs_shapes(th, V, d, storage, n):
    """Row widths of 1, 2 and 4 chunks per thread, ring refills (more rows
    per group than slots), f32 / f16 / bf16 storage; shapes the ring kernel
    cannot take fall back to the other kernels with the same ids."""
    st = {"f32": th.SVT_F32, "f16": th.SVT_F16, "bf16": th.SVT_BF16}[storage]
    head = th.HeadMatrix.random(V, d, 0x5EED + d, storage=st,
                                dtype_bytes=2 if storage == "f16" else 4)
    W = head.to_host()
    rng = np.random.default_rng(d + n)
    ids = np.sort(rng.choice(V, n, replace=False)).astype(np.uint32)
    dec = _rows_decoder(th, head, ids, materialize=(n % 2 == 0))
    sub = W[ids]
    for t in range(4):
        h = rng.uniform(-1, 1, d).astype(np.float32)
        assert _greedy_hs(dec, h) == orc.greedy_step(sub, h, ids)[0], (V, d, t)


def test_hs_special_values(th):
    """The reference scan rules through the stable-hidden path: zero hidden
    (all rows tie -> row 0), NaN hidden (-> plan row 0), NaN at row 0 and at
    a later row, duplicated maxima (-> lowest row), +-inf, signed zeros,
    near-ties overflowing the per-CTA candidate list."""
    rng = np.random.default_rng(78)
    n, d = 1200, 512
    W = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    W[917] = W[233] = W[1001] = np.abs(W[5]) + 0.5
    ar = np.arange(n, dtype=np.uint32)
    head = th.HeadMatrix.from_host(W)
    dec = _rows_decoder(th, head, ar, remap=False)
    pos = np.ones(d, np.float32)
    assert _greedy_hs(dec, pos) == orc.greedy_step(W, pos, ar)[0] == 233
    zero = np.zeros(d, np.float32)
    assert _greedy_hs(dec, zero) == 0
    nanh = zero.copy()
    nanh[3] = np.nan
    assert _greedy_hs(dec, nanh) == 0
    for r in (0, 7):
        Wn = W.copy()
        Wn[r, 9] = np.nan
        dn = _rows_decoder(th, th.HeadMatrix.from_host(Wn), ar)
        ref = orc.greedy_step(Wn, pos, ar)[0]
        assert _greedy_hs(dn, pos) == ref
        if r == 0:
            assert ref == 0
    Wi = W.copy()
    Wi[40, 0] = Wi[41, 0] = np.inf
    di = _rows_decoder(th, th.HeadMatrix.from_host(Wi), ar)
    assert _greedy_hs(di, pos) == orc.greedy_step(Wi, pos, ar)[0] == 40
    Wz = np.zeros((n, d), np.float32)
    Wz[::2, 0] = -1.0
    dz = _rows_decoder(th, th.HeadMatrix.from_host(Wz), ar)
    assert _greedy_hs(dz, np.zeros(d, np.float32)) == 0
    base = rng.uniform(-1, 1, d).astype(np.float32)
    Wt = np.stack([base[rng.permutation(d)] for _ in range(n)])
    dt = _rows_decoder(th, th.HeadMatrix.from_host(Wt), ar)
    want, wmax = orc.greedy_step(Wt, pos, ar)
    got, gmax = _greedy_hs(dt, pos, want_max=True)
    assert got == want and bits([gmax])[0] == bits([wmax])[0]
    assert _greedy_hs(dt, pos) == want


def test_hs_two_streams_mixed_eager_and_graphs(th):
    """Four cfg1-shaped decoders on two streams (two per stream, token-
    interleaved), resident-hidden calls: stream A replays a CUDA graph while
    stream B runs eagerly, then the roles swap, with no host sync in
    between; every id equals the reference (record slots per workspace,
    grids of both streams competing for the SMs)."""
    V, d, steps, R = 128256, 2048, 24, 4
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, R, 512, 2048, steps)
    W = head.to_host()
    plans = [orc.select(prompts[j], words, V, V).active_ids for j in range(R)]
    want = np.array([[orc.greedy_step(W[plans[j]], hid[t][j], plans[j])[0] for j in range(R)]
                     for t in range(steps)], np.uint32)
    decs = [_rows_decoder(th, head, plans[j]) for j in range(R)]
    hd = torch.from_numpy(np.ascontiguousarray(hid, np.float32)).cuda()
    out = torch.full((steps, R), -1, dtype=torch.int32, device="cuda")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    groups = {0: ([0, 1], sa), 1: ([2, 3], sb)}
    for jobs, st in groups.values():
        for j in jobs:
            decs[j].stream = st

    def run(jobs):
        for t in range(steps):
            for j in jobs:
                decs[j].greedy(hd[t, j], out[t, j], hidden_stable=True)

    for jobs, st in groups.values():  # first calls (epoch kernel), then capture
        with torch.cuda.stream(st):
            run(jobs)
    torch.cuda.synchronize()
    graphs = {}
    for k, (jobs, st) in groups.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run(jobs)
        graphs[k] = g
    for rnd in range(3):
        out.fill_(-1)
        torch.cuda.synchronize()
        ka, kb = (0, 1) if rnd % 2 == 0 else (1, 0)
        with torch.cuda.stream(groups[ka][1]):
            graphs[ka].replay()
        with torch.cuda.stream(groups[kb][1]):
            run(groups[kb][0])
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want), rnd
    for dcd in decs:
        dcd.stream = None
