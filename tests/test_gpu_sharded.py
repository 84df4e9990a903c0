"""Vocab-shard through the C-ABI (svt_sharded_greedy over an NCCL
communicator made by svt_nccl_*): identity and tailored plans, exact maxima,
a 64-step decode captured in one CUDA graph (kernel + ncclAllGather +
combine per step), and tailored-plan slices at G = 2, 4, 8 on the cfg4 head.
One GPU per call here, so the communicator has one rank; the G-way combine
is covered by the single-process slice emulation and the world-size-2 gloo
protocol test (tests/test_sharding_gloo.py). Reference semantics:
head.cpp:203-217 over the whole plan; row-parallel slices per SPEC.md:508."""
import numpy as np
import pytest
import torch

from oracle.oracle import c_oracle, words_from_ids

pytestmark = pytest.mark.gpu

orc = c_oracle()


@pytest.fixture(scope="module")
def th():
    from paper_2508_15229_b200 import tailored_head

    torch.cuda.set_device(0)
    return tailored_head


@pytest.fixture(scope="module")
def comm(th):
    from paper_2508_15229_b200 import sharded

    c = sharded.NcclComm(1, 0)
    yield c
    c.close()


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def test_sharded_cabi_identity_and_tailored(th, comm):
    from paper_2508_15229_b200 import sharded, synth

    V, d = 24000, 512
    rng = np.random.default_rng(8)
    head = th.HeadMatrix.random(V, d, 0x5EED, storage=th.SVT_BF16)
    W = head.to_host()
    words = words_from_ids(rng.choice(V, 900, replace=False), V)
    plan = orc.select(rng.integers(0, V, 400).astype(np.uint32), words, V, V).active_ids
    full = np.arange(V, dtype=np.uint32)
    dec_id = sharded.ShardedDecoder(head, comm)
    dec_tp = sharded.ShardedDecoder(head, comm, plan_ids=plan)
    mx = torch.zeros(1, dtype=torch.float32, device="cuda")
    for t in range(4):
        h = synth.round_bf16(rng.uniform(-1, 1, d).astype(np.float32))
        hd = torch.from_numpy(h).cuda()
        want, wmax = orc.greedy_step(W, h, full)
        assert int(dec_id.step(hd, out_max=mx).item()) & 0xFFFFFFFF == want, t
        assert bits([mx.item()])[0] == bits([wmax])[0]
        want, wmax = orc.greedy_step(W[plan], h, plan)
        assert int(dec_tp.step(hd, out_max=mx).item()) & 0xFFFFFFFF == want, t
        assert bits([mx.item()])[0] == bits([wmax])[0]


def test_sharded_decode_graph_64_steps_cfg1_plan(th, comm):
    """cfg1 head and plan (V=128,256, d=2,048, f32, select over 2,048 static
    + a 512-token prompt) as a one-rank tailored shard: 64 decode steps, each
    certified rows kernel + ncclAllGather + combine, captured in ONE CUDA
    graph and replayed twice; ids equal the reference greedy_step."""
    from paper_2508_15229_b200 import sharded, synth

    V, d, steps = 128256, 2048, 64
    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_F32)
    W = head.to_host()
    words = synth.words_of(synth.static_ids(V, 2048), V)
    plan = orc.select(synth.prompt_ids(V, 512, 0), words, V, V).active_ids
    sub = orc.gather(W, plan)
    hid = synth.head_random(steps, d, synth.SEED_H)
    want = np.array([orc.greedy_step(sub, hid[t], plan)[0] for t in range(steps)], np.uint32)
    dec = sharded.ShardedDecoder(head, comm, plan_ids=plan)
    hd = torch.from_numpy(hid).cuda()
    outs = torch.full((steps,), -1, dtype=torch.int32, device="cuda")
    g = dec.graph(hd, outs)
    for _ in range(2):
        outs.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(outs.cpu().numpy().view(np.uint32), want)


def test_tailored_plan_slices_cfg4_head(th):
    """cfg4 head (V=256,000 x 2,304 bf16) with a tailored plan (2,048 static
    + a 512-token prompt): the plan cut into G = 2, 4, 8 contiguous slices,
    each slice's rows streamed through its ids, the records combined — ids
    equal the reference greedy over the whole plan; plus an exact tie
    straddling every slice boundary (the lower id wins) and NaN at plan
    row 0 (slice 0 wins outright)."""
    from paper_2508_15229_b200 import sharded, synth

    V, d = 256000, 2304
    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
    W = head.to_host()
    words = synth.words_of(synth.static_ids(V, 2048), V)
    plan = orc.select(synth.prompt_ids(V, 512, 3), words, V, V).active_ids
    hid = synth.round_bf16(synth.head_random(2, d, synth.SEED_H))
    sub = orc.gather(W, plan)
    for t in range(2):
        want = orc.greedy_step(sub, hid[t], plan)[0]
        for G in (1, 2, 4, 8):
            got = sharded.sharded_greedy_local(head, hid[t][None, :], G, plan_ids=plan)
            assert int(got[0]) == int(want), (t, G)
    # ties at the slice boundaries and NaN at plan row 0, on a small head
    Vs, ds = 6000, 256
    rng = np.random.default_rng(2)
    Ws = synth.round_bf16(rng.uniform(-1, 1, (Vs, ds)).astype(np.float32))
    ps = np.sort(rng.choice(Vs, 1600, replace=False)).astype(np.uint32)
    h = synth.round_bf16(rng.uniform(-1, 1, ds).astype(np.float32))
    Wt = Ws.copy()
    for G in (2, 4, 8):
        for r0, _ in sharded.shard_ranges(ps.size, G)[1:]:
            Wt[ps[r0 - 1]] = Wt[ps[r0]] = np.sign(h) * 1.0
    Wn = Ws.copy()
    Wn[ps[0], 3] = np.nan
    for Wc in (Wt, Wn):
        hs = th.HeadMatrix.from_host(Wc, storage=th.SVT_BF16)
        want = orc.greedy_step(Wc[ps], h, ps)[0]
        for G in (1, 2, 4, 8):
            got = sharded.sharded_greedy_local(hs, h[None, :], G, plan_ids=ps)
            assert int(got[0]) == int(want), G
