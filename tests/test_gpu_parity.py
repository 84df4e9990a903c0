"""GPU parity: the sm_100a path (libsvt.so, through the C-ABI) against the
oracle and the reference goldens. Bit-exact for ids, plans AND logits — the
kernels keep the reference's accumulation order (head.cpp:194-199)."""
import hashlib

import numpy as np
import pytest
import torch

from conftest import golden_cases
from oracle.oracle import c_oracle, words_from_ids

pytestmark = pytest.mark.gpu

orc = c_oracle()


@pytest.fixture(scope="module")
def th():
    from paper_2508_15229_b200 import tailored_head

    torch.cuda.set_device(0)
    return tailored_head


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def bf16_np(x):
    from paper_2508_15229_b200.synth import round_bf16

    return round_bf16(np.asarray(x, np.float32))


# ---- generator -------------------------------------------------------------------
def test_head_random_matches_reference_generator(th):
    for db, st in [(4, th.SVT_F32), (2, th.SVT_F16), (2, th.SVT_F32)]:
        rt = th.SVT_F16 if db == 2 else th.SVT_F32
        m = th.HeadMatrix.random(61, 37, 0xC0FFEE, dtype_bytes=db, storage=st, round_through=rt)
        assert np.array_equal(bits(m.to_host()), bits(orc.head_random(61, 37, 0xC0FFEE, db)))
    m = th.HeadMatrix.random(33, 50, 0x5EED, storage=th.SVT_BF16)
    assert np.array_equal(bits(m.to_host()), bits(bf16_np(orc.head_random(33, 50, 0x5EED))))


# ---- (a) select ----------------------------------------------------------------
def test_select_known_answers(th):
    plan = th.select([0, 2, 0], th.TokenSet.from_ids(8, [3, 4]), 8)
    assert plan.active_ids.tolist() == [0, 2, 3, 4]
    assert (plan.n_static, plan.n_dynamic, plan.full_vocab_size) == (2, 2, 8)
    again = th.select([0, 2, 0], th.TokenSet.from_ids(8, [3, 4]), 8)
    assert again.active_ids.tolist() == plan.active_ids.tolist()
    p = th.select([7, 3, 3], th.TokenSet(16), 16)
    assert p.active_ids.tolist() == [3, 7] and (p.n_static, p.n_dynamic) == (0, 2)
    p = th.select([2, 1, 2], th.TokenSet.from_ids(8, [1, 2, 5]), 8)
    assert p.active_ids.tolist() == [1, 2, 5] and p.n_dynamic == 0


def test_select_errors(th):
    with pytest.raises(th.IntegrityError, match="input token id 8 out of range"):
        th.select([8], th.TokenSet(8), 8)
    with pytest.raises(th.IntegrityError):
        th.select([0], th.TokenSet(4), 8)
    # first offending id in input order is the one named
    with pytest.raises(th.IntegrityError, match="input token id 12 "):
        th.select([1, 12, 3, 9, 15], th.TokenSet(9), 9)


def test_select_randomised_against_oracle(th):
    rng = np.random.default_rng(11)
    for V in [1, 63, 64, 65, 1000, 4097, 128256, 151936, 256000]:
        for _ in range(3):
            t = np.unique(rng.integers(0, V, int(rng.integers(0, min(V, 3000) + 1))))
            ids = rng.integers(0, V, int(rng.integers(0, 2500))).astype(np.uint32)
            got = th.select(ids, th.TokenSet.from_ids(V, t) if t.size < 400 else _fast_set(th, V, t), V)
            want = orc.select(ids, words_from_ids(t, V), V, V)
            assert np.array_equal(got.active_ids, want.active_ids)
            assert (got.n_static, got.n_dynamic) == (want.n_static, want.n_dynamic)


def _fast_set(th, V, ids):
    s = th.TokenSet(V)
    s.words = words_from_ids(ids, V)
    return s


def test_union_plans(th):
    t = th.TokenSet.from_ids(8, [5])
    u = th.union_plans([th.select([0], t, 8), th.select([2, 3], t, 8)])
    assert u.active_ids.tolist() == [0, 2, 3, 5] and (u.n_static, u.n_dynamic) == (1, 3)
    with pytest.raises(th.ConfigError):
        th.union_plans([])
    rng = np.random.default_rng(3)
    V = 151936
    T = _fast_set(th, V, rng.integers(0, V, 2048))
    plans = [th.select(rng.integers(0, V, 512).astype(np.uint32), T, V) for _ in range(8)]
    want = orc.union_plans([_oplan(p) for p in plans])
    got = th.union_plans(plans)
    assert np.array_equal(got.active_ids, want.active_ids) and got.n_dynamic == want.n_dynamic


def _oplan(p):
    from oracle.oracle import Plan

    return Plan(p.active_ids, p.n_static, p.n_dynamic, p.full_vocab_size)


# ---- (b) gather, (c) logits, (d) greedy_step: reference-shaped calls ------------
def test_gather_copies_rows_exactly(th):
    head = th.HeadMatrix.random(8, 4, 1234)
    sub = th.gather(head, th.SelectionPlan(np.array([0, 2, 3, 4], np.uint32), 0, 4, 8))
    assert np.array_equal(bits(sub.to_host()), bits(head.to_host()[[0, 2, 3, 4]]))
    h6 = th.HeadMatrix.random(6, 3, 9)
    ident = th.gather(h6, th.SelectionPlan(np.arange(6, dtype=np.uint32), 0, 6, 6))
    assert np.array_equal(bits(ident.to_host()), bits(h6.to_host()))
    assert th.gather(h6, th.SelectionPlan(np.zeros(0, np.uint32), 0, 0, 6)).rows() == 0
    with pytest.raises(th.IntegrityError):
        th.gather(h6, th.SelectionPlan(np.array([6], np.uint32), 0, 1, 8))


def test_logits_basics(th):
    head = th.HeadMatrix.from_host(np.array([[2.0], [3.0]], np.float32))
    assert th.logits(head, [5.0]).tolist() == [10.0, 15.0]
    r = th.HeadMatrix.random(4, 8, 7)
    assert (th.logits(r, np.zeros(8, np.float32)) == 0).all()
    with pytest.raises(th.IntegrityError):
        th.logits(r, [1.0])


@pytest.mark.parametrize("storage", ["f32", "f16", "bf16"])
def test_logits_bitwise_against_oracle(th, storage):
    st = {"f32": th.SVT_F32, "f16": th.SVT_F16, "bf16": th.SVT_BF16}[storage]
    rng = np.random.default_rng(17)
    # odd dims take the generic kernel, multiples of 8 the bulk-copy ring kernel
    for rows, dim in [(1, 1), (5, 3), (33, 7), (100, 16), (257, 64), (1000, 896), (70, 2048),
                      (64, 2304), (40, 3072), (31, 1000)]:
        db = 2 if st == th.SVT_F16 else 4
        head = th.HeadMatrix.random(rows, dim, int(rng.integers(0, 2**62)), dtype_bytes=db,
                                    storage=st)
        hv = rng.uniform(-2, 2, dim).astype(np.float32)
        if st == th.SVT_BF16:
            hv = bf16_np(hv)
        got = th.logits(head, hv)
        want = orc.logits(head.to_host(), hv)
        assert np.array_equal(bits(got), bits(want)), (rows, dim)


@pytest.mark.parametrize("sig_bits", [12, 13, 14, 24])
def test_f16_head_short_hidden_bitwise(th, sig_bits):
    # f16 weights with full 11-bit significands against hidden values with
    # 12..14 significant bits: 14 + 11 > 24, so w*h is not exact in f32 and
    # the exact-FMA shortcut must not fire (the mask was 0x3FF)
    rng = np.random.default_rng(0xF16 + sig_bits)
    rows, dim = 300, 512
    mant = rng.integers(0x3FF - 64, 0x400, (rows, dim)).astype(np.uint16)  # near-full significands
    expo = rng.integers(13, 17, (rows, dim)).astype(np.uint16)
    sign = rng.integers(0, 2, (rows, dim)).astype(np.uint16)
    w = ((sign << 15) | (expo << 10) | mant).view(np.float16).astype(np.float32)
    head = th.HeadMatrix.from_host(w, dtype_bytes=2, storage=th.SVT_F16)
    h = rng.uniform(-2, 2, dim).astype(np.float32)
    hb = h.view(np.uint32) | np.uint32((1 << 23) - 1)  # all-ones significand
    hb &= ~np.uint32((1 << (24 - sig_bits)) - 1)
    h = hb.view(np.float32)
    want = orc.logits(w, h)
    assert np.array_equal(bits(th.logits(head, h)), bits(want))
    plan = th.SelectionPlan(np.arange(rows, dtype=np.uint32), 0, rows, rows)
    assert th.greedy_step(head, h, plan) == orc.argmax_first(want)


def test_sub_head_logits_equal_full_head_bitwise(th):
    # test_head.cpp:73-93 on the GPU: logits(gather(head, plan)) == logits(head)[plan]
    rng = np.random.default_rng(0x10617)
    for _ in range(150):
        rows, dim = int(rng.integers(1, 33)), int(rng.integers(1, 17))
        head = th.HeadMatrix.random(rows, dim, int(rng.integers(0, 2**62)))
        picked = np.flatnonzero(rng.integers(0, 2, rows)).astype(np.uint32)
        plan = th.SelectionPlan(picked, 0, picked.size, rows)
        h = rng.uniform(-1, 1, dim).astype(np.float32)
        full = th.logits(head, h)
        sub = th.logits(th.gather(head, plan), h)
        assert np.array_equal(bits(sub), bits(full[picked]))
        assert np.array_equal(bits(full), bits(orc.logits(head.to_host(), h)))


def test_greedy_step_known_answers(th):
    plan = th.SelectionPlan(np.array([0, 2, 4], np.uint32), 0, 3, 8)
    sub = th.HeadMatrix.from_host(np.array([[1.0], [3.0], [2.0]], np.float32))
    assert th.greedy_step(sub, [1.0], plan) == 2
    flat = th.HeadMatrix.from_host(np.ones((3, 1), np.float32))
    assert th.greedy_step(flat, [1.0], plan) == 0
    with pytest.raises(th.IntegrityError, match="empty sub-head"):
        th.greedy_step(th.HeadMatrix(0, 1), [1.0], th.SelectionPlan())
    with pytest.raises(th.IntegrityError):
        th.greedy_step(sub, [1.0], th.SelectionPlan(np.array([0, 2], np.uint32), 0, 2, 8))


def test_greedy_special_values(th):
    nan, inf = np.float32("nan"), np.float32("inf")
    ids = np.array([3, 5, 9, 11], np.uint32)
    plan = th.SelectionPlan(ids, 0, 4, 16)
    for scores, want in [([nan, 5, 7, 1], 3), ([1, nan, 7, 7], 9), ([-0.0, 0.0, -1, -2], 3),
                         ([0.0, -0.0, -1, -2], 3), ([-inf, inf, inf, 0], 5),
                         ([-inf, -inf, -inf, -inf], 3), ([1, nan, nan, nan], 3)]:
        sub = th.HeadMatrix.from_host(np.array(scores, np.float32).reshape(4, 1))
        assert th.greedy_step(sub, [1.0], plan) == want, scores


def test_greedy_agrees_with_full_argmax_when_in_plan(th):
    rng = np.random.default_rng(0xA26A)
    for _ in range(100):
        head = th.HeadMatrix.random(16, 8, int(rng.integers(0, 2**62)))
        picked = np.flatnonzero(rng.integers(0, 2, 16)).astype(np.uint32)
        if picked.size == 0:
            continue
        plan = th.SelectionPlan(picked, 0, picked.size, 16)
        h = rng.uniform(-1, 1, 8).astype(np.float32)
        full = th.logits(head, h)
        arg = orc.argmax_first(full)
        got = th.greedy_step(th.gather(head, plan), h, plan)
        if plan.global_to_local(arg) is not None:
            assert got == arg
        ohead = head.to_host()
        assert got == orc.greedy_step(ohead[picked], h, picked)[0]


# ---- golden fixtures from the real reference ---------------------------------
@pytest.mark.parametrize("name,case", golden_cases(), ids=[n for n, _ in golden_cases()])
@pytest.mark.parametrize("fused", [False, True])
def test_batched_engine_reproduces_reference_goldens(th, name, case, fused):
    V, d, db = int(case["V"]), int(case["d"]), int(case["dtype_bytes"])
    st = th.SVT_BF16 if bool(case["bf16"]) else (th.SVT_F16 if db == 2 else th.SVT_F32)
    head = th.HeadMatrix.random(V, d, int(case["W_seed"]), dtype_bytes=db, storage=st)
    assert hashlib.sha256(bits(head.to_host()).tobytes()).hexdigest() == str(case["W_sha256"])
    words = words_from_ids(case["static_ids"], V)
    poff = case["prompt_off"]
    B = len(poff) - 1
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(),
                                len(case["static_ids"]), V,
                                torch.from_numpy(np.concatenate([case["prompts"], [0]]).astype(
                                    np.uint32).view(np.int32)).cuda(), poff)
    off = case["plan_off"]
    for b in range(B):
        p = tb.plan(b)
        assert np.array_equal(p.active_ids, case["plan_ids"][off[b]:off[b + 1]])
        assert (p.n_static, p.n_dynamic) == (int(case["n_static"][b]), int(case["n_dynamic"][b]))
    tb.gather(head)
    ld = (d + 3) // 4 * 4
    hid = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
    hid[:, :d] = torch.from_numpy(case["hidden_bits"].view(np.float32).reshape(B, d)).cuda()
    lg = tb.logits(hid, fused=fused).cpu().numpy()
    out = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    tb.greedy(hid, out, fused=fused)
    got = out.cpu().numpy().view(np.uint32)
    lo = 0
    for b in range(B):
        n = off[b + 1] - off[b]
        o = int(tb.act_off_h[b])
        assert np.array_equal(bits(lg[o:o + n]), case["logit_bits"][lo:lo + n])
        lo += n
        if n:
            assert got[b] == case["greedy"][b]


# ---- the BASELINE shapes ---------------------------------------------------------
def _build_workload(th, V, d, st, B, L, nT, steps, seed_off=0):
    from paper_2508_15229_b200 import synth

    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=st,
                                round_through=st if st != th.SVT_F16 else th.SVT_F16)
    t_ids = synth.static_ids(V, nT)
    words = synth.words_of(t_ids, V)
    prompts = [synth.prompt_ids(V, L, seed_off + r) for r in range(B)]
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), nT, V,
                                torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(),
                                off)
    tb.gather(head)
    hid = synth.head_random(steps * B, d, synth.SEED_H).reshape(steps, B, d)
    if st == th.SVT_BF16:
        hid = synth.round_bf16(hid)
    return head, words, prompts, tb, hid


@pytest.mark.parametrize("fused", [False, True])
def test_cfg1_llama1b_shape_bit_exact(th, fused):
    """cfg1: V=128256, d=2048, fp32, one 512-token prompt + 2048 static."""
    V, d = 128256, 2048
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, 1, 512, 2048, 4)
    W = head.to_host()
    plan = orc.select(prompts[0], words, V, V)
    assert np.array_equal(tb.plan(0).active_ids, plan.active_ids)
    sub = orc.gather(W, plan.active_ids)
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    for t in range(hid.shape[0]):
        h = torch.from_numpy(hid[t]).cuda()
        tb.greedy(h, out, fused=fused)
        assert int(out.item()) == orc.greedy_step(sub, hid[t][0], plan.active_ids)[0]
    lg = tb.logits(torch.from_numpy(hid[0]).cuda(), fused=fused).cpu().numpy()
    assert np.array_equal(bits(lg[: plan.active_ids.size]), bits(orc.logits(sub, hid[0][0])))


@pytest.mark.parametrize("fused", [False, True])
def test_cfg2_qwen05b_shape_bit_exact(th, fused):
    """cfg2: V=151936, d=896, bf16, 64 requests with their own plans."""
    V, d, B = 151936, 896, 64
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_BF16, B, 512, 2048, 2)
    W = head.to_host()
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    mx = torch.empty(B, dtype=torch.float32, device="cuda")
    for t in range(hid.shape[0]):
        tb.greedy(torch.from_numpy(hid[t]).cuda(), out, mx, fused=fused)
        got = out.cpu().numpy().view(np.uint32)
        for b in range(0, B, 7 if t else 1):
            plan = orc.select(prompts[b], words, V, V)
            if t == 0:
                gp = tb.plan(b)
                assert np.array_equal(gp.active_ids, plan.active_ids)
                assert gp.n_static + gp.n_dynamic == gp.size()
            want, wmax = orc.greedy_step(orc.gather(W, plan.active_ids), hid[t][b],
                                         plan.active_ids)
            assert got[b] == want
            assert bits(mx.cpu().numpy()[b]) == bits(np.float32(wmax))


def test_decode_is_replayable_and_graph_capturable(th):
    V, d, B = 151936, 896, 16
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_BF16, B, 512, 2048, 1)
    h = torch.from_numpy(hid[0]).cuda()
    outs = []
    for _ in range(5):
        o = torch.empty(B, dtype=torch.int32, device="cuda")
        tb.greedy(h, o)
        outs.append(o.cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs)
    # CUDA-graph capture of the decode step replays bit-identically
    o = torch.empty(B, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    tb.stream = s
    with torch.cuda.stream(s):
        tb.greedy(h, o)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tb.greedy(h, o)
    o.fill_(-1)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(o.cpu().numpy(), outs[0])


def test_vocab_sharded_combine(th):
    """Contiguous row shards of one plan + per-shard greedy with row_base +
    svt_shard_combine == whole-plan greedy."""
    from paper_2508_15229_b200 import sharded

    V, d = 20000, 256
    head = th.HeadMatrix.random(V, d, 77, storage=th.SVT_BF16)
    rng = np.random.default_rng(9)
    hid = bf16_np(rng.uniform(-1, 1, (3, d)).astype(np.float32))
    full_ids = np.arange(V, dtype=np.uint32)
    want = [orc.greedy_step(head.to_host(), hid[b], full_ids)[0] for b in range(3)]
    for G in (1, 2, 3, 8):
        got = sharded.sharded_greedy_local(head, hid, G)
        assert got.tolist() == want, G


def test_embedding_lookup_paths(th):
    from paper_2508_15229_b200 import offload

    rows, dim = 5000, 896
    table = np.random.default_rng(1).standard_normal((rows, dim)).astype(np.float32)
    ids = np.random.default_rng(2).integers(0, rows, 700).astype(np.uint32)
    emb = offload.HostEmbedding(table, th.SVT_BF16)
    want = bf16_np(table[ids])
    for mode in ("zero_copy", "staged"):
        got = emb.lookup(ids, mode=mode).float().cpu().numpy()
        assert np.array_equal(bits(got), bits(want)), mode
    with pytest.raises(th.IntegrityError):
        emb.lookup(np.array([rows], np.uint32), mode="staged")


def test_session_host_api_matches_batched_engine(th):
    from paper_2508_15229_b200 import session

    V, d, B = 151936, 896, 8
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_BF16, B, 512, 2048, 2)
    with session.Session(head, max_batch=B) as s:
        off = np.zeros(B + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in prompts])
        s.prepare(words, V, np.concatenate(prompts), off)
        for t in range(2):
            ids = s.greedy(hid[t])
            o = torch.empty(B, dtype=torch.int32, device="cuda")
            tb.greedy(torch.from_numpy(hid[t]).cuda(), o)
            assert np.array_equal(ids, o.cpu().numpy().view(np.uint32))
        with pytest.raises(th.IntegrityError, match="out of range"):
            s.prepare(words, V, np.array([V + 5], np.uint32), np.array([0, 1], np.int64))


def test_certified_greedy_matches_exact_ids(th):
    """svt_greedy_certified (split-K + bounds + exact recompute of candidates)
    returns the reference ids: random steps, exact ties (every row equal),
    zero hidden, NaN hidden, and near-tie rows."""
    from paper_2508_15229_b200 import synth

    for V, d, st, B, steps in [(128256, 2048, th.SVT_F32, 1, 6), (151936, 896, th.SVT_BF16, 16, 3)]:
        head, words, prompts, tb, hid = _build_workload(th, V, d, st, B, 512, 2048, steps)
        W = head.to_host()
        ld = (d + 3) // 4 * 4
        for t in range(steps):
            h = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
            h[:, :d] = torch.from_numpy(hid[t]).cuda()
            a = torch.empty(B, dtype=torch.int32, device="cuda")
            c = torch.empty(B, dtype=torch.int32, device="cuda")
            tb.greedy(h, a)
            tb.greedy_certified(h, c)
            assert np.array_equal(a.cpu().numpy(), c.cpu().numpy()), (V, t)
        plan = orc.select(prompts[0], words, V, V)
        want = orc.greedy_step(orc.gather(W, plan.active_ids), hid[0][0], plan.active_ids)[0]
        h = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
        h[:, :d] = torch.from_numpy(hid[0]).cuda()
        c = torch.empty(B, dtype=torch.int32, device="cuda")
        tb.greedy_certified(h, c)
        assert int(c[0].item()) == want
        # zero hidden: every logit is +0.0 -> lowest row of each plan
        z = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
        tb.greedy_certified(z, c)
        for b in range(B):
            assert int(c[b].item()) & 0xFFFFFFFF == int(tb.plan(b).active_ids[0])
        # NaN hidden: non-finite -> all rows recomputed -> row 0 (s[0] is NaN)
        n = z.clone()
        n[:, 0] = float("nan")
        tb.greedy_certified(n, c)
        a = torch.empty(B, dtype=torch.int32, device="cuda")
        tb.greedy(n, a)
        assert np.array_equal(a.cpu().numpy(), c.cpu().numpy())
        fast, slow = tb.certified_stats()
        assert fast + slow >= steps + 3


def test_certified_near_ties_recompute(th):
    """Rows whose logits differ in the last bits (sum order decides): the
    certified path must fall back to the exact recompute and still match."""
    rows, d = 96, 64
    rng = np.random.default_rng(5)
    base = rng.uniform(-1, 1, d).astype(np.float32)
    W = np.tile(base, (rows, 1))
    # permute columns per row: same multiset of products, different order
    for r in range(1, rows):
        W[r] = base[rng.permutation(d)]
    h = np.ones(d, np.float32)
    head = th.HeadMatrix.from_host(W)
    ids = np.arange(rows, dtype=np.uint32)
    words = words_from_ids(ids[:0], rows)
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 0, rows,
                                torch.from_numpy(ids.view(np.int32)).cuda(),
                                np.array([0, rows], np.int64))
    tb.gather(head)
    hd = torch.from_numpy(h).cuda().view(1, d)
    a = torch.empty(1, dtype=torch.int32, device="cuda")
    c = torch.empty(1, dtype=torch.int32, device="cuda")
    tb.greedy(hd, a)
    tb.greedy_certified(hd, c)
    want = orc.greedy_step(W, h, ids)[0]
    assert int(a.item()) == want and int(c.item()) == want


@pytest.fixture(params=[(1, 4, "1"), (0, 1, "1"), (1, 3, "0"), (0, 8, "0"), (1, 0, "1")],
                ids=lambda t: f"pair{t[0]}_split{t[1]}_smallN{t[2]}")
def prefill_tuning(request, monkeypatch):
    """GEMM tuning: CTA pair or single CTA, N splits (0 = automatic), and
    whether launches with few 256-row N tiles may switch to 64-row tiles."""
    from paper_2508_15229_b200 import prefill

    old = prefill.PrefillScorer.tuning()
    prefill.PrefillScorer.set_tuning(request.param[0], request.param[1])
    monkeypatch.setenv("SVT_PREFILL_SMALL_N", request.param[2])
    yield request.param
    prefill.PrefillScorer.set_tuning(*old)


@pytest.mark.parametrize("S,P,d,V,nT,L", [(3, 128, 256, 6000, 500, 400), (2, 256, 512, 20000, 900, 700),
                                          (2, 512, 192, 9000, 2500, 1200)])
@pytest.mark.parametrize("fused", [False, True], ids=["gathered", "gather4"])
def test_prefill_scoring_tcgen05_ids_exact(th, prefill_tuning, S, P, d, V, nT, L, fused):
    """cfg3-style batched prefill scoring on tcgen05: every position's id
    equals the reference greedy id over its sequence's plan; the tensor-core
    top-1 logit lies within the certification bound of the exact logit.
    Runs the single-CTA and CTA-pair GEMMs with 1-8 N-range splits (ragged
    splits included: some splits own no N tile)."""
    from paper_2508_15229_b200 import prefill, synth

    head = th.HeadMatrix.random(V, d, 0x5EED, storage=th.SVT_BF16)
    W = head.to_host()
    rng = np.random.default_rng(S * 1000 + d)
    words = words_from_ids(rng.choice(V, nT, replace=False), V)
    plans = [orc.select(rng.integers(0, V, L).astype(np.uint32), words, V, V).active_ids
             for _ in range(S)]
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in plans])
    ids = torch.from_numpy(np.concatenate(plans).view(np.int32)).cuda()
    sc = prefill.PrefillScorer(head, ids, off, P, fused=fused)
    hid = synth.round_bf16(rng.uniform(-1, 1, (S * P, d)).astype(np.float32))
    hdev = torch.from_numpy(hid).cuda().to(torch.bfloat16)
    out = torch.empty(S * P, dtype=torch.int32, device="cuda")
    sc.score(hdev, out)
    got = out.cpu().numpy().view(np.uint32)
    tv, tr = sc.top8()
    tv, tr = tv.cpu().numpy(), tr.cpu().numpy().view(np.uint32)
    best = tv.argmax(1)
    tv = tv[np.arange(len(tv)), best][:, None]
    tr = tr[np.arange(len(tr)), best][:, None]
    u = 2.0 ** -24
    gam = lambda n: n * u / (1 - n * u)  # noqa: E731
    worst = 0.0
    for s in range(S):
        sub = orc.gather(W, plans[s])
        wmax = np.sqrt((sub.astype(np.float64) ** 2).sum(1)).max()
        for p in range(P):
            pos = s * P + p
            want, _ = orc.greedy_step(sub, hid[pos], plans[s])
            assert got[pos] == want, (s, p)
            exact = float(orc.logits(sub[tr[pos, 0]: tr[pos, 0] + 1], hid[pos])[0])
            bound = (gam(2 * d) + gam(d)) * np.sqrt((hid[pos].astype(np.float64) ** 2).sum()) * wmax
            worst = max(worst, abs(float(tv[pos, 0]) - exact) / bound)
    assert worst < 1.0, worst
    print("max |tc - exact| / bound =", worst, "stats", sc.stats())


@pytest.mark.parametrize("fused", [False, True], ids=["gathered", "gather4"])
@pytest.mark.parametrize("case", ["duplicate_rows", "nonfinite", "tiny", "tiny_subnormal"])
def test_prefill_scoring_all_rows_fallback(th, prefill_tuning, case, fused):
    """Positions the top-8 cannot certify — more than eight rows tied at the
    maximum (duplicated head rows) or non-finite logits (overflowing hidden
    states) — go through the grid-wide all-rows recompute and still match the
    reference greedy ids (first max, NaN rules of head.cpp:203-217)."""
    from paper_2508_15229_b200 import prefill, synth

    V, d, S, P = 3000, 128, 2, 256
    rng = np.random.default_rng(11)
    base = synth.round_bf16(rng.uniform(-1, 1, (100, d)).astype(np.float32))
    W = base[np.arange(V) % 100] if case == "duplicate_rows" else \
        synth.round_bf16(rng.uniform(-1, 1, (V, d)).astype(np.float32))
    head = th.HeadMatrix.from_host(W, dtype_bytes=2, storage=th.SVT_BF16)
    W = head.to_host()
    plans = [np.sort(rng.choice(V, 1500, replace=False)).astype(np.uint32) for _ in range(S)]
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in plans])
    ids = torch.from_numpy(np.concatenate(plans).view(np.int32)).cuda()
    sc = prefill.PrefillScorer(head, ids, off, P, fused=fused)
    hid = synth.round_bf16(rng.uniform(-1, 1, (S * P, d)).astype(np.float32))
    if case == "nonfinite":
        hid[::7] *= np.float32(3e38)  # products overflow: ±inf and inf-inf NaN logits
        hid[3, :] = np.float32(np.inf)
        hid = synth.round_bf16(hid)
    if case.startswith("tiny"):
        # logits near the smallest normal (products partly subnormal) or
        # entirely subnormal: the reference underflows gradually, the
        # certification's absolute slack must cover it and any flush
        hid = synth.round_bf16(hid * np.float32(2.0 ** (-124 if case == "tiny" else -130)))
    hdev = torch.from_numpy(hid).cuda().to(torch.bfloat16)
    out = torch.empty(S * P, dtype=torch.int32, device="cuda")
    sc.score(hdev, out)
    got = out.cpu().numpy().view(np.uint32)
    for s in range(S):
        sub = orc.gather(W, plans[s])
        for p in range(P):
            want, _ = orc.greedy_step(sub, hid[s * P + p], plans[s])
            assert got[s * P + p] == want, (case, s, p)
    st = sc.stats()
    if not case.startswith("tiny"):
        assert st[1] > 0, st  # candidates were recomputed (all rows or the top-8 ones)


@pytest.mark.parametrize("fused", [False, True], ids=["gathered", "gather4"])
def test_prefill_from_device_batch_matches_reference(th, fused):
    """select (device) -> svt_gather_plans (capacity-CSR) -> prefill scoring:
    ids equal the reference greedy over each request's own plan
    (selector.cpp:16-43 then head.cpp:203-217), no host round trip."""
    from paper_2508_15229_b200 import prefill, synth

    V, d, S, P = 7000, 128, 3, 256
    rng = np.random.default_rng(5)
    head = th.HeadMatrix.random(V, d, 0xC0FFEE, storage=th.SVT_BF16)
    W = head.to_host()
    words = words_from_ids(rng.choice(V, 600, replace=False), V)
    prompts = [rng.integers(0, V, L).astype(np.uint32) for L in (300, 17, 900)]
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in prompts])
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 600, V,
                                torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(),
                                off)
    sc = prefill.PrefillScorer.from_batch(head, tb, P, fused=fused)
    hid = synth.round_bf16(rng.uniform(-1, 1, (S * P, d)).astype(np.float32))
    out = torch.empty(S * P, dtype=torch.int32, device="cuda")
    sc.score(torch.from_numpy(hid).cuda().to(torch.bfloat16), out)
    got = out.cpu().numpy().view(np.uint32)
    for s in range(S):
        plan = orc.select(prompts[s], words, V, V).active_ids
        sub = orc.gather(W, plan)
        for p in range(P):
            want, _ = orc.greedy_step(sub, hid[s * P + p], plan)
            assert got[s * P + p] == want, (s, p)
    assert int(sc.bad.item()) == 0


@pytest.mark.parametrize("case,nT", [("random", 600), ("random", 512), ("duplicate_rows", 600),
                                     ("nonfinite", 300)])
def test_prefill_split_matches_reference(th, prefill_tuning, case, nT):
    """Static/dynamic split (svt_prefill_split_plans + svt_prefill_score_split):
    the shared static rows scored from one block, only D_s \\ T gathered per
    sequence; ids equal the reference greedy over each full plan. Covers the
    static padding (|T| not a multiple of the N tile), ties between static
    and dynamic rows (duplicated head rows: the lower id wins), non-finite
    logits (NaN at the plan's smallest id), an empty prompt, and a plan
    rewritten to miss part of T (its static block is masked, every row
    dynamic)."""
    from paper_2508_15229_b200 import prefill, synth

    V, d, S, P = 5000, 128, 4, 256
    rng = np.random.default_rng(nT * 7 + len(case))
    if case == "duplicate_rows":
        base = synth.round_bf16(rng.uniform(-1, 1, (150, d)).astype(np.float32))
        head = th.HeadMatrix.from_host(base[np.arange(V) % 150], dtype_bytes=2,
                                       storage=th.SVT_BF16)
    else:
        head = th.HeadMatrix.random(V, d, 0xBEEF + nT, storage=th.SVT_BF16)
    W = head.to_host()
    t_ids = rng.choice(V, nT, replace=False)
    words = words_from_ids(t_ids, V)
    prompts = [rng.integers(0, V, L).astype(np.uint32) for L in (400, 0, 1300, 90)]
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in prompts])
    flat = np.concatenate(prompts) if off[-1] else np.zeros(1, np.uint32)
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), nT, V,
                                torch.from_numpy(flat.view(np.int32)).cuda(), off)
    plans = [orc.select(prompts[s], words, V, V).active_ids for s in range(S)]
    # request 3: a plan that misses part of T (explicit rows)
    p3 = plans[3][::2].copy()
    o3 = int(tb.act_off_h[3])
    tb.active[o3: o3 + p3.size].copy_(torch.from_numpy(p3.view(np.int32)))
    tb.n_active[3] = p3.size
    plans[3] = p3
    sc = prefill.PrefillScorer.from_batch(head, tb, P, split=True)
    assert sc.split
    assert sc.st_valid.cpu().tolist() == [nT, nT, nT, 0]
    hid = synth.round_bf16(rng.uniform(-1, 1, (S * P, d)).astype(np.float32))
    if case == "nonfinite":
        hid[::5] *= np.float32(3e38)
        hid[7, :] = np.float32(np.inf)
        hid = synth.round_bf16(hid)
    out = torch.empty(S * P, dtype=torch.int32, device="cuda")
    mx = torch.empty(S * P, dtype=torch.float32, device="cuda")
    sc.score(torch.from_numpy(hid).cuda().to(torch.bfloat16), out, mx)
    got = out.cpu().numpy().view(np.uint32)
    for s in range(S):
        sub = orc.gather(W, plans[s])
        for p in range(P):
            want, _ = orc.greedy_step(sub, hid[s * P + p], plans[s])
            assert got[s * P + p] == want, (case, s, p)
    assert int(sc.bad.item()) == 0
    print("split stats", sc.stats())


@pytest.mark.parametrize("case", ["random_bf16", "random_f32_d100", "duplicate_rows", "nonfinite",
                                  "bf16_d100", "tiny_bf16", "tiny_edge_bf16"])
def test_split_decode_matches_reference(th, case):
    """Split decode (svt_decode_split_plans + svt_greedy_split): the static rows
    scored once for the whole batch, the dynamic rows per request; ids and the
    exact winning logit equal the reference greedy_step over each full plan
    (head.cpp:203-217), across steps and a re-select. Covers ties between
    static and dynamic rows (duplicated head rows: the lower id wins), NaN
    logits (the plan's smallest id wins, static or dynamic), empty prompts,
    a prompt inside T, partial 16-byte chunks (d = 100) and f32 heads."""
    V, B = 20000, 7
    d = 100 if case.endswith("d100") else 256
    storage = th.SVT_F32 if "f32" in case else th.SVT_BF16
    rng = np.random.default_rng(len(case) * 13 + d)
    if case == "duplicate_rows":
        base = bf16_np(rng.uniform(-1, 1, (120, d)).astype(np.float32))
        head = th.HeadMatrix.from_host(base[np.arange(V) % 120], dtype_bytes=2, storage=storage)
    else:
        head = th.HeadMatrix.random(V, d, 0xD00D + d, storage=storage)
    W = head.to_host()
    t_ids = rng.choice(V, 333, replace=False)
    words = words_from_ids(t_ids, V)
    lens = [200, 0, 50, 300, 1, 120, 64]
    prompts = [rng.integers(0, V, L).astype(np.uint32) for L in lens]
    prompts[4] = np.array([int(np.sort(t_ids)[5])], np.uint32)  # entirely inside T
    prompts[6][0] = 0  # id 0 makes the dynamic rows start this plan
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in prompts])
    d_prompts = torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda()
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 333, V, d_prompts,
                                off)
    dec = th.SplitDecoder(tb, head)
    ld = (d + 3) // 4 * 4
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    mx = torch.empty(B, dtype=torch.float32, device="cuda")
    for rnd in range(2):
        for t in range(3):
            h = bf16_np(rng.uniform(-1, 1, (B, d)).astype(np.float32))
            if case == "nonfinite":
                h[t % B] *= np.float32(3e38)
                h[(t + 3) % B, :] = np.float32(np.inf)
            if case.startswith("tiny"):
                # logits in the subnormal range (tiny) or straddling the
                # smallest normal (edge): the reference's f32 chain has
                # gradual underflow, the certification bound must cover
                # every flushed or underflowed partial
                e = -150 if case == "tiny_bf16" else -128
                h = bf16_np(h * np.float32(2.0 ** e / (np.abs(W[:64]).mean() * np.sqrt(d))))
            hl = np.zeros((B, ld), np.float32)
            hl[:, :d] = h
            hd = torch.from_numpy(hl).cuda()
            dec.greedy(hd, out)  # ids only (certified: interval hand-off to the combine)
            got_ids = out.cpu().numpy().view(np.uint32).copy()
            dec.greedy(hd, out, mx)
            got = out.cpu().numpy().view(np.uint32)
            gmx = mx.cpu().numpy()
            assert np.array_equal(got_ids, got), (case, rnd, t)
            for b in range(B):
                plan = orc.select(prompts[b], words, V, V).active_ids
                want, wmax = orc.greedy_step(W[plan], h[b], plan)
                assert got[b] == want, (case, rnd, t, b)
                assert (np.isnan(wmax) and np.isnan(gmx[b])) or gmx[b] == wmax, (case, b)
        prompts = [rng.integers(0, V, L).astype(np.uint32) for L in lens]
        d_prompts.copy_(torch.from_numpy(np.concatenate(prompts).view(np.int32)))
        tb.run_select()
        dec.prepare()
    assert int(dec.bad.item()) == 0
    one, more = dec.stats()
    if storage == th.SVT_BF16 and d % 64 == 0:
        # the certified static half ran: every (step, request) with static
        # rows was decided, mostly from a single candidate's exact chain
        assert one + more > 0
        if case not in ("nonfinite", "duplicate_rows") and not case.startswith("tiny"):
            assert one >= more, (one, more)
    else:
        assert (one, more) == (0, 0)


def test_split_decode_certified_many_requests(th):
    """The certified static half with more than one 64-request block (B =
    150: three blocks, the last partial), |T| not a multiple of the 128-row
    tile and d = 384 (three 128-wide K slices): ids-only calls and calls
    with the exact logit equal the reference greedy_step."""
    V, B, d, nT = 30000, 150, 384, 700
    rng = np.random.default_rng(150)
    head = th.HeadMatrix.random(V, d, 0xB150, storage=th.SVT_BF16)
    W = head.to_host()
    t_ids = rng.choice(V, nT, replace=False)
    words = words_from_ids(t_ids, V)
    prompts = [rng.integers(0, V, int(rng.integers(0, 90))).astype(np.uint32) for _ in range(B)]
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in prompts])
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), nT, V,
                                torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(), off)
    dec = th.SplitDecoder(tb, head)
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    mx = torch.empty(B, dtype=torch.float32, device="cuda")
    plans = [orc.select(prompts[b], words, V, V).active_ids for b in range(B)]
    for t in range(2):
        h = bf16_np(rng.uniform(-1, 1, (B, d)).astype(np.float32))
        hd = torch.from_numpy(h).cuda()
        dec.greedy(hd, out)
        ids_only = out.cpu().numpy().view(np.uint32).copy()
        dec.greedy(hd, out, mx)
        got = out.cpu().numpy().view(np.uint32)
        gmx = mx.cpu().numpy()
        assert np.array_equal(ids_only, got), t
        for b in range(B):
            want, wmax = orc.greedy_step(W[plans[b]], h[b], plans[b])
            assert got[b] == want and bits([gmx[b]])[0] == bits([wmax])[0], (t, b)
    one, more = dec.stats()
    assert one + more == 4 * B and one >= more, (one, more)


def test_split_decode_two_streams(th):
    """Two split decoders on two streams, launched back to back without a
    host sync between them: each stream's static half runs on its own side
    stream and joins its own caller (no shared events), so both batches get
    the reference ids."""
    V, d, B = 12000, 256, 5
    head = th.HeadMatrix.random(V, d, 0xAB, storage=th.SVT_BF16)
    W = head.to_host()
    rng = np.random.default_rng(77)
    decs, hids, refs = [], [], []
    for j in range(2):
        words = words_from_ids(rng.choice(V, 250 + 50 * j, replace=False), V)
        prompts = [rng.integers(0, V, 150).astype(np.uint32) for _ in range(B)]
        off = np.zeros(B + 1, np.int64)
        off[1:] = np.cumsum([len(q) for q in prompts])
        tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(),
                                    250 + 50 * j, V,
                                    torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(),
                                    off)
        decs.append(th.SplitDecoder(tb, head))
        h = bf16_np(rng.uniform(-1, 1, (B, d)).astype(np.float32))
        hids.append(torch.from_numpy(h).cuda())
        refs.append([orc.greedy_step(W[orc.select(prompts[b], words, V, V).active_ids], h[b],
                                     orc.select(prompts[b], words, V, V).active_ids)[0]
                     for b in range(B)])
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty(B, dtype=torch.int32, device="cuda") for _ in range(2)]
    for rep in range(4):
        for j in range(2):
            decs[j].stream = streams[j]
            with torch.cuda.stream(streams[j]):
                decs[j].greedy(hids[j], outs[j])
    torch.cuda.synchronize()
    for j in range(2):
        assert outs[j].cpu().numpy().view(np.uint32).tolist() == refs[j], j


# ---- certified batch-1 decode over row-major rows (cfg1 latency path) ----------
def _rows_decoder(th, head, ids, materialize=True, **kw):
    d_ids = torch.from_numpy(np.ascontiguousarray(ids, np.uint32).view(np.int32)).cuda()
    return th.RowDecoder(head, d_ids, len(ids), materialize=materialize, **kw)


def _rows_greedy(dec, h, want_max=False):
    hd = torch.from_numpy(np.ascontiguousarray(h, np.float32)).cuda()
    out = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    mx = torch.full((1,), -7.0, dtype=torch.float32, device="cuda") if want_max else None
    dec.greedy(hd, out, mx)
    got = int(out.item()) & 0xFFFFFFFF
    return (got, float(mx.item())) if want_max else got


@pytest.mark.parametrize("materialize", [True, False])
def test_rows_certified_cfg1_shape(th, materialize):
    """cfg1 (V=128256, d=2048, f32, 512-token prompt + 2048 static): ids and
    the exact winning logit equal the reference greedy_step bit for bit."""
    V, d = 128256, 2048
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, 1, 512, 2048, 12)
    W = head.to_host()
    plan = orc.select(prompts[0], words, V, V)
    sub = orc.gather(W, plan.active_ids)
    dec = _rows_decoder(th, head, plan.active_ids, materialize)
    for t in range(hid.shape[0]):
        want, wmax = orc.greedy_step(sub, hid[t][0], plan.active_ids)
        assert _rows_greedy(dec, hid[t][0]) == want
        if t < 3:
            got, gmax = _rows_greedy(dec, hid[t][0], want_max=True)
            assert got == want and bits([gmax])[0] == bits([wmax])[0]
    fast, slow = dec.stats()
    assert fast + slow == hid.shape[0] + 3 and slow >= 3


def test_rows_cfg1_all_64_steps_graph_and_exact_logits(th):
    """cfg1 at full shape, all 64 decode steps: (i) back-to-back in CUDA
    graphs (programmatic launches, no host sync between tokens) for two
    jobs token-interleaved and for one job alone, replayed twice — ids equal
    the reference greedy_step; (ii) every step's exact winning logit equals
    the reference's bit for bit."""
    from paper_2508_15229_b200 import synth

    V, d, steps = 128256, 2048, 64
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, 2, 512, 2048, steps)
    W = head.to_host()
    plans = [orc.select(prompts[j], words, V, V).active_ids for j in range(2)]
    subs = [orc.gather(W, p) for p in plans]
    want = np.zeros((steps, 2), np.uint32)
    wmax = np.zeros((steps, 2), np.float32)
    for j in range(2):
        for t in range(steps):
            want[t, j], wmax[t, j] = orc.greedy_step(subs[j], hid[t][j], plans[j])
    decs = [_rows_decoder(th, head, plans[j]) for j in range(2)]
    hd = torch.from_numpy(np.ascontiguousarray(hid, np.float32)).cuda()
    out = torch.full((steps, 2), -1, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    for dcd in decs:
        dcd.stream = st

    def run(jobs):
        for t in range(steps):
            for j in jobs:
                decs[j].greedy(hd[t, j], out[t, j])

    for jobs in ([0, 1], [0]):
        with torch.cuda.stream(st):
            run(jobs)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run(jobs)
        for _ in range(2):
            out.fill_(-1)
            with torch.cuda.stream(st):
                g.replay()
            torch.cuda.synchronize()
            got = out.cpu().numpy().view(np.uint32)
            assert np.array_equal(got[:, jobs], want[:, jobs]), jobs
    for dcd in decs:
        dcd.stream = None
    for t in range(steps):
        for j in range(2):
            gid, gmax = _rows_greedy(decs[j], hid[t][j], want_max=True)
            assert gid == want[t, j] and bits([gmax])[0] == bits([wmax[t, j]])[0], (t, j)


def test_session_prepare_many(th):
    """svt_session_prepare_host_many (one sync for every session) prepares
    the same plans as per-session prepares: five batch-1 sessions on one
    stream then decode_host equals the reference; an out-of-range prompt id
    in the third session raises the reference's IntegrityError."""
    from paper_2508_15229_b200 import session

    V, d, steps, R = 128256, 2048, 4, 5
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, R, 512, 2048, steps)
    W = head.to_host()
    plans = [orc.select(prompts[j], words, V, V).active_ids for j in range(R)]
    want = np.array([[orc.greedy_step(W[plans[j]], hid[t][j], plans[j])[0] for j in range(R)]
                     for t in range(steps)], np.uint32)
    st = torch.cuda.Stream()
    sess = [session.Session(head, max_batch=1, stream=st) for _ in range(R)]
    offs = [np.array([0, len(p)], np.int64) for p in prompts]
    try:
        for rnd in range(2):
            session.prepare_many(sess, words, V, prompts, offs)
            ids = session.decode_host(sess, np.ascontiguousarray(hid, np.float32), steps)
            assert np.array_equal(ids, want), rnd
            # batch-1 plans: counts computed on the host, ids by the select
            for j in range(R):
                op = orc.select(prompts[j], words, V, V)
                n_act, n_st, n_dyn, pids, _ = sess[j].plans()
                assert (int(n_act[0]), int(n_st[0]), int(n_dyn[0])) == (
                    len(op.active_ids), op.n_static, op.n_dynamic), (rnd, j)
                assert np.array_equal(pids, op.active_ids), (rnd, j)
        bad = [p.copy() for p in prompts]
        bad[2][7] = V + 3
        with pytest.raises(th.IntegrityError, match=f"input token id {V + 3} out of range"):
            session.prepare_many(sess, words, V, bad, offs)
    finally:
        for s_ in sess:
            s_.close()


def test_session_batch1_rows_and_decode_host(th):
    """Batch-1 sessions run the certified rows kernel (row-major gather per
    prepare); svt_session_decode_host over three sessions sharing a stream
    (batches 1, 1 and 3) equals the reference for every step, and a single
    session's per-step host call agrees."""
    from paper_2508_15229_b200 import session

    V, d, steps = 128256, 2048, 5
    head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_F32, 5, 512, 2048, steps)
    W = head.to_host()
    plans = [orc.select(prompts[j], words, V, V).active_ids for j in range(5)]
    subs = [orc.gather(W, p) for p in plans]
    want = np.array([[orc.greedy_step(subs[j], hid[t][j], plans[j])[0] for j in range(5)]
                     for t in range(steps)], np.uint32)
    st = torch.cuda.Stream()
    groups = [[0], [1], [2, 3, 4]]
    sess = [session.Session(head, max_batch=len(g), stream=st) for g in groups]
    try:
        for s_, g in zip(sess, groups):
            off = np.zeros(len(g) + 1, np.int64)
            off[1:] = np.cumsum([len(prompts[j]) for j in g])
            s_.prepare(words, V, np.concatenate([prompts[j] for j in g]), off)
        ids = session.decode_host(sess, np.ascontiguousarray(hid, np.float32), steps)
        assert np.array_equal(ids, want)
        ids2 = session.decode_host(sess, torch.from_numpy(hid).pin_memory(), steps)
        assert np.array_equal(ids2, want)
        for t in range(steps):
            assert int(sess[0].greedy(hid[t][:1])[0]) == want[t, 0]
        mx = np.zeros(1, np.float32)
        got = sess[1].greedy(hid[0][1:2], out_max=mx)
        assert int(got[0]) == want[0, 1]
        assert bits(mx)[0] == bits([orc.greedy_step(subs[1], hid[0][1], plans[1])[1]])[0]
    finally:
        for s_ in sess:
            s_.close()


@pytest.mark.parametrize("V,d,storage,n", [(151936, 896, "bf16", 2600), (256000, 2304, "bf16", 4000),
                                           (5000, 256, "f16", 700), (3000, 64, "f32", 300),
                                           (9000, 8192, "f32", 333), (40000, 1024, "bf16", 40000)])
def test_rows_certified_shapes(th, V, d, storage, n):
    """Every team shape (warps per row 1/2/4/8, chunks per lane 1..8), f32 /
    f16 / bf16 storage, and multi-batch CTAs (n = 40000 identity rows)."""
    st = {"f32": th.SVT_F32, "f16": th.SVT_F16, "bf16": th.SVT_BF16}[storage]
    head = th.HeadMatrix.random(V, d, 0x5EED + d, storage=st,
                                dtype_bytes=2 if storage == "f16" else 4)
    W = head.to_host()
    rng = np.random.default_rng(d)
    ids = np.arange(V, dtype=np.uint32) if n == V else np.sort(
        rng.choice(V, n, replace=False)).astype(np.uint32)
    dec = _rows_decoder(th, head, ids, materialize=(n % 2 == 0))
    sub = W[ids]
    for t in range(4):
        h = rng.uniform(-1, 1, d).astype(np.float32)
        assert _rows_greedy(dec, h) == orc.greedy_step(sub, h, ids)[0], (V, d, t)


def test_rows_certified_special_values(th):
    """Reference scan rules through the certified path: zero hidden (all rows
    tie -> lowest), NaN hidden (-> plan row 0), NaN at row 0 / later rows,
    duplicated maxima (-> lowest row), -0.0 vs +0.0, +-inf, and repeated
    calls (the control words reset themselves)."""
    rng = np.random.default_rng(77)
    n, d = 600, 128
    W = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    W[417] = W[233] = W[501] = np.abs(W[5]) + 0.5  # identical maxima for h = +1
    ids = (np.arange(n, dtype=np.uint32) * 3 + 11)
    head = th.HeadMatrix.from_host(W)
    dec = _rows_decoder(th, head, np.arange(n, dtype=np.uint32), remap=False)
    dmap = _rows_decoder(th, head, np.arange(n, dtype=np.uint32))
    pos = np.ones(d, np.float32)
    assert _rows_greedy(dec, pos) == orc.greedy_step(W, pos, np.arange(n, dtype=np.uint32))[0] == 233
    zero = np.zeros(d, np.float32)
    assert _rows_greedy(dec, zero) == 0
    nanh = zero.copy()
    nanh[3] = np.nan
    assert _rows_greedy(dec, nanh) == 0
    for r, want in [(0, 0), (7, None)]:
        Wn = W.copy()
        Wn[r, 9] = np.nan
        hn = th.HeadMatrix.from_host(Wn)
        dn = _rows_decoder(th, hn, ids[:n] * 0 + np.arange(n, dtype=np.uint32))
        ref = orc.greedy_step(Wn, pos, np.arange(n, dtype=np.uint32))[0]
        assert _rows_greedy(dn, pos) == ref
        if want is not None:
            assert ref == want
    Wi = W.copy()
    Wi[40, 0] = np.inf
    Wi[41, 0] = np.inf
    hi = th.HeadMatrix.from_host(Wi)
    di = _rows_decoder(th, hi, np.arange(n, dtype=np.uint32))
    assert _rows_greedy(di, pos) == orc.greedy_step(Wi, pos, np.arange(n, dtype=np.uint32))[0] == 40
    # signed zeros: every row's logit is -0.0 or +0.0 -> row 0
    Wz = np.zeros((n, d), np.float32)
    Wz[::2, 0] = -1.0
    hz = th.HeadMatrix.from_host(Wz)
    dz = _rows_decoder(th, hz, np.arange(n, dtype=np.uint32))
    e1 = np.zeros(d, np.float32)
    e1[0] = 0.0
    assert _rows_greedy(dz, e1) == 0
    # remap through plan ids and repeated calls
    dm = _rows_decoder(th, head, np.arange(n, dtype=np.uint32))
    dm.ids.copy_(torch.from_numpy(ids.view(np.int32)).cuda())
    h = rng.uniform(-1, 1, d).astype(np.float32)
    want = orc.greedy_step(W, h, ids)[0]
    for _ in range(3):
        assert _rows_greedy(dm, h) == want
    assert dmap is not None


def test_rows_certified_candidate_overflow_paths(th):
    """Many candidates: > 16 per CTA (per-CTA overflow -> rescan of that
    CTA's rows) and > 1024 in total (every row recomputed)."""
    for n in (500, 3000):
        d = 64
        rng = np.random.default_rng(n)
        base = rng.uniform(-1, 1, d).astype(np.float32)
        W = np.stack([base[rng.permutation(d)] for _ in range(n)])  # near-ties
        head = th.HeadMatrix.from_host(W)
        ids = np.arange(n, dtype=np.uint32)
        dec = _rows_decoder(th, head, ids)
        h = np.ones(d, np.float32)
        want, wmax = orc.greedy_step(W, h, ids)
        got, gmax = _rows_greedy(dec, h, want_max=True)
        assert got == want and bits([gmax])[0] == bits([wmax])[0]
        assert _rows_greedy(dec, h) == want


def test_rows_certified_slice_row_base(th):
    """Identity-plan slice (vocab-shard use): rows [r0, r1) of the head, ids
    returned as row_base + row; plan_start=0 disables the NaN-at-row-0 rule."""
    V, d = 20000, 512
    head = th.HeadMatrix.random(V, d, 0xABC, storage=th.SVT_BF16)
    W = head.to_host()
    r0, r1 = 7000, 13000
    sl = th.HeadMatrix(0, d, 2, th.SVT_BF16, data=head.data[r0:r1])
    dummy = torch.zeros(1, dtype=torch.int32, device="cuda")
    dec = th.RowDecoder(sl, dummy, r1 - r0, materialize=False, row_base=r0, plan_start=0,
                        remap=False)
    dec._pre = (sl.data.data_ptr(), sl.storage, r1 - r0, d, None, r1 - r0)
    rng = np.random.default_rng(3)
    for _ in range(3):
        h = rng.uniform(-1, 1, d).astype(np.float32)
        want = orc.greedy_step(W[r0:r1], h, np.arange(r0, r1, dtype=np.uint32))[0]
        assert _rows_greedy(dec, h) == want


@pytest.mark.parametrize("storage", ["bf16", "f32"])
def test_explicit_plans_large_subsets(th, storage):
    """TailoredBatch.from_plans (cfg5's explicit subsets, up to 16k rows per
    request, one shared plan among them) through the interleaved and the
    fused-gather decode: ids equal the reference greedy_step."""
    V, d = 40000, 256
    st = th.SVT_BF16 if storage == "bf16" else th.SVT_F32
    head = th.HeadMatrix.random(V, d, 0x5EED, storage=st)
    W = head.to_host()
    rng = np.random.default_rng(9)
    shared = np.sort(rng.choice(V, 16384, replace=False)).astype(np.uint32)
    plans = [shared, np.sort(rng.choice(V, 1000, replace=False)).astype(np.uint32),
             np.arange(V, dtype=np.uint32)[:12345], shared]
    B = len(plans)
    hid = rng.uniform(-1, 1, (B, d)).astype(np.float32)
    if storage == "bf16":
        hid = bf16_np(hid)
    hd = torch.from_numpy(hid).cuda()
    for fused in (False, True):
        tb = th.TailoredBatch.from_plans(V, plans)
        if fused:
            tb.attach(head)
        else:
            tb.gather(head)
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        tb.greedy(hd, out, fused=fused)
        got = out.cpu().numpy().view(np.uint32)
        for b in range(B):
            want = orc.greedy_step(W[plans[b]], hid[b], plans[b])[0]
            assert got[b] == want, (fused, b)
    with pytest.raises(th.IntegrityError):
        th.TailoredBatch.from_plans(V, [np.array([V], np.uint32)])


def test_vocab_sharded_certified_batch1(th):
    """Batch 1 vocab shards run the certified rows kernel with exact shard
    records: random steps, an exact tie straddling shard boundaries (lowest
    global id wins), NaN at global row 0 (shard 0 wins outright) and an
    all-zero hidden state (every row ties -> row 0)."""
    from paper_2508_15229_b200 import sharded

    V, d = 24000, 512
    rng = np.random.default_rng(21)
    W = bf16_np(rng.uniform(-1, 1, (V, d)).astype(np.float32))
    h = bf16_np(rng.uniform(-1, 1, d).astype(np.float32))
    top = np.abs(W).max() * 0 + 1.0
    Wt = W.copy()
    for r in (11999, 12000, 17999):  # straddles the G=2 and G=4 boundaries
        Wt[r] = np.sign(h) * top
    Wn = W.copy()
    Wn[0, 5] = np.nan
    full = np.arange(V, dtype=np.uint32)
    cases = [(W, rng.uniform(-1, 1, d).astype(np.float32)), (W, h), (Wt, h), (Wn, h),
             (W, np.zeros(d, np.float32))]
    for Wc, hc in cases:
        hc = bf16_np(hc)
        head = th.HeadMatrix.from_host(Wc, storage=th.SVT_BF16)
        want = orc.greedy_step(Wc, hc, full)[0]
        for G in (1, 2, 3, 4):
            got = sharded.sharded_greedy_local(head, hc[None, :], G)
            assert int(got[0]) == int(want), (G, want, got)


@pytest.mark.parametrize("split", ["1", "0"], ids=["split", "unsplit"])
@pytest.mark.parametrize("zero_copy", ["1", "0"], ids=["zero_copy", "step_graph"])
def test_session_step_graph_pinned_buffers(th, monkeypatch, zero_copy, split):
    """Pinned host buffers take the zero-copy step (a pull kernel reads the
    hidden states over PCIe while the PDL-launched GEMV streams weights; the
    finalize writes the ids into host memory) or, with
    SVT_SESSION_ZERO_COPY=0, the per-session step graph (H2D -> GEMV ->
    finalize -> D2H, memcpy nodes re-pointed per call): ids equal the batched
    engine across steps with different buffers, a pageable call in between,
    strided pinned rows with the maxima, and a re-prepare with another batch."""
    from paper_2508_15229_b200 import session

    monkeypatch.setenv("SVT_SESSION_ZERO_COPY", zero_copy)
    monkeypatch.setenv("SVT_SESSION_SPLIT", split)  # shared static rows, or every row per request

    V, d = 151936, 896
    for B, steps in ((8, 3), (5, 2)):
        head, words, prompts, tb, hid = _build_workload(th, V, d, th.SVT_BF16, B, 512, 2048,
                                                        steps, seed_off=B)
        hid_pinned = torch.from_numpy(hid).pin_memory()
        outs = torch.empty((steps, B), dtype=torch.int32).pin_memory()
        with session.Session(head, max_batch=8) as s:
            off = np.zeros(B + 1, np.int64)
            off[1:] = np.cumsum([len(p) for p in prompts])
            for rep in range(2):  # prepare twice: graph dropped and rebuilt
                s.prepare(words, V, np.concatenate(prompts), off)
                for t in range(steps):
                    s.greedy(hid_pinned[t], outs[t])
                    o = torch.empty(B, dtype=torch.int32, device="cuda")
                    tb.greedy(torch.from_numpy(hid[t]).cuda(), o)
                    assert torch.equal(outs[t], o.cpu()), (B, rep, t)
                    assert np.array_equal(s.greedy(hid[t]), o.cpu().numpy().view(np.uint32))
                    # strided pinned rows (ld > d) with pinned maxima
                    wide = torch.zeros((B, d + 64), dtype=torch.float32).pin_memory()
                    wide[:, :d] = torch.from_numpy(hid[t])
                    ids2 = torch.empty(B, dtype=torch.int32).pin_memory()
                    mx2 = torch.empty(B, dtype=torch.float32).pin_memory()
                    s.greedy(wide, ids2, mx2)
                    assert torch.equal(ids2, o.cpu()), (B, rep, t, "strided")
                    mref = torch.empty(B, dtype=torch.float32, device="cuda")
                    tb.greedy(torch.from_numpy(hid[t]).cuda(), o, mref)
                    assert torch.equal(mx2, mref.cpu()), (B, rep, t, "max")


@pytest.mark.parametrize("fused", [False, True])
def test_decode_steps_across_reselect(th, fused):
    """Decode steps stream their weights ahead of the programmatic-dependency
    wait only while the sub-heads are unchanged: after run_select() on new
    prompts (+ gather) the next step must see the new plans and rows."""
    V, d, B = 20000, 256, 6
    head = th.HeadMatrix.random(V, d, 0x77, storage=th.SVT_BF16)
    W = head.to_host()
    rng = np.random.default_rng(31)
    words = words_from_ids(rng.choice(V, 300, replace=False), V)
    prompts = [rng.integers(0, V, 200).astype(np.uint32) for _ in range(B)]
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in prompts])
    d_prompts = torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda()
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 300, V, d_prompts,
                                off)
    if fused:
        tb.attach(head)
    else:
        tb.gather(head)
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    for rnd in range(3):
        for t in range(3):
            h = bf16_np(rng.uniform(-1, 1, (B, d)).astype(np.float32))
            tb.greedy(torch.from_numpy(h).cuda(), out, fused=fused)
            got = out.cpu().numpy().view(np.uint32)
            for b in range(B):
                plan = orc.select(prompts[b], words, V, V).active_ids
                assert got[b] == orc.greedy_step(W[plan], h[b], plan)[0], (rnd, t, b)
        # new prompts in place, re-select (+ re-gather)
        prompts = [rng.integers(0, V, 200).astype(np.uint32) for _ in range(B)]
        d_prompts.copy_(torch.from_numpy(np.concatenate(prompts).view(np.int32)))
        tb.run_select()
        if not fused:
            tb.gather(head)


@pytest.mark.gpu
def test_session_batch1_host_counts_edge_cases(th):
    """Batch-1 prepares compute the plan counts and the out-of-range check on
    the host (no read-back): empty prompt, a prompt inside T, duplicates,
    ids 0 and V-1, an empty static set, and bad ids at the first and last
    position (the reference's first offending id in input order); every
    plan, count and decoded id equals the oracle, and a failed prepare
    leaves the session usable for the next one."""
    from paper_2508_15229_b200 import session

    V, d = 5000, 256
    rng = np.random.default_rng(0xC0DE)
    head = th.HeadMatrix.random(V, d, 0x77, storage=th.SVT_F32)
    W = head.to_host()
    t_ids = rng.choice(V, 300, replace=False)
    words = words_from_ids(t_ids, V)
    empty = words_from_ids(np.array([], np.int64), V)
    cases = [
        ("empty prompt", words, np.array([], np.uint32)),
        ("inside T", words, t_ids[:40].astype(np.uint32)),
        ("duplicates", words, np.array([7, 7, 9, 7, 9, 11, 11], np.uint32)),
        ("ends", words, np.array([0, V - 1, 0, V - 1], np.uint32)),
        ("no static", empty, rng.integers(0, V, 64).astype(np.uint32)),
        ("random", words, rng.integers(0, V, 500).astype(np.uint32)),
    ]
    with session.Session(head, max_batch=1) as s:
        for name, w, p in cases:
            s.prepare(w, V, p, np.array([0, len(p)], np.int64))
            op = orc.select(p, w, V, V)
            n_act, n_st, n_dyn, pids, _ = s.plans()
            assert (int(n_act[0]), int(n_st[0]), int(n_dyn[0])) == (
                len(op.active_ids), op.n_static, op.n_dynamic), name
            assert np.array_equal(pids, op.active_ids), name
            if len(op.active_ids):
                h = rng.uniform(-1, 1, (1, d)).astype(np.float32)
                got = s.greedy(h)
                want, _ = orc.greedy_step(W[op.active_ids], h[0], op.active_ids)
                assert int(got[0]) == want, name
        for bad_pos in (0, 5):
            p = rng.integers(0, V, 6).astype(np.uint32)
            p[bad_pos] = V + bad_pos
            p[5] = V + 100 if bad_pos == 0 else p[5]
            with pytest.raises(th.IntegrityError, match=f"input token id {V + bad_pos} out of range"):
                s.prepare(words, V, p, np.array([0, len(p)], np.int64))
        p = rng.integers(0, V, 30).astype(np.uint32)
        s.prepare(words, V, p, np.array([0, len(p)], np.int64))
        op = orc.select(p, words, V, V)
        assert np.array_equal(s.plans()[3], op.active_ids)


def test_session_decode_host_graph_batched(th):
    """svt_session_decode_host over a batched (split) session with pinned
    host buffers runs as one cached CUDA graph once a layout repeats (the
    first call of a layout is eager, the second captures): repeated calls with
    re-prepares of the same shape and with DIFFERENT pinned hidden / output
    buffers (the memcpy nodes are re-pointed), then a prepare with other
    prompt lengths (a new layout: the graph is rebuilt), and a pageable
    call in between (eager) all return the reference ids."""
    from paper_2508_15229_b200 import session

    V, d, B, steps = 20000, 256, 12, 5
    rng = np.random.default_rng(0x6A)
    head = th.HeadMatrix.random(V, d, 0x6A, storage=th.SVT_BF16)
    W = head.to_host()
    words = words_from_ids(rng.choice(V, 400, replace=False), V)

    def prompts_of(lo, hi):
        return [rng.integers(0, V, int(rng.integers(lo, hi))).astype(np.uint32) for _ in range(B)]

    def want(prompts, hid):
        plans = [orc.select(p, words, V, V).active_ids for p in prompts]
        return np.array([[orc.greedy_step(W[plans[b]], hid[t, b], plans[b])[0] for b in range(B)]
                         for t in range(steps)], np.uint32)

    with session.Session(head, max_batch=B) as s:
        prompts = prompts_of(20, 120)
        flat = np.concatenate(prompts)
        off = np.zeros(B + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in prompts])
        for rnd in range(4):
            s.prepare(words, V, flat, off)
            hid = bf16_np(rng.uniform(-1, 1, (steps, B, d)).astype(np.float32))
            if rnd == 2:  # pageable: the eager path
                got = session.decode_host([s], hid, steps)
            else:
                hp = torch.from_numpy(hid).pin_memory()
                out = torch.empty((steps, B), dtype=torch.int32).pin_memory()
                session.decode_host([s], hp, steps, out)
                got = out.numpy().view(np.uint32)
            assert np.array_equal(got, want(prompts, hid)), rnd
        prompts = prompts_of(130, 200)  # other lengths: a new layout
        flat = np.concatenate(prompts)
        off[1:] = np.cumsum([len(p) for p in prompts])
        for rnd in range(3):  # eager, capture, replay of the new layout
            s.prepare(words, V, flat, off)
            hid = bf16_np(rng.uniform(-1, 1, (steps, B, d)).astype(np.float32))
            hp = torch.from_numpy(hid).pin_memory()
            out = torch.empty((steps, B), dtype=torch.int32).pin_memory()
            session.decode_host([s], hp, steps, out)
            assert np.array_equal(out.numpy().view(np.uint32), want(prompts, hid)), rnd
