"""Full-shape parity pins (VERDICT r1 "next" 1): each BASELINE config's own
path checked against the oracle at the config's real shape, not a reduced
stand-in.

* cfg2: the split decode (static rows once per step) at V=151,936, d=896,
  B=64, |T|=2,048, L=512 — ids and exact winning logits of sampled requests
  against the reference greedy_step (head.cpp:203-217) over each full plan
  (selector.cpp:16-43), every request against the unsplit exact GEMV;
* cfg3: the tcgen05 prefill scorer at d=3,072, V=128,256, |S| ~ 4k (2,048
  static + a 2,048-token prompt) and an adversarial head/hidden pair
  (exactly cancelling products spread over 2^-30..2^16 plus a normal part:
  the reference's own rounding decides the argmax) — ids exact, tensor-core
  top-1 within the certification bound;
* cfg4: the vocab-sharded head at V=256,000 x 2,304 (bf16, identity plan)
  for G = 2, 4, 8, two tokens each.

The oracle (oracle/svt_oracle.c) runs threaded over positions: ctypes
releases the GIL, every call is the same single-threaded restatement."""
from concurrent.futures import ThreadPoolExecutor

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


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _pmap(fn, items):
    with ThreadPoolExecutor(max_workers=8) as ex:
        return list(ex.map(fn, items))


def _workload(th, V, d, st, B, L, nT, steps):
    from paper_2508_15229_b200 import synth

    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=st)
    t_ids = synth.static_ids(V, nT)
    words = synth.words_of(t_ids, V)
    prompts = [synth.prompt_ids(V, L, r) for r in range(B)]
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), nT, V,
                                torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(),
                                off)
    hid = synth.head_random(steps * B, d, synth.SEED_H).reshape(steps, B, d)
    if st == th.SVT_BF16:
        hid = synth.round_bf16(hid)
    return head, words, prompts, tb, hid


def test_split_decode_cfg2_full_shape(th):
    """cfg2 (V=151,936, d=896, bf16, B=64, |T|=2,048, L=512), 4 decode steps
    through SplitDecoder: 8 requests per step (a different 8 each step, 32
    distinct) against the oracle with the exact winning logit; all 64
    against the unsplit exact-order GEMV."""
    V, d, B, steps = 151936, 896, 64, 4
    head, words, prompts, tb, hid = _workload(th, V, d, th.SVT_BF16, B, 512, 2048, steps)
    tb.gather(head)
    W = head.to_host()
    dec = th.SplitDecoder(tb, head)
    assert dec.nT == 2048
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    mx = torch.empty(B, dtype=torch.float32, device="cuda")
    ref = torch.empty(B, dtype=torch.int32, device="cuda")
    plans = {}
    for t in range(steps):
        h = torch.from_numpy(hid[t]).cuda()
        dec.greedy(h, out)  # ids only: certified intervals handed to the combine
        ids_only = out.cpu().numpy().view(np.uint32).copy()
        dec.greedy(h, out, mx)
        tb.greedy(h, ref)
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(ids_only, got), t
        gmx = mx.cpu().numpy()
        assert np.array_equal(got, ref.cpu().numpy().view(np.uint32)), t
        reqs = list(range(t, B, 8))

        def one(b):
            if b not in plans:
                plans[b] = orc.select(prompts[b], words, V, V).active_ids
            p = plans[b]
            return orc.greedy_step(W[p], hid[t][b], p)

        for b, (want, wmax) in zip(reqs, _pmap(one, reqs)):
            assert got[b] == want, (t, b)
            assert bits([gmx[b]])[0] == bits([wmax])[0], (t, b)
    assert int(dec.bad.item()) == 0
    # the certified static half decided every request of every step, almost
    # always with the exact chain of a single candidate row
    one, more = dec.stats()
    assert one + more == 2 * steps * B and one >= 0.8 * 2 * steps * B, (one, more)


def _check_prefill(th, head, W, plans, hid, S, P, sc):
    d = W.shape[1]
    hdev = torch.from_numpy(hid).cuda().to(torch.bfloat16)
    out = torch.empty(S * P, dtype=torch.int32, device="cuda")
    sc.score(hdev, out)
    got = out.cpu().numpy().view(np.uint32)
    tv, tr = sc.top8()
    tv, tr = tv.cpu().numpy(), tr.cpu().numpy().view(np.uint32)
    u = 2.0 ** -24
    gam = lambda n: n * u / (1 - n * u)  # noqa: E731
    subs = [orc.gather(W, p) for p in plans]

    def one(pos):
        s = pos // P
        want, _ = orc.greedy_step(subs[s], hid[pos], plans[s])
        return want

    wants = _pmap(one, range(S * P))
    assert np.array_equal(got, np.array(wants, np.uint32)), \
        np.flatnonzero(got != np.array(wants, np.uint32))[:8]
    # the tensor-core top-1 (a split's best; plan rows / head ids depending on
    # the layout) stays inside the certification bound of its exact logit
    worst = 0.0
    if sc.split:  # split records name virtual rows [T padded, D_s \\ T]
        vids = sc.vids.cpu().numpy().view(np.uint32)
        voff = sc.vid_off.cpu().numpy()
    for s in range(S):
        wmax = np.sqrt((subs[s].astype(np.float64) ** 2).sum(1)).max()
        for p in range(P):
            pos = s * P + p
            k = int(np.argmax(tv[pos]))
            r = int(tr[pos, k])
            row = W[vids[voff[s] + r]] if sc.split else subs[s][r]
            exact = float(orc.logits(row[None, :].copy(), hid[pos])[0])
            if not np.isfinite(exact):
                continue
            bound = (gam(2 * d) + gam(d)) * np.sqrt((hid[pos].astype(np.float64) ** 2).sum()) * wmax
            worst = max(worst, abs(float(tv[pos, k]) - exact) / bound)
    assert worst < 1.0, worst
    return worst


@pytest.mark.parametrize("split", [True, False], ids=["split", "per_sequence"])
def test_prefill_scorer_cfg3_full_shape(th, split):
    """cfg3 shape (V=128,256, d=3,072, bf16; |T|=2,048 + a 2,048-token prompt
    per sequence, |S| ~ 4k), 2 sequences x 128 positions through the
    tcgen05 scorer: every id equals the reference greedy_step."""
    from paper_2508_15229_b200 import prefill, synth

    V, d, S, P = 128256, 3072, 2, 128
    head, words, prompts, tb, _ = _workload(th, V, d, th.SVT_BF16, S, 2048, 2048, 1)
    W = head.to_host()
    plans = [orc.select(prompts[s], words, V, V).active_ids for s in range(S)]
    assert all(3900 < p.size < 4200 for p in plans), [p.size for p in plans]
    sc = prefill.PrefillScorer.from_batch(head, tb, P, split=split)
    assert sc.split == split
    hid = synth.round_bf16(synth.head_random(S * P, d, synth.SEED_H))
    worst = _check_prefill(th, head, W, plans, hid, S, P, sc)
    assert int(sc.bad.item()) == 0
    print("cfg3 full shape: max |tc - exact| / bound =", worst, "stats", sc.stats())


@pytest.mark.parametrize("emax", [16, 0], ids=["noise_dominated", "mostly_certified"])
def test_prefill_scorer_d3072_adversarial_cancellation(th, emax):
    """d=3,072, rows whose first 2,048 coordinates come in exactly cancelling
    pairs (w, -w) against hidden pairs (x, x) with |x| spread over
    2^-30..2^emax (emax 16: noise-dominated, every position recomputed; emax
    0: most positions certified straight from the tensor cores), the other 1,024 coordinates ordinary: the exact dot is the
    ordinary part, but the reference's sequential sum carries rounding noise
    of the large cancelling terms, which decides near-ties. Stresses the
    tensor-core accumulation model (wide exponent spread inside K blocks,
    heavy cancellation) behind the certification; ids must still be the
    reference's bit for bit."""
    from paper_2508_15229_b200 import prefill, synth

    V, d, S, P, nT, L = 12000, 3072, 2, 128, 1000, 1500
    rng = np.random.default_rng(3072)
    npair = 1024
    a = synth.round_bf16(rng.uniform(-1, 1, (V, npair)).astype(np.float32))
    W = np.empty((V, d), np.float32)
    W[:, 0:2 * npair:2] = a
    W[:, 1:2 * npair:2] = -a
    W[:, 2 * npair:] = synth.round_bf16(rng.uniform(-1, 1, (V, d - 2 * npair)).astype(np.float32))
    head = th.HeadMatrix.from_host(W, dtype_bytes=2, storage=th.SVT_BF16)
    W = head.to_host()
    words = words_from_ids(rng.choice(V, nT, replace=False), V)
    prompts = [rng.integers(0, V, L).astype(np.uint32) for _ in range(S)]
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in prompts])
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), nT, V,
                                torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(),
                                off)
    plans = [orc.select(prompts[s], words, V, V).active_ids for s in range(S)]
    e = rng.integers(-30, emax + 1, (S * P, npair)).astype(np.float32)
    x = (np.sign(rng.uniform(-1, 1, (S * P, npair))) * np.exp2(e) *
         rng.uniform(1, 2, (S * P, npair))).astype(np.float32)
    hid = np.empty((S * P, d), np.float32)
    hid[:, 0:2 * npair:2] = x
    hid[:, 1:2 * npair:2] = x
    hid[:, 2 * npair:] = rng.uniform(-1, 1, (S * P, d - 2 * npair))
    hid = synth.round_bf16(hid)
    for split in (True, False):
        sc = prefill.PrefillScorer.from_batch(head, tb, P, split=split)
        worst = _check_prefill(th, head, W, plans, hid, S, P, sc)
        st = sc.stats()
        print("adversarial emax", emax, "split" if split else "per-seq", "worst", worst,
              "stats", st)
        assert int(sc.bad.item()) == 0


def test_vocab_shard_cfg4_full_head(th):
    """cfg4: the full V=256,000 x d=2,304 bf16 head (identity plan) cut into
    G = 2, 4, 8 contiguous shards, each shard's certified rows kernel with an
    exact record, then svt_shard_combine: two tokens, ids equal the reference
    greedy_step over the whole vocabulary (head.cpp:203-217)."""
    from paper_2508_15229_b200 import sharded, synth

    V, d = 256000, 2304
    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
    W = head.to_host()
    hid = synth.round_bf16(synth.head_random(2, d, synth.SEED_H))
    full = np.arange(V, dtype=np.uint32)
    # the oracle over row slices (contiguous, ascending: first max of the
    # slices' first maxima == the whole scan's)
    want = []
    for t in range(2):
        parts = _pmap(lambda r: orc.greedy_step(W[r[0]:r[1]], hid[t], full[r[0]:r[1]]),
                      sharded.shard_ranges(V, 8))
        # orc.greedy_step over the slice returns (id, max); pick the first max
        best = 0
        for g, (gid, gmax) in enumerate(parts):
            if g == 0 or gmax > parts[best][1]:
                best = g
        want.append(parts[best][0])
    # and pin that slice combination against the unsharded oracle once
    assert orc.greedy_step(W, hid[0], full)[0] == want[0]
    for G in (1, 2, 4, 8):
        got = sharded.sharded_greedy_local(head, hid, G)
        assert got.tolist() == want, (G, got, want)
