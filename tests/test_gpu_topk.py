"""Top-k over each request's plan on the GPU (svt_topk_logits over the exact
reference-order logits) against the oracle's definition (orc_topk: value
desc, id asc, the scan's NaN rules; entry 0 == greedy_step) — at the cfg2
shape and on special values. Ids and values bit-exact."""
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


def same_values(a, b):
    """Bit-equal, except that any NaN matches any NaN (the payload of a NaN
    produced by arithmetic differs between the CPU and the GPU)."""
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    nan = np.isnan(a) & np.isnan(b)
    return bool(np.all(nan | (bits(a) == bits(b))))


@pytest.mark.parametrize("k", [1, 8, 64, 256])
def test_topk_cfg2_shape(th, k):
    from paper_2508_15229_b200 import synth

    V, d, B = 151936, 896, 64
    head = th.HeadMatrix.random(V, d, synth.SEED_W, storage=th.SVT_BF16)
    W = head.to_host()
    words = synth.words_of(synth.static_ids(V, 2048), V)
    prompts = [synth.prompt_ids(V, 512, r) for r in range(B)]
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 2048, V,
                                torch.from_numpy(np.concatenate(prompts).view(np.int32)).cuda(),
                                off)
    tb.gather(head)
    hid = synth.round_bf16(synth.head_random(B, d, synth.SEED_H))
    hd = torch.from_numpy(hid).cuda()
    ids, vals = tb.topk(hd, k)
    greedy = torch.empty(B, dtype=torch.int32, device="cuda")
    tb.greedy(hd, greedy)
    ids = ids.cpu().numpy().view(np.uint32)
    vals = vals.cpu().numpy()
    assert np.array_equal(ids[:, 0], greedy.cpu().numpy().view(np.uint32))
    for b in range(0, B, 9):
        plan = orc.select(prompts[b], words, V, V).active_ids
        wid, wv = orc.topk(W[plan], hid[b], plan, k)
        assert np.array_equal(ids[b], wid), b
        assert same_values(vals[b], wv), b


def test_topk_special_values_and_small_plans(th):
    """Exact ties (duplicated rows: the lower id first), NaN at plan row 0
    (first) and elsewhere (last), -0.0 == +0.0, +-inf, k larger than a plan
    (tail 0xFFFFFFFF / NaN), an empty prompt."""
    rng = np.random.default_rng(12)
    V, d = 4000, 128
    base = rng.uniform(-1, 1, (40, d)).astype(np.float32)
    W = base[np.arange(V) % 40].copy()  # 100 copies of each row: ties everywhere
    W[5, 0] = np.nan
    W[17, :] = 0.0
    W[17, 0] = -0.0
    W[23, 1] = np.inf
    head = th.HeadMatrix.from_host(W)
    W = head.to_host()
    words = words_from_ids(rng.choice(V, 300, replace=False), V)
    prompts = [rng.integers(0, V, L).astype(np.uint32) for L in (200, 0, 3, 500)]
    prompts[2][:] = [0, 5, 17]  # NaN row 5 sits early, row 0 is plan row 0
    off = np.zeros(len(prompts) + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    flat = np.concatenate(prompts)
    tb = th.TailoredBatch.build(torch.from_numpy(words.view(np.int64)).cuda(), 300, V,
                                torch.from_numpy(flat.view(np.int32)).cuda(), off)
    tb.gather(head)
    for trial in range(3):
        hid = rng.uniform(-1, 1, (len(prompts), d)).astype(np.float32)
        if trial == 1:
            hid[:, 0] = np.nan  # every row NaN: plan row 0 first, then by row
        if trial == 2:
            hid[:, :] = 0.0  # all logits +-0: ties to the lowest ids
        hd = torch.from_numpy(hid).cuda()
        for k in (1, 7, 256):
            ids, vals = tb.topk(hd, k)
            ids = ids.cpu().numpy().view(np.uint32)
            vals = vals.cpu().numpy()
            for b in range(len(prompts)):
                plan = orc.select(prompts[b], words, V, V).active_ids
                wid, wv = orc.topk(W[plan], hid[b], plan, k)
                assert np.array_equal(ids[b], wid), (trial, k, b)
                assert same_values(vals[b], wv), (trial, k, b)
