"""Pin the CPU oracle (oracle/svt_oracle.c) before trusting it.

1. Known-answer tests copied in meaning from the reference's own suite
   (tests/test_selector.cpp, test_head.cpp, test_token_set.cpp,
   acceptance.cpp criteria 4 and 6, fixtures/golden/plan_aca.json).
2. The committed golden fixtures (tests/golden/*.npz), produced by the real
   reference compiled from /root/reference (tests/golden/make_golden.py).
3. When oracle/_ref is built (this container), live differential checks
   against the reference on seeded inputs.
"""
import hashlib

import numpy as np
import pytest

from conftest import golden_cases
from oracle.oracle import OracleError, c_oracle, ref_available, ref_lib, words_from_ids

orc = c_oracle()


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


# ---- select / remap / union (test_selector.cpp) ---------------------------
def test_select_fixture_aca():
    # "aca" encodes to [0, 2, 0] with the toy tokenizer; T = {3, 4}
    # (test_selector.cpp:37-52, fixtures/golden/plan_aca.json)
    p = orc.select([0, 2, 0], words_from_ids([3, 4], 8), 8, 8)
    assert p.active_ids.tolist() == [0, 2, 3, 4]
    assert (p.n_static, p.n_dynamic, p.full_vocab_size) == (2, 2, 8)


def test_select_empty_static_and_inside_static():
    p = orc.select([7, 3, 3], words_from_ids([], 16), 16, 16)
    assert p.active_ids.tolist() == [3, 7] and p.n_dynamic == 2 and p.n_static == 0
    p = orc.select([2, 1, 2], words_from_ids([1, 2, 5], 8), 8, 8)
    assert p.active_ids.tolist() == [1, 2, 5] and p.n_dynamic == 0


def test_select_rejects_out_of_range():
    with pytest.raises(OracleError) as e:
        orc.select([8], words_from_ids([], 8), 8, 8)
    assert e.value.code == 4
    with pytest.raises(OracleError) as e:
        orc.select([0], words_from_ids([], 4), 4, 8)
    assert e.value.code == 4


def test_remap_and_global_to_local():
    p = orc.select([0, 2], words_from_ids([3, 4], 8), 8, 8)
    assert orc.remap_out(p.active_ids, 0) == 0 and orc.remap_out(p.active_ids, 3) == 4
    with pytest.raises(OracleError):
        orc.remap_out(p.active_ids, 4)
    for k, g in enumerate(p.active_ids):
        assert orc.global_to_local(p.active_ids, int(g)) == k
    assert orc.global_to_local(p.active_ids, 1) is None


def test_union_plans():
    t = words_from_ids([5], 8)
    u = orc.union_plans([orc.select([0], t, 8, 8), orc.select([2, 3], t, 8, 8)])
    assert u.active_ids.tolist() == [0, 2, 3, 5] and u.n_static == 1 and u.n_dynamic == 3
    with pytest.raises(OracleError) as e:
        orc.union_plans([])
    assert e.value.code == 2


# ---- head (test_head.cpp) ----------------------------------------------------
def test_logits_basics():
    assert orc.logits(np.array([[2.0], [3.0]], np.float32), [5.0]).tolist() == [10.0, 15.0]
    r = orc.head_random(4, 8, 7)
    assert (orc.logits(r, np.zeros(8, np.float32)) == 0).all()
    with pytest.raises(OracleError):
        orc.logits(r, [1.0])


def test_gather_exact_and_bounds():
    head = orc.head_random(8, 4, 1234)
    sub = orc.gather(head, [0, 2, 3, 4])
    assert np.array_equal(bits(sub), bits(head[[0, 2, 3, 4]]))
    assert orc.gather(head, []).shape == (0, 4)
    with pytest.raises(OracleError):
        orc.gather(orc.head_random(6, 3, 9), [6])


def test_greedy_step_kats():
    sub = np.array([[1.0], [3.0], [2.0]], np.float32)
    assert orc.greedy_step(sub, [1.0], [0, 2, 4])[0] == 2
    assert orc.greedy_step(np.ones((3, 1), np.float32), [1.0], [0, 2, 4])[0] == 0
    with pytest.raises(OracleError):
        orc.greedy_step(np.zeros((0, 1), np.float32), [1.0], [])


def test_argmax_nan_and_signed_zero_rules():
    nan = np.float32("nan")
    assert orc.argmax_first(np.array([nan, 5, 7], np.float32)) == 0   # s[0] NaN -> 0
    assert orc.argmax_first(np.array([1, nan, 7], np.float32)) == 2   # later NaN skipped
    assert orc.argmax_first(np.array([-0.0, 0.0], np.float32)) == 0   # -0 == +0
    assert orc.argmax_first(np.array([-np.inf, np.inf, np.inf], np.float32)) == 1


def test_sub_head_logits_equal_full_head_bitwise():
    # test_head.cpp:73-93 / acceptance criterion 4, seeded numpy stream
    rng = np.random.default_rng(0x10617)
    for _ in range(500):
        rows, dim = int(rng.integers(1, 33)), int(rng.integers(1, 17))
        head = orc.head_random(rows, dim, int(rng.integers(0, 2**63)))
        picked = np.flatnonzero(rng.integers(0, 2, rows)).astype(np.uint32)
        hid = rng.uniform(-1, 1, dim).astype(np.float32)
        full = orc.logits(head, hid)
        sub = orc.logits(orc.gather(head, picked), hid)
        assert np.array_equal(bits(sub), bits(full[picked]))


def test_memory_report_arithmetic():
    fh, sh, eg, eh, saved = orc.memory_report(128000, 2048, 2, 105)
    assert (sh, fh, eg, eh) == (430080, 524288000, 0, 524288000) and saved > 0.99
    assert orc.memory_report(1000, 64, 4, 1000)[4] == 0.5
    assert orc.memory_report(1000, 64, 4, 0)[4] == 1.0
    with pytest.raises(OracleError) as e:
        orc.memory_report(10, 10, 3, 1)
    assert e.value.code == 2


def test_half_conversions_every_pattern():
    for h in range(0x10000):
        if ((h >> 10) & 0x1F) == 0x1F and (h & 0x3FF):
            continue
        assert orc.float_to_half(orc.half_to_float(h)) == h
    assert orc.half_to_float(0x3C00) == 1.0 and orc.half_to_float(0xC000) == -2.0
    assert orc.float_to_half(0.5) == 0x3800


# ---- golden fixtures from the real reference ----------------------------------
@pytest.mark.parametrize("name,case", golden_cases(), ids=[n for n, _ in golden_cases()])
def test_oracle_reproduces_reference_goldens(name, case):
    V, d, db = int(case["V"]), int(case["d"]), int(case["dtype_bytes"])
    W = orc.head_random(V, d, int(case["W_seed"]), db)
    if bool(case["bf16"]):
        W = np.vectorize(orc.round_bf16, otypes=[np.float32])(W)
    assert hashlib.sha256(bits(W).tobytes()).hexdigest() == str(case["W_sha256"])
    words = words_from_ids(case["static_ids"], V)
    hid = case["hidden_bits"].view(np.float32)
    poff, off = case["prompt_off"], case["plan_off"]
    lo = 0
    for b in range(len(poff) - 1):
        p = orc.select(case["prompts"][poff[b]:poff[b + 1]], words, V, V)
        assert np.array_equal(p.active_ids, case["plan_ids"][off[b]:off[b + 1]])
        assert (p.n_static, p.n_dynamic) == (int(case["n_static"][b]), int(case["n_dynamic"][b]))
        sub = orc.gather(W, p.active_ids)
        lg = orc.logits(sub, hid[b])
        assert np.array_equal(bits(lg), case["logit_bits"][lo:lo + len(lg)])
        lo += len(lg)
        if len(p.active_ids):
            assert orc.greedy_step(sub, hid[b], p.active_ids)[0] == int(case["greedy"][b])


# ---- live differential checks against oracle/_ref -------------------------------
needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_random_head_matches_reference():
    ref = ref_lib()
    for db in (4, 2):
        a, b = orc.head_random(37, 29, 0xABC, db), ref.head_random(37, 29, 0xABC, db)
        assert np.array_equal(bits(a), bits(b))


@needs_ref
def test_select_union_greedy_match_reference_randomised():
    ref = ref_lib()
    rng = np.random.default_rng(5)
    for _ in range(60):
        V = int(rng.integers(1, 3000))
        t = np.unique(rng.integers(0, V, int(rng.integers(0, min(V, 300) + 1))))
        w = words_from_ids(t, V)
        ids = rng.integers(0, V, int(rng.integers(0, 200))).astype(np.uint32)
        a, b = orc.select(ids, w, V, V), ref.select(ids, w, V, V)
        assert np.array_equal(a.active_ids, b.active_ids)
        assert (a.n_static, a.n_dynamic) == (b.n_static, b.n_dynamic)
        d = int(rng.integers(1, 40))
        W = orc.head_random(V, d, int(rng.integers(0, 2**62)))
        h = rng.uniform(-2, 2, d).astype(np.float32)
        if a.active_ids.size:
            sub = orc.gather(W, a.active_ids)
            assert np.array_equal(bits(orc.logits(sub, h)), bits(ref.logits(sub, h)))
            assert orc.greedy_step(sub, h, a.active_ids)[0] == ref.greedy_step(sub, h, a.active_ids)
    plans = [orc.select(rng.integers(0, 500, 30).astype(np.uint32), words_from_ids([1, 9], 500),
                        500, 500) for _ in range(5)]
    assert np.array_equal(orc.union_plans(plans).active_ids, ref.union_plans(plans).active_ids)


@needs_ref
def test_offload_model_matches_reference():
    ref = ref_lib()
    hw = (16e9, 4e12, 50e-9)
    for plan, dim, b, L, f in [(0, 2048, 2, 512, 2e9), (1000, 2048, 4, 100, 1e9),
                               (123456, 896, 2, 2048, 3e9), (5, 1, 2, 0, 0.0)]:
        assert orc.simulate(*hw, plan, dim, b, L, f) == ref.simulate(*hw, plan, dim, b, L, f)
    for dim, b, L, f in [(2048, 2, 512, 2e9), (896, 4, 64, 5e8), (3072, 2, 2048, 6e9)]:
        assert orc.breakeven_rows(*hw, dim, b, L, f) == ref.breakeven_rows(*hw, dim, b, L, f)
    for h in range(0, 0x10000, 7):
        assert orc.half_to_float(h) == ref.half_to_float(h) or (
            np.isnan(orc.half_to_float(h)) and np.isnan(ref.half_to_float(h)))


# ---- top-k (north_star (d); defined, not in the reference) --------------------
def _topk_brute(scores, ids, k):
    """(value desc, id asc) with the scan's NaN rules, by Python sorting."""
    s = np.asarray(scores, np.float32)

    def rank(r):
        v = float(s[r])
        if np.isnan(v):
            return (2, 0.0, r) if r == 0 else (0, 0.0, r)
        return (1, v + 0.0, r)  # -0.0 == +0.0

    order = sorted(range(len(s)), key=lambda r: (-rank(r)[0], -rank(r)[1], r))
    return [int(ids[r]) for r in order[:k]]


def _score_cases(rng):
    yield rng.uniform(-1, 1, 300).astype(np.float32)
    yield np.round(rng.uniform(-3, 3, 200)).astype(np.float32)  # many exact ties
    s = rng.uniform(-1, 1, 50).astype(np.float32)
    s[[0, 7]] = np.nan
    yield s
    s = rng.uniform(-1, 1, 50).astype(np.float32)
    s[[3, 9, 11]] = np.nan
    yield s
    yield np.array([-0.0, 0.0, -0.0, -1.0, np.inf, -np.inf, np.inf], np.float32)
    yield np.full(5, np.nan, np.float32)


def test_topk_definition_brute_force_and_top1_is_greedy():
    rng = np.random.default_rng(17)
    for s in _score_cases(rng):
        n = s.size
        ids = np.sort(rng.choice(10 * n, n, replace=False)).astype(np.uint32)
        # an identity "head" whose logits are exactly the scores: row r = e_r * s_r
        W = np.zeros((n, n), np.float32)
        W[np.arange(n), np.arange(n)] = s
        h = np.ones(n, np.float32)
        sc = orc.logits(W, h)
        for k in (1, 3, n, n + 4):
            got, vals = orc.topk(W, h, ids, k)
            want = _topk_brute(sc, ids, k)
            assert got[:len(want)].tolist() == want, (k, s)
            assert all(x == 0xFFFFFFFF for x in got[len(want):])
            assert got[0] == orc.greedy_step(W, h, ids)[0]
            for j, gid in enumerate(want):
                r = int(np.searchsorted(ids, gid))
                assert bits([vals[j]])[0] == bits([sc[r]])[0]


@needs_ref
def test_topk_top1_matches_reference_greedy():
    ref = ref_lib()
    rng = np.random.default_rng(23)
    for _ in range(40):
        V, d = int(rng.integers(2, 2000)), int(rng.integers(1, 64))
        W = orc.head_random(V, d, int(rng.integers(0, 2**62)))
        plan = np.sort(rng.choice(V, int(rng.integers(1, V + 1)), replace=False)).astype(np.uint32)
        h = rng.uniform(-1, 1, d).astype(np.float32)
        sub = orc.gather(W, plan)
        ids, _ = orc.topk(sub, h, plan, 5)
        assert ids[0] == ref.greedy_step(sub, h, plan)
