"""(f1) Plan wire format (artifacts.cpp:169-192): host-only C-ABI, no GPU.

Pinned against the reference's golden plan file (fixtures/golden/plan_aca.json,
copied to tests/golden/plan_aca.json by tests/golden/make_golden.py) and, for
arbitrary plans, against Python's json module, which writes exactly
nlohmann::json's text for objects of unsigned integers (sorted keys,
', '/': ' separators with indent, none compact)."""
import json

import numpy as np
import pytest

from paper_2508_15229_b200 import _lib
from paper_2508_15229_b200.tailored_head import (IntegrityError, ParseError, SelectionPlan,
                                                 plan_from_json, plan_to_json)

GOLDEN = __file__.replace("test_plan_json.py", "golden/plan_aca.json")


def _ref_text(plan, indent):
    obj = {"active_ids": [int(x) for x in plan.active_ids], "n_static": plan.n_static,
           "n_dynamic": plan.n_dynamic, "full_vocab_size": plan.full_vocab_size}
    if indent is None:
        return json.dumps(obj, sort_keys=True, separators=(",", ":"))
    return json.dumps(obj, sort_keys=True, indent=indent)


def test_golden_plan_aca_bytes():
    plan = SelectionPlan(np.array([0, 2, 3, 4], np.uint32), 2, 2, 8)
    want = open(GOLDEN).read()
    assert plan_to_json(plan, indent=2) + "\n" == want  # save_json: dump(2) + '\n'
    back = plan_from_json(want, "plan_aca.json")
    assert back.active_ids.tolist() == [0, 2, 3, 4]
    assert (back.n_static, back.n_dynamic, back.full_vocab_size) == (2, 2, 8)
    assert plan_to_json(plan) == ('{"active_ids":[0,2,3,4],"full_vocab_size":8,'
                                  '"n_dynamic":2,"n_static":2}')


@pytest.mark.parametrize("indent", [None, 0, 2, 4])
def test_random_plans_match_nlohmann_text(indent):
    rng = np.random.default_rng(indent or 7)
    for n in (0, 1, 5, 2547, 20000):
        full = 151936
        ids = np.sort(rng.choice(full, n, replace=False)).astype(np.uint32)
        plan = SelectionPlan(ids, int(rng.integers(0, n + 1)), int(rng.integers(0, 9)), full)
        text = plan_to_json(plan, indent)
        assert text == _ref_text(plan, indent)
        back = plan_from_json(text)
        assert np.array_equal(back.active_ids, ids)
        assert (back.n_static, back.n_dynamic, back.full_vocab_size) == (
            plan.n_static, plan.n_dynamic, full)


def test_plan_from_json_errors_follow_the_reference():
    ok = {"active_ids": [0, 2], "full_vocab_size": 8, "n_dynamic": 1, "n_static": 1}
    with pytest.raises(IntegrityError, match="strictly increasing"):
        plan_from_json(json.dumps(dict(ok, active_ids=[2, 2])))
    with pytest.raises(IntegrityError, match="active id 9 out of range for full_vocab_size 8"):
        plan_from_json(json.dumps(dict(ok, active_ids=[2, 9])))
    bad = dict(ok)
    del bad["n_static"]
    with pytest.raises(ParseError, match=r'plan\.json: missing field "n_static"'):
        plan_from_json(json.dumps(bad), "plan.json")
    # require() order: active_ids, n_static, n_dynamic, full_vocab_size
    with pytest.raises(ParseError, match='missing field "active_ids"'):
        plan_from_json("{}")
    with pytest.raises(ParseError, match='missing field "n_dynamic"'):
        plan_from_json('{"active_ids": [], "n_static": 0}')
    with pytest.raises(ParseError):
        plan_from_json('{"active_ids": [1,')
    with pytest.raises(ParseError):
        plan_from_json('{"active_ids": [-1], "full_vocab_size": 8, "n_dynamic": 0, "n_static": 0}')
    # unknown fields are ignored, whitespace is free
    text = '{ "meta": {"x": [1, "a", null]}, "n_static": 0, "active_ids": [ 3 ],\n' \
           ' "n_dynamic": 1, "full_vocab_size": 4 }'
    assert plan_from_json(text).active_ids.tolist() == [3]


def test_plans_to_jsonl_capacity_csr():
    import ctypes as C
    ids = np.array([1, 5, 9, 99, 0, 2, 7], np.uint32)
    off = np.array([0, 4], np.int64)      # capacity-CSR starts (request 0 has slack)
    na = np.array([3, 3], np.int64)
    ns = np.array([1, 0], np.int64)
    nd = np.array([2, 3], np.int64)
    need = C.c_size_t()
    args = (ids.ctypes.data, off.ctypes.data, na.ctypes.data, ns.ctypes.data, nd.ctypes.data, 2,
            10)
    _lib.call("svt_plans_to_jsonl", *args, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    _lib.call("svt_plans_to_jsonl", *args, buf, need.value, None)
    lines = buf.value.decode().splitlines()
    assert lines == ['{"active_ids":[1,5,9],"full_vocab_size":10,"n_dynamic":2,"n_static":1}',
                     '{"active_ids":[0,2,7],"full_vocab_size":10,"n_dynamic":3,"n_static":0}']
