"""World-size-2 (gloo, CPU) tests of the multi-GPU protocol host logic.

The device kernels need a GPU; what is checked here is the protocol the
kernels implement: contiguous ascending row shards, the packed
(orderable max, ~row) key of each shard (the host restatement
sharded.pack_key_np of svt_common.cuh make_key), an all-gather of the
records, and the largest-key combine — against the oracle's whole-plan
greedy (head.cpp:203-217), including ties that straddle a shard boundary,
NaN at plan row 0 and signed zeros. Also the batch-shard timing reduction
(max over ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import c_oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cases():
    orc = c_oracle()
    rng = np.random.default_rng(4)
    cases = []
    for V, d in [(777, 16), (64, 8), (1000, 33)]:
        W = orc.head_random(V, d, int(rng.integers(0, 2**62)))
        h = rng.uniform(-1, 1, d).astype(np.float32)
        cases.append((f"random_{V}_{d}", orc.logits(W, h)))
    s = np.zeros(10, np.float32)
    s[[3, 7]] = 5.0  # tie straddling the 2-way split at 5
    cases.append(("tie_across_boundary", s))
    s = np.array([np.nan, 1, 2, 3, 9, 4], np.float32)
    cases.append(("nan_at_row0", s))
    s = np.array([-1, np.nan, -2, -3, np.nan, -1], np.float32)
    cases.append(("nan_elsewhere", s))
    s = np.array([-0.0, -1, -2, 0.0, -5], np.float32)
    cases.append(("signed_zero", s))
    s = np.full(9, -np.inf, np.float32)
    cases.append(("all_minus_inf", s))
    return cases


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_15229_b200 import sharded

    results = []
    for name, scores in _cases():
        ids = np.arange(len(scores), dtype=np.uint32) * 3 + 1  # a strictly increasing plan
        r0, r1 = sharded.shard_ranges(len(scores), world)[rank]
        key, gid = sharded.shard_record_np(scores[r0:r1], r0, rank == 0, ids[r0:r1])
        rec = torch.tensor([key & 0xFFFFFFFF, key >> 32, gid], dtype=torch.int64)
        out = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(out, rec)
        keys = np.array([[(int(o[1]) << 32) | int(o[0])] for o in out], dtype=np.uint64)
        gids = np.array([[int(o[2])] for o in out], dtype=np.int64)
        results.append((name, int(sharded.combine_np(keys, gids)[0])))
    # batch-shard timing: max over ranks
    t = torch.tensor([1.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    results.append(("timing_max", float(t.item())))
    dist.destroy_process_group()
    q.put((rank, results))


@pytest.mark.parametrize("world", [2])
def test_vocab_shard_protocol_matches_whole_plan_greedy(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = c_oracle()
    for rank in range(world):
        res = dict(got[rank])
        assert res.pop("timing_max") == float(world)
        for name, scores in _cases():
            ids = np.arange(len(scores), dtype=np.uint32) * 3 + 1
            want = int(ids[orc.argmax_first(scores)])
            assert res[name] == want, (name, rank)


def test_shard_ranges_cover_contiguously():
    from paper_2508_15229_b200.sharded import shard_ranges

    for n in (0, 1, 7, 256000):
        for G in (1, 2, 3, 8):
            r = shard_ranges(n, G)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
