"""Multi-GPU partitioning of the tailored head.

* batch-shard: requests are split across ranks; every rank runs the whole
  single-GPU path on its own requests; no collective.
* vocab-shard: the plan (or the full vocabulary for the identity plan) is
  cut into G contiguous ascending row ranges; rank g streams only its rows,
  reduces a packed (orderable max << 32 | ~global_row) key per request on
  the device, and one all-gather of (key, id, max) records over NCCL lets
  every rank pick the winner with svt_shard_combine. Because shards are
  contiguous and ascending, "largest key" == the reference scan's first
  maximum (head.cpp:213-215) over the whole plan.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call
from .tailored_head import HeadMatrix, _stream


def shard_ranges(n: int, G: int):
    """Contiguous near-equal row ranges [r0, r1) for G shards."""
    base, extra = divmod(n, G)
    out, r = [], 0
    for g in range(G):
        k = base + (1 if g < extra else 0)
        out.append((r, r + k))
        r += k
    return out


class RowShard:
    """Rows [r0, r1) of a head (a view into the full head, or a rank-local
    copy) scored for B hidden states per step with the fused greedy kernel.
    Source rows are contiguous, so no plan ids are read (identity plan)."""

    def __init__(self, head: HeadMatrix, r0: int, r1: int, B: int, plan_start: bool,
                 local_rows: torch.Tensor = None):
        self.storage = head.storage
        self.dim = head.dim()
        self.r0, self.n, self.B = r0, r1 - r0, B
        self.rows = local_rows if local_rows is not None else head.data[r0:r1]
        self.plan_start = 1 if plan_start else 0
        g = (self.n + 31) // 32
        self.max_groups = g * B
        dev = "cuda"
        n_active = torch.full((max(B, 1),), self.n, dtype=torch.int64, device=dev)
        self.group_begin = torch.zeros(B + 1, dtype=torch.int64, device=dev)
        self.group_meta = torch.zeros((max(1, self.max_groups), 8), dtype=torch.int32, device=dev)
        # identity plan over the slice: no id offsets (row == id index)
        call("svt_plan_layout", n_active.data_ptr(), None, B, self.group_begin.data_ptr(),
             self.group_meta.data_ptr(), self.max_groups, _stream(None))
        self.ws = torch.empty(max(1, _lib.lib.svt_greedy_workspace_bytes(B, self.max_groups)),
                              dtype=torch.uint8, device=dev)
        self.keys = torch.zeros(B, dtype=torch.int64, device=dev)
        self.ids = torch.zeros(B, dtype=torch.int32, device=dev)
        self.max = torch.zeros(B, dtype=torch.float32, device=dev)

    def step(self, hidden: torch.Tensor, stream=None):
        """hidden [B, ld] f32 on the device -> (keys, ids, max) of this shard."""
        if self.n == 0:
            self.keys.zero_()
            return self.keys, self.ids, self.max
        call("svt_greedy_fused", self.rows.data_ptr(), self.storage, self.n, self.dim,
             self.group_begin.data_ptr(), self.group_meta.data_ptr(), None, self.B,
             self.max_groups, hidden.data_ptr(), hidden.stride(0), self.r0,
             self.plan_start, self.ids.data_ptr(), self.max.data_ptr(), self.keys.data_ptr(),
             self.ws.data_ptr(), _stream(stream))
        return self.keys, self.ids, self.max


def combine(keys: torch.Tensor, ids: torch.Tensor, mx: torch.Tensor, out_ids: torch.Tensor,
            out_max: torch.Tensor = None, stream=None):
    """keys/ids/max: [G, B] gathered records -> per-request winner (device)."""
    G, B = keys.shape
    call("svt_shard_combine", keys.data_ptr(), ids.data_ptr(), mx.data_ptr(), G, B,
         out_ids.data_ptr(), None if out_max is None else out_max.data_ptr(), _stream(stream))
    return out_ids


def combine_np(keys: np.ndarray, ids: np.ndarray):
    """Host restatement of svt_shard_combine (largest key, first shard on
    equal keys) — used by the gloo tests of the collective protocol."""
    keys = np.asarray(keys, np.uint64)
    g = np.argmax(keys, axis=0)  # first maximal shard
    return np.asarray(ids)[g, np.arange(keys.shape[1])]


def pack_key_np(value: float, row: int, plan_row0: bool = False) -> int:
    """Host restatement of the device key (svt_common.cuh make_key)."""
    v = np.float32(value)
    if np.isnan(v):
        return 0xFFFFFFFFFFFFFFFF if plan_row0 else 0
    if v == 0:
        v = np.float32(0.0)
    u = int(np.array(v, np.float32).view(np.uint32))
    o = (~u & 0xFFFFFFFF) if (u & 0x80000000) else (u | 0x80000000)
    return (o << 32) | (0xFFFFFFFF - row)


def sharded_greedy_local(head: HeadMatrix, hidden: np.ndarray, G: int) -> np.ndarray:
    """Single-process emulation of the vocab-sharded step (every shard on this
    GPU, the all-gather replaced by a stack): used by tests."""
    B, d = hidden.shape
    ld = (d + 3) // 4 * 4
    h = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
    h[:, :d] = torch.from_numpy(np.ascontiguousarray(hidden, np.float32)).cuda()
    recs = []
    for g, (r0, r1) in enumerate(shard_ranges(head.rows(), G)):
        sh = RowShard(head, r0, r1, B, plan_start=(g == 0))
        k, i, m = sh.step(h)
        recs.append((k.clone(), i.clone(), m.clone()))
    keys = torch.stack([r[0] for r in recs])
    ids = torch.stack([r[1] for r in recs])
    mx = torch.stack([r[2] for r in recs])
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    combine(keys, ids, mx, out)
    return out.cpu().numpy().view(np.uint32)
