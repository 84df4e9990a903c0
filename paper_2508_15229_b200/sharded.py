"""Multi-GPU partitioning of the tailored head.

* batch-shard: requests are split across ranks; every rank runs the whole
  single-GPU path on its own requests; no collective on the data path.
* vocab-shard: the plan (here: the full vocabulary, the identity plan) is
  cut into G contiguous ascending row ranges; rank g streams only its rows
  and reduces one 16-byte record per request on the device
  {u64 key = orderable(max) << 32 | ~global_row, u32 id, f32 max}; a single
  all-gather of the records over NCCL (NVLink/NVSwitch) lets every rank pick
  the winner with svt_shard_combine. Because the shards are contiguous and
  ascending, "largest key" is exactly the reference's first-maximum scan
  (head.cpp:213-215) over the whole plan, including its NaN / signed-zero
  rules (plan row 0 lives on shard 0, which alone sets plan_start).
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from ._lib import call
from .tailored_head import HeadMatrix, _stream

RECORD_WORDS = 4  # int32 words per shard record


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
    """Rows [r0, r1) of a head — a view into a full device head, or a rank's
    own slice — scored against B hidden states per step by the fused exact
    GEMV (identity plan: rows are streamed in place, no ids)."""

    def __init__(self, head: HeadMatrix, r0: int, r1: int, B: int, plan_start: bool,
                 local_rows: torch.Tensor = None, stream=None):
        self.storage = head.storage
        self.dim = head.dim()
        self.r0, self.n, self.B = r0, r1 - r0, B
        self.rows = local_rows if local_rows is not None else head.data[r0:r1]
        self.plan_start = 1 if plan_start else 0
        self.stream = stream
        g = (self.n + 31) // 32
        self.max_groups = g * B
        dev = "cuda"
        n_active = torch.full((max(B, 1),), self.n, dtype=torch.int64, device=dev)
        self.group_begin = torch.zeros(B + 1, dtype=torch.int64, device=dev)
        self.group_meta = torch.zeros((max(1, self.max_groups), 8), dtype=torch.int32, device=dev)
        if B:
            call("svt_plan_layout", n_active.data_ptr(), None, B, self.group_begin.data_ptr(),
                 self.group_meta.data_ptr(), self.max_groups, _stream(stream))
        self.ws = torch.empty(max(1, _lib.lib.svt_greedy_workspace_bytes(B, self.max_groups)),
                              dtype=torch.uint8, device=dev)
        self.ids = torch.zeros(max(B, 1), dtype=torch.int32, device=dev)
        self.records = torch.zeros((max(B, 1), RECORD_WORDS), dtype=torch.int32, device=dev)
        # batch 1: the certified single-request kernel (split-K at HBM speed,
        # exact winner value for the record); otherwise the exact-order GEMV
        esize = 4 if self.storage == 0 else 2
        self.certified = (B == 1 and self.n > 0 and (self.dim * esize) % 16 == 0
                          and self.dim <= 8192 and self.rows.data_ptr() % 16 == 0
                          and not os.environ.get("SVT_SHARD_EXACT"))
        self._stable = 0
        if self.certified:
            self.cws = torch.zeros(_lib.lib.svt_greedy_rows_workspace_bytes(self.n),
                                   dtype=torch.uint8, device=dev)

    def step(self, hidden: torch.Tensor) -> torch.Tensor:
        """hidden [B, ld] f32 on the device -> records [B, 4] int32."""
        if self.n == 0:
            self.records.zero_()  # key 0 never wins
            return self.records
        if self.certified:
            # the shard's rows are written once, long before any step
            call("svt_greedy_certified_rows", self.rows.data_ptr(), self.storage, self.n,
                 self.dim, None, self.n, hidden.data_ptr(), None, self.r0, self.plan_start,
                 self._stable, self.ids.data_ptr(), None, self.records.data_ptr(),
                 self.cws.data_ptr(), _stream(self.stream))
            self._stable = 1
            return self.records
        call("svt_greedy_fused", self.rows.data_ptr(), self.storage, self.n, self.dim,
             self.group_begin.data_ptr(), self.group_meta.data_ptr(), None, self.B,
             self.max_groups, hidden.data_ptr(), hidden.stride(0), self.r0, self.plan_start,
             self._stable, self.ids.data_ptr(), None, self.records.data_ptr(),
             self.ws.data_ptr(), _stream(self.stream))
        self._stable = 1
        return self.records


def combine(records: torch.Tensor, out_ids: torch.Tensor, out_max: torch.Tensor = None,
            stream=None) -> torch.Tensor:
    """records [G, B, 4] int32 (all-gathered) -> per-request winner ids."""
    G, B = records.shape[0], records.shape[1]
    call("svt_shard_combine", records.data_ptr(), G, B, out_ids.data_ptr(),
         None if out_max is None else out_max.data_ptr(), _stream(stream))
    return out_ids


class VocabShardedHead:
    """One rank's part of a vocab-sharded head under torch.distributed (NCCL):
    rows shard_ranges(V, world)[rank] held locally; step() = local exact GEMV
    + argmax -> all_gather_into_tensor of the records -> combine."""

    def __init__(self, head: HeadMatrix, B: int, group=None, local_only: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        r0, r1 = shard_ranges(head.rows(), self.world)[self.rank]
        self.shard = RowShard(head, r0, r1, B, plan_start=(self.rank == 0))
        self.B = B
        # flat [world * B, 4] so every backend accepts it (gloo insists on
        # concatenation along dim 0); viewed as [world, B, 4] for the combine
        self.gathered = torch.zeros((self.world * max(B, 1), RECORD_WORDS), dtype=torch.int32,
                                    device="cuda")
        self.out = torch.zeros(max(B, 1), dtype=torch.int32, device="cuda")

    def step(self, hidden: torch.Tensor) -> torch.Tensor:
        rec = self.shard.step(hidden)
        if self.world > 1:
            self.dist.all_gather_into_tensor(self.gathered, rec, group=self.group)
            return combine(self.gathered.view(self.world, -1, RECORD_WORDS), self.out)
        return combine(rec.view(1, *rec.shape), self.out)


# ---- host restatements (used by the gloo tests of the protocol) -------------
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


def shard_record_np(scores: np.ndarray, row_base: int, plan_start: bool, ids=None):
    """(key, id) of one shard's scores, as the device finalize computes it."""
    best = 0
    for k, s in enumerate(np.asarray(scores, np.float32)):
        key = pack_key_np(s, row_base + k, plan_start and k == 0)
        best = max(best, key)
    if best == 0:
        return 0, 0xFFFFFFFF
    row = 0xFFFFFFFF - (best & 0xFFFFFFFF)
    return best, (int(ids[row - row_base]) if ids is not None else row)


def combine_np(keys: np.ndarray, ids: np.ndarray):
    """Host restatement of svt_shard_combine: largest key, first shard on ties."""
    keys = np.asarray(keys, np.uint64)
    g = np.argmax(keys, axis=0)
    return np.asarray(ids)[g, np.arange(keys.shape[1])]


def sharded_greedy_local(head: HeadMatrix, hidden: np.ndarray, G: int) -> np.ndarray:
    """Single-process emulation of the vocab-sharded step (every shard on this
    GPU, the all-gather replaced by a stack): used by the parity tests."""
    B, d = hidden.shape
    ld = (d + 3) // 4 * 4
    h = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
    h[:, :d] = torch.from_numpy(np.ascontiguousarray(hidden, np.float32)).cuda()
    recs = []
    for g, (r0, r1) in enumerate(shard_ranges(head.rows(), G)):
        sh = RowShard(head, r0, r1, B, plan_start=(g == 0))
        recs.append(sh.step(h).clone())
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    combine(torch.stack(recs), out)
    return out.cpu().numpy().view(np.uint32)
