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


# ---- the C-ABI path: svt_sharded_greedy over an NCCL communicator ----------
class NcclComm:
    """An NCCL communicator made through the C-ABI (svt_nccl_*), so the
    sharded step needs no torch.distributed on its data path: rank 0 makes
    the unique id, ``exchange`` ships it to every rank (torch.distributed
    broadcast of 128 bytes when a process group exists; any transport
    works), each rank initialises its communicator on its current device."""

    def __init__(self, world: int = 1, rank: int = 0, unique_id: bytes = None, exchange=None):
        import ctypes

        self.world, self.rank = world, rank
        if unique_id is None and rank == 0:
            buf = ctypes.create_string_buffer(128)
            call("svt_nccl_get_unique_id", buf, 128)
            unique_id = buf.raw
        if exchange is not None:
            unique_id = exchange(unique_id)
        elif world > 1:
            import torch.distributed as dist

            obj = [unique_id]
            dist.broadcast_object_list(obj, src=0)
            unique_id = obj[0]
        self.unique_id = unique_id
        comm = ctypes.c_void_p()
        call("svt_nccl_comm_init", ctypes.byref(comm), world, rank,
             ctypes.create_string_buffer(unique_id, 128))
        self.ptr = comm.value

    def close(self):
        if self.ptr:
            call("svt_nccl_comm_destroy", self.ptr)
            self.ptr = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class ShardedDecoder:
    """This rank's slice of a vocab-sharded plan, decoded through
    svt_sharded_greedy (certified rows kernel -> ncclAllGather -> combine).

    * identity plan (``plan_ids=None``): rows [r0, r1) of
      shard_ranges(n_plan, world)[rank]; ``head`` is the whole head, or, with
      ``local_rows=True``, only this rank's rows (as cfg4 materialises them;
      then ``n_plan`` = the full vocabulary).
    * tailored plan (``plan_ids``: the plan's ascending ids, host array): the
      plan is cut into contiguous ascending slices;
      this rank gathers only its slice's rows into a row-major block and
      remaps winners through the slice's ids.
    Batch 1. ``graph(hiddens, outs)`` captures a whole decode loop (kernel +
    all-gather + combine per step) in one CUDA graph."""

    def __init__(self, head: HeadMatrix, comm: "NcclComm" = None, plan_ids=None,
                 n_plan: int = None, local_rows: bool = False, stream=None):
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.comm = comm
        self.head, self.stream = head, stream
        self.dim = head.dim()
        esize = 4 if head.storage == 0 else 2
        dev = "cuda"
        if plan_ids is None:
            n_plan = head.rows() if n_plan is None else n_plan
            r0, r1 = shard_ranges(n_plan, self.world)[self.rank]
            self.rows = head.data if local_rows else head.data[r0:r1]
            self.ids = None
        else:
            plan = np.ascontiguousarray(plan_ids, np.uint32)
            r0, r1 = shard_ranges(plan.size, self.world)[self.rank]
            self.ids = torch.from_numpy(plan[r0:r1].view(np.int32).copy()).to(dev)
            self.rows = torch.empty((max(1, r1 - r0), self.dim), dtype=head.data.dtype, device=dev)
            if r1 > r0:
                bad = torch.zeros(1, dtype=torch.int32, device=dev)
                call("svt_gather_rows", head.data.data_ptr(), head.storage, head.rows(), self.dim,
                     self.ids.data_ptr(), r1 - r0, self.rows.data_ptr(), bad.data_ptr(),
                     _stream(stream))
        self.r0, self.n = r0, r1 - r0
        assert self.rows.data_ptr() % 16 == 0 and (self.dim * esize) % 16 == 0
        nb = _lib.lib.svt_sharded_workspace_bytes(self.n, self.world)
        self._ws_buf = torch.zeros(nb + 256, dtype=torch.uint8, device=dev)
        off = (-self._ws_buf.data_ptr()) % 256
        self.ws = self._ws_buf[off:off + nb]
        self.out = torch.zeros(1, dtype=torch.int32, device=dev)
        self._stable = 0

    def step(self, hidden: torch.Tensor, out_id: torch.Tensor = None,
             out_max: torch.Tensor = None) -> torch.Tensor:
        """hidden: f32 [dim] on the device (16-byte aligned) -> global id."""
        out_id = self.out if out_id is None else out_id
        call("svt_sharded_greedy", self.rows.data_ptr(), self.head.storage, max(1, self.n),
             self.dim, None, self.n, hidden.data_ptr(),
             None if self.ids is None else self.ids.data_ptr(), self.r0, self._stable,
             self.comm.ptr if self.comm is not None else None, self.world, out_id.data_ptr(),
             None if out_max is None else out_max.data_ptr(), self.ws.data_ptr(),
             _stream(self.stream))
        self._stable = 1  # the slice's rows are written once, before any step
        return out_id

    def graph(self, hiddens: torch.Tensor, outs: torch.Tensor):
        """Capture len(hiddens) steps (hiddens [T, ld] f32, outs [T] int32) in
        one CUDA graph on a side stream; returns the graph (replay() it)."""
        st = torch.cuda.Stream()
        old = self.stream
        self.stream = st
        with torch.cuda.stream(st):  # warm: stable weights from the 2nd step
            for t in range(min(2, hiddens.shape[0])):
                self.step(hiddens[t], outs[t])
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for t in range(hiddens.shape[0]):
                self.step(hiddens[t], outs[t])
        self.stream = old
        return g


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


def sharded_greedy_local(head: HeadMatrix, hidden: np.ndarray, G: int,
                         plan_ids: np.ndarray = None) -> np.ndarray:
    """Single-process emulation of the vocab-sharded step (every shard on this
    GPU, the all-gather replaced by a stack): used by the parity tests.
    plan_ids (ascending, host): a tailored plan, cut into contiguous slices
    whose rows are gathered per shard; default: the identity plan."""
    B, d = hidden.shape
    ld = (d + 3) // 4 * 4
    h = torch.zeros((B, ld), dtype=torch.float32, device="cuda")
    h[:, :d] = torch.from_numpy(np.ascontiguousarray(hidden, np.float32)).cuda()
    recs = []
    if plan_ids is not None and B == 1:
        plan = np.ascontiguousarray(plan_ids, np.uint32)
        for g, (r0, r1) in enumerate(shard_ranges(plan.size, G)):
            rec = torch.zeros(4, dtype=torch.int32, device="cuda")
            if r1 > r0:
                sl = torch.from_numpy(plan[r0:r1].view(np.int32).copy()).cuda()
                ws = torch.zeros(_lib.lib.svt_greedy_rows_workspace_bytes(r1 - r0),
                                 dtype=torch.uint8, device="cuda")
                oid = torch.zeros(1, dtype=torch.int32, device="cuda")
                # rows through the slice ids straight from the head (fused gather)
                call("svt_greedy_certified_rows", head.data.data_ptr(), head.storage, head.rows(),
                     d, sl.data_ptr(), r1 - r0, h.data_ptr(), sl.data_ptr(), r0,
                     1 if r0 == 0 else 0, 0, oid.data_ptr(), None, rec.data_ptr(),
                     ws.data_ptr(), None)
            recs.append(rec.view(1, 4).clone())
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        combine(torch.stack(recs), out)
        return out.cpu().numpy().view(np.uint32)
    for g, (r0, r1) in enumerate(shard_ranges(head.rows(), G)):
        sh = RowShard(head, r0, r1, B, plan_start=(g == 0))
        recs.append(sh.step(h).clone())
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    combine(torch.stack(recs), out)
    return out.cpu().numpy().view(np.uint32)
