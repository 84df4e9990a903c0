"""Host-side mirror of the reference's tailored-head API over the C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/subvocab/{token_set,selector,head,offload_sim}.hpp
so the parity tests read like the reference's own tests
(tests/test_head.cpp, test_selector.cpp, test_token_set.cpp). All compute
goes through libsvt.so (sm_100a CUDA); PyTorch only provides device memory
and streams. There is no CPU fallback.

Two layers:
  * reference-shaped single-plan calls: select, remap_out, union_plans,
    gather, logits, greedy_step, memory_report, simulate, breakeven_rows;
  * the batched device engine (``TailoredBatch``): one plan per request,
    select -> plan layout -> lane-interleaved gather -> fused greedy decode,
    with no host synchronisation inside a decode step.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import (SVT_BF16, SVT_F16, SVT_F32, SVT_ROWS_HIDDEN_STABLE, SVT_WEIGHTS_STABLE,
                   ConfigError, Error,
                   IntegrityError, ParseError, call)

__all__ = [
    "Error", "ConfigError", "ParseError", "IntegrityError", "TokenSet", "SelectionPlan",
    "HeadMatrix", "select", "remap_out", "union_plans", "gather", "logits", "greedy_step",
    "memory_report", "simulate", "breakeven_rows", "TailoredBatch", "SVT_F32", "SVT_F16",
    "SVT_BF16", "dtype_of", "torch_dtype", "SplitDecoder",
]

_TORCH = {SVT_F32: torch.float32, SVT_F16: torch.float16, SVT_BF16: torch.bfloat16}


def torch_dtype(dt: int) -> torch.dtype:
    return _TORCH[dt]


def dtype_of(t: torch.dtype) -> int:
    for k, v in _TORCH.items():
        if v == t:
            return k
    raise ConfigError(f"unsupported storage dtype {t}")


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _require_cuda():
    if _lib.lib.svt_device_count() == 0 or not torch.cuda.is_available():
        raise Error("no CUDA device available: the tailored-head path has no CPU fallback")


# --------------------------------------------------------------------------
# TokenSet (token_set.hpp:17-64): host bitmap; shipped to the device as words
# --------------------------------------------------------------------------
class TokenSet:
    def __init__(self, universe_size: int = 0):
        self._universe = int(universe_size)
        self.words = np.zeros((self._universe + 63) // 64, dtype=np.uint64)

    @staticmethod
    def from_ids(universe_size: int, ids) -> "TokenSet":
        s = TokenSet(universe_size)
        for i in np.asarray(ids, dtype=np.int64).reshape(-1):
            s.insert(int(i))
        return s

    def universe_size(self) -> int:
        return self._universe

    def size(self) -> int:
        return int(sum(bin(int(w)).count("1") for w in self.words))

    def empty(self) -> bool:
        return not self.words.any()

    def contains(self, tid: int) -> bool:
        if tid < 0 or tid >= self._universe:
            return False
        return bool((int(self.words[tid // 64]) >> (tid % 64)) & 1)

    def insert(self, tid: int) -> None:
        if tid < 0 or tid >= self._universe:
            raise IntegrityError(
                f"token id {tid} out of range for universe of size {self._universe}")
        self.words[tid // 64] |= np.uint64(1 << (tid % 64))

    def erase(self, tid: int) -> None:
        if 0 <= tid < self._universe:
            self.words[tid // 64] &= ~np.uint64(1 << (tid % 64))

    def to_ids(self) -> np.ndarray:
        bits = np.unpackbits(self.words.view(np.uint8), bitorder="little")
        return np.flatnonzero(bits[: self._universe]).astype(np.uint32)

    def __eq__(self, other) -> bool:
        return (isinstance(other, TokenSet) and self._universe == other._universe
                and np.array_equal(self.words, other.words))


# --------------------------------------------------------------------------
# SelectionPlan (selector.hpp:16-24)
# --------------------------------------------------------------------------
@dataclass
class SelectionPlan:
    active_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    n_static: int = 0
    n_dynamic: int = 0
    full_vocab_size: int = 0

    def size(self) -> int:
        return int(len(self.active_ids))

    def global_to_local(self, tid: int) -> Optional[int]:
        k = int(np.searchsorted(self.active_ids, tid, side="left"))
        if k == len(self.active_ids) or int(self.active_ids[k]) != tid:
            return None
        return k


def _dev(a, dtype) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.size == 0:
        a = np.zeros(1, dtype=a.dtype)
    return torch.from_numpy(a).to(device="cuda", dtype=dtype)


def select(input_ids, static_members: TokenSet, full_vocab_size: int) -> SelectionPlan:
    """select (selector.cpp:16-43) on the GPU bitmap builder."""
    _require_cuda()
    if static_members.universe_size() != full_vocab_size:
        raise IntegrityError(
            f"static vocabulary universe {static_members.universe_size()} does not match full "
            f"vocabulary size {full_vocab_size}")
    ids = np.ascontiguousarray(np.asarray(input_ids, dtype=np.int64).reshape(-1))
    if ids.size and (ids.min() < 0 or ids.max() >= 2**32):
        bad = int(ids[(ids < 0) | (ids >= 2**32)][0])
        raise IntegrityError(
            f"input token id {bad} out of range for vocabulary of size {full_vocab_size}")
    ids = ids.astype(np.uint32)
    batch = TailoredBatch.select_only(static_members.words, full_vocab_size, [ids])
    first_bad = int(batch.first_bad[0])
    if first_bad >= 0:
        raise IntegrityError(f"input token id {int(ids[first_bad])} out of range for vocabulary "
                             f"of size {full_vocab_size}")
    return batch.plan(0)


def remap_out(plan: SelectionPlan, local_id: int) -> int:
    """remap_out (selector.cpp:50-56)."""
    if local_id < 0 or local_id >= plan.size():
        raise IntegrityError(
            f"local row {local_id} out of range for a plan of {plan.size()} rows")
    return int(plan.active_ids[local_id])


def union_plans(plans: Sequence[SelectionPlan]) -> SelectionPlan:
    """union_plans (selector.cpp:58-77), the union computed on the GPU."""
    if not plans:
        raise ConfigError("cannot union an empty batch of plans")
    full, ns = plans[0].full_vocab_size, plans[0].n_static
    for p in plans:
        if p.full_vocab_size != full or p.n_static != ns:
            raise IntegrityError("plans in one micro-batch must share the static vocabulary and "
                                 "full vocabulary size")
    _require_cuda()
    ids = np.concatenate([np.asarray(p.active_ids, np.uint32) for p in plans])
    off = np.zeros(len(plans) + 1, np.int64)
    off[1:] = np.cumsum([p.size() for p in plans])
    d_ids, d_off = _dev(ids, torch.int32), _dev(off, torch.int64)
    words = torch.zeros(max(1, (full + 63) // 64), dtype=torch.int64, device="cuda")
    out = torch.empty(max(1, full), dtype=torch.int32, device="cuda")
    n_out = torch.zeros(1, dtype=torch.int64, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    call("svt_union_plans", d_ids.data_ptr(), d_off.data_ptr(), len(plans), full,
         words.data_ptr(), out.data_ptr(), n_out.data_ptr(), bad.data_ptr(), _stream())
    if int(bad.item()):
        raise IntegrityError("plan id out of range for the full vocabulary")
    n = int(n_out.item())
    act = out[:n].cpu().numpy().view(np.uint32).copy()
    return SelectionPlan(act, ns, n - ns, full)  # n - ns as in selector.cpp:73


# --------------------------------------------------------------------------
# HeadMatrix (head.hpp:17-45): device resident; storage f32 / f16 / bf16
# --------------------------------------------------------------------------
class HeadMatrix:
    """LM-head weights [rows x dim] in HBM. ``dtype_bytes`` keeps the
    reference's accounting tag (2 or 4); ``storage`` is the device element
    type (SVT_F32, SVT_F16 — the reference's 2-byte type — or SVT_BF16)."""

    def __init__(self, rows: int = 0, dim: int = 0, dtype_bytes: int = 4,
                 storage: Optional[int] = None, data: Optional[torch.Tensor] = None):
        if dtype_bytes not in (2, 4):
            raise ConfigError(f"dtype_bytes must be 2 or 4; got {dtype_bytes}")
        self.dtype_bytes = dtype_bytes
        self.storage = storage if storage is not None else (SVT_F32 if dtype_bytes == 4 else SVT_F16)
        if data is None:
            _require_cuda()
            data = torch.zeros((rows, dim), dtype=_TORCH[self.storage], device="cuda")
        self.data = data

    @staticmethod
    def random(rows: int, dim: int, seed: int, dtype_bytes: int = 4,
               storage: Optional[int] = None, round_through: Optional[int] = None,
               stream=None) -> "HeadMatrix":
        """HeadMatrix::random (head.cpp:89-107) regenerated on the device.
        dtype_bytes==2 quantizes through binary16 as the reference does;
        storage/round_through SVT_BF16 gives the bf16 configs' weights."""
        if dtype_bytes not in (2, 4):
            raise ConfigError(f"dtype_bytes must be 2 or 4; got {dtype_bytes}")
        st = storage if storage is not None else (SVT_F32 if dtype_bytes == 4 else SVT_F16)
        rt = round_through if round_through is not None else (
            SVT_F16 if dtype_bytes == 2 else (SVT_BF16 if st == SVT_BF16 else SVT_F32))
        m = HeadMatrix(rows, dim, dtype_bytes, st)
        call("svt_head_random", m.data.data_ptr(), st, rt, 0, rows * dim, seed & (2**64 - 1),
             _stream(stream))
        return m

    @staticmethod
    def from_host(values, dtype_bytes: int = 4, storage: Optional[int] = None) -> "HeadMatrix":
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float32))
        if v.ndim == 1:
            v = v.reshape(-1, 1) if v.size else v.reshape(0, 0)
        m = HeadMatrix(v.shape[0], v.shape[1], dtype_bytes, storage)
        if v.size:
            f = torch.from_numpy(v).cuda()
            call("svt_convert_from_f32", f.data_ptr(), m.data.data_ptr(), m.storage, v.size,
                 _stream())
        return m

    def rows(self) -> int:
        return int(self.data.shape[0])

    def dim(self) -> int:
        return int(self.data.shape[1])

    def to_host(self) -> np.ndarray:
        if self.data.numel() == 0:
            return np.zeros(tuple(self.data.shape), np.float32)
        out = torch.empty(tuple(self.data.shape), dtype=torch.float32, device="cuda")
        call("svt_convert_to_f32", self.data.data_ptr(), self.storage, out.data_ptr(),
             self.data.numel(), _stream())
        return out.cpu().numpy()


def gather(head: HeadMatrix, plan: SelectionPlan) -> HeadMatrix:
    """gather (head.cpp:176-187): row-major sub-head of the plan's rows."""
    ids = np.asarray(plan.active_ids, np.uint32)
    if ids.size and int(ids[-1]) >= head.rows():
        raise IntegrityError(f"plan selects row {int(ids[-1])} but the head has only "
                             f"{head.rows()} rows")
    sub = HeadMatrix(ids.size, head.dim(), head.dtype_bytes, head.storage)
    if ids.size and head.dim():
        d_ids = _dev(ids.view(np.int32), torch.int32)
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        call("svt_gather_rows", head.data.data_ptr(), head.storage, head.rows(), head.dim(),
             d_ids.data_ptr(), ids.size, sub.data.data_ptr(), bad.data_ptr(), _stream())
        if int(bad.item()):
            raise IntegrityError("plan selects a row beyond the head")
    return sub


def _hidden_dev(hidden, dim: int) -> torch.Tensor:
    if isinstance(hidden, torch.Tensor):
        h = hidden.detach().to(device="cuda", dtype=torch.float32).reshape(-1).contiguous()
    else:
        h = torch.from_numpy(np.ascontiguousarray(np.asarray(hidden, np.float32).reshape(-1))).cuda()
    if h.numel() != dim:
        raise IntegrityError(f"hidden state dimension {h.numel()} does not match head "
                             f"dimension {dim}")
    return h if h.numel() else torch.zeros(4, device="cuda")


def logits(head: HeadMatrix, hidden) -> np.ndarray:
    """logits (head.cpp:189-201), bit-exact ascending-column order."""
    h = _hidden_dev(hidden, head.dim())
    out = torch.empty(max(head.rows(), 1), dtype=torch.float32, device="cuda")
    if head.rows():
        call("svt_logits", head.data.data_ptr(), head.storage, head.rows(), head.dim(),
             h.data_ptr(), out.data_ptr(), _stream())
    return out[: head.rows()].cpu().numpy()


_WS_CACHE: dict = {}


def _workspace(batch: int, groups: int) -> torch.Tensor:
    dev = torch.cuda.current_device()
    key = (dev, batch, groups)
    ws = _WS_CACHE.get(key)
    if ws is None:
        ws = torch.empty(max(1, _lib.lib.svt_greedy_workspace_bytes(batch, groups)),
                         dtype=torch.uint8, device="cuda")
        _WS_CACHE[key] = ws
    return ws


def greedy_step(subhead: HeadMatrix, hidden, plan: SelectionPlan) -> int:
    """greedy_step (head.cpp:203-217): fused logits + first-max argmax + remap."""
    if subhead.rows() == 0:
        raise IntegrityError("greedy step over an empty sub-head")
    if subhead.rows() != plan.size():
        raise IntegrityError(f"sub-head has {subhead.rows()} rows but the plan names "
                             f"{plan.size()}")
    h = _hidden_dev(hidden, subhead.dim())
    ids = _dev(np.asarray(plan.active_ids, np.uint32).view(np.int32), torch.int32)
    out = torch.empty(2, dtype=torch.int32, device="cuda")
    mx = torch.empty(2, dtype=torch.float32, device="cuda")
    call("svt_greedy_step", subhead.data.data_ptr(), subhead.storage, subhead.rows(),
         subhead.dim(), h.data_ptr(), ids.data_ptr(), out.data_ptr(), mx.data_ptr(),
         _workspace(1, (subhead.rows() + 31) // 32).data_ptr(), _stream())
    return int(out[0].item()) & 0xFFFFFFFF



# --------------------------------------------------------------------------
# (f1) plan wire format (artifacts.cpp:169-192)
# --------------------------------------------------------------------------
def plan_to_json(plan: SelectionPlan, indent: Optional[int] = None) -> str:
    """artifacts::to_json(plan).dump(indent): nlohmann's text, byte for byte
    (indent None = compact, the CLI's plans file line)."""
    ids = np.ascontiguousarray(plan.active_ids, np.uint32)
    need = C.c_size_t()
    args = (ids.ctypes.data if ids.size else None, ids.size, plan.n_static, plan.n_dynamic,
            plan.full_vocab_size, -1 if indent is None else int(indent))
    call("svt_plan_to_json", *args, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    call("svt_plan_to_json", *args, buf, need.value, None)
    return buf.value.decode()


def plan_from_json(text: str, origin: str = "<mem>") -> SelectionPlan:
    """artifacts::plan_from_json: ParseError on malformed JSON / a missing
    field, IntegrityError on unsorted or out-of-range ids."""
    raw = text.encode()
    n, ns, nd, full = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
    call("svt_plan_from_json", raw, len(raw), origin.encode(), None, 0, C.byref(n), None, None,
         None)
    ids = np.zeros(max(1, n.value), np.uint32)
    call("svt_plan_from_json", raw, len(raw), origin.encode(), ids.ctypes.data, ids.size,
         C.byref(n), C.byref(ns), C.byref(nd), C.byref(full))
    return SelectionPlan(ids[: n.value].copy(), ns.value, nd.value, full.value)

class SplitDecoder:
    """Batched greedy decode over a select()-built batch with the static rows
    shared (svt_decode_split_plans + svt_greedy_split).

    Each plan is T ∪ D_b; the static rows T are gathered once into one
    lane-interleaved block and scored for every request from it (exact
    reference-order chains), only D_b \\ T is gathered per request and
    streamed by the exact-order GEMV, and the two halves meet in a (value,
    id) combine. Ids are those of ``TailoredBatch.greedy`` over the full
    plans. :meth:`prepare` re-splits and re-gathers after ``tb.run_select()``.
    """

    def __init__(self, tb: "TailoredBatch", head: HeadMatrix, stream=None):
        words = getattr(tb, "_words", None)
        if words is None:
            raise ConfigError("the split decoder needs a batch built by select over a static set")
        self.tb, self.head, self.stream = tb, head, stream
        B, V, d = tb.B, tb.V, head.dim()
        w = words.cpu().numpy().view(np.uint64)
        bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:V]
        st = np.flatnonzero(bits).astype(np.uint32)
        if st.size == 0:
            raise ConfigError("the split decoder needs a non-empty static set")
        self.nT = int(st.size)
        dev = "cuda"
        self.st_ids = torch.from_numpy(st.view(np.int32)).to(dev)
        # the static block: T as one plan, lane-interleaved
        self.st_groups = (self.nT + 31) // 32
        self.st_gb = torch.zeros(2, dtype=torch.int64, device=dev)
        self.st_gm = torch.zeros((self.st_groups, 8), dtype=torch.int32, device=dev)
        n_st = torch.tensor([self.nT], dtype=torch.int64, device=dev)
        off0 = torch.zeros(2, dtype=torch.int64, device=dev)
        call("svt_plan_layout", n_st.data_ptr(), off0.data_ptr(), 1, self.st_gb.data_ptr(),
             self.st_gm.data_ptr(), self.st_groups, _stream(stream))
        self.st_sub = torch.empty(
            max(16, _lib.lib.svt_subhead_bytes(head.storage, d, self.st_groups)),
            dtype=torch.uint8, device=dev)
        self.bad = torch.zeros(1, dtype=torch.int32, device=dev)
        call("svt_gather_interleaved", head.data.data_ptr(), head.storage, head.rows(), d,
             self.st_ids.data_ptr(), self.st_gb.data_ptr(), self.st_gm.data_ptr(), 1,
             self.st_groups, self.st_sub.data_ptr(), self.bad.data_ptr(), _stream(stream))
        # the dynamic halves (capacity layout of the batch's plans)
        self.dyn_ids = torch.empty_like(tb.active)
        self.meta = torch.zeros((2, max(B, 1)), dtype=torch.int64, device=dev)
        self.n_dyn, self.st_valid = self.meta
        self.first_ids = torch.zeros(max(B, 1), dtype=torch.int32, device=dev)
        self.dyn_starts = torch.zeros(max(B, 1), dtype=torch.uint8, device=dev)
        # dynamic rows per request <= its plan capacity (any plan missing part
        # of T keeps every row dynamic); when that capacity's sub-heads would
        # be huge, size for select-built plans (T inside every plan: at most
        # capacity - |T| dynamic rows) and check the static-valid flags
        self.max_groups = tb.max_groups
        self._strict = False
        if _lib.lib.svt_subhead_bytes(head.storage, d, self.max_groups) > (4 << 30):
            caps = np.diff(tb.act_off_h)
            self.max_groups = max(1, int(sum((max(0, int(c) - self.nT) + 31) // 32
                                              for c in caps)))
            self._strict = True
        self.gb = torch.zeros(B + 1, dtype=torch.int64, device=dev)
        self.gm = torch.zeros((max(1, self.max_groups), 8), dtype=torch.int32, device=dev)
        self.sub = torch.empty(
            max(16, _lib.lib.svt_subhead_bytes(head.storage, d, self.max_groups)),
            dtype=torch.uint8, device=dev)
        self.ws = torch.zeros(max(1, _lib.lib.svt_greedy_split_workspace_bytes(
            B, self.max_groups, self.nT, d)), dtype=torch.uint8, device=dev)
        self._stable = False
        self.prepare()

    def prepare(self):
        """Split the batch's current plans and gather their dynamic rows."""
        tb, head, st = self.tb, self.head, _stream(self.stream)
        call("svt_decode_split_plans", tb.active.data_ptr(), tb.act_off.data_ptr(),
             tb.n_active.data_ptr(), tb.B, tb._words.data_ptr(), tb.V, self.st_ids.data_ptr(),
             self.nT, self.dyn_ids.data_ptr(), self.n_dyn.data_ptr(), self.st_valid.data_ptr(),
             self.first_ids.data_ptr(), self.dyn_starts.data_ptr(), st)
        if (self._strict and not torch.cuda.is_current_stream_capturing()
                and self._flags_missing_static(st)):
            raise IntegrityError("split decode sized for select-built plans: a plan is missing "
                                 "static rows")
        call("svt_plan_layout", self.n_dyn.data_ptr(), tb.act_off.data_ptr(), tb.B,
             self.gb.data_ptr(), self.gm.data_ptr(), self.max_groups, st)
        call("svt_gather_interleaved", head.data.data_ptr(), head.storage, head.rows(),
             head.dim(), self.dyn_ids.data_ptr(), self.gb.data_ptr(), self.gm.data_ptr(), tb.B,
             self.max_groups, self.sub.data_ptr(), self.bad.data_ptr(), st)
        self._stable = False
        return self

    def _flags_missing_static(self, st) -> bool:
        # (host check of the split's static-valid flags, on the split's stream)
        _lib.lib.svt_stream_synchronize(st)
        return bool((self.st_valid[: self.tb.B] == 0).any())

    def greedy(self, hidden: torch.Tensor, out_ids: torch.Tensor,
               out_max: Optional[torch.Tensor] = None) -> torch.Tensor:
        """hidden: [B, ld] float32 on the device (ld % 4 == 0, ld >= dim)."""
        flags = SVT_WEIGHTS_STABLE if self._stable else 0
        self._stable = True
        h = self.head
        call("svt_greedy_split", self.st_sub.data_ptr(), h.storage, self.nT, h.dim(),
             self.st_ids.data_ptr(), self.st_valid.data_ptr(), self.first_ids.data_ptr(),
             self.sub.data_ptr(), self.gb.data_ptr(), self.gm.data_ptr(), self.dyn_ids.data_ptr(),
             self.n_dyn.data_ptr(), self.dyn_starts.data_ptr(), self.tb.B, self.max_groups,
             hidden.data_ptr(), hidden.stride(0), flags, out_ids.data_ptr(), _ptr(out_max),
             self.ws.data_ptr(), _stream(self.stream))
        return out_ids

    def stats(self):
        """Certified static half (bf16 heads): (requests whose static
        maximum had one candidate, requests that needed more exact chains),
        accumulated since the decoder was built; (0, 0) on the exact path."""
        w = self.ws[-256:-248].view(torch.int32).cpu().tolist()
        return w[0], w[1]

    def algorithmic_decode_bytes(self, esize: int, dim: int) -> int:
        """Bytes one split decode step must move from HBM: the static block
        once, each request's dynamic rows, the hidden states and the outputs."""
        nd = self.n_dyn.cpu().numpy()
        return (self.nT + int(nd.sum())) * dim * esize + self.tb.B * (dim * 4 + 8)


class RowDecoder:
    """Batch-1 greedy decode over ONE plan (BASELINE cfg1): the plan's rows
    are gathered row-major once (gather, head.cpp:176-187) and every token is
    one svt_greedy_certified_rows launch — a split-K pass at HBM speed with
    rigorous bounds, exact reference-order recompute of the rows that can
    still win. Ids equal greedy_step (head.cpp:203-217) + remap_out.

    ``materialize=False`` streams the rows straight from the head through the
    plan ids (fused gather) instead of a gathered sub-head."""

    def __init__(self, head: HeadMatrix, plan_ids: torch.Tensor, n_rows: int,
                 materialize: bool = True, stream=None, row_base: int = 0,
                 plan_start: int = 1, remap: bool = True):
        if n_rows <= 0:
            raise IntegrityError("greedy step over an empty sub-head")
        self.head, self.n, self.stream = head, int(n_rows), stream
        self.ids = plan_ids
        self.ws = torch.zeros(_lib.lib.svt_greedy_rows_workspace_bytes(self.n),
                              dtype=torch.uint8, device="cuda")
        esize = 4 if head.storage == SVT_F32 else 2
        if materialize:
            self.sub = torch.empty(self.n * head.dim() * esize + 16, dtype=torch.uint8,
                                   device="cuda")
            self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")
            self.gather()
            src, src_ids, rows = self.sub.data_ptr(), None, self.n
        else:
            self.sub = None
            src, src_ids, rows = head.data.data_ptr(), plan_ids.data_ptr(), head.rows()
        self._fn = _lib.lib.svt_greedy_certified_rows
        self._pre = (src, head.storage, rows, head.dim(), src_ids, self.n)
        self._post = ((plan_ids.data_ptr() if remap else None), row_base, plan_start)
        # the first step after a (re)gather must not prefetch rows before the
        # dependency wait; later steps may (SVT_ROWS_WEIGHTS_STABLE)
        self._stable = 0

    def gather(self):
        """(Re)materialise the row-major sub-head (svt_gather_rows)."""
        self._stable = 0
        h = self.head
        call("svt_gather_rows", h.data.data_ptr(), h.storage, h.rows(), h.dim(),
             self.ids.data_ptr(), self.n, self.sub.data_ptr(), self.bad.data_ptr(),
             _stream(self.stream))
        return self

    def greedy(self, hidden: torch.Tensor, out_id: torch.Tensor,
               out_max: Optional[torch.Tensor] = None,
               out_record: Optional[torch.Tensor] = None,
               hidden_stable: bool = False) -> torch.Tensor:
        """hidden: f32 [dim] on the device (16-byte aligned); out_id: one
        int32; out_max (optional): the exact reference logit of the winner;
        out_record (optional, 4 int32): the vocab-shard record for
        svt_shard_combine. hidden_stable: ``hidden`` was not written by the
        kernel queued right before this call (SVT_ROWS_HIDDEN_STABLE: the
        step then overlaps the previous one on every SM)."""
        flags = self._stable | (SVT_ROWS_HIDDEN_STABLE if hidden_stable else 0)
        st = self._fn(*self._pre, hidden.data_ptr(), *self._post, flags,
                      out_id.data_ptr(), _ptr(out_max), _ptr(out_record), self.ws.data_ptr(),
                      _stream(self.stream))
        _lib.check(st, "svt_greedy_certified_rows")
        self._stable = 1
        return out_id

    def stats(self):
        """(tokens certified directly, tokens with an exact recompute)."""
        w = self.ws[:32].view(torch.int32).cpu().tolist()
        return w[4], w[5]


# --------------------------------------------------------------------------
# accounting / offload model (head.cpp:219-237, offload_sim.cpp:44-87)
# --------------------------------------------------------------------------
class _MemRep(C.Structure):
    _fields_ = [("full_head_bytes", C.c_uint64), ("sub_head_bytes", C.c_uint64),
                ("embedding_bytes_gpu", C.c_uint64), ("embedding_bytes_host", C.c_uint64),
                ("saved_fraction", C.c_double)]


class _Timeline(C.Structure):
    _fields_ = [("transfer_time", C.c_double), ("prefill_time", C.c_double),
                ("embedding_time", C.c_double), ("exposed_latency", C.c_double),
                ("hidden", C.c_int32)]


@dataclass
class MemoryReport:
    full_head_bytes: int
    sub_head_bytes: int
    embedding_bytes_gpu: int
    embedding_bytes_host: int
    saved_fraction: float


@dataclass
class OverlapTimeline:
    transfer_time: float
    prefill_time: float
    embedding_time: float
    exposed_latency: float
    hidden: bool


def memory_report(full_size, dim, dtype_bytes, plan_size) -> MemoryReport:
    r = _MemRep()
    call("svt_memory_report", full_size, dim, dtype_bytes, plan_size, C.addressof(r))
    return MemoryReport(r.full_head_bytes, r.sub_head_bytes, r.embedding_bytes_gpu,
                        r.embedding_bytes_host, r.saved_fraction)


def simulate(hw, plan_size, dim, dtype_bytes, prompt_len, flops_per_token) -> OverlapTimeline:
    """hw = (link_bandwidth, device_flops, host_lookup_latency)."""
    t = _Timeline()
    call("svt_simulate", hw[0], hw[1], hw[2], plan_size, dim, dtype_bytes, prompt_len,
         flops_per_token, C.addressof(t))
    return OverlapTimeline(t.transfer_time, t.prefill_time, t.embedding_time,
                           t.exposed_latency, bool(t.hidden))


def breakeven_rows(hw, dim, dtype_bytes, prompt_len, flops_per_token) -> int:
    r = C.c_size_t()
    call("svt_breakeven_rows", hw[0], hw[1], hw[2], dim, dtype_bytes, prompt_len,
         flops_per_token, C.addressof(r))
    return int(r.value)


ILLUSTRATIVE_HW = (16.0e9, 4.0e12, 50e-9)  # offload_sim.cpp:11-17


# --------------------------------------------------------------------------
# Batched device engine: one plan per request, no host sync per step
# --------------------------------------------------------------------------
class TailoredBatch:
    """A micro-batch of requests, each with its own plan S_b = T ∪ prompt_b.

    Device state: plan ids in capacity-CSR order (request b at act_off[b],
    capacity |T| + len_b), per-request counters, the row-group layout and
    (after :meth:`gather`) the lane-interleaved sub-heads.
    """

    def __init__(self, V: int, B: int, caps: np.ndarray, stream=None):
        self.V, self.B = V, B
        self.stream = stream
        self.act_off_h = np.zeros(B + 1, np.int64)
        self.act_off_h[1:] = np.cumsum(caps)
        self.max_groups = int(sum((int(c) + 31) // 32 for c in caps))
        dev = "cuda"
        self.active = torch.empty(max(1, int(self.act_off_h[-1])), dtype=torch.int32, device=dev)
        self.act_off = torch.from_numpy(self.act_off_h).to(dev)
        self.meta = torch.zeros((4, max(B, 1)), dtype=torch.int64, device=dev)
        self.n_active, self.n_static, self.n_dynamic, self.first_bad_d = self.meta
        self.group_begin = torch.zeros(B + 1, dtype=torch.int64, device=dev)
        # one 32-byte GroupMeta record per 32-row group (svt_plan_layout)
        self.group_meta = torch.zeros((max(1, self.max_groups), 8), dtype=torch.int32, device=dev)
        self.sub: Optional[torch.Tensor] = None
        self.head: Optional[HeadMatrix] = None
        self.ws = torch.empty(max(1, _lib.lib.svt_greedy_workspace_bytes(B, self.max_groups)),
                              dtype=torch.uint8, device=dev)
        self._first_bad_h: Optional[np.ndarray] = None

    # ---- (a) select + layout -------------------------------------------
    @classmethod
    def build(cls, static_words_dev: torch.Tensor, n_static: int, V: int,
              prompts_dev: torch.Tensor, prompt_off_h: np.ndarray, stream=None) -> "TailoredBatch":
        B = len(prompt_off_h) - 1
        caps = n_static + np.diff(prompt_off_h)
        tb = cls(V, B, caps, stream)
        tb._prompt_off = torch.from_numpy(np.ascontiguousarray(prompt_off_h, np.int64)).cuda()
        tb._prompts = prompts_dev
        tb._words = static_words_dev
        tb.run_select()
        return tb

    @classmethod
    def from_plans(cls, V: int, plans, stream=None) -> "TailoredBatch":
        """A batch over explicit plans (strictly increasing id arrays, e.g.
        produced elsewhere or loaded from plan files) — no select; the plan
        counters report every row as dynamic."""
        B = len(plans)
        caps = np.array([len(q) for q in plans], np.int64)
        tb = cls(V, B, caps, stream)
        if B and int(caps.sum()):
            flat = np.concatenate([np.asarray(q, np.uint32) for q in plans])
            if int(flat.max()) >= V:
                raise IntegrityError(f"plan id {int(flat.max())} out of range for vocabulary "
                                     f"size {V}")
            tb.active[: flat.size].copy_(torch.from_numpy(flat.view(np.int32)))
        if B:
            n = torch.from_numpy(caps).cuda()
            tb.n_active.copy_(n)
            tb.n_dynamic.copy_(n)
            tb.n_static.zero_()
            tb.first_bad_d.fill_(-1)
        call("svt_plan_layout", tb.n_active.data_ptr(), tb.act_off.data_ptr(), B,
             tb.group_begin.data_ptr(), tb.group_meta.data_ptr(), tb.max_groups,
             _stream(stream))
        tb._stable = False
        return tb

    def attach(self, head: HeadMatrix):
        """Use ``head`` for the fused (no sub-head) decode without gathering."""
        self.head = head
        self._fast = None
        self._stable = False
        return self

    def run_select(self, layout: bool = True):
        """select (a) for every request; ``layout=False`` skips the row-group
        layout the interleaved paths use (row-major / batch-1 decoders)."""
        self._stable = False
        call("svt_select_batched", self._words.data_ptr(), self.V, self.V,
             self._prompts.data_ptr(), self._prompt_off.data_ptr(), self.B,
             self.active.data_ptr(), self.act_off.data_ptr(), self.n_active.data_ptr(),
             self.n_static.data_ptr(), self.n_dynamic.data_ptr(), self.first_bad_d.data_ptr(),
             _stream(self.stream))
        if not layout:
            self._first_bad_h = None
            return
        call("svt_plan_layout", self.n_active.data_ptr(), self.act_off.data_ptr(), self.B,
             self.group_begin.data_ptr(), self.group_meta.data_ptr(), self.max_groups,
             _stream(self.stream))
        self._first_bad_h = None

    @classmethod
    def select_only(cls, static_words: np.ndarray, V: int, prompts) -> "TailoredBatch":
        words = np.ascontiguousarray(static_words, np.uint64)
        n_static = int(sum(bin(int(w)).count("1") for w in words))
        off = np.zeros(len(prompts) + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in prompts])
        flat = (np.concatenate([np.asarray(p, np.uint32) for p in prompts])
                if len(prompts) else np.zeros(0, np.uint32))
        return cls.build(_dev(words.view(np.int64), torch.int64), n_static, V,
                         _dev(flat.view(np.int32), torch.int32), off)

    @property
    def first_bad(self) -> np.ndarray:
        if self._first_bad_h is None:
            self._first_bad_h = self.first_bad_d.cpu().numpy()
        return self._first_bad_h

    def plan(self, b: int) -> SelectionPlan:
        meta = self.meta[:, b].cpu().numpy()
        n = int(meta[0])
        o = int(self.act_off_h[b])
        ids = self.active[o:o + n].cpu().numpy().view(np.uint32).copy()
        return SelectionPlan(ids, int(meta[1]), int(meta[2]), self.V)

    def plans(self):
        return [self.plan(b) for b in range(self.B)]

    def plans_jsonl(self) -> str:
        """The batch's device-selected plans as the CLI's plans file: one
        compact JSON object per line (subvocab.cpp:413), one D2H copy."""
        meta = self.meta.cpu().numpy()
        ids = self.active.cpu().numpy().view(np.uint32)
        off = np.ascontiguousarray(self.act_off_h[:-1] if self.B else np.zeros(1, np.int64))
        na, ns, nd = (np.ascontiguousarray(meta[i]) for i in range(3))
        need = C.c_size_t()
        args = (ids.ctypes.data, off.ctypes.data, na.ctypes.data, ns.ctypes.data,
                nd.ctypes.data, self.B, self.V)
        call("svt_plans_to_jsonl", *args, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        call("svt_plans_to_jsonl", *args, buf, need.value, None)
        return buf.value.decode()

    # ---- (b) interleaved gather ------------------------------------------
    def gather(self, head: HeadMatrix):
        if self.head is not head or self.sub is None:
            self.head = head
            nbytes = _lib.lib.svt_subhead_bytes(head.storage, head.dim(), self.max_groups)
            if self.sub is None or self.sub.numel() < nbytes:
                self.sub = torch.empty(max(16, nbytes), dtype=torch.uint8, device="cuda")
            # sticky error flag: set by the kernel when a plan id is >= rows
            self.gather_bad = torch.zeros(1, dtype=torch.int32, device="cuda")
            self._fast = None
        self._stable = False
        call("svt_gather_interleaved", head.data.data_ptr(), head.storage, head.rows(),
             head.dim(), self.active.data_ptr(), self.group_begin.data_ptr(),
             self.group_meta.data_ptr(), self.B, self.max_groups, self.sub.data_ptr(),
             self.gather_bad.data_ptr(), _stream(self.stream))
        return self

    def _fast_args(self):
        """Pointer tuples for the per-step decode call, resolved once so the
        host side of a decode step is a single ctypes call."""
        if getattr(self, "_fast", None) is None:
            h = self.head
            common = (self.group_begin.data_ptr(), self.group_meta.data_ptr(),
                      self.active.data_ptr(), self.B, self.max_groups)
            self._fast = {
                False: (_lib.lib.svt_greedy_interleaved,
                        ((self.sub.data_ptr() if self.sub is not None else None), h.storage,
                         h.dim()) + common),
                True: (_lib.lib.svt_greedy_fused,
                       (h.data.data_ptr(), h.storage, h.rows(), h.dim()) + common),
            }
        return self._fast

    # ---- (c)+(d) fused greedy ----------------------------------------------
    def greedy(self, hidden: torch.Tensor, out_ids: torch.Tensor,
               out_max: Optional[torch.Tensor] = None, fused: bool = False,
               out_keys: Optional[torch.Tensor] = None, row_base: int = 0,
               plan_start: int = 1) -> torch.Tensor:
        """hidden: [B, ld] float32 on the device (ld % 4 == 0, ld >= dim)."""
        # SVT_WEIGHTS_STABLE from the second step after a select / gather on:
        # the sub-heads and group records are then not written by the kernel
        # the step depends on, so its first weight stages stream early
        flags = SVT_WEIGHTS_STABLE if getattr(self, "_stable", False) else 0
        self._stable = True
        if out_max is None and out_keys is None and row_base == 0 and plan_start == 1 and (
                fused or self.sub is not None):
            fn, pre = self._fast_args()[bool(fused)]
            st = fn(*pre, hidden.data_ptr(), hidden.stride(0), 0, 1, flags, out_ids.data_ptr(),
                    None, None, self.ws.data_ptr(), _stream(self.stream))
            _lib.check(st, "greedy")
            return out_ids
        head = self.head
        if fused:
            call("svt_greedy_fused", head.data.data_ptr(), head.storage, head.rows(), head.dim(),
                 self.group_begin.data_ptr(), self.group_meta.data_ptr(), self.active.data_ptr(),
                 self.B, self.max_groups, hidden.data_ptr(), hidden.stride(0), row_base,
                 plan_start, flags, out_ids.data_ptr(), _ptr(out_max), _ptr(out_keys),
                 self.ws.data_ptr(), _stream(self.stream))
        else:
            call("svt_greedy_interleaved", self.sub.data_ptr(), head.storage, head.dim(),
                 self.group_begin.data_ptr(), self.group_meta.data_ptr(), self.active.data_ptr(),
                 self.B, self.max_groups, hidden.data_ptr(), hidden.stride(0), row_base,
                 plan_start, flags, out_ids.data_ptr(), _ptr(out_max), _ptr(out_keys),
                 self.ws.data_ptr(), _stream(self.stream))
        return out_ids

    def greedy_certified(self, hidden: torch.Tensor, out_ids: torch.Tensor,
                         out_max: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Same ids as greedy(): split-K fast pass + error bounds + exact
        recompute of the candidate rows only (svt_greedy_certified)."""
        if getattr(self, "cws", None) is None:
            self.cws = torch.zeros(
                max(1, _lib.lib.svt_certified_workspace_bytes(self.B, self.max_groups)),
                dtype=torch.uint8, device="cuda")
        head = self.head
        call("svt_greedy_certified", self.sub.data_ptr(), head.storage, head.dim(),
             self.group_begin.data_ptr(), self.group_meta.data_ptr(), self.active.data_ptr(),
             self.B, self.max_groups, hidden.data_ptr(), hidden.stride(0), out_ids.data_ptr(),
             _ptr(out_max), self.cws.data_ptr(), _stream(self.stream))
        return out_ids

    def certified_stats(self):
        """(steps certified without recompute, steps that recomputed)."""
        if getattr(self, "cws", None) is None:
            return 0, 0
        st = self.cws[-256:].view(torch.int32)[:2].cpu().tolist()
        return st[0], st[1]

    def logits(self, hidden: torch.Tensor, fused: bool = False) -> torch.Tensor:
        """Per-request logits, CSR by plan size (offsets = capacity CSR)."""
        head = self.head
        out = torch.empty(max(1, int(self.act_off_h[-1])), dtype=torch.float32, device="cuda")
        if fused:
            call("svt_logits_rows", head.data.data_ptr(), head.storage, head.rows(), head.dim(),
                 self.group_begin.data_ptr(), self.group_meta.data_ptr(), self.active.data_ptr(),
                 self.B, self.max_groups, hidden.data_ptr(), hidden.stride(0), out.data_ptr(),
                 self.act_off.data_ptr(), _stream(self.stream))
        else:
            call("svt_logits_interleaved", self.sub.data_ptr(), head.storage, head.dim(),
                 self.group_begin.data_ptr(), self.group_meta.data_ptr(), self.B,
                 self.max_groups, hidden.data_ptr(), hidden.stride(0), out.data_ptr(),
                 self.act_off.data_ptr(), _stream(self.stream))
        return out

    def topk(self, hidden: torch.Tensor, k: int, fused: bool = False):
        """Top-k per request (svt_topk_logits over the exact logits): ids
        [B, k] (global, remapped through the plans) and values [B, k], value
        descending, ties to the lower id; entry 0 == greedy()'s id."""
        lg = self.logits(hidden, fused=fused)
        ids = torch.empty((self.B, k), dtype=torch.int32, device="cuda")
        vals = torch.empty((self.B, k), dtype=torch.float32, device="cuda")
        call("svt_topk_logits", lg.data_ptr(), self.act_off.data_ptr(), self.n_active.data_ptr(),
             self.active.data_ptr(), self.act_off.data_ptr(), self.B, k, 1, ids.data_ptr(),
             vals.data_ptr(), _stream(self.stream))
        return ids, vals

    def stats(self):
        """Certified static half (bf16 heads): (requests whose static
        maximum had one candidate, requests that needed more exact chains),
        accumulated since the decoder was built; (0, 0) on the exact path."""
        w = self.ws[-256:-248].view(torch.int32).cpu().tolist()
        return w[0], w[1]

    def algorithmic_decode_bytes(self, esize: int, dim: int) -> int:
        """Bytes one decode step must move: Σ_b |S_b|·d·b_W
        + d·4 (hidden) + 8 (id + max out)."""
        n = self.n_active.cpu().numpy()
        return int(n.sum()) * dim * esize + self.B * (dim * 4 + 8)
