"""Batched prefill-scoring over per-sequence tailored heads (BASELINE cfg3)
on the tcgen05 tensor cores, with certified reference-exact ids
(svt_prefill_score)."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import call
from .tailored_head import HeadMatrix, SVT_BF16, _stream


class PrefillScorer:
    """Plans (one per sequence) + their gathered row-major bf16 sub-heads.

    Two ways in:
      * ``PrefillScorer(head, plan_ids, id_offsets, positions)``: concatenated
        plan ids (device u32 / int32 view) and host id_offsets [S+1];
      * ``PrefillScorer.from_batch(head, tb, positions)``: the capacity-CSR
        plans a :class:`TailoredBatch` selected on the device (no host sync);
        :meth:`regather` refreshes the sub-heads after ``tb.run_select()``.
    positions must be a multiple of 128 and d of 64."""

    def __init__(self, head: HeadMatrix, plan_ids: torch.Tensor, id_offsets: np.ndarray,
                 positions: int, stream=None, fused: bool = False):
        n_rows = np.diff(id_offsets).astype(np.int64)
        self.fused = fused
        self.split = False
        self._setup(head, positions, len(id_offsets) - 1, 0 if fused else int(n_rows.sum()),
                    stream)
        self.n_rows = torch.from_numpy(n_rows).cuda()
        self.row_off = torch.from_numpy(np.ascontiguousarray(id_offsets[:-1], np.int64)).cuda()
        self.id_off = self.row_off
        self.plan_ids = plan_ids
        if fused:
            return
        call("svt_gather_rows", head.data.data_ptr(), head.storage, head.rows(), self.d,
             plan_ids.data_ptr(), self.total, self.sub.data_ptr(), self.bad.data_ptr(),
             _stream(stream))

    @classmethod
    def from_batch(cls, head: HeadMatrix, tb, positions: int, stream=None,
                   fused: bool = False, split: bool = False) -> "PrefillScorer":
        """fused=True: no sub-heads; the GEMM gathers the plan rows from the
        head itself (svt_prefill_score_fused, TMA tile::gather4).
        split=True (a batch built by select over a static set): the static
        rows are gathered once and shared by every sequence, only each
        plan's dynamic rows are gathered (svt_prefill_score_split)."""
        if fused and split:
            raise _lib.ConfigError("the fused and split scorers are exclusive")
        self = cls.__new__(cls)
        self.fused = fused
        self.split = False
        self._setup(head, positions, tb.B, 0 if fused else int(tb.act_off_h[-1]), stream)
        self.n_rows = tb.n_active            # device int64 [S]
        self.row_off = tb.act_off            # device int64 [S+1] (capacity offsets)
        self.id_off = tb.act_off
        self.plan_ids = tb.active
        self._tb = tb
        if split:
            words = getattr(tb, "_words", None)
            if words is None:
                raise _lib.ConfigError("the split scorer needs a batch built from a static set")
            w = words.cpu().numpy().view(np.uint64)
            bits = np.unpackbits(w.view(np.uint8), bitorder="little")[: tb.V]
            st = np.flatnonzero(bits).astype(np.uint32)
            if st.size:
                self.split = True
                self.nT = int(st.size)
                self.nTp = int(_lib.lib.svt_prefill_static_pad(self.nT))
                self.st_ids = torch.from_numpy(st.view(np.int32)).cuda()
                self.st_rows = torch.empty((self.nT, self.d), dtype=torch.bfloat16, device="cuda")
                S = tb.B
                self.dyn_ids = torch.empty(max(1, self.total), dtype=torch.int32, device="cuda")
                self.vids = torch.empty(max(1, self.total + S * self.nTp), dtype=torch.int32,
                                        device="cuda")
                self.split_meta = torch.zeros((4, max(1, S)), dtype=torch.int64, device="cuda")
                self.n_dyn, self.vid_off, self.vrows, self.st_valid = self.split_meta
        self.regather()
        return self

    def regather(self):
        """Re-gather the sub-heads from the batch's current plans (device
        only; nothing to do for the fused scorer)."""
        if self.fused:
            return
        tb = self._tb
        if self.split:
            st = _stream(self.stream)
            call("svt_prefill_split_plans", tb.active.data_ptr(), tb.act_off.data_ptr(),
                 tb.n_active.data_ptr(), tb.B, tb._words.data_ptr(), tb.V,
                 self.st_ids.data_ptr(), self.nT, self.dyn_ids.data_ptr(), self.n_dyn.data_ptr(),
                 self.vids.data_ptr(), self.vid_off.data_ptr(), self.vrows.data_ptr(),
                 self.st_valid.data_ptr(), st)
            call("svt_gather_rows", self.head.data.data_ptr(), self.head.storage,
                 self.head.rows(), self.d, self.st_ids.data_ptr(), self.nT,
                 self.st_rows.data_ptr(), self.bad.data_ptr(), st)
            call("svt_gather_plans", self.head.data.data_ptr(), self.head.storage,
                 self.head.rows(), self.d, self.dyn_ids.data_ptr(), tb.act_off.data_ptr(),
                 self.n_dyn.data_ptr(), tb.B, self.total, self.sub.data_ptr(),
                 self.bad.data_ptr(), st)
            return
        call("svt_gather_plans", self.head.data.data_ptr(), self.head.storage, self.head.rows(),
             self.d, tb.active.data_ptr(), tb.act_off.data_ptr(), tb.n_active.data_ptr(), tb.B,
             self.total, self.sub.data_ptr(), self.bad.data_ptr(), _stream(self.stream))

    def _setup(self, head: HeadMatrix, positions: int, S: int, total: int, stream):
        if head.storage != SVT_BF16:
            raise _lib.ConfigError("prefill scoring runs on bf16 heads")
        self.head, self.P, self.stream, self.S, self.total = head, positions, stream, S, total
        self.d = head.dim()
        self.sub = torch.empty((max(1, total), self.d), dtype=torch.bfloat16, device="cuda")
        self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.ws = torch.zeros(_lib.lib.svt_prefill_workspace_bytes(S, positions),
                              dtype=torch.uint8, device="cuda")
        # per-head row norms (once per head) bound Σ|w h| in the certification
        if getattr(head, "row_norms", None) is None:
            head.row_norms = torch.empty(head.rows(), dtype=torch.float32, device="cuda")
            call("svt_row_norms_bf16", head.data.data_ptr(), head.rows(), self.d,
                 head.row_norms.data_ptr(), _stream(stream))

    def score(self, hidden: torch.Tensor, out_ids: torch.Tensor, out_max=None) -> torch.Tensor:
        """hidden: bf16 [S*P, d] on the device -> out_ids int32 [S*P]."""
        if self.fused:
            call("svt_prefill_score_fused", hidden.data_ptr(), self.head.data.data_ptr(),
                 self.head.rows(), self.n_rows.data_ptr(), self.plan_ids.data_ptr(),
                 self.id_off.data_ptr(), self.head.row_norms.data_ptr(), self.S, self.P, self.d,
                 out_ids.data_ptr(), None if out_max is None else out_max.data_ptr(),
                 self.ws.data_ptr(), _stream(self.stream))
            return out_ids
        if self.split:
            call("svt_prefill_score_split", hidden.data_ptr(), self.st_rows.data_ptr(), self.nT,
                 self.st_valid.data_ptr(), self.sub.data_ptr(), self.total,
                 self.row_off.data_ptr(), self.vrows.data_ptr(), self.vids.data_ptr(),
                 self.vid_off.data_ptr(), self.head.row_norms.data_ptr(), self.S, self.P, self.d,
                 out_ids.data_ptr(), None if out_max is None else out_max.data_ptr(),
                 self.ws.data_ptr(), _stream(self.stream))
            return out_ids
        call("svt_prefill_score", hidden.data_ptr(), self.sub.data_ptr(), self.total,
             self.row_off.data_ptr(), self.n_rows.data_ptr(), self.plan_ids.data_ptr(),
             self.id_off.data_ptr(), self.head.row_norms.data_ptr(), self.S, self.P, self.d,
             out_ids.data_ptr(),
             None if out_max is None else out_max.data_ptr(), self.ws.data_ptr(),
             _stream(self.stream))
        return out_ids

    @staticmethod
    def tuning():
        """(pair, nsplit) of the prefill GEMM (svt_prefill_get_tuning)."""
        pr, ns = ctypes.c_int32(), ctypes.c_int32()
        _lib.lib.svt_prefill_get_tuning(ctypes.byref(pr), ctypes.byref(ns))
        return pr.value, ns.value

    @staticmethod
    def set_tuning(pair: bool = True, nsplit: int = 0):
        call("svt_prefill_set_tuning", int(pair), int(nsplit))

    def _offsets(self):
        out = (ctypes.c_int64 * 4)()
        _lib.lib.svt_prefill_offsets(self.S, self.P, out)
        return list(out)

    def top8(self):
        """Partial top-8 records of the last score(): (values f32
        [S*P, nsplit*8], plan rows u32-as-int32 [S*P, nsplit*8])."""
        npos = self.S * self.P
        mo = _lib.lib.svt_prefill_meta_offset(self.S, self.P)
        ns = int(self.ws[mo: mo + 4].view(torch.int32).item())  # splits the last call used
        o = self._offsets()
        v = self.ws[o[0]: o[0] + npos * ns * 32].view(torch.float32).view(npos, ns * 8)
        r = self.ws[o[1]: o[1] + npos * ns * 32].view(torch.int32).view(npos, ns * 8)
        return v, r

    def stats(self):
        """Counters of the last score(): (certified directly, recomputed,
        recomputed over all rows, with a non-finite logit, candidate pairs)."""
        o = self._offsets()
        st = self.ws[o[2]: o[2] + 32].view(torch.int32).cpu().tolist()
        return st[0], st[1], st[2], st[3], st[6]

    def profile_counters(self):
        """SVT_PREFILL_MODE bit 3 cycle counters of the last score()."""
        o = self._offsets()
        return self.ws[o[3]: o[3] + 64].view(torch.int64).cpu().tolist()
