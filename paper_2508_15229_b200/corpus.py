"""(f3, f4) The static builder's data-parallel parts on the GPU:
the corpus profiler (profiler.cpp:56-178) and the tolerance filter
(static_builder.cpp:79-121), with the reference's names, result types and
error behaviour. Document ids and df counts are uploaded once; the kernels
are svt_profile_batch / svt_profile_merge / svt_tolerance_filter."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import ConfigError, IntegrityError, ParseError, call
from .tailored_head import TokenSet, _dev, _stream


@dataclass
class Document:
    """vocab.hpp:52-56."""
    input_ids: np.ndarray
    output_ids: np.ndarray
    doc_index: int = 0


@dataclass
class DocStats:
    doc_index: int
    distinct_input: int
    overlap_occurrence: float
    overlap_distinct: float


@dataclass
class ProfiledCorpus:
    """profiler.hpp:15-32 (df dense over the vocabulary, per_doc by doc_index)."""
    vocab_size: int
    doc_count: int
    df: np.ndarray
    input_union: TokenSet
    output_union: TokenSet
    per_doc: List[DocStats] = field(default_factory=list)


@dataclass
class OverlapStats:
    doc_count: int
    mean_overlap: float
    mean_overlap_distinct: float
    mean_input_size: float
    union_input_size: int
    locality_ratio: float


@dataclass
class ToleranceResult:
    """static_builder.hpp:62-66."""
    kept: TokenSet
    pruned: np.ndarray
    pruned_df_sum: int


def _set_from_words(words: np.ndarray, universe: int) -> TokenSet:
    s = TokenSet(universe)
    s.words[:] = words[: s.words.size]
    return s


class Profiler:
    """Streaming accumulator (profiler.hpp:46-60) with device-resident df and
    union bitmaps; add_batch() profiles many documents in one launch."""

    def __init__(self, vocab_size: int, stream=None):
        self.V = int(vocab_size)
        self.stream = stream
        nw = (self.V + 63) // 64
        self.df = torch.zeros(max(self.V, 1), dtype=torch.int32, device="cuda")
        self.in_union = torch.zeros(max(nw, 1), dtype=torch.int64, device="cuda")
        self.out_union = torch.zeros(max(nw, 1), dtype=torch.int64, device="cuda")
        self.doc_count = 0
        self.stats: List[DocStats] = []

    def add(self, doc: Document) -> None:
        self.add_batch([doc])

    def add_batch(self, docs: Sequence[Document]) -> None:
        n = len(docs)
        if n == 0:
            return
        ins = [np.asarray(d.input_ids, np.uint32) for d in docs]
        outs = [np.asarray(d.output_ids, np.uint32) for d in docs]
        ioff = np.zeros(n + 1, np.int64)
        ioff[1:] = np.cumsum([a.size for a in ins])
        ooff = np.zeros(n + 1, np.int64)
        ooff[1:] = np.cumsum([a.size for a in outs])
        d_in = _dev(np.concatenate(ins).view(np.int32) if ioff[-1] else np.zeros(1, np.int32),
                    torch.int32)
        d_out = _dev(np.concatenate(outs).view(np.int32) if ooff[-1] else np.zeros(1, np.int32),
                     torch.int32)
        d_ioff, d_ooff = _dev(ioff, torch.int64), _dev(ooff, torch.int64)
        distinct = torch.empty(n, dtype=torch.int32, device="cuda")
        occ = torch.empty(n, dtype=torch.float64, device="cuda")
        dis = torch.empty(n, dtype=torch.float64, device="cuda")
        err = torch.zeros(n, dtype=torch.int32, device="cuda")
        err_id = torch.zeros(n, dtype=torch.int32, device="cuda")
        call("svt_profile_batch", self.V, d_in.data_ptr(), d_ioff.data_ptr(), d_out.data_ptr(),
             d_ooff.data_ptr(), n, self.df.data_ptr(), self.in_union.data_ptr(),
             self.out_union.data_ptr(), distinct.data_ptr(), occ.data_ptr(), dis.data_ptr(),
             err.data_ptr(), err_id.data_ptr(), _stream(self.stream))
        e = err.cpu().numpy()
        bad = np.flatnonzero(e)
        if bad.size:  # the reference throws at the first failing add()
            k = int(bad[0])
            idx = docs[k].doc_index
            bid = int(err_id[k].item()) & 0xFFFFFFFF
            if e[k] == 3:
                raise ParseError(f"document {idx} has an empty output; its overlap ratio is "
                                 "undefined")
            side = "input" if e[k] == 1 else "output"
            raise IntegrityError(f"document {idx}: {side} token id {bid} out of range for "
                                 f"vocabulary of size {self.V}")
        dc, oc, ds = distinct.cpu().numpy(), occ.cpu().numpy(), dis.cpu().numpy()
        for k, d in enumerate(docs):
            self.stats.append(DocStats(int(d.doc_index), int(dc[k]), float(oc[k]), float(ds[k])))
        self.doc_count += n

    def finish(self) -> ProfiledCorpus:
        """profiler.cpp:99-104 (per_doc sorted by doc_index)."""
        per_doc = sorted(self.stats, key=lambda s: s.doc_index)
        return ProfiledCorpus(self.V, self.doc_count,
                              self.df[: self.V].cpu().numpy().view(np.uint32).copy(),
                              _set_from_words(self.in_union.cpu().numpy().view(np.uint64),
                                              self.V),
                              _set_from_words(self.out_union.cpu().numpy().view(np.uint64),
                                              self.V),
                              per_doc)


def profile(docs: Sequence[Document], vocab_size: int) -> ProfiledCorpus:
    """profiler.cpp:129-133."""
    p = Profiler(vocab_size)
    p.add_batch(list(docs))
    return p.finish()


def merge(a: ProfiledCorpus, b: ProfiledCorpus) -> ProfiledCorpus:
    """Profiler::merge (profiler.cpp:106-127): df and unions on the device,
    per-document records merged by doc_index with the duplicate check."""
    if a.vocab_size != b.vocab_size:
        raise IntegrityError("cannot merge profiles over different vocabulary sizes: "
                             f"{a.vocab_size} vs {b.vocab_size}")
    V = a.vocab_size
    df = torch.from_numpy(a.df.view(np.int32).copy()).cuda()
    dfb = torch.from_numpy(b.df.view(np.int32).copy()).cuda()
    iu = torch.from_numpy(a.input_union.words.view(np.int64).copy()).cuda()
    iub = torch.from_numpy(b.input_union.words.view(np.int64).copy()).cuda()
    ou = torch.from_numpy(a.output_union.words.view(np.int64).copy()).cuda()
    oub = torch.from_numpy(b.output_union.words.view(np.int64).copy()).cuda()
    call("svt_profile_merge", V, df.data_ptr(), dfb.data_ptr(), iu.data_ptr(), iub.data_ptr(),
         ou.data_ptr(), oub.data_ptr(), _stream())
    per_doc = sorted(a.per_doc + b.per_doc, key=lambda s: s.doc_index)
    for i in range(1, len(per_doc)):
        if per_doc[i].doc_index == per_doc[i - 1].doc_index:
            raise IntegrityError(f"duplicate doc_index {per_doc[i].doc_index} across merged "
                                 "profile shards")
    return ProfiledCorpus(V, a.doc_count + b.doc_count, df.cpu().numpy().view(np.uint32).copy(),
                          _set_from_words(iu.cpu().numpy().view(np.uint64), V),
                          _set_from_words(ou.cpu().numpy().view(np.uint64), V), per_doc)


def _sorted_mean(values) -> float:
    """profiler.cpp:24-31: sum a sorted copy (order-independent)."""
    if len(values) == 0:
        return 0.0
    s = 0.0
    for v in sorted(values):
        s += float(v)
    return s / float(len(values))


def locality_report(p: ProfiledCorpus) -> OverlapStats:
    """profiler.cpp:154-178."""
    if p.doc_count == 0:
        raise ConfigError("locality report requires a non-empty corpus")
    mi = _sorted_mean([d.distinct_input for d in p.per_doc])
    union = p.input_union.size()
    return OverlapStats(p.doc_count, _sorted_mean([d.overlap_occurrence for d in p.per_doc]),
                        _sorted_mean([d.overlap_distinct for d in p.per_doc]), mi, union,
                        float(union) / mi if mi > 0.0 else 1.0)


def tolerance_filter(candidates: TokenSet, df, doc_count: int, tau: float,
                     always_keep: Optional[TokenSet] = None) -> ToleranceResult:
    """static_builder.cpp:79-121 on the GPU (svt_tolerance_filter)."""
    if doc_count < 1:
        raise ConfigError("tolerance filtering requires at least one profiled document")
    U = candidates.universe_size()
    nw = max(1, (U + 63) // 64)
    df = np.ascontiguousarray(np.asarray(df, np.uint32))
    d_cand = _dev(candidates.words.view(np.int64), torch.int64)
    d_keep = (_dev(always_keep.words.view(np.int64), torch.int64)
              if always_keep is not None and always_keep.universe_size() > 0 else None)
    d_df = _dev(df.view(np.int32) if df.size else np.zeros(1, np.int32), torch.int32)
    kept = torch.zeros(nw, dtype=torch.int64, device="cuda")
    pruned = torch.empty(max(1, candidates.size()), dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.int64, device="cuda")
    call("svt_tolerance_filter", d_cand.data_ptr(), None if d_keep is None else d_keep.data_ptr(),
         U, d_df.data_ptr(), df.size, int(doc_count), float(tau), kept.data_ptr(),
         pruned.data_ptr(), scal.data_ptr(), scal.data_ptr() + 8, _stream())
    n, s = (int(x) for x in scal.cpu().tolist())
    return ToleranceResult(_set_from_words(kept.cpu().numpy().view(np.uint64), U),
                           pruned[:n].cpu().numpy().view(np.uint32).copy(), s & (2**64 - 1))
