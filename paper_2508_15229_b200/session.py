"""Python view of the host-buffer session C-ABI (svt_session_*): the call an
external runtime makes with HOST buffers — H2D inside, D2H of the ids, one
synchronisation per call. bench.py's e2e leg measures through this."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import call
from .tailored_head import HeadMatrix


class Session:
    def __init__(self, head: HeadMatrix, max_batch: int, max_plan_rows: int = 0, stream=None):
        self.head = head
        h = C.c_void_p()
        call("svt_session_create", C.byref(h), head.data.data_ptr(), head.storage, head.rows(),
             head.dim(), max_batch, max_plan_rows, None if stream is None else stream.cuda_stream)
        self.h = h
        self.B = 0

    def close(self):
        if self.h:
            _lib.lib.svt_session_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def prepare(self, static_words: np.ndarray, V: int, prompts: np.ndarray,
                offsets: np.ndarray):
        w = np.ascontiguousarray(static_words, np.uint64)
        p = np.ascontiguousarray(prompts, np.uint32)
        o = np.ascontiguousarray(offsets, np.int64)
        call("svt_session_prepare_host", self.h, w.ctypes.data, V,
             p.ctypes.data if p.size else None, o.ctypes.data, len(o) - 1)
        self.B = len(o) - 1

    def plans(self):
        B = self.B
        na = np.zeros(B, np.int64)
        ns, nd = np.zeros(B, np.int64), np.zeros(B, np.int64)
        call("svt_session_plans_host", self.h, na.ctypes.data, ns.ctypes.data, nd.ctypes.data,
             None, None)
        ids = np.zeros(max(1, int(na.sum())), np.uint32)
        off = np.zeros(B + 1, np.int64)
        call("svt_session_plans_host", self.h, None, None, None, ids.ctypes.data, off.ctypes.data)
        return na, ns, nd, ids[: int(na.sum())], off

    def greedy(self, hidden, out_ids: np.ndarray = None, out_max: np.ndarray = None):
        """hidden: host array [B, >=dim] float32 (pinned or pageable)."""
        if hasattr(hidden, "data_ptr"):  # pinned torch tensor
            ptr, ld = hidden.data_ptr(), hidden.stride(0)
        else:
            hidden = np.ascontiguousarray(hidden, np.float32)
            ptr, ld = hidden.ctypes.data, hidden.shape[1]
        if out_ids is None:
            out_ids = np.empty(self.B, np.uint32)
        optr = out_ids.data_ptr() if hasattr(out_ids, "data_ptr") else out_ids.ctypes.data
        mptr = None if out_max is None else (
            out_max.data_ptr() if hasattr(out_max, "data_ptr") else out_max.ctypes.data)
        call("svt_session_greedy_host", self.h, ptr, ld, optr, mptr)
        return out_ids


def prepare_many(sessions, static_words: np.ndarray, V: int, prompts, offsets):
    """svt_session_prepare_host_many: prepare every session (session i over
    prompts[i] / offsets[i]); batch-1 sessions do not synchronise (their
    plan counts are computed on the host)."""
    w = np.ascontiguousarray(static_words, np.uint64)
    ps = [np.ascontiguousarray(p, np.uint32) for p in prompts]
    os_ = [np.ascontiguousarray(o, np.int64) for o in offsets]
    n = len(sessions)
    arr = (C.c_void_p * n)(*[s.h.value for s in sessions])
    pid = (C.c_void_p * n)(*[p.ctypes.data if p.size else None for p in ps])
    poff = (C.c_void_p * n)(*[o.ctypes.data for o in os_])
    bs = (C.c_int32 * n)(*[len(o) - 1 for o in os_])
    call("svt_session_prepare_host_many", arr, n, w.ctypes.data, V, pid, poff, bs)
    for s_, o in zip(sessions, os_):
        s_.B = len(o) - 1


def decode_host(sessions, hidden, steps: int, out_ids=None):
    """svt_session_decode_host: `steps` token-interleaved decode steps over
    prepared sessions sharing one stream. hidden: host [steps][sum B][dim]
    float32 (a pinned torch tensor or a numpy array); returns the ids
    [steps][sum B] (uint32 numpy array or the given buffer)."""
    rows = sum(s.B for s in sessions)
    arr = (C.c_void_p * len(sessions))(*[s.h.value for s in sessions])
    if hasattr(hidden, "data_ptr"):
        hptr = hidden.data_ptr()
    else:
        hidden = np.ascontiguousarray(hidden, np.float32)
        hptr = hidden.ctypes.data
    if out_ids is None:
        out_ids = np.empty((steps, rows), np.uint32)
    optr = out_ids.data_ptr() if hasattr(out_ids, "data_ptr") else out_ids.ctypes.data
    call("svt_session_decode_host", arr, len(sessions), hptr, steps, optr)
    return out_ids

