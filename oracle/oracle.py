"""oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-ends for the two checkers of the tailored-head path:

* ``C``   — ``oracle/libsvt_oracle.so``, the plain-C restatement
  (``oracle/svt_oracle.c``; every routine cites its reference file:line).
* ``Ref`` — ``oracle/_ref/libsubvocab_ref.so``, the UNMODIFIED reference
  TUs from ``/root/reference/proj/src`` compiled by ``oracle/Makefile`` with
  ``oracle/ref_shim.cpp`` (extern "C" calls into the reference API).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module, and only as the checker / the timed CPU baseline. The
product path (``paper_2508_15229_b200``) never imports it.

Status codes follow ``subvocab::Error::exit_code()`` (error.hpp:10-38).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libsvt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsubvocab_ref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_szp = np.ctypeslib.ndpointer(np.uintp, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_P = C.POINTER


class OracleError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


@dataclass
class Plan:
    active_ids: np.ndarray
    n_static: int
    n_dynamic: int
    full_vocab_size: int


def words_from_ids(ids, universe: int) -> np.ndarray:
    """TokenSet bitmap words (token_set.hpp:17-64 layout: bit id%64 of word id/64)."""
    w = np.zeros((universe + 63) // 64, dtype=np.uint64)
    ids = np.asarray(ids, dtype=np.uint64)
    if ids.size:
        np.bitwise_or.at(w, (ids // 64).astype(np.int64), np.left_shift(np.uint64(1), ids % 64))
    return w


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing — run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


class _COracle:
    def __init__(self):
        L = self.L = _load(ORACLE_SO)
        L.orc_head_random.argtypes = [_f32p, _sz, _sz, C.c_uint64, C.c_int]
        L.orc_head_random_slice.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.orc_float_to_half.argtypes = [C.c_float]
        L.orc_float_to_half.restype = C.c_uint16
        L.orc_half_to_float.argtypes = [C.c_uint16]
        L.orc_half_to_float.restype = C.c_float
        L.orc_round_bf16.argtypes = [C.c_float]
        L.orc_round_bf16.restype = C.c_float
        L.orc_select.argtypes = [_u32p, _sz, _u64p, _sz, _sz, _u32p, _P(_sz), _P(_sz), _P(_sz),
                                 _P(C.c_uint32)]
        L.orc_remap_out.argtypes = [_u32p, _sz, _sz, _P(C.c_uint32)]
        L.orc_global_to_local.argtypes = [_u32p, _sz, C.c_uint32]
        L.orc_global_to_local.restype = C.c_int64
        L.orc_union_plans.argtypes = [_u32p, _i64p, _szp, _szp, _sz, _u32p, _P(_sz), _P(_sz),
                                      _P(_sz)]
        L.orc_gather.argtypes = [_f32p, _sz, _sz, _u32p, _sz, _f32p]
        L.orc_logits.argtypes = [_f32p, _sz, _sz, _f32p, _sz, _f32p]
        L.orc_greedy_step.argtypes = [_f32p, _sz, _sz, _f32p, _sz, _u32p, _sz, _P(C.c_uint32),
                                      _P(C.c_float)]
        L.orc_topk.argtypes = [_f32p, _sz, _sz, _f32p, _sz, _u32p, _sz, _sz, _u32p, _f32p]
        L.orc_argmax_first.argtypes = [_f32p, _sz]
        L.orc_argmax_first.restype = _sz
        L.orc_memory_report.argtypes = [_sz, _sz, C.c_int, _sz] + [_P(C.c_uint64)] * 4 + [
            _P(C.c_double)]
        L.orc_simulate.argtypes = [C.c_double] * 3 + [_sz, _sz, C.c_int, _sz, C.c_double] + [
            _P(C.c_double)] * 4 + [_P(C.c_int)]
        L.orc_breakeven_rows.argtypes = [C.c_double] * 3 + [_sz, C.c_int, _sz, C.c_double,
                                                            _P(_sz)]
        L.orc_static_ids.argtypes = [C.c_uint64, _sz, _sz, _u32p]
        L.orc_prompt_ids.argtypes = [C.c_uint64, _sz, _sz, _u32p]

    # -- generators -------------------------------------------------------
    def head_random(self, rows, dim, seed, dtype_bytes=4):
        out = np.empty(rows * dim, np.float32)
        st = self.L.orc_head_random(out, rows, dim, seed, dtype_bytes)
        if st:
            raise OracleError(st)
        return out.reshape(rows, dim)

    def head_random_slice(self, first, count, seed, dtype_bytes=4):
        out = np.empty(count, np.float32)
        self.L.orc_head_random_slice(out, first, count, seed, dtype_bytes)
        return out

    def static_ids(self, seed, V, n):
        out = np.empty(n, np.uint32)
        self.L.orc_static_ids(seed, V, n, out)
        return out

    def prompt_ids(self, seed, V, L):
        out = np.empty(L, np.uint32)
        self.L.orc_prompt_ids(seed, V, L, out)
        return out

    def float_to_half(self, f):
        return self.L.orc_float_to_half(f)

    def half_to_float(self, h):
        return self.L.orc_half_to_float(h)

    def round_bf16(self, f):
        return self.L.orc_round_bf16(f)

    # -- path -------------------------------------------------------------
    def select(self, ids, static_words, static_universe, V) -> Plan:
        ids = np.ascontiguousarray(ids, np.uint32)
        static_words = np.ascontiguousarray(static_words, np.uint64)
        out = np.empty(static_universe + ids.size + 1, np.uint32)
        na, ns, nd, bad = _sz(), _sz(), _sz(), C.c_uint32()
        st = self.L.orc_select(ids, ids.size, static_words, static_universe, V, out,
                               C.byref(na), C.byref(ns), C.byref(nd), C.byref(bad))
        if st:
            raise OracleError(st, f"bad id {bad.value}")
        return Plan(out[: na.value].copy(), ns.value, nd.value, V)

    def remap_out(self, ids, local):
        ids = np.ascontiguousarray(ids, np.uint32)
        o = C.c_uint32()
        st = self.L.orc_remap_out(ids, ids.size, local, C.byref(o))
        if st:
            raise OracleError(st)
        return o.value

    def global_to_local(self, ids, gid):
        ids = np.ascontiguousarray(ids, np.uint32)
        r = self.L.orc_global_to_local(ids, ids.size, gid)
        return None if r < 0 else r

    def union_plans(self, plans) -> Plan:
        if not plans:
            ids = np.zeros(1, np.uint32)
            off = np.zeros(1, np.int64)
            fs = np.zeros(1, np.uintp)
            ns = np.zeros(1, np.uintp)
        else:
            ids = np.concatenate([np.asarray(p.active_ids, np.uint32) for p in plans] + [
                np.zeros(1, np.uint32)])
            off = np.zeros(len(plans) + 1, np.int64)
            off[1:] = np.cumsum([len(p.active_ids) for p in plans])
            fs = np.array([p.full_vocab_size for p in plans], np.uintp)
            ns = np.array([p.n_static for p in plans], np.uintp)
        cap = max(1, max((p.full_vocab_size for p in plans), default=1))
        out = np.empty(cap, np.uint32)
        na, nst, nd = _sz(), _sz(), _sz()
        st = self.L.orc_union_plans(ids, off, fs, ns, len(plans), out, C.byref(na),
                                    C.byref(nst), C.byref(nd))
        if st:
            raise OracleError(st)
        return Plan(out[: na.value].copy(), nst.value, nd.value, int(fs[0]))

    def gather(self, head, ids):
        head = np.ascontiguousarray(head, np.float32)
        ids = np.ascontiguousarray(ids, np.uint32)
        rows, dim = head.shape
        out = np.empty((max(ids.size, 1), dim), np.float32)
        st = self.L.orc_gather(head.reshape(-1), rows, dim, ids, ids.size, out.reshape(-1))
        if st:
            raise OracleError(st)
        return out[: ids.size]

    def logits(self, head, hidden):
        head = np.ascontiguousarray(head, np.float32)
        hidden = np.ascontiguousarray(hidden, np.float32)
        rows, dim = head.shape
        out = np.empty(max(rows, 1), np.float32)
        st = self.L.orc_logits(head.reshape(-1) if head.size else np.zeros(1, np.float32), rows,
                               dim, hidden if hidden.size else np.zeros(1, np.float32),
                               hidden.size, out)
        if st:
            raise OracleError(st)
        return out[:rows]

    def greedy_step(self, sub, hidden, plan_ids):
        sub = np.ascontiguousarray(sub, np.float32)
        hidden = np.ascontiguousarray(hidden, np.float32)
        plan_ids = np.ascontiguousarray(plan_ids, np.uint32)
        rows, dim = sub.shape
        o, m = C.c_uint32(), C.c_float()
        st = self.L.orc_greedy_step(sub.reshape(-1) if sub.size else np.zeros(1, np.float32),
                                    rows, dim, hidden if hidden.size else np.zeros(1, np.float32),
                                    hidden.size,
                                    plan_ids if plan_ids.size else np.zeros(1, np.uint32),
                                    plan_ids.size, C.byref(o), C.byref(m))
        if st:
            raise OracleError(st)
        return o.value, m.value

    def argmax_first(self, scores):
        s = np.ascontiguousarray(scores, np.float32)
        return self.L.orc_argmax_first(s, s.size)

    def topk(self, sub, hidden, plan_ids, k):
        """(ids, values) of the k best plan rows: value desc, id asc (not a
        reference function; svt_oracle.c orc_topk)."""
        sub = np.ascontiguousarray(sub, np.float32)
        hidden = np.ascontiguousarray(hidden, np.float32)
        plan_ids = np.ascontiguousarray(plan_ids, np.uint32)
        rows, dim = sub.shape
        ids = np.zeros(max(k, 1), np.uint32)
        vals = np.zeros(max(k, 1), np.float32)
        st = self.L.orc_topk(sub.reshape(-1) if sub.size else np.zeros(1, np.float32), rows, dim,
                             hidden if hidden.size else np.zeros(1, np.float32), hidden.size,
                             plan_ids if plan_ids.size else np.zeros(1, np.uint32), plan_ids.size,
                             k, ids, vals)
        if st:
            raise OracleError(st)
        return ids[:k], vals[:k]

    def memory_report(self, full, dim, dtype_bytes, plan):
        a, b, c, d = (C.c_uint64() for _ in range(4))
        s = C.c_double()
        st = self.L.orc_memory_report(full, dim, dtype_bytes, plan, C.byref(a), C.byref(b),
                                      C.byref(c), C.byref(d), C.byref(s))
        if st:
            raise OracleError(st)
        return a.value, b.value, c.value, d.value, s.value

    def simulate(self, link, flops, lat, plan, dim, b, L, fpt):
        t, p, e, x = (C.c_double() for _ in range(4))
        h = C.c_int()
        st = self.L.orc_simulate(link, flops, lat, plan, dim, b, L, fpt, C.byref(t), C.byref(p),
                                 C.byref(e), C.byref(x), C.byref(h))
        if st:
            raise OracleError(st)
        return t.value, p.value, e.value, x.value, bool(h.value)

    def breakeven_rows(self, link, flops, lat, dim, b, L, fpt):
        r = _sz()
        st = self.L.orc_breakeven_rows(link, flops, lat, dim, b, L, fpt, C.byref(r))
        if st:
            raise OracleError(st)
        return r.value


class _RefLib:
    """The real reference, compiled from /root/reference (oracle/_ref)."""

    def __init__(self):
        L = self.L = _load(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_head_random.argtypes = [_f32p, _sz, _sz, C.c_uint64, C.c_int]
        L.ref_float_to_half.argtypes = [C.c_float]
        L.ref_float_to_half.restype = C.c_uint16
        L.ref_half_to_float.argtypes = [C.c_uint16]
        L.ref_half_to_float.restype = C.c_float
        L.ref_select.argtypes = [_u32p, _sz, _u64p, _sz, _sz, _u32p, _P(_sz), _P(_sz), _P(_sz)]
        L.ref_remap_out.argtypes = [_u32p, _sz, _sz, _P(C.c_uint32)]
        L.ref_global_to_local.argtypes = [_u32p, _sz, C.c_uint32]
        L.ref_global_to_local.restype = C.c_int64
        L.ref_union_plans.argtypes = [_u32p, _i64p, _szp, _szp, _sz, _u32p, _P(_sz), _P(_sz),
                                      _P(_sz)]
        L.ref_gather.argtypes = [_f32p, _sz, _sz, _u32p, _sz, _f32p]
        L.ref_logits.argtypes = [_f32p, _sz, _sz, _f32p, _sz, _f32p]
        L.ref_greedy_step.argtypes = [_f32p, _sz, _sz, _f32p, _sz, _u32p, _sz, _P(C.c_uint32)]
        L.ref_memory_report.argtypes = [_sz, _sz, C.c_int, _sz] + [_P(C.c_uint64)] * 4 + [
            _P(C.c_double)]
        L.ref_simulate.argtypes = [C.c_double] * 3 + [_sz, _sz, C.c_int, _sz, C.c_double] + [
            _P(C.c_double)] * 4 + [_P(C.c_int)]
        L.ref_breakeven_rows.argtypes = [C.c_double] * 3 + [_sz, C.c_int, _sz, C.c_double,
                                                            _P(_sz)]
        L.ref_head_new.argtypes = [_f32p, _sz, _sz, C.c_int]
        L.ref_head_new.restype = C.c_void_p
        L.ref_head_new_random.argtypes = [_sz, _sz, C.c_uint64, C.c_int]
        L.ref_head_new_random.restype = C.c_void_p
        L.ref_head_free.argtypes = [C.c_void_p]
        L.ref_head_copy_out.argtypes = [C.c_void_p, _f32p]
        L.ref_head_assign.argtypes = [C.c_void_p, _f32p]
        L.ref_batch_new.restype = C.c_void_p
        L.ref_batch_free.argtypes = [C.c_void_p]
        L.ref_batch_prepare.argtypes = [C.c_void_p, C.c_void_p, _u64p, _sz, _u32p, _i64p, C.c_int,
                                        C.c_int]
        L.ref_batch_plan_size.argtypes = [C.c_void_p, C.c_int]
        L.ref_batch_plan_size.restype = C.c_int64
        L.ref_batch_plan_ids.argtypes = [C.c_void_p, C.c_int, _u32p, _P(C.c_int64),
                                         _P(C.c_int64)]
        L.ref_batch_greedy.argtypes = [C.c_void_p, _f32p, _sz, C.c_int, C.c_int, _u32p]
        L.ref_slice_argmax.argtypes = [C.c_void_p, _sz, _sz, _f32p, _P(C.c_uint32),
                                       _P(C.c_float)]
        L.ref_jobs_run.argtypes = [C.c_void_p, _u64p, _sz, _u32p, _i64p, C.c_int, _f32p,
                                   C.c_int, C.c_int, _u32p, _P(C.c_double), _P(C.c_double)]

    def jobs_run(self, head, words, V, flat, off, hidden, steps, threads):
        """ref_jobs_run: J = len(off) - 1 cfg1 jobs (select -> gather ->
        `steps` greedy steps each) on `threads` host threads. Returns (ids
        [steps][J], (select, gather, decode) seconds summed over jobs, wall s)."""
        J = len(off) - 1
        ids = np.zeros((steps, J), np.uint32)
        ph = (C.c_double * 3)()
        wall = C.c_double()
        self._chk(self.L.ref_jobs_run(head, np.ascontiguousarray(words, np.uint64), V,
                                      np.ascontiguousarray(flat, np.uint32),
                                      np.ascontiguousarray(off, np.int64), J,
                                      np.ascontiguousarray(hidden, np.float32), steps, threads,
                                      ids, ph, C.byref(wall)))
        return ids, tuple(ph), wall.value

    def _chk(self, st):
        if st:
            raise OracleError(st, self.L.ref_last_error().decode())

    def head_random(self, rows, dim, seed, dtype_bytes=4):
        out = np.empty(rows * dim, np.float32)
        self._chk(self.L.ref_head_random(out, rows, dim, seed, dtype_bytes))
        return out.reshape(rows, dim)

    def float_to_half(self, f):
        return self.L.ref_float_to_half(f)

    def half_to_float(self, h):
        return self.L.ref_half_to_float(h)

    def select(self, ids, static_words, static_universe, V) -> Plan:
        ids = np.ascontiguousarray(ids, np.uint32)
        static_words = np.ascontiguousarray(static_words, np.uint64)
        out = np.empty(static_universe + ids.size + 1, np.uint32)
        na, ns, nd = _sz(), _sz(), _sz()
        self._chk(self.L.ref_select(ids if ids.size else np.zeros(1, np.uint32), ids.size,
                                    static_words if static_words.size else np.zeros(1, np.uint64),
                                    static_universe, V, out, C.byref(na), C.byref(ns),
                                    C.byref(nd)))
        return Plan(out[: na.value].copy(), ns.value, nd.value, V)

    def remap_out(self, ids, local):
        ids = np.ascontiguousarray(ids, np.uint32)
        o = C.c_uint32()
        self._chk(self.L.ref_remap_out(ids if ids.size else np.zeros(1, np.uint32), ids.size,
                                       local, C.byref(o)))
        return o.value

    def global_to_local(self, ids, gid):
        ids = np.ascontiguousarray(ids, np.uint32)
        r = self.L.ref_global_to_local(ids if ids.size else np.zeros(1, np.uint32), ids.size, gid)
        return None if r < 0 else r

    def union_plans(self, plans) -> Plan:
        ids = np.concatenate([np.asarray(p.active_ids, np.uint32) for p in plans] + [
            np.zeros(1, np.uint32)])
        off = np.zeros(len(plans) + 1, np.int64)
        off[1:] = np.cumsum([len(p.active_ids) for p in plans]) if plans else []
        fs = np.array([p.full_vocab_size for p in plans] or [0], np.uintp)
        ns = np.array([p.n_static for p in plans] or [0], np.uintp)
        cap = max(1, max((p.full_vocab_size for p in plans), default=1))
        out = np.empty(cap, np.uint32)
        na, nst, nd = _sz(), _sz(), _sz()
        self._chk(self.L.ref_union_plans(ids, off, fs, ns, len(plans), out, C.byref(na),
                                         C.byref(nst), C.byref(nd)))
        return Plan(out[: na.value].copy(), nst.value, nd.value, int(fs[0]))

    def gather(self, head, ids):
        head = np.ascontiguousarray(head, np.float32)
        ids = np.ascontiguousarray(ids, np.uint32)
        rows, dim = head.shape
        out = np.empty((max(ids.size, 1), dim), np.float32)
        self._chk(self.L.ref_gather(head.reshape(-1) if head.size else np.zeros(1, np.float32),
                                    rows, dim, ids if ids.size else np.zeros(1, np.uint32),
                                    ids.size, out.reshape(-1) if out.size else np.zeros(
                                        1, np.float32)))
        return out[: ids.size]

    def logits(self, head, hidden):
        head = np.ascontiguousarray(head, np.float32)
        hidden = np.ascontiguousarray(hidden, np.float32)
        rows, dim = head.shape
        out = np.empty(max(rows, 1), np.float32)
        self._chk(self.L.ref_logits(head.reshape(-1) if head.size else np.zeros(1, np.float32),
                                    rows, dim, hidden if hidden.size else np.zeros(1, np.float32),
                                    hidden.size, out))
        return out[:rows]

    def greedy_step(self, sub, hidden, plan_ids):
        sub = np.ascontiguousarray(sub, np.float32)
        hidden = np.ascontiguousarray(hidden, np.float32)
        plan_ids = np.ascontiguousarray(plan_ids, np.uint32)
        rows, dim = sub.shape
        o = C.c_uint32()
        self._chk(self.L.ref_greedy_step(sub.reshape(-1) if sub.size else np.zeros(1, np.float32),
                                         rows, dim,
                                         hidden if hidden.size else np.zeros(1, np.float32),
                                         hidden.size,
                                         plan_ids if plan_ids.size else np.zeros(1, np.uint32),
                                         plan_ids.size, C.byref(o)))
        return o.value

    def memory_report(self, full, dim, dtype_bytes, plan):
        a, b, c, d = (C.c_uint64() for _ in range(4))
        s = C.c_double()
        self._chk(self.L.ref_memory_report(full, dim, dtype_bytes, plan, C.byref(a), C.byref(b),
                                           C.byref(c), C.byref(d), C.byref(s)))
        return a.value, b.value, c.value, d.value, s.value

    def simulate(self, link, flops, lat, plan, dim, b, L, fpt):
        t, p, e, x = (C.c_double() for _ in range(4))
        h = C.c_int()
        self._chk(self.L.ref_simulate(link, flops, lat, plan, dim, b, L, fpt, C.byref(t),
                                      C.byref(p), C.byref(e), C.byref(x), C.byref(h)))
        return t.value, p.value, e.value, x.value, bool(h.value)

    def breakeven_rows(self, link, flops, lat, dim, b, L, fpt):
        r = _sz()
        self._chk(self.L.ref_breakeven_rows(link, flops, lat, dim, b, L, fpt, C.byref(r)))
        return r.value


_c = None
_ref = None


def c_oracle() -> _COracle:
    global _c
    if _c is None:
        _c = _COracle()
    return _c


def ref_lib() -> _RefLib:
    global _ref
    if _ref is None:
        _ref = _RefLib()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
