"""(f3) corpus profiler and (f4) tolerance filter.

CPU (not gpu): the C restatement (oracle/svt_oracle.c) against the
UNMODIFIED reference (oracle/_ref/libsubvocab_ref_static.so, built from
/root/reference by oracle/Makefile) on seeded cases, including the
reference's edge cases (negative / NaN / infinite budgets, protected ids, df
shorter than the universe, empty outputs, out-of-range ids).
GPU: svt_tolerance_filter and svt_profile_batch / svt_profile_merge against
the oracle, bit for bit (ids, counts and the per-document doubles)."""
import ctypes as C
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC = C.CDLL(os.path.join(ROOT, "oracle", "libsvt_oracle.so"))
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libsubvocab_ref_static.so")
REF = C.CDLL(REF_PATH) if os.path.exists(REF_PATH) else None
_p = lambda a: a.ctypes.data if a is not None else None  # noqa: E731

for L, pre in ((ORC, "orc_"), (REF, "refs_")):
    if L is None:
        continue
    getattr(L, pre + "tolerance_filter").argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                           C.c_size_t, C.c_int64, C.c_double, C.c_void_p,
                                           C.c_void_p, C.POINTER(C.c_size_t),
                                           C.POINTER(C.c_uint64)]
ORC.orc_profile_doc.argtypes = [C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
if REF is not None:
    REF.refs_profile.argtypes = [C.c_size_t] + [C.c_void_p] * 5 + [C.c_size_t] + [C.c_void_p] * 3 + [
        C.POINTER(C.c_int64)] + [C.c_void_p] * 4
    REF.refs_last_error.restype = C.c_char_p


def words_of(ids, U):
    w = np.zeros(max(1, (U + 63) // 64), np.uint64)
    for i in np.asarray(ids, np.int64):
        w[i // 64] |= np.uint64(1) << np.uint64(i % 64)
    return w


def tol(L, pre, cand, keep, U, df, M, tau):
    kept = np.zeros(max(1, (U + 63) // 64), np.uint64)
    pruned = np.zeros(max(1, U), np.uint32)
    n, s = C.c_size_t(), C.c_uint64()
    st = getattr(L, pre + "tolerance_filter")(_p(cand), _p(keep), U, _p(df), df.size, M, tau, _p(kept),
                                     _p(pruned), C.byref(n), C.byref(s))
    return st, kept, pruned[: n.value].copy(), s.value


def tol_cases():
    rng = np.random.default_rng(1234)
    out = []
    for k in range(40):
        U = int(rng.integers(1, 5000))
        cand = np.unique(rng.integers(0, U, int(rng.integers(0, U + 1))))
        keep = (np.unique(rng.choice(cand, int(rng.integers(0, cand.size + 1)), replace=False))
                if cand.size and k % 3 == 0 else None)
        ndf = int(rng.integers(0, U + 10)) if k % 5 else U
        hi = [1, 3, 50, 10**6][k % 4]
        df = rng.integers(0, hi + 1, ndf).astype(np.uint32)
        M = int(rng.integers(1, 2000))
        tau = [0.0, 0.01, 0.1, 0.5, 1.0, 2.5, -0.1, float("nan"), float("inf"), 1e-9][k % 10]
        out.append((words_of(cand, U), None if keep is None else words_of(keep, U), U, df, M, tau))
    return out


@pytest.mark.skipif(REF is None, reason="reference static library not built")
def test_oracle_tolerance_matches_reference():
    for cand, keep, U, df, M, tau in tol_cases():
        a = tol(ORC, "orc_", cand, keep, U, df, M, tau)
        b = tol(REF, "refs_", cand, keep, U, df, M, tau)
        assert a[0] == b[0] == 0
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3], tau
    # ConfigError for doc_count < 1
    st = tol(REF, "refs_", words_of([1], 8), None, 8, np.ones(8, np.uint32), 0, 0.5)[0]
    assert st == tol(ORC, "orc_", words_of([1], 8), None, 8, np.ones(8, np.uint32), 0, 0.5)[0] == 2


def profile_docs(rng, V, n, bad=None, long_every=0):
    docs = []
    for d in range(n):
        li, lo = int(rng.integers(0, 300)), int(rng.integers(1, 200))
        if long_every and d % long_every == 0:  # past the register-staged size
            li, lo = int(rng.integers(1000, 3000)), int(rng.integers(500, 1500))
        pool = rng.integers(0, V, 64)  # shared ids make copies likely
        inp = np.where(rng.random(li) < 0.5, rng.choice(pool, li), rng.integers(0, V, li))
        out = np.where(rng.random(lo) < 0.5, rng.choice(pool, lo), rng.integers(0, V, lo))
        docs.append((inp.astype(np.uint32), out.astype(np.uint32), int(rng.integers(0, 10**6)) * 7 + d))
    return docs


def orc_profile(V, docs):
    df = np.zeros(V, np.uint32)
    iu, ou = np.zeros((V + 63) // 64, np.uint64), np.zeros((V + 63) // 64, np.uint64)
    stats = []
    for inp, out, idx in docs:
        di, oc, od, bid, side = C.c_uint32(), C.c_double(), C.c_double(), C.c_uint32(), C.c_int()
        st = ORC.orc_profile_doc(V, _p(inp), inp.size, _p(out), out.size, _p(df), _p(iu), _p(ou),
                                 C.byref(di), C.byref(oc), C.byref(od), C.byref(bid),
                                 C.byref(side))
        if st:
            return st, (idx, bid.value, side.value)
        stats.append((idx, di.value, oc.value, od.value))
    stats.sort(key=lambda s: s[0])
    return 0, (df, iu, ou, stats)


def csr(docs):
    ins = [d[0] for d in docs]
    outs = [d[1] for d in docs]
    io = np.concatenate([[0], np.cumsum([a.size for a in ins])]).astype(np.int64)
    oo = np.concatenate([[0], np.cumsum([a.size for a in outs])]).astype(np.int64)
    cat = lambda xs: np.concatenate(xs).astype(np.uint32) if sum(x.size for x in xs) else np.zeros(1, np.uint32)  # noqa: E731
    return cat(ins), io, cat(outs), oo, np.array([d[2] for d in docs], np.int64)


@pytest.mark.skipif(REF is None, reason="reference static library not built")
def test_oracle_profiler_matches_reference():
    rng = np.random.default_rng(77)
    for V in (1, 97, 5000):
        docs = profile_docs(rng, V, 25)
        st, (df, iu, ou, stats) = orc_profile(V, docs)
        assert st == 0
        ii, io, oi, oo, idx = csr(docs)
        n = len(docs)
        rdf = np.zeros(V, np.uint32)
        riu, rou = np.zeros((V + 63) // 64, np.uint64), np.zeros((V + 63) // 64, np.uint64)
        cnt = C.c_int64()
        si = np.zeros(n, np.int64)
        di = np.zeros(n, np.uint32)
        oc = np.zeros(n, np.float64)
        od = np.zeros(n, np.float64)
        assert REF.refs_profile(V, _p(ii), _p(io), _p(oi), _p(oo), _p(idx), n, _p(rdf), _p(riu),
                                _p(rou), C.byref(cnt), _p(si), _p(di), _p(oc), _p(od)) == 0
        assert cnt.value == n and np.array_equal(df, rdf)
        assert np.array_equal(iu, riu) and np.array_equal(ou, rou)
        assert [s[0] for s in stats] == si.tolist() and [s[1] for s in stats] == di.tolist()
        assert np.array_equal(np.array([s[2] for s in stats]).view(np.uint64), oc.view(np.uint64))
        assert np.array_equal(np.array([s[3] for s in stats]).view(np.uint64), od.view(np.uint64))
    # errors: the first failing document, input before output, then empty output
    for mut, code, word in ((lambda d: d[0].__setitem__(0, 999), 4, "input"),
                            (lambda d: d[1].__setitem__(0, 999), 4, "output"),
                            (None, 3, "empty")):
        docs = profile_docs(np.random.default_rng(5), 50, 4)
        docs[2] = (docs[2][0].copy(), docs[2][1].copy() if mut else np.zeros(0, np.uint32),
                   docs[2][2])
        if mut:
            if docs[2][0].size == 0:
                docs[2] = (np.array([1], np.uint32), docs[2][1], docs[2][2])
            mut(docs[2])
        st, info = orc_profile(50, docs)
        ii, io, oi, oo, idx = csr(docs)
        bufs = [np.zeros(50, np.uint32), np.zeros(64, np.uint64), np.zeros(64, np.uint64),
                np.zeros(4, np.int64), np.zeros(4, np.uint32), np.zeros(4), np.zeros(4)]
        cnt = C.c_int64()
        rst = REF.refs_profile(50, _p(ii), _p(io), _p(oi), _p(oo), _p(idx), 4, _p(bufs[0]),
                               _p(bufs[1]), _p(bufs[2]), C.byref(cnt), _p(bufs[3]), _p(bufs[4]),
                               _p(bufs[5]), _p(bufs[6]))
        assert st == rst == code
        msg = REF.refs_last_error().decode()
        assert f"document {docs[2][2]}" in msg and word in msg


# ---- GPU --------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("ctas", [None, "3", "1"], ids=["auto", "3ctas", "1cta"])
def test_gpu_tolerance_filter_matches_oracle(monkeypatch, ctas):
    from paper_2508_15229_b200 import corpus
    from paper_2508_15229_b200.tailored_head import TokenSet

    if ctas is not None:  # the multi-CTA cooperative kernel or the single-CTA one
        monkeypatch.setenv("SVT_TOLERANCE_CTAS", ctas)
    for cand, keep, U, df, M, tau in tol_cases():
        st, kept, pruned, s = tol(ORC, "orc_", cand, keep, U, df, M, tau)
        c = TokenSet(U)
        c.words[:] = cand[: c.words.size]
        k = None
        if keep is not None:
            k = TokenSet(U)
            k.words[:] = keep[: k.words.size]
        r = corpus.tolerance_filter(c, df, M, tau, k)
        assert np.array_equal(r.kept.words, kept[: r.kept.words.size]), (U, tau)
        assert np.array_equal(r.pruned, pruned) and r.pruned_df_sum == s, (U, tau, M)
    # a large case: the full Llama-3.2-1B vocabulary with a heavy-tailed df
    rng = np.random.default_rng(3)
    U = 128256
    cand = np.unique(rng.integers(0, U, 60000))
    df = np.minimum(rng.zipf(1.3, U), 10**6).astype(np.uint32)
    for tau in (0.001, 0.05, 0.3):
        st, kept, pruned, s = tol(ORC, "orc_", words_of(cand, U), None, U, df, 200000, tau)
        c = TokenSet(U)
        c.words[:] = words_of(cand, U)
        r = corpus.tolerance_filter(c, df, 200000, tau)
        assert np.array_equal(r.pruned, pruned) and r.pruned_df_sum == s
    # df values across the whole u32 range (every radix level picks a
    # non-zero digit) with a large budget; sums stay below 2^53
    U = 70000
    cand = np.unique(rng.integers(0, U, 40000))
    df = rng.integers(0, 2**32, U, dtype=np.uint64).astype(np.uint32)
    df[::7] = rng.integers(0, 300, df[::7].size).astype(np.uint32)
    for M, tau in ((10**9, 1e-3), (10**9, 7.0), (10**12, 0.5), (10**15, 1.0)):
        st, kept, pruned, s = tol(ORC, "orc_", words_of(cand, U), None, U, df, M, tau)
        c = TokenSet(U)
        c.words[:] = words_of(cand, U)
        r = corpus.tolerance_filter(c, df, M, tau)
        assert np.array_equal(r.pruned, pruned) and r.pruned_df_sum == s, (M, tau)
        assert np.array_equal(r.kept.words, kept[: r.kept.words.size])
    with pytest.raises(corpus.ConfigError):
        corpus.tolerance_filter(TokenSet(8), np.zeros(8, np.uint32), 0, 0.5)


@pytest.mark.gpu
def test_gpu_profiler_matches_oracle():
    from paper_2508_15229_b200 import corpus

    rng = np.random.default_rng(99)
    for V in (1, 97, 151936, 256000):
        docs = profile_docs(rng, V, 60)
        st, (df, iu, ou, stats) = orc_profile(V, docs)
        p = corpus.profile([corpus.Document(a, b, i) for a, b, i in docs], V)
        assert p.doc_count == 60 and np.array_equal(p.df, df)
        assert np.array_equal(p.input_union.words, iu) and np.array_equal(p.output_union.words, ou)
        got = [(s.doc_index, s.distinct_input, s.overlap_occurrence, s.overlap_distinct)
               for s in p.per_doc]
        assert got == stats  # doubles compared exactly
    # long documents (the global-memory path) interleaved with short ones
    for V in (3000, 151936):
        docs = profile_docs(rng, V, 90, long_every=4)
        st, (df, iu, ou, stats) = orc_profile(V, docs)
        p = corpus.profile([corpus.Document(a, b, i) for a, b, i in docs], V)
        assert np.array_equal(p.df, df)
        assert np.array_equal(p.input_union.words, iu) and np.array_equal(p.output_union.words, ou)
        assert [(s.doc_index, s.distinct_input, s.overlap_occurrence, s.overlap_distinct)
                for s in p.per_doc] == stats
    # shard merge == one profile of all documents; duplicates rejected
    docs = profile_docs(np.random.default_rng(8), 5000, 40)
    a = corpus.profile([corpus.Document(*d) for d in docs[:15]], 5000)
    b = corpus.profile([corpus.Document(*d) for d in docs[15:]], 5000)
    whole = corpus.profile([corpus.Document(*d) for d in docs], 5000)
    m = corpus.merge(a, b)
    assert np.array_equal(m.df, whole.df) and m.per_doc == whole.per_doc
    assert corpus.locality_report(m) == corpus.locality_report(whole)
    with pytest.raises(corpus.IntegrityError, match="duplicate doc_index"):
        corpus.merge(a, a)
    # errors name the first failing document
    bad = [corpus.Document(*d) for d in docs[:5]]
    bad[3] = corpus.Document(bad[3].input_ids, np.zeros(0, np.uint32), bad[3].doc_index)
    bad[4] = corpus.Document(np.array([6000], np.uint32), bad[4].output_ids, bad[4].doc_index)
    with pytest.raises(corpus.ParseError, match=f"document {docs[3][2]} has an empty output"):
        corpus.profile(bad, 5000)
    with pytest.raises(corpus.IntegrityError,
                       match=f"document {docs[4][2]}: input token id 6000 out of range"):
        corpus.profile(bad[4:], 5000)
    # errors inside long documents: the first offending position wins
    li = np.arange(2500, dtype=np.uint32) % 5000
    lo = np.arange(1200, dtype=np.uint32) % 5000
    li2, lo2 = li.copy(), lo.copy()
    lo2[900], lo2[1100] = 7001, 7002
    with pytest.raises(corpus.IntegrityError, match="output token id 7001 out of range"):
        corpus.profile([corpus.Document(li, lo, 0), corpus.Document(li2, lo2, 1)], 5000)
    li2[2100], li2[2300] = 8001, 8002
    with pytest.raises(corpus.IntegrityError, match="input token id 8001 out of range"):
        corpus.profile([corpus.Document(li, lo, 0), corpus.Document(li2, lo2, 1)], 5000)
