"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/svt.h declares, the host-only accounting entry points
agree with the oracle, and compute entry points fail loudly (no CPU fallback)
when no CUDA device is present."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle.oracle import c_oracle

HEADER = os.path.join(ROOT, "include", "svt.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2508_15229_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, missing
    # and the binding declares a signature for each of them
    assert set(syms) <= set(_lib.EXPORTED), set(syms) - set(_lib.EXPORTED)
    assert _lib.lib.svt_abi_version() == 1


def test_dropin_library_loads_and_links_the_cabi():
    import ctypes

    so = os.path.join(ROOT, "paper_2508_15229_b200", "lib", "libsubvocab_b200.so")
    if not os.path.exists(so):
        pytest.skip("C++ drop-in not built")
    ctypes.CDLL(so)


def test_kernels_are_sm100a():
    import subprocess

    so = os.path.join(ROOT, "paper_2508_15229_b200", "lib", "libsvt.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                          text=True).stdout
    assert "UBLKCP" in sass  # bulk-copy (TMA engine) staging in the GEMV ring


def test_host_accounting_matches_oracle():
    from paper_2508_15229_b200 import tailored_head as th

    orc = c_oracle()
    for args in [(128000, 2048, 2, 105), (1000, 64, 4, 1000), (1000, 64, 4, 0), (0, 0, 2, 0),
                 (151936, 896, 2, 2552)]:
        r = th.memory_report(*args)
        assert (r.full_head_bytes, r.sub_head_bytes, r.embedding_bytes_gpu,
                r.embedding_bytes_host, r.saved_fraction) == orc.memory_report(*args)
    with pytest.raises(th.ConfigError):
        th.memory_report(10, 10, 3, 1)
    hw = th.ILLUSTRATIVE_HW
    for plan, dim, b, L, f in [(0, 2048, 2, 512, 2e9), (2555, 2048, 4, 512, 2.4e9),
                               (4047, 3072, 2, 2048, 6e9)]:
        t = th.simulate(hw, plan, dim, b, L, f)
        assert (t.transfer_time, t.prefill_time, t.embedding_time, t.exposed_latency,
                t.hidden) == orc.simulate(*hw, plan, dim, b, L, f)
    for dim, b, L, f in [(2048, 2, 512, 2e9), (896, 4, 64, 5e8)]:
        assert th.breakeven_rows(hw, dim, b, L, f) == orc.breakeven_rows(*hw, dim, b, L, f)
    with pytest.raises(th.ConfigError):
        th.simulate((0.0, 1.0, 1.0), 1, 1, 2, 1, 1.0)
    with pytest.raises(th.ConfigError):
        th.simulate(hw, 1, 0, 2, 1, 1.0)


def test_compute_entry_points_fail_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2508_15229_b200 import _lib

    assert _lib.lib.svt_device_count() == 0
    st = _lib.lib.svt_logits(None, 0, 4, 4, None, None, None)
    assert st == 1 and "no CUDA device" in _lib.last_error()


def test_synthetic_streams_match_oracle_generators():
    from paper_2508_15229_b200 import synth

    orc = c_oracle()
    assert np.array_equal(synth.head_random(7, 13, 0x5EED).view(np.uint32),
                          orc.head_random(7, 13, 0x5EED).view(np.uint32))
    assert np.array_equal(synth.head_random(2, 5, 3, first=11).reshape(-1).view(np.uint32),
                          orc.head_random_slice(11, 10, 3).view(np.uint32))
    assert np.array_equal(synth.static_ids(151936, 2048), orc.static_ids(0x57A7, 151936, 2048))
    assert np.array_equal(synth.prompt_ids(128256, 512, 5), orc.prompt_ids(0x9A0 + 5, 128256, 512))
    x = np.random.default_rng(0).standard_normal(1000).astype(np.float32)
    assert np.array_equal(synth.round_bf16(x).view(np.uint32),
                          np.array([orc.round_bf16(v) for v in x], np.float32).view(np.uint32))
