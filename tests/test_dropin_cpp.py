"""Run the C++ drop-in test program (tests/cpp/test_dropin.cpp, linked against
lib/libsubvocab_b200.so -> lib/libsvt.so) on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "paper_2508_15229_b200", "lib", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_api():
    assert os.path.exists(BIN), "build with __graft_entry__.build()"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_dropin_built():
    assert os.path.exists(BIN)
