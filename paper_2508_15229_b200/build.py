"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

* lib/libsvt.so          — the sm_100a CUDA kernels + C-ABI (include/svt.h)
* lib/libsubvocab_b200.so — the C++ drop-in of the reference API
                            (include/subvocab/*.hpp) over the C-ABI

Compiled with ``-gencode arch=compute_100a,code=sm_100a`` (NOT ``-arch=sm_100a``,
which also embeds compute_100 PTX that ptxas rejects for tcgen05/bulk ops).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
HOST = os.path.join(CSRC, "host")
LIB = os.path.join(HERE, "lib")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "--expt-relaxed-constexpr"]


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_svt(force=False):
    """One object per translation unit, compiled in parallel (only the stale
    ones), then one shared-library link."""
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(LIB, exist_ok=True)
    obj_dir = os.path.join(LIB, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    out = os.path.join(LIB, "libsvt.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "svt.h")]
    objs = [os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(o, [s] + headers)]

    def compile_one(so):
        src, obj = so
        _run([NVCC, *NVFLAGS, *ARCH, "-c", "-I", INCLUDE, "-I", CSRC, src, "-o", obj])

    if todo:
        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(compile_one, todo))
    if force or todo or _stale(out, objs):
        _run([NVCC, *ARCH, "-shared", *objs, "-o", out, "-lcudart", "-ldl"])
    return out


def build_dropin(force=False):
    out = os.path.join(LIB, "libsubvocab_b200.so")
    srcs = sorted(glob.glob(os.path.join(HOST, "*.cpp")))
    if not srcs:
        return None
    deps = srcs + glob.glob(os.path.join(INCLUDE, "subvocab", "*.hpp")) + [
        os.path.join(INCLUDE, "svt.h"), os.path.join(LIB, "libsvt.so")]
    if force or _stale(out, deps):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-I", INCLUDE,
              *srcs, "-o", out, "-L", LIB, "-lsvt", "-Wl,-rpath,$ORIGIN"])
    return out


def build_dropin_test(force=False):
    """C++ test of the drop-in API (tests/cpp), run on the GPU by
    tests/test_dropin_cpp.py."""
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    out = os.path.join(LIB, "test_dropin")
    if not os.path.exists(src):
        return None
    deps = [src, os.path.join(ROOT, "tests", "cpp", "mini_test.hpp"),
            os.path.join(LIB, "libsubvocab_b200.so")]
    if force or _stale(out, deps):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=c++20", "-O2", "-ffp-contract=off", "-I", INCLUDE, src, "-o", out,
              "-L", LIB, "-lsubvocab_b200", "-lsvt", "-Wl,-rpath,$ORIGIN"])
    return out


def build_dropin_bench(force=False):
    """C++ drop-in timing at cfg1 (tests/cpp/bench_dropin_cfg1.cpp)."""
    src = os.path.join(ROOT, "tests", "cpp", "bench_dropin_cfg1.cpp")
    out = os.path.join(LIB, "bench_dropin_cfg1")
    deps = [src, os.path.join(LIB, "libsubvocab_b200.so")]
    if force or _stale(out, deps):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=c++20", "-O2", "-I", INCLUDE, src, "-o", out, "-L", LIB,
              "-lsubvocab_b200", "-lsvt", "-Wl,-rpath,$ORIGIN"])
    return out


def build_all(force=False):
    build_svt(force)
    build_dropin(force)
    build_dropin_test(force)
    build_dropin_bench(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
