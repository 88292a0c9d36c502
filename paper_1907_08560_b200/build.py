"""Build libghsvd.so (the C-ABI library) in-tree with nvcc for sm_100a.

Usage: python -m paper_1907_08560_b200.build [--force]
Objects are compiled in parallel into build/ and linked with the static
CUDA runtime; NCCL is loaded at run time with dlopen (comm.cpp), so the
library loads on hosts without a GPU or NCCL (CPU tests check its symbols).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "ghsvd")
LIB = os.path.join(HERE, "libghsvd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "ghsvd.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    # GHSVD_NVCC_EXTRA: extra nvcc flags for A/B builds of the tools (e.g. -DGHSVD_GRAM_RT=48)
    cmd = [NVCC] + ARCH + FLAGS + os.environ.get("GHSVD_NVCC_EXTRA", "").split() + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    tmp = LIB + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


DEMO_SRC = os.path.join(ROOT, "examples", "c_demo.c")
DEMO = os.path.join(ROOT, "build", "c_demo")


def build_c_demo(force: bool = False) -> str:
    """examples/c_demo.c: a plain-C99 program against include/ghsvd.h and libghsvd.so
    (proves the boundary is usable without Python; run by a GPU test)."""
    lib = build()
    if not force and os.path.exists(DEMO) and os.path.getmtime(DEMO) >= max(
            os.path.getmtime(lib), os.path.getmtime(DEMO_SRC), os.path.getmtime(os.path.join(ROOT, "include", "ghsvd.h"))):
        return DEMO
    os.makedirs(os.path.dirname(DEMO), exist_ok=True)
    cuda = os.path.dirname(os.path.dirname(NVCC))
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-pedantic", DEMO_SRC, "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(cuda, "include"), "-L" + HERE, "-lghsvd", "-L" + os.path.join(cuda, "lib64"),
           "-lcudart", "-lm", "-Wl,-rpath," + HERE, "-o", DEMO]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"c_demo build failed:\n{r.stdout}\n{r.stderr}")
    return DEMO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
