"""CPU checks of the C-ABI boundary: libghsvd.so loads without a GPU and exports
every function include/ghsvd.h declares; host-side argument checks."""
import ctypes
import os
import re

import pytest

from paper_1907_08560_b200 import build, ghsvd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return ghsvd.load()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ghsvd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ghsvd_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_five_north_star_calls():
    fns = header_functions()
    for f in ("ghsvd_create", "ghsvd_factor", "ghsvd_reduce", "ghsvd_sweep", "ghsvd_extract"):
        assert f in fns


def test_every_declared_symbol_is_exported(lib):
    fns = header_functions()
    assert sorted(fns) == sorted(ghsvd.EXPORTS)
    for f in fns:
        assert hasattr(lib, f), f


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ghsvd.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_options_and_workspace(lib):
    o = ghsvd.Options()
    lib.ghsvd_default_options(ctypes.byref(o))
    assert o.world_size == 1 and o.max_sweeps == 30 and o.variant == 0 and o.use_graph == 1
    b1 = lib.ghsvd_workspace_bytes(ctypes.byref(o), 512, 256, 0)
    b2 = lib.ghsvd_workspace_bytes(ctypes.byref(o), 1024, 256, 0)
    assert b1 > 3 * 512 * 256 * 16 and b2 > b1
    # invalid sizes / options -> 0
    assert lib.ghsvd_workspace_bytes(ctypes.byref(o), 10, 20, 0) == 0      # m < n
    o.max_sweeps = 0
    assert lib.ghsvd_workspace_bytes(ctypes.byref(o), 10, 5, 0) == 0
    o.max_sweeps = 30
    o.nblocks = 3                                                          # odd block count
    assert lib.ghsvd_workspace_bytes(ctypes.byref(o), 10, 5, 0) == 0
    o.nblocks = 0
    o.world_size = 2                                                       # no nccl id
    assert lib.ghsvd_workspace_bytes(ctypes.byref(o), 10, 5, 0) == 0


def test_create_rejects_bad_args_before_touching_cuda(lib):
    o = ghsvd.Options()
    lib.ghsvd_default_options(ctypes.byref(o))
    h = ctypes.c_void_p()
    assert lib.ghsvd_create(ctypes.byref(o), 16, 8, 0, None, 0, ctypes.byref(h)) == -1
    need = lib.ghsvd_workspace_bytes(ctypes.byref(o), 16, 8, 0)
    buf = ctypes.create_string_buffer(16)
    assert lib.ghsvd_create(ctypes.byref(o), 16, 8, 0, buf, need - 1, ctypes.byref(h)) == -5
    assert lib.ghsvd_last_error(None) == b"null context"
    assert lib.ghsvd_sweep(None, None) == -1
    lib.ghsvd_destroy(None)
    assert b"sm_100a" in lib.ghsvd_version()


def test_c_demo_builds_as_plain_c99():
    """The public header is plain C: examples/c_demo.c compiles with gcc -std=c99 -pedantic
    -Wall -Wextra against include/ghsvd.h and links libghsvd.so (run on the GPU by
    tests/test_gpu_c_demo.py)."""
    from paper_1907_08560_b200 import build
    exe = build.build_c_demo(force=True)
    assert os.path.exists(exe) and os.access(exe, os.X_OK)
