"""The C-ABI library: builds, loads, exports every symbol of include/sfk.h,
and its host-only entry points behave (CPU — no kernel is launched)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1711_02473_b200 import compile_kernel, runtime
from paper_1711_02473_b200.errors import NativeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "sfk.h")).read()
    return sorted(set(re.findall(r"\b(sfk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = runtime.load_library()
    declared = _header_functions()
    assert set(declared) == set(runtime.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sfk_abi_version() == 1


def test_plan_create_sizes_destroy_on_host():
    lib = runtime.load_library()
    plan = compile_kernel("action_laplace", "hex", 3)
    h = runtime.native_plan(plan)
    vals = [ctypes.c_int64() for _ in range(4)]
    assert lib.sfk_plan_sizes(h, *[ctypes.byref(v) for v in vals]) == 0
    assert [v.value for v in vals] == [24, 64, 0, 64]


def test_error_paths_without_gpu():
    lib = runtime.load_library()
    out = ctypes.c_void_p()
    z = np.zeros(64)
    p = z.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    # unknown kind -> SFK_EINVAL with a message
    rc = lib.sfk_plan_create(99, 3, 1, 2, 2, 0, p, p, p, p, p, p, None, 0, ctypes.byref(out))
    assert rc == 1
    buf = ctypes.create_string_buffer(256)
    lib.sfk_last_error(buf, 256)
    assert b"unknown kind" in buf.value
    # too many dofs per axis -> SFK_EUNSUPPORTED
    rc = lib.sfk_plan_create(1, 3, 30, 31, 31, 0, p, p, p, p, p, p, None, 0, ctypes.byref(out))
    assert rc == 2
    # NULL plan / negative count -> SFK_EINVAL; zero cells is a no-op
    assert lib.sfk_eval(None, 1, None, None, None, None, None) == 1
    plan = compile_kernel("action_laplace", "hex", 1)
    h = runtime.native_plan(plan)
    assert lib.sfk_eval(h, -1, None, None, None, None, None) == 1
    assert lib.sfk_eval(h, 0, None, None, None, None, None) == 0
    with pytest.raises(NativeError):
        runtime._check(1)


def test_mesh_error_paths_without_gpu():
    """sfk_mesh_* validate before touching the device (include/sfk.h)."""
    lib = runtime.load_library()
    out = ctypes.c_void_p()
    assert lib.sfk_mesh_create(10, 7, ctypes.byref(out)) == 1          # coords_size 24 or 8
    assert lib.sfk_mesh_create(-1, 24, ctypes.byref(out)) == 1
    assert lib.sfk_mesh_create(10, 24, None) == 1
    assert lib.sfk_mesh_upload(None, None) == 1
    assert lib.sfk_mesh_coords(None) is None
    assert lib.sfk_mesh_destroy(None) == 0
    plan = compile_kernel("action_laplace", "hex", 2)
    h = runtime.native_plan(plan)
    assert lib.sfk_eval_host_mesh(h, None, 0, 1, None, None, None, 0, 1) == 1
