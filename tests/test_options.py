"""Host-side contracts of the C library that need no GPU: the explicit
tuning-option API (sfk_set_option, which replaced the round-1 environment
switches) and the kernel instance table that compile_kernel consults so an
unsupported request raises at compile time (reference cli.py:155-208)."""

import pytest

from paper_1711_02473_b200 import compile_kernel, runtime
from paper_1711_02473_b200.errors import NativeError, Unsupported


def test_option_roundtrip_and_restore():
    assert runtime.get_option("c2_kernel") == 0
    with runtime.options(c2_kernel="v5", c2_g=2):
        assert runtime.get_option("c2_kernel") == runtime.C2_KERNELS["v5"]
        assert runtime.get_option("c2_g") == 2
    assert runtime.get_option("c2_kernel") == 0 and runtime.get_option("c2_g") == 0


def test_unknown_option_raises():
    with pytest.raises(NativeError, match="unknown option"):
        runtime.set_option("no_such_option", 1)
    with pytest.raises(NativeError):
        runtime.get_option("SFK_C2_KERNEL")


def test_options_from_env_maps_round1_switches():
    env = {"SFK_C2_KERNEL": "v4", "SFK_COLLOC_WARPS": "0", "SFK_C5_P3": "phase",
           "SFK_LIBRARY": "/x.so", "PATH": "/bin"}
    try:
        got = runtime.options_from_env(env)
        assert got == {"c2_kernel": 6, "colloc_warps": -1, "c5_p3": 1}
    finally:
        for k in ("c2_kernel", "colloc_warps", "c5_p3"):
            runtime.set_option(k, 0)


def test_library_reads_no_dispatch_environment():
    import glob
    import os
    import re

    csrc = os.path.join(os.path.dirname(runtime.__file__), "csrc")
    hits = []
    for f in glob.glob(os.path.join(csrc, "*.c*")):
        for m in re.finditer(r'getenv\("([A-Z_0-9]+)"\)', open(f).read()):
            hits.append(m.group(1))
    assert hits == ["SFK_NVRTC"], hits   # a library search path, not a dispatch switch


@pytest.mark.parametrize("form,cell,p,kw", [
    ("action_mass", "hex", 1, {}), ("action_mass", "hex", 8, {}),
    ("action_mass", "hex", 3, {"quadrature": 5}),
    ("action_mass", "hex", 6, {"variant": "spectral_gll", "quadrature": "collocated-gll"}),
    ("action_laplace", "hex", 9, {}), ("action_laplace", "quad", 8, {}),
    ("action_laplace", "quad", 16, {}), ("action_mass", "quad", 12, {}),
    ("laplace", "hex", 4, {}), ("laplace", "hex", 5, {}), ("laplace", "hex", 8, {}),
    ("action_laplace", "hex", 16, {"variant": "spectral_gll", "quadrature": "collocated-gll"}),
])
def test_supported_requests_compile(form, cell, p, kw):
    plan = compile_kernel(form, cell, p, **kw)
    assert runtime.kernel_available(plan.kind, plan.dim, plan.n, plan.m, plan.collocated)


@pytest.mark.parametrize("form,cell,p,kw", [
    ("action_laplace", "quad", 17, {}),       # quad kernel stops at n = 17 (p = 16)
    ("action_mass", "quad", 3, {"quadrature": 5}),   # quad: m == n only
    ("laplace", "hex", 9, {}),                # local matrices: p <= 8
    ("laplace", "hex", 2, {"quadrature": 4}),  # matrices need m == n
    ("action_laplace", "hex", 10, {}),        # n = 11 > the line-kernel table
    ("action_laplace", "hex", 2, {"quadrature": 7}),
])
def test_unsupported_requests_raise_at_compile(form, cell, p, kw):
    with pytest.raises(Unsupported):
        compile_kernel(form, cell, p, **kw)


def test_plan_create_rejects_what_the_table_rejects():
    import ctypes

    import numpy as np

    lib = runtime.load_library()
    z = np.zeros(18 * 18)
    ptr = z.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    out = ctypes.c_void_p()
    # hex laplace matrix at n = 10 (p = 9): no kernel -> SFK_EUNSUPPORTED at create
    assert lib.sfk_kernel_available(4, 3, 10, 10, 0) == 0
    assert lib.sfk_kernel_available(4, 3, 9, 9, 0) == 1
    rc = lib.sfk_plan_create(4, 3, 9, 10, 10, 0, ptr, ptr, ptr, ptr, ptr, ptr, None, 0,
                             ctypes.byref(out))
    assert rc == 2 and not out.value
    assert lib.sfk_kernel_available(3, 3, 4, 4, 0) == 1   # hex action_mass
