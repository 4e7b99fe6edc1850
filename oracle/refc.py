"""ctypes driver of oracle/_ref (the reference's own emitted C, compiled with
an OpenMP cell loop by oracle/gen_ref.py) — TEST/BASELINE INFRASTRUCTURE
ONLY (see oracle/__init__.py).  Used by bench.py as the "reference" CPU arm
and by tests as a third oracle when present."""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
_libs = {}


def key_for(plan):
    name, cell, p = plan.name, plan.meta["cell"], plan.degree
    if cell == "hex" and name == "action_laplace" and not plan.collocated and plan.m == plan.n \
            and plan.meta.get("variant") == "equispaced":
        return "c2_p%d" % p
    if cell == "hex" and name == "laplace" and plan.m == plan.n:
        return "c5_p%d" % p
    if cell == "quad" and p == 3 and plan.m == 4:
        return "c1_%s" % name
    if cell == "hex" and name == "action_weighted_laplace" and plan.collocated:
        return "c3_p%d" % p
    if cell == "hex" and name == "neohookean_residual" and plan.m == plan.n + 1:
        return "c4_p%d" % p
    return None


def available(plan, build="parity"):
    k = key_for(plan)
    sfx = "_fast" if build == "fast" else ""
    return k is not None and os.path.exists(os.path.join(OUT, "libref_%s%s.so" % (k, sfx)))


def _lib(key, build="parity"):
    """build: "parity" (-O3 -march=native -ffp-contract=off) or "fast"
    (-ffast-math, the paper's flags)."""
    if (key, build) not in _libs:
        path = os.path.join(OUT, "libref_%s%s.so" % (key, "_fast" if build == "fast" else ""))
        L = ctypes.CDLL(path)
        L.sumfact_ref_run.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 4
        L.sumfact_ref_threads.restype = ctypes.c_int
        if hasattr(L, "sumfact_ref_set_threads"):
            L.sumfact_ref_set_threads.argtypes = [ctypes.c_int]
        meta = json.load(open(os.path.join(OUT, "src", key + ".json")))
        _libs[(key, build)] = (L, meta)
    return _libs[(key, build)]


def threads(plan, build="parity"):
    return _lib(key_for(plan), build)[0].sumfact_ref_threads()


def set_threads(plan, n, build="parity"):
    """OpenMP threads of the cell loop (0 = all host cores)."""
    L = _lib(key_for(plan), build)[0]
    if not hasattr(L, "sumfact_ref_set_threads"):
        raise RuntimeError("oracle/_ref predates the thread control; rerun build()")
    L.sumfact_ref_set_threads(int(n))


def evaluate(plan, inputs, out=None, build="parity"):
    """Run the reference's emitted kernel over every cell (OpenMP)."""
    key = key_for(plan)
    L, meta = _lib(key, build)
    assert [tuple(a) for a in meta["arguments"]] == [tuple(a) for a in plan.arguments], \
        (meta["arguments"], plan.arguments)
    arrs = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in inputs.items()}
    ncells = arrs["coords"].shape[0]
    if out is None:
        out = np.empty((ncells, plan.return_size))
    ptr = lambda k: arrs[k].ctypes.data if k in arrs else None  # noqa: E731
    L.sumfact_ref_run(ncells, out.ctypes.data, ptr("coords"), ptr("w0"), ptr("w1"))
    return out
