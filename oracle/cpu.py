"""ctypes driver of oracle/liboracle.so — TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).  Builds the library with gcc on first use."""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sumfact_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
# Parity build of the reference's emitted C: no FMA
# contraction, so the oracle's rounding is the plain C semantics.
CFLAGS = ["-O3", "-march=native", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared"]

_lib = None
_lock = threading.Lock()
_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_ci = ctypes.c_int
_cd = ctypes.c_double


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.run(["gcc"] + CFLAGS + ["-o", tmp, SRC, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                build()
                L = ctypes.CDLL(LIB)
                L.oracle_hex_laplace_action.argtypes = [_ci, _ci] + [_dp] * 5 + [_i64, _dp, _dp, _dp]
                L.oracle_hex_colloc_action.argtypes = [_ci] + [_dp] * 4 + [_i64, _dp, _dp, _dp, _dp]
                L.oracle_quad_action.argtypes = [_ci, _ci, _ci] + [_dp] * 5 + [_i64, _dp, _dp, _dp]
                L.oracle_hex_laplace_matrix.argtypes = [_ci, _ci] + [_dp] * 5 + [_i64, _dp, _dp]
                L.oracle_hex_neohookean.argtypes = ([_ci, _ci] + [_dp] * 5 + [_cd, _cd, _i64]
                                                    + [_dp] * 3)
                L.oracle_num_threads.restype = _ci
                _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads():
    return lib().oracle_num_threads()


def evaluate(plan, inputs):
    """Evaluate a KernelPlan on host arrays with the C oracle."""
    L = lib()
    coords = _c(inputs["coords"])
    ncells = coords.shape[0]
    B, D, w, Bc, Dc = (_c(plan.B), _c(plan.D), _c(plan.wq), _c(plan.Bc), _c(plan.Dc))
    out = np.empty((ncells, plan.return_size))
    name, cell = plan.name, plan.meta["cell"]
    if cell == "hex" and name == "action_laplace" and not plan.collocated:
        L.oracle_hex_laplace_action(plan.n, plan.m, _p(B), _p(D), _p(w), _p(Bc), _p(Dc),
                                    ncells, _p(coords), _p(_c(inputs["w0"])), _p(out))
    elif cell == "hex" and name in ("action_laplace", "action_weighted_laplace") and plan.collocated:
        kappa = _c(inputs["w1"]) if name == "action_weighted_laplace" else None
        L.oracle_hex_colloc_action(plan.n, _p(D), _p(w), _p(Bc), _p(Dc), ncells, _p(coords),
                                   _p(_c(inputs["w0"])), _p(kappa), _p(out))
    elif cell == "quad" and name in ("action_mass", "action_laplace"):
        L.oracle_quad_action(0 if name == "action_mass" else 1, plan.n, plan.m, _p(B), _p(D),
                             _p(w), _p(Bc), _p(Dc), ncells, _p(coords),
                             _p(_c(inputs["w0"])), _p(out))
    elif cell == "hex" and name == "laplace":
        L.oracle_hex_laplace_matrix(plan.n, plan.m, _p(B), _p(D), _p(w), _p(Bc), _p(Dc),
                                    ncells, _p(coords), _p(out))
    elif cell == "hex" and name == "neohookean_residual":
        mu, lam = plan.params
        L.oracle_hex_neohookean(plan.n, plan.m, _p(B), _p(D), _p(w), _p(Bc), _p(Dc), mu, lam,
                                ncells, _p(coords), _p(_c(inputs["w0"])), _p(out))
    else:
        raise NotImplementedError("no oracle for %r" % plan)
    return out
