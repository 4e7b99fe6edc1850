"""Host tabulation and plan metadata vs the reference (CPU).

Pins (SURVEY.md §8(c) 'What pins the results'):
* GL/GLL points and weights, 1D Lagrange tables: np.array_equal with the
  reference's own arrays (tests/golden/tables.npz, made by make_golden.py);
* known answers of SPEC.md:136-145 (GL(1), GL(2), GLL(2), GLL(3));
* plan ABI metadata identical to the reference LoopProgram's
  (name, arguments, return_buffer, meta; scheduling.py:87-95);
* reference flop counts (tests/golden/flops.json) = our F formulas.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1711_02473_b200 import (REGISTRY, UsageError, action_form, compile_form,
                                   compile_kernel, gauss_legendre,
                                   gauss_lobatto_legendre, lagrange_interval,
                                   lagrange_tables, neohookean_residual_form)
from paper_1711_02473_b200.errors import InvalidArity, Unsupported

T = np.load(os.path.join(GOLDEN, "tables.npz"))


@pytest.mark.parametrize("m", range(1, 19))
def test_gauss_legendre_bit_exact(m):
    r = gauss_legendre(m)
    assert np.array_equal(r.point_set.points, T["gl_x_%d" % m])
    assert np.array_equal(r.weights, T["gl_w_%d" % m])


@pytest.mark.parametrize("m", range(2, 19))
def test_gauss_lobatto_bit_exact(m):
    r = gauss_lobatto_legendre(m)
    assert np.array_equal(r.point_set.points, T["gll_x_%d" % m])
    assert np.array_equal(r.weights, T["gll_w_%d" % m])


def _combos():
    for key in T.files:
        if key.startswith("B_"):
            yield key[2:]


@pytest.mark.parametrize("key", sorted(_combos()))
def test_lagrange_tables_bit_exact(key):
    variant, rest = key.rsplit("_p", 1)
    p, fam = rest.split("_")
    p = int(p)
    m = int(fam[3:] if fam.startswith("gll") else fam[2:])
    rule = gauss_lobatto_legendre(m) if fam.startswith("gll") else gauss_legendre(m)
    el = lagrange_interval(p, variant)
    assert np.array_equal(el.nodes, T["nodes_" + key])
    t = lagrange_tables(el.nodes, rule.point_set.points, 1)
    assert np.array_equal(t[0], T["B_" + key])
    assert np.array_equal(t[1], T["D_" + key])


def test_known_quadrature_answers():
    # SPEC.md:136-145
    r = gauss_legendre(1)
    assert r.point_set.points.tolist() == [0.5] and r.weights.tolist() == [1.0]
    r = gauss_legendre(2)
    s = 1 / np.sqrt(3)
    assert np.allclose(r.point_set.points, [(1 - s) / 2, (1 + s) / 2], atol=1e-15)
    assert np.allclose(r.weights, [0.5, 0.5], atol=1e-15)
    r = gauss_lobatto_legendre(2)
    assert r.point_set.points.tolist() == [0.0, 1.0]
    r = gauss_lobatto_legendre(3)
    assert np.allclose(r.point_set.points, [0, 0.5, 1], atol=1e-15)
    assert np.allclose(r.weights, [1 / 6, 2 / 3, 1 / 6], atol=1e-15)
    with pytest.raises(InvalidArity):
        gauss_legendre(0)
    with pytest.raises(InvalidArity):
        gauss_lobatto_legendre(1)


@pytest.mark.parametrize("m", [2, 5, 9, 17])
def test_quadrature_exactness(m):
    # GL(m) exact to degree 2m-1, GLL(m) to 2m-3 on [0,1]
    r = gauss_legendre(m)
    x, w = r.point_set.points, r.weights
    for k in range(2 * m):
        assert abs(np.dot(w, x ** k) - 1 / (k + 1)) < 1e-13
    r = gauss_lobatto_legendre(m)
    x, w = r.point_set.points, r.weights
    for k in range(2 * m - 2):
        assert abs(np.dot(w, x ** k) - 1 / (k + 1)) < 1e-13


def test_plan_metadata_matches_reference_loopprogram():
    # reference: cli.compile_kernel('action_laplace','hex',p,'spectral') has
    # arguments [('coords', 24), ('w0', (p+1)**3)], return ('A', (p+1)**3)
    for p in range(1, 9):
        plan = compile_kernel("action_laplace", "hex", p, "spectral")
        assert plan.name == "action_laplace"
        assert plan.arguments == [("coords", 24), ("w0", (p + 1) ** 3)]
        assert plan.return_buffer == ("A", (p + 1) ** 3)
        assert plan.meta == {"form": "action_laplace", "cell": "hex", "degree": p,
                             "mode": "spectral", "variant": "equispaced"}
        assert plan.n == p + 1 and plan.m == p + 1 and not plan.collocated
    plan = compile_kernel("laplace", "hex", 2, "spectral")
    assert plan.arguments == [("coords", 24)] and plan.return_buffer == ("A", 729)
    plan = compile_kernel("action_mass", "quad", 3, "spectral")
    assert plan.arguments == [("coords", 8), ("w0", 16)] and plan.return_buffer == ("A", 16)
    spec = action_form(REGISTRY["weighted_laplace"])
    plan = compile_form(spec, "hex", 4, "spectral", "spectral_gll", "collocated-gll")
    assert plan.name == "action_weighted_laplace"
    assert plan.arguments == [("coords", 24), ("w0", 125), ("w1", 125)]
    assert plan.collocated and np.array_equal(plan.B, np.eye(5))
    plan = compile_form(neohookean_residual_form(), "hex", 3, quadrature=5)
    assert plan.arguments == [("coords", 24), ("w0", 192)]
    assert plan.return_buffer == ("A", 192) and plan.m == 5


def test_reference_flop_counts_pinned():
    with open(os.path.join(GOLDEN, "flops.json")) as f:
        ref = json.load(f)
    for p in range(1, 9):
        assert compile_kernel("action_laplace", "hex", p).reference_flops == ref["C2_p%d" % p]
    for p in range(1, 5):
        assert compile_kernel("laplace", "hex", p).reference_flops == ref["C5_p%d" % p]
    for form in ("action_mass", "action_laplace"):
        assert compile_kernel(form, "quad", 3).reference_flops == ref["C1_" + form]


def test_usage_errors_mirror_reference():
    with pytest.raises(UsageError):
        compile_kernel("nope", "hex", 1)
    with pytest.raises(UsageError):
        compile_kernel("laplace", "cube", 1)
    with pytest.raises(UsageError):
        compile_kernel("laplace", "hex", 1, "fast")
    with pytest.raises(UsageError):
        compile_kernel("laplace", "hex", 0)
    with pytest.raises(UsageError):
        compile_kernel("action_laplace", "hex", 2, quadrature="collocated-gll")
    with pytest.raises(UsageError):
        compile_kernel("action_laplace", "hex", 2, quadrature="x")
    with pytest.raises(Unsupported):
        compile_kernel("stokes_momentum", "hex", 2)
    with pytest.raises(Unsupported):
        compile_kernel("laplace", "triangle", 2)
