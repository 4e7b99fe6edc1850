"""The CPU oracles (oracle/cpu.py C restatement, oracle/dense.py numpy
restatement) against the reference's own outputs (tests/golden, produced by
reference forms.evaluate_kernel) and the analytic known answers of
SPEC.md:611-618 / SURVEY.md §4.  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from oracle import cpu, dense
from paper_1711_02473_b200 import (REGISTRY, action_form, compile_form, compile_kernel,
                                   neohookean_residual_form, workloads)

TOL = 1e-13


@pytest.mark.parametrize("p", range(1, 9))
def test_c2_golden(p):
    g = np.load(os.path.join(GOLDEN, "c2.npz"))
    plan = compile_kernel("action_laplace", "hex", p)
    inp = {"coords": g["coords"], "w0": g["w0_p%d" % p]}
    assert rel_err(cpu.evaluate(plan, inp), g["A_p%d" % p]) < TOL
    assert rel_err(dense.evaluate(plan, inp), g["A_p%d" % p]) < TOL


@pytest.mark.parametrize("p", [1, 2, 4, 6, 8, 12, 16])
def test_c3_golden(p):
    g = np.load(os.path.join(GOLDEN, "c3.npz"))
    spec = action_form(REGISTRY["weighted_laplace"])
    plan = compile_form(spec, "hex", p, "spectral", "spectral_gll", "collocated-gll")
    inp = {"coords": g["coords"], "w0": g["w0_p%d" % p], "w1": g["w1_p%d" % p]}
    assert rel_err(cpu.evaluate(plan, inp), g["A_p%d" % p]) < TOL
    if p <= 8:
        assert rel_err(dense.evaluate(plan, inp), g["A_p%d" % p]) < TOL
    plan2 = compile_kernel("action_laplace", "hex", p, "spectral", "spectral_gll",
                           "collocated-gll")
    assert rel_err(cpu.evaluate(plan2, inp), g["Alap_p%d" % p]) < TOL


@pytest.mark.parametrize("p", range(1, 7))
def test_c4_golden(p):
    g = np.load(os.path.join(GOLDEN, "c4.npz"))
    plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
    with np.errstate(invalid="ignore"):
        for s in ("", "b"):
            inp = {"coords": g["coords"], "w0": g["w0%s_p%d" % (s, p)]}
            ref = g["A%s_p%d" % (s, p)]
            out = cpu.evaluate(plan, inp)
            # the config's own draw inverts elements at p=6: NaN where the
            # reference is NaN (ln of a negative J), equal elsewhere
            assert np.array_equal(np.isnan(out), np.isnan(ref))
            ok = ~np.isnan(ref).any(axis=1)
            if ok.any():
                assert rel_err(out[ok], ref[ok]) < TOL
                assert rel_err(dense.evaluate(plan, inp)[ok], ref[ok]) < TOL


@pytest.mark.parametrize("p", range(1, 5))
def test_c5_golden(p):
    g = np.load(os.path.join(GOLDEN, "c5.npz"))
    plan = compile_kernel("laplace", "hex", p)
    assert rel_err(cpu.evaluate(plan, {"coords": g["coords"]}), g["A_p%d" % p]) < TOL
    assert rel_err(dense.evaluate(plan, {"coords": g["coords"]}), g["A_p%d" % p]) < TOL


def test_c1_golden():
    g = np.load(os.path.join(GOLDEN, "c1.npz"))
    for form in ("action_mass", "action_laplace"):
        plan = compile_kernel(form, "quad", 3)
        inp = {"coords": g["coords"], "w0": g["w0"]}
        assert rel_err(cpu.evaluate(plan, inp), g["A_" + form]) < TOL
        assert rel_err(dense.evaluate(plan, inp), g["A_" + form]) < TOL


def test_analytic_q1_matrices():
    # Q1 quad stiffness = K(x)M + M(x)K, hex analogue
    M = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    K = np.array([[1.0, -1.0], [-1.0, 1.0]])
    g = np.load(os.path.join(GOLDEN, "c5.npz"))
    plan = compile_kernel("laplace", "hex", 1)
    A = cpu.evaluate(plan, {"coords": g["ref_coords"]}).reshape(8, 8)
    expect = (np.kron(np.kron(K, M), M) + np.kron(np.kron(M, K), M)
              + np.kron(np.kron(M, M), K))
    assert np.abs(A - expect).max() < 1e-14
    assert np.abs(A - g["A_ref_p1"].reshape(8, 8)).max() < 1e-15
    # quad mass on the unit square via the action with unit vectors
    plan = compile_kernel("action_mass", "quad", 1)
    sq = np.array([[0.0, 0.0, 0.0, 1.0, 1.0, 0.0, 1.0, 1.0]])
    cols = [cpu.evaluate(plan, {"coords": sq, "w0": e[None]})[0] for e in np.eye(4)]
    assert np.abs(np.array(cols).T - np.kron(M, M)).max() < 1e-15


def test_properties_patch_symmetry_consistency():
    coords = workloads.lattice_coords(2, 2, 2)
    p = 2
    mat = cpu.evaluate(compile_kernel("laplace", "hex", p), {"coords": coords})
    A = mat.reshape(-1, 27, 27)
    assert np.abs(A.sum(axis=2)).max() < 1e-13           # patch test
    assert np.abs(A - A.transpose(0, 2, 1)).max() < 1e-15  # symmetry
    u = workloads.uniform_dofs(coords.shape[0], 27)
    act = cpu.evaluate(compile_kernel("action_laplace", "hex", p),
                       {"coords": coords, "w0": u})
    assert rel_err(act, np.einsum("cij,cj->ci", A, u)) < 1e-13


MASS_CASES = ([("gl", p) for p in range(1, 9)] + [("glp2", p) for p in (1, 2, 4)]
              + [("gll", p) for p in (2, 4, 7)])


def mass_plan(tag, p):
    if tag == "gl":
        return compile_kernel("action_mass", "hex", p)
    if tag == "glp2":
        return compile_kernel("action_mass", "hex", p, quadrature=p + 2)
    return compile_kernel("action_mass", "hex", p, "spectral", "spectral_gll", "collocated-gll")


@pytest.mark.parametrize("tag,p", MASS_CASES)
def test_hex_mass_golden(tag, p):
    """Hex action_mass: the dense numpy restatement against the reference's
    own eval_expr outputs (tests/golden/make_golden.py mass_hex)."""
    g = np.load(os.path.join(GOLDEN, "mass_hex.npz"))
    plan = mass_plan(tag, p)
    inp = {"coords": g["coords"], "w0": g["w0_%s_p%d" % (tag, p)]}
    assert rel_err(dense.evaluate(plan, inp), g["A_%s_p%d" % (tag, p)]) < TOL


def _refc_or_skip(plan):
    from oracle import refc
    if not refc.available(plan):
        pytest.skip("oracle/_ref (reference emitted C) not generated")
    return refc


@pytest.mark.parametrize("cfg,p", [("C2", p) for p in range(1, 9)] + [("C3", p) for p in (4, 8, 12, 16)]
                         + [("C4", p) for p in range(2, 7)] + [("C5", p) for p in range(1, 5)])
def test_oracle_port_vs_reference_emitted_c(cfg, p):
    """The C restatement (oracle/cpu.py) against the reference's OWN emitted
    C (oracle/_ref, built by gen_ref.py through the reference API) on 256
    cells of each config's generator — a larger pin than the golden cells."""
    if cfg == "C2":
        plan = compile_kernel("action_laplace", "hex", p)
        inp = workloads.c2_inputs(p, dims=(4, 8, 8))
    elif cfg == "C3":
        plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p, "spectral",
                            "spectral_gll", "collocated-gll")
        inp = workloads.c3_inputs(p, dims=(4, 8, 8))
    elif cfg == "C4":
        plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
        inp = workloads.c4_inputs(p, dims=(4, 8, 8))
    else:
        plan = compile_kernel("laplace", "hex", p)
        inp = workloads.c5_inputs(0, 1, (2, 4, 8))
    refc = _refc_or_skip(plan)
    with np.errstate(invalid="ignore"):
        ref = refc.evaluate(plan, inp)
        out = cpu.evaluate(plan, inp)
    assert np.array_equal(np.isnan(out), np.isnan(ref))
    ok = ~np.isnan(ref).any(axis=1)
    if ok.any():
        # C4 p = 5: cells the config's draw nearly inverts amplify rounding
        tol = 1e-12 if cfg == "C4" and p == 5 else TOL
        assert rel_err(out[ok], ref[ok]) < tol
