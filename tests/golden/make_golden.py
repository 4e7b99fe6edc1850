"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are frozen here
as small .npz fixtures:

* tables.npz     GL/GLL points+weights (quadrature.py:221-240) and the 1D
                 Lagrange tables (elements.py:163-177) for every (variant, n,
                 points) the B200 kernels use — pins the host tabulation
                 bit-for-bit;
* c1.npz .. c5_*.npz   a few seeded cells per config and degree with the
                 reference tier-1 oracle output ``forms.evaluate_kernel`` of
                 the unoptimised lowering (forms.py:431-447, interpreter
                 eval_expr) — the ground truth of SURVEY.md §8(c);
* flops.json     ``scheduling.count_flops`` of the spectral-mode program
                 (scheduling.py:416-437) for the registry configs — pins the
                 F_alg formulas of SURVEY.md §8(d).

C4 (neo-Hookean) has no reference form: its builder below
composes reference IR nodes exactly as SURVEY.md §8(a) row a17 prescribes,
and the reference lowering + eval_expr evaluates it.  That pins our kernels
to the reference's semantics of the formula, not to a published result
("parity unpinned" in the sense of SURVEY.md §8(c)).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")

from sumfact import cli, elements, forms, quadrature, scheduling  # noqa: E402
from sumfact import ir  # noqa: E402

from paper_1711_02473_b200 import workloads  # noqa: E402

NCELLS = 4


def tables():
    out = {}
    for m in range(1, 19):
        x, w = quadrature._gl_cache.get(m) or (None, None)
        r = quadrature.gauss_legendre(m)
        out["gl_x_%d" % m] = np.array(r.point_set.points)
        out["gl_w_%d" % m] = np.array(r.weights)
        if m >= 2:
            r = quadrature.gauss_lobatto_legendre(m)
            out["gll_x_%d" % m] = np.array(r.point_set.points)
            out["gll_w_%d" % m] = np.array(r.weights)
    combos = []
    for p in range(1, 10):
        combos.append(("equispaced", p, "gl", p + 1))
        combos.append(("equispaced", p, "gl", p + 2))
    for p in range(1, 17):
        combos.append(("spectral_gll", p, "gll", p + 1))
        combos.append(("spectral_gll", p, "gl", p + 1))
    for p in range(0, 9):
        combos.append(("spectral_gl", p, "gl", p + 1))
    for variant, p, fam, m in combos:
        el = elements.lagrange_interval(p, variant)
        pts = (quadrature.gauss_legendre(m) if fam == "gl"
               else quadrature.gauss_lobatto_legendre(m)).point_set.points
        t = elements._lagrange_tables(el.nodes, pts, 1)
        key = "%s_p%d_%s%d" % (variant, p, fam, m)
        out["nodes_" + key] = np.array(el.nodes)
        out["B_" + key] = t[0]
        out["D_" + key] = t[1]
    # P1 coordinate tables at GL/GLL points
    for m in range(1, 19):
        el = elements.lagrange_interval(1)
        for fam in ("gl", "gll"):
            if fam == "gll" and m < 2:
                continue
            pts = (quadrature.gauss_legendre(m) if fam == "gl"
                   else quadrature.gauss_lobatto_legendre(m)).point_set.points
            t = elements._lagrange_tables(el.nodes, pts, 1)
            out["Bc_%s%d" % (fam, m)] = t[0]
            out["Dc_%s%d" % (fam, m)] = t[1]
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)
    print("tables.npz: %d arrays" % len(out))


def _evaluate(kernel, coords, w0=None, w1=None):
    outs = []
    for c in range(coords.shape[0]):
        inputs = {"coords": coords[c]}
        if w0 is not None:
            inputs["w0"] = w0[c]
        if w1 is not None:
            inputs["w1"] = w1[c]
        outs.append(forms.evaluate_kernel(kernel, inputs))
    return np.array(outs)


def _small_lattice():
    # first NCELLS cells of a (2, 2, 1)-lattice drawn with the config seeds
    return workloads.lattice_coords(2, 2, 1)[:NCELLS]


def _request(form, cell, p, variant="equispaced", quadrature=None):
    return cli.build_request(form, cell, p, "spectral", variant, quadrature)


def neohookean_spec(mu=1.0, lam=10.0):
    """Builder-supplied FormSpec of SURVEY.md §8(a) row a17 in reference IR."""
    from sumfact.ir import Division, Literal, MathFunction, Product, Sum

    def neg(e):
        return Product(Literal(-1.0), e)

    def builder(ctx, v, u):
        d = 3
        F = [[None] * d for _ in range(d)]
        for a in range(d):
            for k in range(d):
                g = forms._physical_grad(ctx, u, k, (a,))
                F[a][k] = Sum(Literal(1.0), g) if a == k else g

        def minor(r, c):
            rs = [x for x in range(3) if x != r]
            cs = [x for x in range(3) if x != c]
            return Sum(Product(F[rs[0]][cs[0]], F[rs[1]][cs[1]]),
                       neg(Product(F[rs[0]][cs[1]], F[rs[1]][cs[0]])))

        J = Sum(Sum(Product(F[0][0], minor(0, 0)), neg(Product(F[0][1], minor(0, 1)))),
                Product(F[0][2], minor(0, 2)))
        lnJ = MathFunction("ln", J)
        total = None
        for a in range(d):
            for k in range(d):
                cof = minor(a, k)
                if (a + k) % 2:
                    cof = neg(cof)
                finvT = Division(cof, J)
                P = Sum(Product(Literal(mu), Sum(F[a][k], neg(finvT))),
                        Product(Product(Literal(lam), lnJ), finvT))
                term = Product(P, forms._physical_grad(ctx, v, k, (a,)))
                total = term if total is None else Sum(total, term)
        return total

    return forms.FormSpec("neohookean_residual", 1, 1, builder, family="vector",
                          cells=("hex",), coefficient_slots=((1, "vector"),))


def c1():
    coords = workloads.quad_coords(1024)[:NCELLS]
    w0 = workloads.uniform_dofs(1024, 16)[:NCELLS]
    out = {"coords": coords, "w0": w0}
    for form in ("action_mass", "action_laplace"):
        k = _request(form, "quad", 3)
        out["A_" + form] = _evaluate(k, coords, w0)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)


def c2(degrees=range(1, 9)):
    coords = _small_lattice()
    out = {"coords": coords}
    for p in degrees:
        n = p + 1
        w0 = workloads.uniform_dofs(NCELLS, n ** 3)
        k = _request("action_laplace", "hex", p)
        out["w0_p%d" % p] = w0
        out["A_p%d" % p] = _evaluate(k, coords, w0)
    np.savez_compressed(os.path.join(HERE, "c2.npz"), **out)


def c3(degrees=(1, 2, 4, 6, 8, 12, 16)):
    coords = _small_lattice()[:2]
    out = {"coords": coords}
    spec = forms.action_form(forms.REGISTRY["weighted_laplace"])
    for p in degrees:
        n = p + 1
        w0 = workloads.uniform_dofs(2, n ** 3)
        w1 = workloads.uniform_dofs(2, n ** 3, 0.5, 2.0, seed=workloads.SEED_KAPPA)
        el = forms.form_element(spec, "hex", p, "spectral_gll")
        rule = forms.default_quadrature("hex", p, collocated_gll=True)
        ce = [forms.coefficient_element(spec, fam, "hex", p, "spectral_gll")
              for (_o, fam) in spec.coefficient_slots]
        k = forms.lower_form(spec, el, rule, "hex", coeff_elements=ce)
        t0 = time.time()
        out["w0_p%d" % p] = w0
        out["w1_p%d" % p] = w1
        out["A_p%d" % p] = _evaluate(k, coords, w0, w1)
        # plain action_laplace through the CLI collocated path
        k2 = _request("action_laplace", "hex", p, "spectral_gll", "collocated-gll")
        out["Alap_p%d" % p] = _evaluate(k2, coords, w0)
        print("c3 p=%d %.1fs" % (p, time.time() - t0))
    np.savez_compressed(os.path.join(HERE, "c3.npz"), **out)


def c4(degrees=(1, 2, 3, 4, 5, 6)):
    coords = _small_lattice()[:2]
    out = {"coords": coords}
    spec = neohookean_spec()
    for p in degrees:
        n = p + 1
        w0 = workloads.uniform_dofs(2, 3 * n ** 3, -0.01, 0.01, scale=workloads.H)
        el = forms.form_element(spec, "hex", p)
        rule = forms.default_quadrature("hex", p, points_per_direction=p + 2)
        ce = [forms.coefficient_element(spec, fam, "hex", p)
              for (_o, fam) in spec.coefficient_slots]
        k = forms.lower_form(spec, el, rule, "hex", coeff_elements=ce)
        t0 = time.time()
        out["w0_p%d" % p] = w0
        out["A_p%d" % p] = _evaluate(k, coords, w0)
        # The config's own draw U(-0.01, 0.01)*h inverts elements at p >= 5
        # (J <= 0 somewhere, ln J = NaN in the reference too).  A second draw
        # with amplitude 0.03*h/p^2 keeps J > 0 at every degree while still
        # exercising the nonlinearity.
        amp = 0.03 / p ** 2
        w0b = workloads.uniform_dofs(2, 3 * n ** 3, -amp, amp, seed=99,
                                     scale=workloads.H)
        out["w0b_p%d" % p] = w0b
        out["Ab_p%d" % p] = _evaluate(k, coords, w0b)
        print("c4 p=%d %.1fs" % (p, time.time() - t0))
    np.savez_compressed(os.path.join(HERE, "c4.npz"), **out)


def c5(degrees=(1, 2, 3, 4)):
    coords = _small_lattice()[:2]
    out = {"coords": coords}
    for p in degrees:
        k = _request("laplace", "hex", p)
        out["A_p%d" % p] = _evaluate(k, coords)
    # the reference cell: analytic K(x)M(x)M + M(x)K(x)M + M(x)M(x)K at p=1
    out["ref_coords"] = np.array(
        [[x, y, z] for x in (0.0, 1.0) for y in (0.0, 1.0) for z in (0.0, 1.0)]).reshape(1, 24)
    k = _request("laplace", "hex", 1)
    out["A_ref_p1"] = _evaluate(k, out["ref_coords"])
    np.savez_compressed(os.path.join(HERE, "c5.npz"), **out)


def mass_hex():
    """Hex ``action_mass`` (registry, forms.py:173, 261-263): GL(p+1) and
    GL(p+2) equispaced, and the GLL-collocated variant (B = Delta)."""
    coords = _small_lattice()[:3]
    out = {"coords": coords}
    cases = [("gl", p, "equispaced", None) for p in range(1, 9)]
    cases += [("glp2", p, "equispaced", p + 2) for p in (1, 2, 4)]
    cases += [("gll", p, "spectral_gll", "collocated-gll") for p in (2, 4, 7)]
    for tag, p, variant, quad in cases:
        n = p + 1
        w0 = workloads.uniform_dofs(3, n ** 3)
        k = _request("action_mass", "hex", p, variant, quad)
        out["w0_%s_p%d" % (tag, p)] = w0
        out["A_%s_p%d" % (tag, p)] = _evaluate(k, coords, w0)
    np.savez_compressed(os.path.join(HERE, "mass_hex.npz"), **out)


def flops():
    rec = {}
    for p in range(1, 9):
        prog = cli.compile_kernel("action_laplace", "hex", p, "spectral")
        rec["C2_p%d" % p] = scheduling.count_flops(prog).total_flops
        assert prog.arguments == [("coords", 24), ("w0", (p + 1) ** 3)]
        assert tuple(prog.return_buffer) == ("A", (p + 1) ** 3)
    for p in range(1, 5):
        prog = cli.compile_kernel("laplace", "hex", p, "spectral")
        rec["C5_p%d" % p] = scheduling.count_flops(prog).total_flops
    for form in ("action_mass", "action_laplace"):
        prog = cli.compile_kernel(form, "quad", 3, "spectral")
        rec["C1_" + form] = scheduling.count_flops(prog).total_flops
    with open(os.path.join(HERE, "flops.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    print(rec)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tables", "c1", "c2", "c3", "c4", "c5", "flops"]
    for w in which:
        t0 = time.time()
        globals()[w]()
        print("%s done in %.1fs" % (w, time.time() - t0))
