"""Plan construction: the drop-in for ``cli.compile_kernel``.

Reference tier 1 of the boundary: ``compile_kernel(form,
cell, degree, mode, variant='equispaced', quadrature=None,
element_spec=None)`` (reference cli.py:155-217) validates a request, builds
element and quadrature, lowers and optimises the form, and returns a
``LoopProgram`` whose ``name`` / ``return_buffer`` / ``arguments`` / ``meta``
define the per-cell ABI of the emitted C function (scheduling.py:87-95,
731-735).

Here the optimisation pipeline is not re-run at all: its spectral-mode output
for the supported (form, cell) families *is* the contraction schedule the
sm_100a kernels implement by hand.  What the plan
carries instead is the data those kernels need — reference-bit-exact 1D
tables, weights and points — plus the identical ABI metadata, so a caller can
swap ``compile_kernel`` + its C cell loop for ``compile_kernel`` +
``evaluate_batched`` unchanged.
"""

from __future__ import annotations

import numpy as np

from .elements import CELL_DIMENSION, coordinate_element, lagrange_tables
from .errors import (ArityMismatch, InvalidDegree, Unsupported,
                     UnsupportedCell, UsageError)
from .forms import (CELLS, REGISTRY, FormSpec, coefficient_element,
                    default_quadrature, form_element)

__all__ = ["MODES", "KernelPlan", "compile_kernel", "compile_form",
           "reference_flops", "algorithmic_flops", "compulsory_bytes"]

MODES = ("spectral", "coffee", "vanilla")   # reference passes.py:45

# C-ABI kind codes (include/sfk.h, enum sfk_kind)
KIND_ACTION_LAPLACE = 1
KIND_ACTION_WEIGHTED_LAPLACE = 2
KIND_ACTION_MASS = 3
KIND_LAPLACE_MATRIX = 4
KIND_NEOHOOKEAN_RESIDUAL = 5

_KIND_OF_BUILDER = {
    ("action", "laplace"): KIND_ACTION_LAPLACE,
    ("action", "weighted_laplace"): KIND_ACTION_WEIGHTED_LAPLACE,
    ("action", "mass"): KIND_ACTION_MASS,
    ("matrix", "laplace"): KIND_LAPLACE_MATRIX,
    ("residual", "neohookean"): KIND_NEOHOOKEAN_RESIDUAL,
}


class KernelPlan:
    """A compiled batched kernel.

    ABI metadata identical to the reference ``LoopProgram``:
      name           e.g. ``"action_laplace"``
      return_buffer  ``("A", size)``
      arguments      ``[("coords", 3*2**d), ("w0", nd), ("w1", nd) ...]``
      meta           ``{form, cell, degree, mode, variant}``
    Device data (host copies, passed by value to every launch):
      B, D           1D basis / derivative tables, shape (n, m), basis-major
      wq, xq         1D quadrature weights / points, shape (m,)
      Bc, Dc         P1 coordinate tables at the points, shape (2, m)
    """

    def __init__(self, name, return_size, arguments, meta, kind, dim, n, m,
                 collocated, B, D, wq, xq, Bc, Dc, params=()):
        self.name = name
        self.return_buffer = ("A", int(return_size))
        self.arguments = list(arguments)
        self.meta = dict(meta)
        self.kind = kind
        self.dim = dim
        self.n = n
        self.m = m
        self.collocated = bool(collocated)
        self.B = np.ascontiguousarray(B, dtype=np.float64)
        self.D = np.ascontiguousarray(D, dtype=np.float64)
        self.wq = np.ascontiguousarray(wq, dtype=np.float64)
        self.xq = np.ascontiguousarray(xq, dtype=np.float64)
        self.Bc = np.ascontiguousarray(Bc, dtype=np.float64)
        self.Dc = np.ascontiguousarray(Dc, dtype=np.float64)
        self.params = tuple(float(p) for p in params)
        self._native = {}

    @property
    def degree(self):
        return self.meta.get("degree")

    @property
    def return_size(self):
        return self.return_buffer[1]

    def argument_size(self, name):
        for a, s in self.arguments:
            if a == name:
                return s
        raise KeyError(name)

    @property
    def reference_flops(self):
        return reference_flops(self)

    @property
    def algorithmic_flops(self):
        return algorithmic_flops(self)

    @property
    def compulsory_bytes(self):
        return compulsory_bytes(self)

    def __repr__(self):
        return ("KernelPlan(%s, cell=%s, degree=%s, n=%d, m=%d%s)"
                % (self.name, self.meta.get("cell"), self.degree, self.n,
                   self.m, ", collocated" if self.collocated else ""))


def _kind_for(spec):
    tag = spec.builder if isinstance(spec.builder, str) else None
    if spec.rank == 1 and spec.coefficient_slots and tag != "neohookean":
        key = ("action", tag)
    elif spec.rank == 2:
        key = ("matrix", tag)
    elif tag == "neohookean":
        key = ("residual", tag)
    else:
        key = (None, tag)
    kind = _KIND_OF_BUILDER.get(key)
    if kind is None:
        raise Unsupported("no B200 kernel family for form %r (supported: "
                          "action_laplace, action_weighted_laplace, "
                          "action_mass, laplace, neohookean_residual)"
                          % spec.name)
    return kind


def compile_form(spec, cell, degree, mode="spectral", variant="equispaced",
                 quadrature=None, points_per_direction=None):
    """Build a plan for an arbitrary ``FormSpec`` (the reference's
    ``lower_form`` + ``run_pipeline`` + ``schedule`` path, forms.py:353-417).

    ``quadrature``: None (GL(degree+1)), an int (GL points per direction) or
    ``"collocated-gll"`` (GLL at the element's own nodes; requires
    ``variant='spectral_gll'``).
    """
    if not isinstance(spec, FormSpec):
        raise UsageError("expected a FormSpec")
    if mode not in MODES:
        raise UsageError("unknown mode %r" % mode)
    if degree < 1:
        raise UsageError("degree must be >= 1")
    if cell not in CELLS:
        raise UsageError("unknown cell %r" % cell)
    collocated = False
    points = points_per_direction
    if quadrature is not None:
        if quadrature == "collocated-gll":
            if variant != "spectral_gll":
                raise UsageError(
                    "--quadrature collocated-gll requires --variant "
                    "spectral_gll: collocation must match the element nodes")
            if cell not in ("interval", "quad", "hex"):
                raise UsageError("collocated-gll quadrature needs a box cell")
            collocated = True
        else:
            try:
                points = int(quadrature)
            except (TypeError, ValueError):
                raise UsageError("--quadrature takes an integer point count "
                                 "per direction or 'collocated-gll'") from None
            if points < 1:
                raise UsageError("quadrature needs at least one point")
    kind = _kind_for(spec)
    if cell not in ("quad", "hex"):
        raise Unsupported("the B200 kernels cover quad and hex cells only")
    try:
        element = form_element(spec, cell, degree, variant)
        rule = default_quadrature(cell, degree, points_per_direction=points,
                                  collocated_gll=collocated)
        coeff_elements = [coefficient_element(spec, fam, cell, degree, variant)
                          for (_o, fam) in spec.coefficient_slots]
    except (UnsupportedCell, InvalidDegree) as e:
        raise UsageError(str(e)) from e

    d = CELL_DIMENSION[cell]
    factors = element.factors_1d
    rules = rule.rules_1d
    if len(factors) != d or len(rules) != d:
        raise ArityMismatch("element/cell dimension mismatch")
    # Q_p on a box: every axis carries the same 1D element and 1D rule.
    f0, r0 = factors[0], rules[0]
    for f, r in zip(factors, rules):
        if not (np.array_equal(f.nodes, f0.nodes)
                and np.array_equal(r.point_set.points, r0.point_set.points)):
            raise Unsupported("anisotropic tensor-product elements are not "
                              "supported by the B200 kernels")
    pts = r0.point_set.points
    tabs = f0.tables(pts, 1)
    is_colloc = f0.is_collocated(pts)
    coord_factor = coordinate_element(cell).factors_1d[0]
    ctabs = coord_factor.tables(pts, 1)

    arguments = [("coords", coordinate_element(cell).space_dimension)]
    for slot, ce in enumerate(coeff_elements):
        arguments.append(("w%d" % slot, ce.space_dimension))
    if spec.rank == 2:
        return_size = element.space_dimension ** 2
    else:
        return_size = element.space_dimension

    if kind == KIND_ACTION_WEIGHTED_LAPLACE and not is_colloc:
        raise Unsupported("action_weighted_laplace is implemented for the "
                          "GLL-collocated variant (BASELINE config C3)")
    if kind == KIND_NEOHOOKEAN_RESIDUAL and cell != "hex":
        raise Unsupported("neo-Hookean residual is hex-only")

    params = ()
    if kind == KIND_NEOHOOKEAN_RESIDUAL:
        params = (spec.parameters.get("mu", 1.0),
                  spec.parameters.get("lambda", 10.0))
    n, m = len(f0.nodes), len(pts)
    from .runtime import kernel_available

    if not kernel_available(kind, d, n, m, is_colloc):
        raise Unsupported(
            "no B200 kernel for %s on %s at degree %d with %d quadrature points per "
            "direction%s (kernel instances: sfk_kernel_available, csrc/sfk_api.cu)"
            % (spec.name, cell, degree, m, ", collocated" if is_colloc else ""))
    meta = {"form": spec.name, "cell": cell, "degree": element.degree,
            "mode": mode, "variant": variant}
    return KernelPlan(spec.name, return_size, arguments, meta, kind, d,
                      n, m, is_colloc, tabs[0], tabs[1],
                      r0.weights, pts, ctabs[0], ctabs[1], params)


def compile_kernel(form, cell, degree, mode="spectral", variant="equispaced",
                   quadrature=None, element_spec=None):
    """Drop-in for reference ``cli.compile_kernel`` (cli.py:211-217).

    ``form`` is a registry name (as in the reference) or a ``FormSpec``.
    """
    if isinstance(form, FormSpec):
        spec = form
    else:
        if form not in REGISTRY:
            raise UsageError("unknown form %r (choose from %s)"
                             % (form, ", ".join(sorted(REGISTRY))))
        spec = REGISTRY[form]
    if cell not in CELLS:
        raise UsageError("unknown cell %r" % cell)
    if mode not in MODES:
        raise UsageError("unknown mode %r" % mode)
    if degree < 1:
        raise UsageError("degree must be >= 1")
    if element_spec is not None:
        raise Unsupported("element specification strings are out of scope "
                          "for the B200 path (SURVEY.md §2, cli.py row)")
    return compile_form(spec, cell, degree, mode, variant, quadrature)


# ---------------------------------------------------------------------------
# flop / byte accounting


def reference_flops(plan):
    """The reference ``count_flops`` of the spectral-mode program (exact
    closed forms fitted in SURVEY.md Appendix B), or None when unknown."""
    n, m = plan.n, plan.m
    name, cell = plan.name, plan.meta["cell"]
    if cell == "hex" and name == "action_laplace" and not plan.collocated and m == n:
        return 33 * n**4 + 134 * n**3 + 72 * n**2 + 96 * n
    if cell == "hex" and name == "laplace" and m == n:
        return 15 * n**7 + 27 * n**6 + 24 * n**5 + 143 * n**3 + 72 * n**2 + 96 * n
    if cell == "hex" and name == "action_weighted_laplace" and plan.collocated:
        return 24 * n**4 + 363 * n**3 + 216 * n**2 + 192 * n
    if cell == "quad" and n == 4 and m == 4:
        return {"action_mass": 944, "action_laplace": 1872}.get(name)
    if cell == "hex" and name == "neohookean_residual":
        return {2: 34788, 3: 78945, 4: 156258, 5: 280371, 6: 467304}.get(plan.degree)
    return None


def algorithmic_flops(plan):
    """F_alg of SURVEY.md §8(d): the per-cell flop figure the roofline uses."""
    n, m = plan.n, plan.m
    name, cell = plan.name, plan.meta["cell"]
    if cell == "hex" and name == "action_weighted_laplace" and plan.collocated:
        return 12 * n**4 + 135 * n**3 + 72 * n**2 + 96 * n
    if cell == "hex" and name == "neohookean_residual":
        return 6 * (4 * m * n**3 + 6 * m**2 * n**2 + 6 * m**3 * n) + 311 * m**3
    return reference_flops(plan)


def compulsory_bytes(plan):
    """Compulsory HBM bytes per cell: every argument read once, A written once."""
    total = plan.return_size
    for _name, size in plan.arguments:
        total += size
    return 8 * total
