"""Weak-form registry, elements and quadrature per request (host side).

Mirrors reference forms.py: the same ``FormSpec`` fields, the same
``REGISTRY`` names (forms.py:246-263), ``action_form`` (forms.py:235-243),
``form_element`` / ``coefficient_element`` (forms.py:266-288) and
``default_quadrature`` (forms.py:291-319).  The difference is what a spec's
``builder`` is: in the reference it composes IR; here it names the pointwise
operator a hand-written sm_100a kernel family implements
(``paper_1711_02473_b200/csrc``).  ``neohookean_residual_form`` adds the
builder-supplied hyperelastic residual of BASELINE config C4 (SURVEY.md §8(a)
row a17), which the reference declares out of scope.
"""

from __future__ import annotations

from .elements import (CELL_DIMENSION, scalar_element, vector_element)
from .errors import ArityMismatch, Unsupported, UnsupportedCell
from .quadrature import gauss_legendre, gauss_lobatto_legendre, tensor_rule

__all__ = ["FormSpec", "REGISTRY", "CELLS", "action_form", "form_element",
           "coefficient_element", "default_quadrature",
           "neohookean_residual_form"]

CELLS = ("interval", "quad", "triangle", "hex", "prism")


class FormSpec:
    """Registry entry: rank, argument derivative order, coefficient slots and
    the pointwise operator tag (reference forms.py:220-232)."""

    def __init__(self, name, rank, arg_order, builder, family="scalar",
                 cells=CELLS, coefficient_slots=(), parameters=None):
        self.name = name
        self.rank = rank
        self.arg_order = arg_order
        self.builder = builder
        self.family = family
        self.cells = tuple(cells)
        self.coefficient_slots = tuple(coefficient_slots)
        self.parameters = dict(parameters or {})

    def __repr__(self):
        return "FormSpec(%r, rank=%d)" % (self.name, self.rank)


def action_form(bilinear):
    """Demote the trial argument of a bilinear form to coefficient slot 0."""
    if bilinear.rank != 2:
        raise ArityMismatch("action needs a bilinear form")
    return FormSpec(
        "action_" + bilinear.name, 1, bilinear.arg_order, bilinear.builder,
        family=bilinear.family, cells=bilinear.cells,
        coefficient_slots=((bilinear.arg_order, bilinear.family),)
        + bilinear.coefficient_slots, parameters=bilinear.parameters)


REGISTRY = {}
for _spec in (
    FormSpec("mass", 2, 0, "mass"),
    FormSpec("weighted_mass", 2, 0, "weighted_mass",
             coefficient_slots=((0, "scalar"),)),
    FormSpec("laplace", 2, 1, "laplace"),
    FormSpec("weighted_laplace", 2, 1, "weighted_laplace",
             coefficient_slots=((0, "scalar"),)),
    FormSpec("vector_mass", 2, 0, "vector_mass", family="vector"),
    FormSpec("stokes_momentum", 2, 1, "stokes_momentum", family="vector"),
    FormSpec("curl_curl", 2, 1, "curl_curl", family="rtcf", cells=("quad",)),
    FormSpec("rhs_source", 1, 0, "rhs_source",
             coefficient_slots=((0, "scalar"),)),
):
    REGISTRY[_spec.name] = _spec
for _name in ("mass", "laplace", "curl_curl"):
    _a = action_form(REGISTRY[_name])
    REGISTRY[_a.name] = _a


def neohookean_residual_form(mu=1.0, lam=10.0):
    """Compressible neo-Hookean residual r(v) = int P(F) : grad v.

    F = I + grad u, J = det F, P = mu (F - F^-T) + lam ln(J) F^-T.
    Vector Q_p test space, displacement u in coefficient slot 0 (first
    derivatives).  Parameters follow BASELINE.json config C4.
    """
    return FormSpec("neohookean_residual", 1, 1, "neohookean",
                    family="vector", cells=("hex",),
                    coefficient_slots=((1, "vector"),),
                    parameters={"mu": float(mu), "lambda": float(lam)})


def form_element(spec, cell, degree, variant="equispaced"):
    """Argument element of a form (reference forms.py:266-282)."""
    if cell not in spec.cells:
        raise UnsupportedCell("form %s is not defined on %s" % (spec.name, cell))
    if spec.family == "scalar":
        return scalar_element(cell, degree, variant)
    if spec.family == "vector":
        return vector_element(scalar_element(cell, degree, variant),
                              CELL_DIMENSION[cell])
    if spec.family == "rtcf":
        raise Unsupported("RTCF (H(div)) elements are out of scope for the "
                          "B200 path (SURVEY.md §2)")
    raise Unsupported("unknown element family %r" % spec.family)


def coefficient_element(spec, family, cell, degree, variant="equispaced"):
    if family == "scalar":
        return scalar_element(cell, degree, variant)
    return form_element(spec, cell, degree, variant)


def default_quadrature(cell, degree, points_per_direction=None,
                       collocated_gll=False):
    """GL(degree+1) per direction unless overridden; GLL(degree+1) for the
    collocated spectral variant (reference forms.py:291-319)."""
    if collocated_gll:
        m = degree + 1
        if cell == "interval":
            return gauss_lobatto_legendre(m)
        if cell == "quad":
            return tensor_rule(gauss_lobatto_legendre(m),
                               gauss_lobatto_legendre(m))
        if cell == "hex":
            return tensor_rule(tensor_rule(gauss_lobatto_legendre(m),
                                           gauss_lobatto_legendre(m)),
                               gauss_lobatto_legendre(m))
        raise UnsupportedCell("collocated GLL quadrature needs a box cell")
    m = points_per_direction or degree + 1
    if cell == "interval":
        return gauss_legendre(m)
    if cell == "quad":
        return tensor_rule(gauss_legendre(m), gauss_legendre(m))
    if cell == "hex":
        return tensor_rule(tensor_rule(gauss_legendre(m), gauss_legendre(m)),
                           gauss_legendre(m))
    if cell in ("triangle", "prism"):
        raise UnsupportedCell("simplex quadrature is out of scope for the "
                              "B200 path")
    raise UnsupportedCell("unknown cell %r" % cell)
