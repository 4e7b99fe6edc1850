"""Tensor-product Lagrange elements as *factored* tabulations (host side).

The reference represents tabulations as IR expressions whose only dense
leaves are the 1D interval tables (reference elements.py:1-9).  On B200 that
structure is the device contract itself: a Q_p element on a quad/hex is a
list of 1D interval factors, and the kernels receive only the 1D tables

    B[i, q] = L_i(xi_q),   D[i, q] = L_i'(xi_q)        (basis-major, n x m)

staged by value into every launch.  Nothing here builds IR; the element
objects carry what the plan builder needs (factors, nodes, dof layout).

Bit-exactness: ``lagrange_tables`` performs exactly the numpy operations of
the reference ``_lagrange_tables`` (elements.py:163-177) — a
``Polynomial.fromroots`` of the other nodes, scaled by the product of node
differences, differentiated with ``.deriv`` and evaluated with ``__call__``.
Those tables deviate from exact values by up to 5e-7 relative at p=16 GLL
(SURVEY.md §8(a) row a4), so the 1e-12 parity target is only reachable with
these exact doubles; the device never regenerates or symmetrises them.

Dof layouts (reference elements.py:397-452):
    scalar hex: (ix*n + iy)*n + iz       quad: ix*n + iy
    vector hex: ((ix*n + iy)*n + iz)*3 + comp
    coordinates: coords[3*v + comp], v = 4a + 2b + c (a,b,c = x,y,z offsets)
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch, InvalidDegree, Unsupported
from .quadrature import (PointSet1D, TensorPointSet, gauss_legendre_points,
                         gauss_lobatto_legendre_points)

__all__ = [
    "lagrange_tables", "IntervalLagrange", "ProductElement",
    "TensorFamilyElement", "lagrange_interval", "tensor_product_element",
    "vector_element", "scalar_element", "coordinate_element",
    "discontinuous_lagrange_interval", "CELL_DIMENSION",
]

CELL_DIMENSION = {"interval": 1, "quad": 2, "hex": 3, "triangle": 2, "prism": 3}


def lagrange_tables(nodes, points, max_order):
    """table[o][i, q] = d^o L_i/dx^o (points[q]) for o = 0..max_order.

    Same operation sequence as reference elements.py:163-177.
    """
    nodes = np.asarray(nodes, dtype=float)
    points = np.asarray(points, dtype=float)
    nf, nq = len(nodes), len(points)
    out = {o: np.empty((nf, nq)) for o in range(max_order + 1)}
    for i in range(nf):
        rest = np.delete(nodes, i)
        if len(rest):
            poly = np.polynomial.Polynomial.fromroots(rest)
            poly = poly / np.prod(nodes[i] - rest)
        else:
            poly = np.polynomial.Polynomial([1.0])
        for o in range(max_order + 1):
            p = poly.deriv(o) if o else poly
            out[o][i, :] = p(points)
    return out


def _equispaced_nodes(n):
    # reference elements.py:180-183
    if n == 0:
        return np.array([0.5])
    return np.linspace(0.0, 1.0, n + 1)


class IntervalLagrange:
    """Nodal Lagrange basis on [0, 1] (reference elements.py:186-220)."""

    dimension = 1

    def __init__(self, degree, nodes, continuity, collocation=False,
                 variant="equispaced"):
        self.degree = degree
        self.nodes = np.asarray(nodes, dtype=float)
        self.nodes.flags.writeable = False
        self.continuity = continuity
        self.collocation = collocation
        self.variant = variant
        self.basis_shape = (len(self.nodes),)
        self.value_shape = ()

    @property
    def space_dimension(self):
        return len(self.nodes)

    @property
    def factors_1d(self):
        return (self,)

    def is_collocated(self, points):
        """True when the value table is the identity (Delta(i, q)); mirrors
        reference elements.py:200-203 (bit-equal node/point arrays)."""
        return bool(self.collocation and len(points) == len(self.nodes)
                    and np.array_equal(points, self.nodes))

    def tables(self, points, max_order=1):
        """Dense 1D tables at ``points``; entry 0 is exactly the identity for a
        collocated element (the device then skips that contraction)."""
        points = np.asarray(points, dtype=float)
        tabs = lagrange_tables(self.nodes, points, max_order)
        if self.is_collocated(points):
            tabs[0] = np.eye(len(self.nodes))
        return tabs


def lagrange_interval(n, variant="equispaced"):
    """Interval Lagrange family (reference elements.py:223-249)."""
    if variant == "equispaced":
        if n < 1:
            raise InvalidDegree("continuous Lagrange needs degree >= 1")
        return IntervalLagrange(n, _equispaced_nodes(n), "C0", variant=variant)
    if variant == "equispaced_discontinuous":
        if n < 0:
            raise InvalidDegree("negative degree")
        return IntervalLagrange(n, _equispaced_nodes(n), "L2", variant=variant)
    if variant == "spectral_gll":
        if n < 1:
            raise InvalidDegree("GLL variant needs degree >= 1")
        return IntervalLagrange(n, gauss_lobatto_legendre_points(n + 1), "C0",
                                collocation=True, variant=variant)
    if variant == "spectral_gl":
        if n < 0:
            raise InvalidDegree("negative degree")
        return IntervalLagrange(n, gauss_legendre_points(n + 1), "L2",
                                collocation=True, variant=variant)
    raise Unsupported("unknown interval variant %r" % variant)


def discontinuous_lagrange_interval(n):
    return lagrange_interval(n, "equispaced_discontinuous")


class ProductElement:
    """Tensor product of two scalar elements; the first factor is the outer
    (slowest) dof axis (reference elements.py:385-414)."""

    def __init__(self, e1, e2):
        if e1.value_shape != () or e2.value_shape != ():
            raise Unsupported("tensor products of non-scalar elements are "
                              "built via the HDiv/HCurl wrappers")
        self.factors = (e1, e2)
        self.dimension = e1.dimension + e2.dimension
        self.degree = max(e1.degree, e2.degree)
        self.basis_shape = e1.basis_shape + e2.basis_shape
        self.value_shape = ()

    @property
    def space_dimension(self):
        return int(np.prod(self.basis_shape))

    @property
    def factors_1d(self):
        out = ()
        for f in self.factors:
            out += f.factors_1d
        return out

    @property
    def variant(self):
        vs = {f.variant for f in self.factors_1d}
        return vs.pop() if len(vs) == 1 else None


def tensor_product_element(e1, e2):
    return ProductElement(e1, e2)


class TensorFamilyElement:
    """Vector/tensor version of a scalar element; value components are the
    innermost dof axis (reference elements.py:425-452)."""

    def __init__(self, scalar, value_shape):
        if scalar.value_shape != ():
            raise Unsupported("vector/tensor elements need a scalar-valued base")
        self.scalar = scalar
        self.dimension = scalar.dimension
        self.degree = scalar.degree
        self.value_shape = tuple(value_shape)
        self.basis_shape = scalar.basis_shape + self.value_shape

    @property
    def space_dimension(self):
        return int(np.prod(self.basis_shape))

    @property
    def factors_1d(self):
        return self.scalar.factors_1d

    @property
    def variant(self):
        return getattr(self.scalar, "variant", None)


def vector_element(scalar, d):
    return TensorFamilyElement(scalar, (d,))


def scalar_element(cell_name, degree, variant="equispaced"):
    """Default scalar element on a box cell (reference elements.py:600-617)."""
    if cell_name == "interval":
        return lagrange_interval(degree, variant)
    if cell_name == "quad":
        return tensor_product_element(lagrange_interval(degree, variant),
                                      lagrange_interval(degree, variant))
    if cell_name == "hex":
        return tensor_product_element(
            tensor_product_element(lagrange_interval(degree, variant),
                                   lagrange_interval(degree, variant)),
            lagrange_interval(degree, variant))
    if cell_name in ("triangle", "prism"):
        raise Unsupported("simplex factors are out of scope for the B200 path "
                          "(SURVEY.md §2, elements.py row)")
    raise Unsupported("unknown cell %r" % cell_name)


def coordinate_element(cell_name):
    """Degree-1 vector element of the coordinate field (elements.py:620-632)."""
    d = CELL_DIMENSION.get(cell_name)
    if cell_name not in ("interval", "quad", "hex"):
        raise Unsupported("unknown or unsupported cell %r" % cell_name)
    if cell_name == "interval":
        return vector_element(lagrange_interval(1), 1)
    return vector_element(scalar_element(cell_name, 1), d)


def point_set_1d(ps):
    """The 1D factors of a (tensor) point set, x-axis first."""
    if isinstance(ps, (PointSet1D, TensorPointSet)):
        return ps.factors_1d
    raise DimensionMismatch("expected a 1D or tensor-product point set")
