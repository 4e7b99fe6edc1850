"""Seeded synthetic inputs of the BASELINE configs.

BASELINE.json names no dataset; every input is synthetic:

* jittered unit-cube lattice, h = 1/64, vertices ``(i,j,k)*h + U(-0.1h, 0.1h)``
  drawn as ``rng_geom.uniform(-0.1*h, 0.1*h, size=(Nx+1, Ny+1, Nz+1, 3))``;
  cell id ``(ix*Ny + iy)*Nz + iz``; coords gathered in reference vertex
  order ``v = 4a + 2b + c`` (geometry.py:119-121), component innermost;
* seeds ``seed_geom = 1711``, ``seed_u = 2473``, ``seed_kappa = 2474``
  (numpy PCG64 ``default_rng``), fixed call order.
"""

from __future__ import annotations

import numpy as np

SEED_GEOM = 1711
SEED_U = 2473
SEED_KAPPA = 2474
H = 1.0 / 64


def lattice_coords(nx, ny, nz, h=H, seed=SEED_GEOM, ix_range=None):
    """(C, 24) hex vertex coordinates of a jittered lattice.

    ``ix_range=(lo, hi)`` keeps only cells with lo <= ix < hi (rank shard of
    BASELINE config C5); the jitter draw always covers the whole lattice so
    shards of one lattice agree with the unsharded lattice.
    """
    rng = np.random.default_rng(seed)
    jit = rng.uniform(-0.1 * h, 0.1 * h, size=(nx + 1, ny + 1, nz + 1, 3))
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                             indexing="ij")
    verts = np.stack([ii, jj, kk], axis=-1) * h + jit
    lo, hi = (0, nx) if ix_range is None else ix_range
    cx = np.arange(lo, hi)
    cy = np.arange(ny)
    cz = np.arange(nz)
    CX, CY, CZ = np.meshgrid(cx, cy, cz, indexing="ij")
    CX, CY, CZ = CX.reshape(-1), CY.reshape(-1), CZ.reshape(-1)
    coords = np.empty((CX.size, 8, 3))
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                coords[:, 4 * a + 2 * b + c, :] = verts[CX + a, CY + b, CZ + c]
    return coords.reshape(-1, 24)


def quad_coords(ncells, seed=SEED_GEOM):
    """(C, 8) jittered unit squares of BASELINE config C1 (v = 2a + b)."""
    rng = np.random.default_rng(seed)
    ref = np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 0.0], [1.0, 1.0]])
    return (ref[None] + rng.uniform(-0.1, 0.1, (ncells, 4, 2))).reshape(ncells, 8)


def uniform_dofs(ncells, size, lo=-1.0, hi=1.0, seed=SEED_U, scale=1.0):
    rng = np.random.default_rng(seed)
    out = rng.uniform(lo, hi, (ncells, size))
    if scale != 1.0:
        out *= scale
    return out


CONFIGS = {
    # name: (description, lattice dims)
    "C1": ("quad Q3 mass+Laplace action, 1024 cells", None),
    "C2": ("hex Q_p Laplace action, GL, 2^18 cells", (64, 64, 64)),
    "C3": ("hex GLL-collocated weighted Laplace action, 2^16 cells", (16, 64, 64)),
    "C4": ("hex Q_p^3 neo-Hookean residual, 2^16 cells", (16, 64, 64)),
    "C5": ("hex Laplace local matrices, 2^16 cells per GPU", (16, 64, 64)),
}


def c2_inputs(degree, dims=(64, 64, 64)):
    n = degree + 1
    coords = lattice_coords(*dims)
    return {"coords": coords, "w0": uniform_dofs(coords.shape[0], n ** 3)}


def c3_inputs(degree, dims=(16, 64, 64)):
    n = degree + 1
    coords = lattice_coords(*dims)
    c = coords.shape[0]
    return {"coords": coords, "w0": uniform_dofs(c, n ** 3),
            "w1": uniform_dofs(c, n ** 3, 0.5, 2.0, seed=SEED_KAPPA)}


def c4_inputs(degree, dims=(16, 64, 64)):
    n = degree + 1
    coords = lattice_coords(*dims)
    return {"coords": coords,
            "w0": uniform_dofs(coords.shape[0], 3 * n ** 3, -0.01, 0.01, scale=H)}


def c5_inputs(rank=0, world=1, dims_per_rank=(16, 64, 64)):
    nx, ny, nz = dims_per_rank
    coords = lattice_coords(nx * world, ny, nz, ix_range=(nx * rank, nx * (rank + 1)))
    return {"coords": coords}


def c1_inputs(ncells=1024):
    coords = quad_coords(ncells)
    return {"coords": coords, "w0": uniform_dofs(ncells, 16)}
