"""Global (assembled) matrix-free operators — SURVEY.md §8(f) item 1.

The reference stops at the per-cell kernel; global assembly is the caller's
job.  The immediate caller of the hot path is the E-vector <->
L-vector map of a conforming mesh: gather a cell's dofs from the global
vector, apply the cell kernel, scatter-add back (PAPER.md:176-189,
1804-1819).  ``GlobalOperator.apply`` does all three in ONE launch of the
C2 line kernel (``sfk_eval_gather_scatter``: gather fused into the x stage,
fp64 atomic scatter fused into the transposed x stage), so the E-vector
never exists in HBM.

``lattice_dof_map`` numbers the continuous Q_p space of the structured
jittered lattice used by the BASELINE configs: cell (cx, cy, cz), local dof
(a, b, c) (reference order (a*n+b)*n+c) -> global grid node
(cx*p + a, cy*p + b, cz*p + c) of the (nx*p+1, ny*p+1, nz*p+1) grid.
"""

from __future__ import annotations

import numpy as np

from .errors import NativeError, ShapeMismatch

__all__ = ["lattice_dof_map", "lattice_boundary_mask", "GlobalOperator", "cg"]


def lattice_dof_map(nx, ny, nz, degree, ix_range=None):
    """(C, (p+1)^3) int32 global dof of every local dof, cells ordered like
    ``workloads.lattice_coords`` ((cx*ny + cy)*nz + cz)."""
    p = degree
    n = p + 1
    gy, gz = ny * p + 1, nz * p + 1
    lo, hi = (0, nx) if ix_range is None else ix_range
    cx, cy, cz = np.meshgrid(np.arange(lo, hi), np.arange(ny), np.arange(nz), indexing="ij")
    a, b, c = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    X = cx.reshape(-1, 1) * p + a.reshape(1, -1)
    Y = cy.reshape(-1, 1) * p + b.reshape(1, -1)
    Z = cz.reshape(-1, 1) * p + c.reshape(1, -1)
    g = (X * gy + Y) * gz + Z
    if g.max() >= 2 ** 31:
        raise ValueError("global dof count exceeds int32")
    return np.ascontiguousarray(g, dtype=np.int32)


def lattice_ndofs(nx, ny, nz, degree):
    p = degree
    return (nx * p + 1) * (ny * p + 1) * (nz * p + 1)


def lattice_boundary_mask(nx, ny, nz, degree):
    """Boolean mask of the global dofs on the lattice boundary."""
    p = degree
    gx, gy, gz = nx * p + 1, ny * p + 1, nz * p + 1
    X, Y, Z = np.meshgrid(np.arange(gx), np.arange(gy), np.arange(gz), indexing="ij")
    m = (X == 0) | (X == gx - 1) | (Y == 0) | (Y == gy - 1) | (Z == 0) | (Z == gz - 1)
    return m.reshape(-1)


class GlobalOperator:
    """y = K x with K = sum_c P_c^T A_c P_c, applied matrix-free on the GPU.

    plan       a hex ``action_laplace`` KernelPlan (GL, m == n)
    cell_dofs  (C, nd) int32 CUDA tensor (``lattice_dof_map``)
    coords     (C, 24) float64 CUDA tensor
    ndofs      length of the global vectors
    """

    def __init__(self, plan, cell_dofs, coords, ndofs):
        import torch

        if cell_dofs.dtype != torch.int32 or not cell_dofs.is_cuda:
            raise TypeError("cell_dofs must be an int32 CUDA tensor")
        if coords.dtype != torch.float64 or not coords.is_cuda:
            raise TypeError("coords must be a float64 CUDA tensor")
        nd = plan.argument_size("w0")
        if tuple(cell_dofs.shape) != (coords.shape[0], nd):
            raise ShapeMismatch("cell_dofs must be (%d, %d)" % (coords.shape[0], nd))
        self.plan = plan
        self.cell_dofs = cell_dofs.contiguous()
        self.coords = coords.contiguous()
        self.ndofs = int(ndofs)

    def apply(self, x, out=None, accumulate=False, stream=None):
        import torch

        from .runtime import _check, load_library, native_plan

        if x.dtype != torch.float64 or not x.is_cuda or x.numel() != self.ndofs:
            raise ShapeMismatch("x must be a float64 CUDA vector of length %d" % self.ndofs)
        x = x.contiguous()
        if out is None:
            out = torch.zeros_like(x)
        elif not accumulate:
            out.zero_()
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        with torch.cuda.device(x.device):
            _check(load_library().sfk_eval_gather_scatter(
                native_plan(self.plan), self.coords.shape[0], self.cell_dofs.data_ptr(),
                x.data_ptr(), out.data_ptr(), self.coords.data_ptr(), stream))
        return out

    __call__ = apply


def cg(op, b, fixed=None, tol=1e-10, maxiter=1000):
    """Conjugate gradients for K x = b with homogeneous Dirichlet rows on
    ``fixed`` (bool CUDA mask): those dofs are held at zero.  Returns
    (x, iterations, relative residual).  Vector algebra in torch; every
    operator application is one fused gather-action-scatter launch."""
    import torch

    free = None if fixed is None else (~fixed).to(b.dtype)

    def K(v):
        y = op.apply(v)
        return y if free is None else y * free

    x = torch.zeros_like(b)
    r = b.clone() if free is None else b * free
    p = r.clone()
    rr = torch.dot(r, r)
    b2 = rr.sqrt()
    if b2.item() == 0.0:
        return x, 0, 0.0
    it = 0
    for it in range(1, maxiter + 1):
        Kp = K(p)
        alpha = rr / torch.dot(p, Kp)
        x += alpha * p
        r -= alpha * Kp
        rr_new = torch.dot(r, r)
        if (rr_new.sqrt() / b2).item() < tol:
            rr = rr_new
            break
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, it, (rr.sqrt() / b2).item()
