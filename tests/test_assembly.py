"""Global gather/scatter operator: dof map on CPU,
fused gather-action-scatter on the GPU vs the oracle assembled on the host."""

import numpy as np
import pytest

from oracle import cpu
from paper_1711_02473_b200 import compile_kernel, workloads
from paper_1711_02473_b200.assembly import (lattice_boundary_mask, lattice_dof_map,
                                            lattice_ndofs)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_dof_map_is_conforming(p):
    nx, ny, nz = 3, 2, 2
    g = lattice_dof_map(nx, ny, nz, p)
    n = p + 1
    assert g.shape == (nx * ny * nz, n ** 3) and g.dtype == np.int32
    assert len(np.unique(g)) == lattice_ndofs(nx, ny, nz, p)
    # neighbours in x share their common face: local (p, b, c) of cell 0 ==
    # local (0, b, c) of the cell next in x
    G = g.reshape(nx, ny, nz, n, n, n)
    assert np.array_equal(G[0, 0, 0, p], G[1, 0, 0, 0])
    assert np.array_equal(G[0, 0, 0, :, p], G[0, 1, 0, :, 0])
    assert np.array_equal(G[0, 0, 0, :, :, p], G[0, 0, 1, :, :, 0])
    # the geometric node of every dof agrees between cells (equispaced Q_p)
    m = lattice_boundary_mask(nx, ny, nz, p)
    assert m.sum() == lattice_ndofs(nx, ny, nz, p) - (nx * p - 1) * (ny * p - 1) * (nz * p - 1)


def _assemble_oracle(plan, coords, cell_dofs, x):
    u = x[cell_dofs]
    A = cpu.evaluate(plan, {"coords": coords, "w0": u})
    y = np.zeros_like(x)
    np.add.at(y, cell_dofs, A)
    return y


@pytest.mark.gpu
@pytest.mark.parametrize("p", range(1, 9))
def test_gather_scatter_matches_oracle(cuda, p):
    torch = cuda
    from paper_1711_02473_b200.assembly import GlobalOperator

    dims = (3, 4, 3)
    plan = compile_kernel("action_laplace", "hex", p)
    coords = workloads.lattice_coords(*dims)
    g = lattice_dof_map(*dims, p)
    nd = lattice_ndofs(*dims, p)
    x = np.random.default_rng(5).uniform(-1, 1, nd)
    op = GlobalOperator(plan, torch.from_numpy(g).cuda(), torch.from_numpy(coords).cuda(), nd)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = _assemble_oracle(plan, coords, g, x)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    # constants are in the kernel of the assembled Laplacian
    one = op.apply(torch.ones(nd, dtype=torch.float64, device="cuda")).cpu().numpy()
    assert np.abs(one).max() < 1e-11 * np.abs(ref).max()


@pytest.mark.gpu
def test_cg_poisson_manufactured(cuda):
    """K x = K x* with Dirichlet x* = 0 on the boundary: CG recovers x*."""
    torch = cuda
    from paper_1711_02473_b200.assembly import GlobalOperator, cg

    dims, p = (4, 4, 4), 3
    plan = compile_kernel("action_laplace", "hex", p)
    coords = torch.from_numpy(workloads.lattice_coords(*dims)).cuda()
    g = torch.from_numpy(lattice_dof_map(*dims, p)).cuda()
    nd = lattice_ndofs(*dims, p)
    fixed = torch.from_numpy(lattice_boundary_mask(*dims, p)).cuda()
    op = GlobalOperator(plan, g, coords, nd)
    xs = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, nd)).cuda()
    xs[fixed] = 0.0
    b = op.apply(xs)
    x, it, res = cg(op, b, fixed=fixed, tol=1e-11, maxiter=2000)
    assert res < 1e-11
    assert (x - xs).abs().max().item() < 1e-8
