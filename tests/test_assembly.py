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


# ---------------------------------------------------------------------------
# assembled CSR matrices


def _scipy_csr(coords, cell_dofs, nd, p):
    """Oracle: dense cell matrices from the CPU oracle, summed by scipy."""
    import scipy.sparse as sp

    plan = compile_kernel("laplace", "hex", p)
    A = cpu.evaluate(plan, {"coords": coords}).reshape(len(cell_dofs), -1)
    n3 = cell_dofs.shape[1]
    rows = np.repeat(cell_dofs, n3, axis=1).reshape(-1)
    cols = np.tile(cell_dofs, (1, n3)).reshape(-1)
    K = sp.coo_matrix((A.reshape(-1), (rows, cols)), shape=(nd, nd)).tocsr()
    K.sum_duplicates()
    K.sort_indices()
    return K


def _permuted_dofs(dims, p, seed=3):
    """Lattice numbering scrambled by a random permutation (rows whose
    columns are not monotone in the local order)."""
    g = lattice_dof_map(*dims, p)
    nd = lattice_ndofs(*dims, p)
    perm = np.random.default_rng(seed).permutation(nd).astype(np.int32)
    return np.ascontiguousarray(perm[g]), nd


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("numbering", ["lattice", "permuted"])
def test_csr_assembly_matches_oracle(cuda, p, numbering):
    torch = cuda
    from paper_1711_02473_b200.assembly import CsrPattern, assemble_csr

    dims = (3, 2, 3)
    coords = workloads.lattice_coords(*dims)
    if numbering == "lattice":
        g, nd = lattice_dof_map(*dims, p), lattice_ndofs(*dims, p)
    else:
        g, nd = _permuted_dofs(dims, p)
    K = _scipy_csr(coords, g, nd, p)
    gd = torch.from_numpy(g).cuda()
    pat = CsrPattern(gd, nd)
    assert pat.nnz == K.nnz and pat.nrows == nd
    assert np.array_equal(pat.row_ptr.cpu().numpy(), K.indptr.astype(np.int64))
    assert np.array_equal(pat.col_idx.cpu().numpy(), K.indices.astype(np.int32))
    vals = assemble_csr(compile_kernel("laplace", "hex", p), gd,
                        torch.from_numpy(coords).cuda(), pat).cpu().numpy()
    assert np.abs(vals - K.data).max() <= 1e-12 * np.abs(K.data).max()
    # the entry-map insertion path: positions, then the same values
    emap = pat.entry_map(gd)
    kk = np.asarray(K[np.repeat(g, g.shape[1], axis=1).reshape(-1),
                      np.tile(g, (1, g.shape[1])).reshape(-1)]).reshape(-1)
    pos = emap.cpu().numpy().reshape(-1)
    assert np.array_equal(K.indices[pos], np.tile(g, (1, g.shape[1])).reshape(-1))
    assert np.array_equal(K.data[pos], kk)
    vm = assemble_csr(compile_kernel("laplace", "hex", p), gd, torch.from_numpy(coords).cuda(),
                      pat, entry_map=emap).cpu().numpy()
    assert np.abs(vm - K.data).max() <= 1e-12 * np.abs(K.data).max()
    # assembling twice into the same values doubles them (accumulate semantics)
    v2 = assemble_csr(compile_kernel("laplace", "hex", p), gd, torch.from_numpy(coords).cuda(),
                      pat, values=torch.from_numpy(vals).cuda()).cpu().numpy()
    assert np.abs(v2 - 2 * K.data).max() <= 2e-12 * np.abs(K.data).max()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_csr_matvec_equals_matrix_free_operator(cuda, p):
    """The assembled matrix and the fused matrix-free operator are the same K."""
    torch = cuda
    from paper_1711_02473_b200.assembly import CsrPattern, GlobalOperator, assemble_csr

    dims = (4, 4, 3)
    coords = torch.from_numpy(workloads.lattice_coords(*dims)).cuda()
    g = torch.from_numpy(lattice_dof_map(*dims, p)).cuda()
    nd = lattice_ndofs(*dims, p)
    pat = CsrPattern(g, nd)
    K = pat.matrix(assemble_csr(compile_kernel("laplace", "hex", p), g, coords, pat))
    x = torch.from_numpy(np.random.default_rng(7).uniform(-1, 1, nd)).cuda()
    y_csr = (K @ x.unsqueeze(1)).squeeze(1)
    y_mf = GlobalOperator(compile_kernel("action_laplace", "hex", p), g, coords, nd).apply(x)
    assert (y_csr - y_mf).abs().max().item() <= 1e-12 * y_mf.abs().max().item()


@pytest.mark.gpu
def test_csr_pattern_edge_cases(cuda):
    torch = cuda
    from paper_1711_02473_b200.assembly import CsrPattern

    empty = CsrPattern(torch.zeros((0, 8), dtype=torch.int32, device="cuda"), 5)
    assert empty.nnz == 0 and empty.row_ptr.cpu().tolist() == [0] * 6
    # one cell, a dof unused by every cell -> empty row
    one = CsrPattern(torch.tensor([[0, 2]], dtype=torch.int32, device="cuda"), 3)
    assert one.row_ptr.cpu().tolist() == [0, 2, 2, 4]
    assert one.col_idx.cpu().tolist() == [0, 2, 0, 2]


# ---------------------------------------------------------------------------
# fused global operators of the other action kernels (sfk_eval_global)


def _assemble_oracle_w(plan, coords, cell_dofs, x, w1=None):
    inp = {"coords": coords, "w0": x[cell_dofs]}
    if w1 is not None:
        inp["w1"] = w1
    with np.errstate(invalid="ignore"):
        A = cpu.evaluate(plan, inp)
    y = np.zeros_like(x)
    np.add.at(y, cell_dofs, A)
    return y


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 4, 7, 12])
@pytest.mark.parametrize("weighted", [False, True])
def test_global_collocated_matches_oracle(cuda, p, weighted):
    torch = cuda
    from paper_1711_02473_b200 import REGISTRY, action_form, compile_form
    from paper_1711_02473_b200.assembly import GlobalOperator

    if weighted:
        plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p, "spectral",
                            "spectral_gll", "collocated-gll")
    else:
        plan = compile_kernel("action_laplace", "hex", p, "spectral", "spectral_gll",
                              "collocated-gll")
    dims = (3, 2, 3)
    coords = workloads.lattice_coords(*dims)
    g = lattice_dof_map(*dims, p)
    nd = lattice_ndofs(*dims, p)
    x = np.random.default_rng(11).uniform(-1, 1, nd)
    w1 = (np.random.default_rng(12).uniform(0.5, 2.0, (coords.shape[0], (p + 1) ** 3))
          if weighted else None)
    op = GlobalOperator(plan, torch.from_numpy(g).cuda(), torch.from_numpy(coords).cuda(), nd,
                        w1=torch.from_numpy(w1).cuda() if weighted else None)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = _assemble_oracle_w(plan, coords, g, x, w1)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 3, 4, 5, 6])
def test_global_neohookean_residual_matches_oracle(cuda, p):
    """Assembled nonlinear residual r(x) = sum_c P_c^T r_c(P_c x)."""
    torch = cuda
    from paper_1711_02473_b200 import compile_form, neohookean_residual_form
    from paper_1711_02473_b200.assembly import GlobalOperator, lattice_vector_dof_map

    plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
    dims = (2, 3, 2)
    coords = workloads.lattice_coords(*dims)
    g = lattice_vector_dof_map(*dims, p)
    nd = 3 * lattice_ndofs(*dims, p)
    x = np.random.default_rng(13).uniform(-1, 1, nd) * 0.03 * workloads.H / p ** 2
    op = GlobalOperator(plan, torch.from_numpy(g).cuda(), torch.from_numpy(coords).cuda(), nd)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = _assemble_oracle_w(plan, coords, g, x)
    assert np.isfinite(ref).all()
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    # zero displacement: F = I, P = 0, zero residual
    z = op.apply(torch.zeros(nd, dtype=torch.float64, device="cuda")).abs().max().item()
    assert z == 0.0


def test_vector_dof_map_layout():
    from paper_1711_02473_b200.assembly import lattice_vector_dof_map

    g = lattice_dof_map(2, 2, 1, 2)
    v = lattice_vector_dof_map(2, 2, 1, 2)
    assert v.shape == (4, 3 * 27) and v.dtype == np.int32
    assert np.array_equal(v[:, 0::3], 3 * g) and np.array_equal(v[:, 2::3], 3 * g + 2)


@pytest.mark.gpu
def test_csr_dmma_epilogue_opt_in(cuda):
    """The DMMA kernels' entry-map CSR epilogue (opt-in, option csr_dmma = 1)
    gives the same assembled matrices."""
    from paper_1711_02473_b200 import runtime

    with runtime.options(csr_dmma=1):
        for p in (3, 4):
            for numbering in ("lattice", "permuted"):
                test_csr_assembly_matches_oracle(cuda, p, numbering)


@pytest.mark.gpu
@pytest.mark.parametrize("gen", [1, 2, 3])
def test_gather_scatter_alternative_generations(cuda, gen):
    """The global operator through the older kernel generations (option
    c2g_kernel = 1: the round-1 selection, 2 / 3: forced v2 / v3; the
    default is the collocation-derivative v6 / tc8c) agrees with the
    assembled oracle too."""
    from paper_1711_02473_b200 import runtime

    with runtime.options(c2g_kernel=gen):
        for p in range(1, 9):
            test_gather_scatter_matches_oracle(cuda, p)


# ---------------------------------------------------------------------------
# CSR insertion of ANY kernel's cell matrices (§8(f) item 3 beyond the fused
# hex-Laplace path): reference LoopProgram fixtures (every cell type, vector
# and mixed forms), a random cell -> dof map with shared and repeated dofs,
# oracle = the reference's own cell matrices summed with np.add.at.

ANY_FORMS = ["mass_triangle_p2", "laplace_prism_p2", "vector_mass_hex_p1",
             "stokes_momentum_quad_p2", "curl_curl_quad_p2", "weighted_laplace_hex_p2",
             "laplace_interval_p2"]


def _program_fixture(key):
    import json
    import os

    from conftest import GOLDEN

    meta = {m["key"]: m for m in json.load(open(os.path.join(GOLDEN, "programs.json")))}[key]
    z = np.load(os.path.join(GOLDEN, "programs.npz"))
    text = bytes(z[key + "__json"]).decode()
    inputs = {a: z["%s__%s" % (key, a)] for a, _ in meta["arguments"]}
    return text, inputs, z[key + "__A"]


@pytest.mark.gpu
@pytest.mark.parametrize("key", ANY_FORMS)
@pytest.mark.parametrize("use_map", [False, True])
def test_insert_csr_any_matrix_form(cuda, key, use_map):
    torch = cuda
    from paper_1711_02473_b200 import load_program
    from paper_1711_02473_b200.assembly import CsrPattern, assemble_csr_from

    text, inputs, ref = _program_fixture(key)
    nc, nd2 = ref.shape
    nd = int(round(nd2 ** 0.5))
    ndofs = max(2 * nd, nc * nd // 3)
    dofs = np.random.default_rng(7).integers(0, ndofs, (nc, nd)).astype(np.int32)
    g = torch.from_numpy(dofs).cuda()
    pat = CsrPattern(g, ndofs)
    emap = pat.entry_map(g) if use_map else None
    vals = assemble_csr_from(load_program(text),
                             {k: torch.from_numpy(v).cuda() for k, v in inputs.items()},
                             g, pat, entry_map=emap)
    got = pat.matrix(vals).to_dense().cpu().numpy()
    K = np.zeros((ndofs, ndofs))
    np.add.at(K, (dofs[:, :, None], dofs[:, None, :]), ref.reshape(nc, nd, nd))
    assert np.abs(got - K).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.gpu
def test_insert_csr_matches_fused_assembly(cuda):
    """Hand C5 cell matrices inserted by sfk_csr_insert == the fused C5 CSR
    epilogue (sfk_assemble_csr) on a lattice numbering."""
    torch = cuda
    from paper_1711_02473_b200 import evaluate_batched
    from paper_1711_02473_b200.assembly import CsrPattern, assemble_csr, insert_csr, lattice_ndofs

    p, dims = 2, (3, 4, 5)
    plan = compile_kernel("laplace", "hex", p)
    coords = torch.from_numpy(workloads.lattice_coords(*dims)).cuda()
    g = torch.from_numpy(lattice_dof_map(*dims, p)).cuda()
    pat = CsrPattern(g, lattice_ndofs(*dims, p))
    fused = assemble_csr(plan, g, coords, pat)
    A = evaluate_batched(plan, {"coords": coords})
    ins = insert_csr(A, g, pat, entry_map=pat.entry_map(g))
    assert torch.allclose(fused, ins, rtol=0, atol=1e-12 * fused.abs().max().item())


def test_insert_csr_validates_arguments():
    """CPU tier: insert_csr rejects host tensors / wrong dtypes before any
    device work (the product path has no CPU fallback)."""
    import torch

    from paper_1711_02473_b200.assembly import insert_csr

    with pytest.raises(TypeError):
        insert_csr(torch.zeros(2, 4, dtype=torch.float64), torch.zeros(2, 2, dtype=torch.int32), None)
    with pytest.raises(TypeError):
        insert_csr(torch.zeros(2, 4, dtype=torch.float32), torch.zeros(2, 2, dtype=torch.int64), None)


@pytest.mark.gpu
def test_global_operator_validates_out_and_map(cuda):
    """GlobalOperator rejects an out that is short, float32, or aliases x, and
    a cell->dof map with entries outside [0, ndofs) (which the fused scatter
    would otherwise turn into out-of-bounds fp64 atomics)."""
    torch = cuda
    from paper_1711_02473_b200.assembly import CsrPattern, GlobalOperator
    from paper_1711_02473_b200.errors import ShapeMismatch

    p = 2
    plan = compile_kernel("action_laplace", "hex", p)
    dims = (2, 3, 2)
    cmap = torch.from_numpy(lattice_dof_map(*dims, p)).cuda()
    coords = torch.from_numpy(workloads.lattice_coords(*dims)).cuda()
    nd = lattice_ndofs(*dims, p)
    op = GlobalOperator(plan, cmap, coords, nd)
    x = torch.rand(nd, dtype=torch.float64, device="cuda")
    with pytest.raises(ShapeMismatch):
        op.apply(x, out=torch.zeros(nd - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ShapeMismatch):
        op.apply(x, out=torch.zeros(nd, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        op.apply(x, out=x)
    y = op.apply(x)
    assert torch.isfinite(y).all()
    bad = cmap.clone()
    bad[0, 0] = nd
    with pytest.raises(ValueError):
        GlobalOperator(plan, bad, coords, nd)
    with pytest.raises(ValueError):
        CsrPattern(bad, nd)
