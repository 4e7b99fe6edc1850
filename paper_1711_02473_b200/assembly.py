"""Global (assembled) operators — SURVEY.md §8(f) items 1 and 3.

The reference stops at the per-cell kernel; global assembly is the caller's
job.  The immediate caller of the hot path is the E-vector <->
L-vector map of a conforming mesh: gather a cell's dofs from the global
vector, apply the cell kernel, scatter-add back (PAPER.md:176-189,
1804-1819).  ``GlobalOperator.apply`` does all three in ONE launch of the
C2 line kernel (``sfk_eval_gather_scatter``: gather fused into the x stage,
fp64 atomic scatter fused into the transposed x stage), so the E-vector
never exists in HBM.

``CsrPattern`` + ``assemble_csr`` (§8(f) item 3) assemble the global
stiffness matrix itself: the CSR pattern is built on the device from the
cell -> dof map (``sfk_csr_create``: radix sort + unique of the (row, col)
pairs) and the C5 local-matrix kernel scatter-adds every cell matrix
straight into the CSR values (``sfk_assemble_csr``), so the (p+1)^6 local
matrices never reach HBM.  ``CsrPattern.matrix`` wraps the result as a
``torch.sparse_csr_tensor`` (cuSPARSE SpMV for the solver).

``lattice_dof_map`` numbers the continuous Q_p space of the structured
jittered lattice used by the BASELINE configs: cell (cx, cy, cz), local dof
(a, b, c) (reference order (a*n+b)*n+c) -> global grid node
(cx*p + a, cy*p + b, cz*p + c) of the (nx*p+1, ny*p+1, nz*p+1) grid.
"""

from __future__ import annotations

import numpy as np

from .errors import NativeError, ShapeMismatch

__all__ = ["lattice_dof_map", "lattice_vector_dof_map", "lattice_boundary_mask",
           "GlobalOperator", "cg",
           "CsrPattern", "assemble_csr", "insert_csr", "assemble_csr_from"]


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


def lattice_vector_dof_map(nx, ny, nz, degree, ix_range=None):
    """(C, 3 (p+1)^3) int32 global dofs of a vector Q_p field in the
    reference's vector layout (local dof = 3*node + comp, global dof =
    3*node + comp of the node lattice)."""
    g = lattice_dof_map(nx, ny, nz, degree, ix_range).astype(np.int64)
    v = 3 * g[:, :, None] + np.arange(3)[None, None, :]
    if v.max() >= 2 ** 31:
        raise ValueError("global dof count exceeds int32")
    return np.ascontiguousarray(v.reshape(g.shape[0], -1), dtype=np.int32)


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
    """y = sum_c P_c^T K_c(P_c x), applied matrix-free on the GPU in ONE
    fused gather -> cell kernel -> scatter launch (``sfk_eval_global``).

    plan       a hex KernelPlan: ``action_laplace`` (GL or collocated GLL),
               ``action_weighted_laplace`` (collocated GLL; pass ``w1``) or
               ``neohookean_residual`` (then y is the assembled nonlinear
               residual r(x) and cell_dofs the vector map)
    cell_dofs  (C, nd) int32 CUDA tensor (``lattice_dof_map`` /
               ``lattice_vector_dof_map``)
    coords     (C, 24) float64 CUDA tensor
    ndofs      length of the global vectors
    w1         (C, n^3) float64 CUDA tensor of per-cell coefficient values
               (kappa) for the weighted Laplacian, not gathered
    """

    def __init__(self, plan, cell_dofs, coords, ndofs, w1=None):
        import torch

        if cell_dofs.dtype != torch.int32 or not cell_dofs.is_cuda:
            raise TypeError("cell_dofs must be an int32 CUDA tensor")
        if coords.dtype != torch.float64 or not coords.is_cuda:
            raise TypeError("coords must be a float64 CUDA tensor")
        nd = plan.argument_size("w0")
        if tuple(cell_dofs.shape) != (coords.shape[0], nd):
            raise ShapeMismatch("cell_dofs must be (%d, %d)" % (coords.shape[0], nd))
        if "w1" in dict(plan.arguments):
            if w1 is None:
                raise ShapeMismatch("plan %s needs w1 (per-cell coefficient)" % plan.name)
            if (w1.dtype != torch.float64 or not w1.is_cuda
                    or tuple(w1.shape) != (coords.shape[0], plan.argument_size("w1"))):
                raise ShapeMismatch("w1 must be a float64 CUDA (%d, %d) tensor"
                                    % (coords.shape[0], plan.argument_size("w1")))
            w1 = w1.contiguous()
        elif w1 is not None:
            raise ShapeMismatch("plan %s takes no w1" % plan.name)
        if coords.device != cell_dofs.device:
            raise ValueError("cell_dofs and coords must be on one device")
        self.plan = plan
        self.cell_dofs = cell_dofs.contiguous()
        self.coords = coords.contiguous()
        self.ndofs = int(ndofs)
        self.w1 = w1
        # one-time map check: an index outside [0, ndofs) would turn into an
        # out-of-bounds fp64 atomic in the fused scatter
        _check_map(self.cell_dofs, self.ndofs)

    def apply(self, x, out=None, accumulate=False, stream=None):
        import torch

        from .runtime import _check, load_library, native_plan

        if x.dtype != torch.float64 or not x.is_cuda or x.numel() != self.ndofs:
            raise ShapeMismatch("x must be a float64 CUDA vector of length %d" % self.ndofs)
        if x.device != self.coords.device:
            raise ValueError("x must be on %s" % self.coords.device)
        x = x.contiguous()
        if out is None:
            out = torch.zeros_like(x)
        else:
            if (not isinstance(out, torch.Tensor) or out.dtype != torch.float64
                    or out.device != x.device or out.numel() != self.ndofs
                    or not out.is_contiguous()):
                raise ShapeMismatch("out must be a contiguous float64 vector of length %d on %s"
                                    % (self.ndofs, x.device))
            if out.data_ptr() == x.data_ptr() or _aliases(out, x):
                raise ValueError("out must not alias x (the gather reads x while the "
                                 "scatter writes out)")
            if not accumulate:
                out.zero_()
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        with torch.cuda.device(x.device):
            _check(load_library().sfk_eval_global(
                native_plan(self.plan), self.coords.shape[0], self.cell_dofs.data_ptr(),
                x.data_ptr(), out.data_ptr(), self.coords.data_ptr(),
                self.w1.data_ptr() if self.w1 is not None else None, stream))
        return out

    __call__ = apply


def _aliases(a, b):
    a0, b0 = a.data_ptr(), b.data_ptr()
    return a0 < b0 + b.numel() * b.element_size() and b0 < a0 + a.numel() * a.element_size()


def _check_map(cell_dofs, ndofs):
    """0 <= cell_dofs < ndofs (one device reduction, checked once)."""
    if cell_dofs.numel() == 0:
        return
    lo = int(cell_dofs.min().item())
    hi = int(cell_dofs.max().item())
    if lo < 0 or hi >= ndofs:
        raise ValueError("cell_dofs entries must lie in [0, %d), got [%d, %d]" % (ndofs, lo, hi))


def _values(values, pattern, device):
    """The CSR value array to accumulate into: zeros, or the caller's
    (checked: float64, contiguous, nnz entries, on the pattern's device)."""
    import torch

    if values is None:
        return torch.zeros(pattern.nnz, dtype=torch.float64, device=device)
    if (not isinstance(values, torch.Tensor) or values.dtype != torch.float64
            or not values.is_contiguous() or values.device != device):
        raise ShapeMismatch("values must be a contiguous float64 tensor on %s" % device)
    if values.numel() != pattern.nnz:
        raise ShapeMismatch("values must have nnz = %d entries" % pattern.nnz)
    return values


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


class _DevArray:
    """__cuda_array_interface__ view of a libsfk-owned device array."""

    def __init__(self, ptr, n, typestr, owner):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3}
        self._owner = owner


class CsrPattern:
    """Sparsity pattern of K = sum_c P_c^T A_c P_c on the device.

    ``row_ptr`` (ndofs + 1, int64) and ``col_idx`` (nnz, int32, sorted per
    row) are torch views of arrays owned by libsfk (freed with the pattern).
    """

    def __init__(self, cell_dofs, ndofs, stream=None):
        import ctypes

        import torch

        from .runtime import _check, load_library

        if cell_dofs.dtype != torch.int32 or not cell_dofs.is_cuda or cell_dofs.dim() != 2:
            raise TypeError("cell_dofs must be a 2D int32 CUDA tensor")
        cell_dofs = cell_dofs.contiguous()
        _check_map(cell_dofs, int(ndofs))
        self._lib = load_library()
        self._h = ctypes.c_void_p()
        if stream is None:
            stream = torch.cuda.current_stream(cell_dofs.device).cuda_stream
        with torch.cuda.device(cell_dofs.device):
            _check(self._lib.sfk_csr_create(cell_dofs.shape[0], cell_dofs.shape[1],
                                            cell_dofs.data_ptr(), int(ndofs), stream,
                                            ctypes.byref(self._h)))
        nrows, nnz = ctypes.c_int64(), ctypes.c_int64()
        rp, ci = ctypes.c_void_p(), ctypes.c_void_p()
        _check(self._lib.sfk_csr_info(self._h, ctypes.byref(nrows), ctypes.byref(nnz),
                                      ctypes.byref(rp), ctypes.byref(ci)))
        self.nrows, self.nnz = nrows.value, nnz.value
        self.device = cell_dofs.device
        with torch.cuda.device(self.device):
            self.row_ptr = torch.as_tensor(_DevArray(rp.value, self.nrows + 1, "<i8", self),
                                           device=self.device)
            self.col_idx = torch.as_tensor(_DevArray(ci.value, self.nnz, "<i4", self),
                                           device=self.device)

    def __del__(self):
        try:
            if self._h:
                self._lib.sfk_csr_destroy(self._h)
        except Exception:
            pass

    def entry_map(self, cell_dofs, stream=None):
        """(C, nd^2) int32 CUDA tensor: position of every cell entry A_c[i][j]
        in ``values`` (``sfk_csr_entry_map``; once per pattern, then every
        ``assemble_csr(..., entry_map=m)`` inserts with one load + one atomic
        per entry instead of a binary search)."""
        import torch

        from .runtime import _check

        cell_dofs = cell_dofs.contiguous()
        nc, nd = cell_dofs.shape
        m = torch.empty((nc, nd * nd), dtype=torch.int32, device=cell_dofs.device)
        if stream is None:
            stream = torch.cuda.current_stream(cell_dofs.device).cuda_stream
        with torch.cuda.device(cell_dofs.device):
            _check(self._lib.sfk_csr_entry_map(self._h, nc, nd, cell_dofs.data_ptr(),
                                               m.data_ptr(), stream))
        return m

    def matrix(self, values):
        """torch.sparse_csr_tensor over this pattern (values length nnz)."""
        import torch

        # torch wants one index dtype for both arrays
        if self.nnz < 2 ** 31:
            crow, col = self.row_ptr.to(torch.int32), self.col_idx
        else:
            crow, col = self.row_ptr, self.col_idx.to(torch.int64)
        return torch.sparse_csr_tensor(crow, col, values, size=(self.nrows, self.nrows),
                                       check_invariants=False)


def assemble_csr(plan, cell_dofs, coords, pattern, values=None, entry_map=None, stream=None):
    """Assembled stiffness matrix values (length pattern.nnz, float64 CUDA):
    values += sum_c P_c^T A_c P_c with A_c the hex ``laplace`` cell matrix of
    ``plan`` (C5 kernels: p <= 4 fused with a binary search or the entry map,
    p = 5..8 the DMMA kernel of hex_matrix_tcn.cu, which inserts through the
    entry map — built here when not given).  ``values`` is zeroed unless given."""
    import torch

    from .runtime import _check, load_library, native_plan

    if cell_dofs.dtype != torch.int32 or not cell_dofs.is_cuda:
        raise TypeError("cell_dofs must be an int32 CUDA tensor")
    if coords.dtype != torch.float64 or not coords.is_cuda:
        raise TypeError("coords must be a float64 CUDA tensor")
    nd = plan.return_size
    n3 = int(round(nd ** 0.5))
    if tuple(cell_dofs.shape) != (coords.shape[0], n3):
        raise ShapeMismatch("cell_dofs must be (%d, %d)" % (coords.shape[0], n3))
    cell_dofs = cell_dofs.contiguous()
    coords = coords.contiguous()
    if entry_map is not None and (entry_map.dtype != torch.int32 or not entry_map.is_contiguous()
                                  or tuple(entry_map.shape) != (coords.shape[0], n3 * n3)):
        raise ShapeMismatch("entry_map must be a contiguous int32 (%d, %d) tensor"
                            % (coords.shape[0], n3 * n3))
    if entry_map is None and n3 > 125:
        entry_map = pattern.entry_map(cell_dofs)
    values = _values(values, pattern, coords.device)
    if stream is None:
        stream = torch.cuda.current_stream(coords.device).cuda_stream
    with torch.cuda.device(coords.device):
        _check(load_library().sfk_assemble_csr(
            native_plan(plan), coords.shape[0], cell_dofs.data_ptr(), coords.data_ptr(),
            pattern.row_ptr.data_ptr(), pattern.col_idx.data_ptr(),
            entry_map.data_ptr() if entry_map is not None else None, values.data_ptr(), stream))
    return values


def insert_csr(cell_matrices, cell_dofs, pattern, values=None, entry_map=None, stream=None):
    """values += sum_c P_c^T A_c P_c for dense cell matrices (C, nd*nd) or
    (C, nd, nd) float64 CUDA, test index outer — what any matrix kernel
    returns (a hand-written family or a generated LoopProgram), so every
    registry matrix form on every cell can be assembled (``sfk_csr_insert``:
    one fp64 atomic per entry, positions from ``entry_map`` or a binary
    search).  ``values`` is zeroed unless given."""
    import torch

    from .runtime import _check, load_library

    if cell_dofs.dtype != torch.int32 or not cell_dofs.is_cuda:
        raise TypeError("cell_dofs must be an int32 CUDA tensor")
    if cell_matrices.dtype != torch.float64 or not cell_matrices.is_cuda:
        raise TypeError("cell_matrices must be a float64 CUDA tensor")
    ncells, nd = cell_dofs.shape
    if cell_matrices.numel() != ncells * nd * nd:
        raise ShapeMismatch("cell_matrices must hold (%d, %d x %d) entries" % (ncells, nd, nd))
    cell_dofs = cell_dofs.contiguous()
    cell_matrices = cell_matrices.contiguous()
    if entry_map is not None and (entry_map.dtype != torch.int32 or not entry_map.is_contiguous()
                                  or entry_map.numel() != ncells * nd * nd):
        raise ShapeMismatch("entry_map must be a contiguous int32 (%d, %d) tensor"
                            % (ncells, nd * nd))
    values = _values(values, pattern, cell_dofs.device)
    if stream is None:
        stream = torch.cuda.current_stream(cell_dofs.device).cuda_stream
    with torch.cuda.device(cell_dofs.device):
        _check(load_library().sfk_csr_insert(
            ncells, nd, cell_matrices.data_ptr(), cell_dofs.data_ptr(),
            pattern.row_ptr.data_ptr(), pattern.col_idx.data_ptr(),
            entry_map.data_ptr() if entry_map is not None else None, values.data_ptr(), stream))
    return values


def assemble_csr_from(plan, inputs, cell_dofs, pattern, values=None, entry_map=None):
    """Assemble any matrix kernel: evaluate the per-cell matrices of ``plan``
    (a ``compile_kernel`` plan or a ``load_program`` LoopProgram plan) on
    ``inputs`` with ``evaluate_batched`` and insert them (``insert_csr``).
    For the hex Laplace matrix at p <= 4 ``assemble_csr`` is the fused path
    (no cell matrices in HBM); this one covers every other form, cell and
    degree."""
    from .runtime import evaluate_batched

    A = evaluate_batched(plan, inputs)
    return insert_csr(A, cell_dofs, pattern, values=values, entry_map=entry_map)
