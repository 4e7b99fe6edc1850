"""numpy restatement of the reference's UNOPTIMISED lowering — TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

This follows ``forms.lower_form`` (reference forms.py:353-417) literally:
the full tensor-product tabulation of every basis function at every point
(elements.py:397-414 product of 1D tables), the Jacobian from the P1
coordinate element (geometry.py:42-64), G = J^-1 and S = |det J|
(geometry.py:71-108), the integrand of the registry builder
(forms.py:173-193) times w_q*S_q, summed over points — with no sum
factorisation at all.  It is therefore independent of both the C oracle's
and the CUDA kernels' contraction schedules; it is O(n^6) per cell and meant
for small batches.
"""

from __future__ import annotations

import numpy as np


def _tab3(T1, T2, T3):
    """(n^3, m^3) product tabulation, x outermost on both axes."""
    n, m = T1.shape
    return np.einsum("ax,by,cz->abcxyz", T1, T2, T3).reshape(n ** 3, m ** 3)


def _tab2(T1, T2):
    n, m = T1.shape
    return np.einsum("ax,by->abxy", T1, T2).reshape(n ** 2, m ** 2)


def hex_tabulation(plan):
    B, D = plan.B, plan.D
    phi = _tab3(B, B, B)
    dphi = np.stack([_tab3(D, B, B), _tab3(B, D, B), _tab3(B, B, D)])
    return phi, dphi


def hex_geometry(plan, coords):
    """J (C, Q, 3, 3), G = J^-1, det (C, Q), weights (Q,)."""
    Bc, Dc = plan.Bc, plan.Dc
    dPhi = np.stack([_tab3(Dc, Bc, Bc), _tab3(Bc, Dc, Bc), _tab3(Bc, Bc, Dc)])  # (3, 8, Q)
    X = coords.reshape(-1, 8, 3)
    J = np.einsum("cva,bvq->cqab", X, dPhi)
    G = np.linalg.inv(J)
    det = np.linalg.det(J)
    w = plan.wq
    wq = np.einsum("x,y,z->xyz", w, w, w).reshape(-1)
    return J, G, det, wq


def quad_geometry(plan, coords):
    Bc, Dc = plan.Bc, plan.Dc
    dPhi = np.stack([_tab2(Dc, Bc), _tab2(Bc, Dc)])
    X = coords.reshape(-1, 4, 2)
    J = np.einsum("cva,bvq->cqab", X, dPhi)
    G = np.linalg.inv(J)
    det = np.linalg.det(J)
    w = plan.wq
    return J, G, det, np.einsum("x,y->xy", w, w).reshape(-1)


def evaluate(plan, inputs):
    name, cell = plan.name, plan.meta["cell"]
    coords = np.asarray(inputs["coords"], dtype=float)
    if cell == "quad":
        B, D = plan.B, plan.D
        phi = _tab2(B, B)
        dphi = np.stack([_tab2(D, B), _tab2(B, D)])
        J, G, det, wq = quad_geometry(plan, coords)
    else:
        phi, dphi = hex_tabulation(plan)
        J, G, det, wq = hex_geometry(plan, coords)
    ws = wq[None, :] * np.abs(det)                       # (C, Q)
    if name == "action_mass":
        uq = np.einsum("iq,ci->cq", phi, inputs["w0"])
        return np.einsum("iq,cq->ci", phi, ws * uq)
    if name in ("action_laplace", "action_weighted_laplace"):
        gref = np.einsum("liq,ci->clq", dphi, inputs["w0"])
        gphys = np.einsum("cqlk,clq->cqk", G, gref)
        if name == "action_weighted_laplace":
            # kappa from its own (collocated GLL) element: kappa(q) = sum_i k_i phi_i(q)
            ws = ws * np.einsum("iq,ci->cq", phi, inputs["w1"])
        f = ws[:, None, :] * np.einsum("cqlk,cqk->clq", G, gphys)
        return np.einsum("liq,clq->ci", dphi, f)
    if name == "laplace":
        K = ws[:, :, None, None] * np.einsum("cqlk,cqrk->cqlr", G, G)
        A = np.einsum("liq,cqlr,rjq->cij", dphi, K, dphi, optimize=True)
        return A.reshape(A.shape[0], -1)
    if name == "neohookean_residual":
        mu, lam = plan.params
        n3 = phi.shape[0]
        u = np.asarray(inputs["w0"]).reshape(-1, n3, 3)
        gref = np.einsum("liq,cia->caql", dphi, u)
        F = np.eye(3)[None, None] + np.einsum("cqlk,caql->cqak", G, gref)
        Jf = np.linalg.det(F)
        FinvT = np.transpose(np.linalg.inv(F), (0, 1, 3, 2))
        P = mu * (F - FinvT) + lam * np.log(Jf)[:, :, None, None] * FinvT
        flux = ws[:, :, None, None] * np.einsum("cqlk,cqak->cqal", G, P)
        r = np.einsum("liq,cqal->cia", dphi, flux)
        return r.reshape(r.shape[0], -1)
    raise NotImplementedError(name)
