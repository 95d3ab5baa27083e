"""Sparse assembly of A_l = a_l + g_l and of the right-hand side.

PAPER.md l.81-87 (Nitsche form a_l), l.91-108 (ghost penalty g_l and
A_l = a_l + g_l), l.109-121 (weak problem, matrix A_l with entries
A_l(phi_j, phi_i)).  The matrix is built by summing cell matrices over
M_{l,Omega} and face matrices over F_G; duplicates are summed by scipy's COO
-> CSR conversion.

Quadrature: n = p+1 Gauss points per direction on uncut cells and on faces
(exact for these polynomial integrands); the rule of oracle.quadrature on cut
cells (reading R6).  Parameters: gamma_D (reading R7), gamma_k and sigma
(reading R5).

Test infrastructure only (see oracle/__init__.py).
"""
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .fe import basis_1d, gauss_legendre, ghost_weight
from .geometry import CUT, INSIDE, OUTSIDE
from .quadrature import cut_cell_rules, tensor_gauss


@dataclass
class Params:
    gamma_D: float = None          # Nitsche penalty; default 5 p (p+1) (R7)
    gamma_k: tuple = None          # ghost coefficients for k = 1..p; default 0.1 (R5)
    sigma: int = -1                # ghost scaling h^(2k+sigma) (R5)
    n_q: int = None                # 1D quadrature points; default p+1

    def resolved(self, p):
        return Params(
            gamma_D=5.0 * p * (p + 1) if self.gamma_D is None else float(self.gamma_D),
            gamma_k=tuple([0.1] * p) if self.gamma_k is None else tuple(float(g) for g in self.gamma_k),
            sigma=int(self.sigma),
            n_q=p + 1 if self.n_q is None else int(self.n_q),
        )


def cell_dofs(lv, i, j):
    """Global DoF ids of cell (i,j), local order l = ky (p+1) + kx."""
    p, nl = lv.p, lv.nl
    ids = []
    for ky in range(p + 1):
        for kx in range(p + 1):
            ids.append(lv.dof_index[(j * p + ky) * nl + (i * p + kx)])
    return np.array(ids, dtype=np.int64)


def eval_basis(lv, i, j, pts):
    """Values and physical gradients of the (p+1)^2 cell basis at points."""
    p, h = lv.p, lv.h
    xl, _, yl, _ = lv.cell_bounds(i, j)
    xi = (pts[:, 0] - xl) / h
    eta = (pts[:, 1] - yl) / h
    bx, by = basis_1d(p, xi), basis_1d(p, eta)
    dx, dy = basis_1d(p, xi, 1) / h, basis_1d(p, eta, 1) / h
    v = (by[:, None, :] * bx[None, :, :]).reshape((p + 1) ** 2, -1)
    gx = (by[:, None, :] * dx[None, :, :]).reshape((p + 1) ** 2, -1)
    gy = (dy[:, None, :] * bx[None, :, :]).reshape((p + 1) ** 2, -1)
    return v, gx, gy


def cell_matrix(lv, i, j, prm):
    """Element matrix of a_l on cell (i,j): (grad u, grad v)_{T∩Omega}
    - (d_n u, v)_{Gamma∩T} - (u, d_n v)_{Gamma∩T} + gamma_D/h (u, v)_{Gamma∩T}
    (PAPER.md eq. cutfem_nitsche, l.81-86)."""
    ct = lv.cell_type[j, i]
    xl, xh, yl, yh = lv.cell_bounds(i, j)
    if ct == INSIDE:
        vp, vw = tensor_gauss(xl, xh, yl, yh, prm.n_q)
        sp_, sw, sn = np.zeros((0, 2)), np.zeros(0), np.zeros((0, 2))
    elif ct == CUT:
        vp, vw, sp_, sw, sn = cut_cell_rules(xl, xh, yl, yh, lv.circle, prm.n_q)
    else:
        raise ValueError("outside cell has no matrix")
    _, gx, gy = eval_basis(lv, i, j, vp) if len(vw) else (None, np.zeros(((lv.p + 1) ** 2, 0)), np.zeros(((lv.p + 1) ** 2, 0)))
    E = (gx * vw) @ gx.T + (gy * vw) @ gy.T
    if len(sw):
        v, sx, sy = eval_basis(lv, i, j, sp_)
        dn = sx * sn[:, 0] + sy * sn[:, 1]
        E += -((v * sw) @ dn.T) - ((dn * sw) @ v.T) + (prm.gamma_D / lv.h) * ((v * sw) @ v.T)
    return E


def ghost_face_matrix(lv, axis, i, j, prm):
    """g_l on one face F(T1,T2): sum_k gamma_k h^(2k+sigma)/(k!)^2
    ([[d_n^k u]], [[d_n^k v]])_F with a (p+1)-point Gauss rule on the full
    face.  Returns (dofs, matrix) over T1 ∪ T2 local
    DoFs (duplicates allowed; summed on assembly)."""
    p, h = lv.p, lv.h
    i2, j2 = (i + 1, j) if axis == 0 else (i, j + 1)
    g, w = gauss_legendre(p + 1)
    wq = w * h
    ones = np.ones_like(g)
    d1 = np.concatenate([cell_dofs(lv, i, j), cell_dofs(lv, i2, j2)])
    M = np.zeros((d1.size, d1.size))
    for k in range(1, p + 1):
        # normal derivative of order k at the face: T1 at xi = 1, T2 at xi = 0
        if axis == 0:
            a1 = (basis_1d(p, ones, k) / h ** k)[None, :, :] * basis_1d(p, g)[:, None, :]
            a2 = (basis_1d(p, 0 * ones, k) / h ** k)[None, :, :] * basis_1d(p, g)[:, None, :]
        else:
            a1 = (basis_1d(p, ones, k) / h ** k)[:, None, :] * basis_1d(p, g)[None, :, :]
            a2 = (basis_1d(p, 0 * ones, k) / h ** k)[:, None, :] * basis_1d(p, g)[None, :, :]
        J = np.concatenate([a1.reshape((p + 1) ** 2, -1), -a2.reshape((p + 1) ** 2, -1)])
        M += ghost_weight(k, h, prm.gamma_k[k - 1], prm.sigma) * ((J * wq) @ J.T)
    return d1, M


def assemble_matrix(lv, prm, with_ghost=True, with_cells=True):
    """Global sparse A_l."""
    prm = prm.resolved(lv.p)
    rows, cols, vals = [], [], []
    n = lv.n
    inside_E = None
    for j in range(n):
        for i in range(n):
            ct = lv.cell_type[j, i]
            if ct == OUTSIDE or not with_cells:
                continue
            if ct == INSIDE:
                if inside_E is None:
                    inside_E = cell_matrix(lv, i, j, prm)   # translation invariant
                E = inside_E
            else:
                E = cell_matrix(lv, i, j, prm)
            d = cell_dofs(lv, i, j)
            rows.append(np.repeat(d, d.size)); cols.append(np.tile(d, d.size)); vals.append(E.ravel())
    if with_ghost:
        from .geometry import ghost_faces
        for axis, i, j in ghost_faces(lv):
            d, M = ghost_face_matrix(lv, axis, i, j, prm)
            rows.append(np.repeat(d, d.size)); cols.append(np.tile(d, d.size)); vals.append(M.ravel())
    if not rows:
        return sp.csr_matrix((lv.n_dofs, lv.n_dofs))
    R, C, V = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    keep = (R >= 0) & (C >= 0)   # nodes without a DoF (fitted boundary: u = 0 strongly) drop out
    A = sp.coo_matrix((V[keep], (R[keep], C[keep])), shape=(lv.n_dofs, lv.n_dofs)).tocsr()
    A.sum_duplicates()
    return A


def assemble_rhs(lv, prm, f, g):
    """b_i = (f, phi_i)_Omega - (g, d_n phi_i)_Gamma + gamma_D/h (g, phi_i)_Gamma.
    PAPER.md l.112 states (f, v)_Omega for homogeneous data; reading R8 adds the
    standard Nitsche consistency terms for inhomogeneous g."""
    prm = prm.resolved(lv.p)
    b = np.zeros(lv.n_dofs)
    for j in range(lv.n):
        for i in range(lv.n):
            ct = lv.cell_type[j, i]
            if ct == OUTSIDE:
                continue
            xl, xh, yl, yh = lv.cell_bounds(i, j)
            if ct == INSIDE:
                vp, vw = tensor_gauss(xl, xh, yl, yh, prm.n_q)
                sp_ = np.zeros((0, 2)); sw = np.zeros(0); sn = np.zeros((0, 2))
            else:
                vp, vw, sp_, sw, sn = cut_cell_rules(xl, xh, yl, yh, lv.circle, prm.n_q)
            d = cell_dofs(lv, i, j)
            ok = d >= 0   # (fitted boundary nodes carry no DoF / test function)
            if len(vw):
                v, _, _ = eval_basis(lv, i, j, vp)
                b[d[ok]] += (v @ (vw * f(vp[:, 0], vp[:, 1])))[ok]
            if len(sw):
                v, sx, sy = eval_basis(lv, i, j, sp_)
                dn = sx * sn[:, 0] + sy * sn[:, 1]
                gv = sw * g(sp_[:, 0], sp_[:, 1])
                b[d[ok]] += (-(dn @ gv) + (prm.gamma_D / lv.h) * (v @ gv))[ok]
    return b


def l2_error(lv, u, exact, n_q):
    """||u_h - u*||_{L2(Omega)} with n_q-point rules (for the convergence pin)."""
    err = 0.0
    for j in range(lv.n):
        for i in range(lv.n):
            ct = lv.cell_type[j, i]
            if ct == OUTSIDE:
                continue
            xl, xh, yl, yh = lv.cell_bounds(i, j)
            if ct == INSIDE:
                vp, vw = tensor_gauss(xl, xh, yl, yh, n_q)
            else:
                vp, vw, _, _, _ = cut_cell_rules(xl, xh, yl, yh, lv.circle, n_q)
            if not len(vw):
                continue
            v, _, _ = eval_basis(lv, i, j, vp)
            d = cell_dofs(lv, i, j)
            uh = np.where(d >= 0, u[np.maximum(d, 0)], 0.0) @ v
            err += float(np.sum(vw * (uh - exact(vp[:, 0], vp[:, 1])) ** 2))
    return np.sqrt(err)
