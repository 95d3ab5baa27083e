"""3D version of the oracle (BASELINE.json configs[2..4]: sphere in a cube).

The paper is 2D (P l.217); the 3D problem is the same method with d = 3:
Q_p on hexahedra with Gauss-Lobatto nodal basis (P l.79), Nitsche + ghost
penalty form A_l (P l.81-108), vertex patches of 2x2x2 cells (P l.143), 8
colours (I, J, K parity; P l.179), Cartesian patches with tensor structure and
cut patches with dense inverses (P l.187-193).  Readings R2-R10 of DESIGN.md
carry over with "circle" -> "sphere"; the 3D cut quadrature is reading R12
(Saye's height-function algorithm for one analytic sphere, `cut_cell_rules3`).

Conventions: cell (i, j, k), arrays indexed [k, j, i]; lattice node
(a, b, c) with flat index (c NL + b) NL + a.

Test infrastructure only (see oracle/__init__.py).
"""
import math
from dataclasses import dataclass
from math import factorial

import numpy as np
import scipy.sparse as sp

from .assemble import Params
from .fe import basis_1d, gauss_legendre, gauss_lobatto_nodes
from .geometry import CARTESIAN, CUT, CUTPATCH, INSIDE, OUTSIDE, Patch, is_fitted


@dataclass(frozen=True)
class Sphere:
    cx: float
    cy: float
    cz: float
    r: float


class Level3:
    def __init__(self, x0, y0, z0, length, n, sphere, p):
        self.x0, self.y0, self.z0 = float(x0), float(y0), float(z0)
        self.length, self.n, self.p = float(length), int(n), int(p)
        self.sphere = sphere
        self.h = self.length / self.n
        self.nl = self.n * self.p + 1
        self.dim = 3
        self.n_colours = 8
        self.cell_type = classify3(self)
        self.dof_mask = node_mask3(self)
        nl = self.nl
        self.dof_index = -np.ones(nl ** 3, dtype=np.int64)
        flat = np.flatnonzero(self.dof_mask.ravel())
        self.dof_index[flat] = np.arange(flat.size)
        self.dof_nodes = flat
        self.n_dofs = flat.size

    def lo(self, i, j, k):
        h = self.h
        return np.array([self.x0 + i * h, self.y0 + j * h, self.z0 + k * h])

    def hi(self, i, j, k):
        """x0 + (i+1) h (reading R2: the same fp64 expression as the
        classification, not lo + h)"""
        h = self.h
        return np.array([self.x0 + (i + 1.0) * h, self.y0 + (j + 1.0) * h, self.z0 + (k + 1.0) * h])

    def ctype(self, i, j, k):
        n = self.n
        if 0 <= i < n and 0 <= j < n and 0 <= k < n:
            return int(self.cell_type[k, j, i])
        return OUTSIDE

    def active(self, i, j, k):
        return self.ctype(i, j, k) != OUTSIDE

    def cells_1d(self, a):
        p, n = self.p, self.n
        if a % p == 0:
            return [c for c in (a // p - 1, a // p) if 0 <= c < n]
        return [a // p]

    def node_support(self, a, b, c):
        return [(i, j, k) for k in self.cells_1d(c) for j in self.cells_1d(b) for i in self.cells_1d(a)
                if self.active(i, j, k)]


def classify3(lv):
    """Reading R2 in 3D: exact fp64 squared distances from the sphere centre
    to the closed cell box, summed in the order x, y, z."""
    s = lv.sphere
    n = lv.n
    if is_fitted(s):
        return np.full((n, n, n), INSIDE, dtype=np.int8)
    idx = np.arange(n, dtype=np.float64)
    out = np.full((n, n, n), CUT, dtype=np.int8)
    q, f = [], []
    for o, c in ((lv.x0, s.cx), (lv.y0, s.cy), (lv.z0, s.cz)):
        lo, hi = o + idx * lv.h, o + (idx + 1.0) * lv.h
        q.append(np.minimum(np.maximum(c, lo), hi) - c)
        f.append(np.maximum(np.abs(lo - c), np.abs(hi - c)))
    dmin2 = (q[0][None, None, :] * q[0][None, None, :] + q[1][None, :, None] * q[1][None, :, None]) \
        + q[2][:, None, None] * q[2][:, None, None]
    dmax2 = (f[0][None, None, :] * f[0][None, None, :] + f[1][None, :, None] * f[1][None, :, None]) \
        + f[2][:, None, None] * f[2][:, None, None]
    r2 = s.r * s.r
    out[dmax2 <= r2] = INSIDE
    out[dmin2 >= r2] = OUTSIDE
    return out


def node_mask3(lv):
    p, n = lv.p, lv.n
    act = lv.cell_type != OUTSIDE
    m = np.zeros((lv.nl,) * 3, dtype=bool)
    for kz in range(p + 1):
        for ky in range(p + 1):
            for kx in range(p + 1):
                m[kz:kz + n * p:p, ky:ky + n * p:p, kx:kx + n * p:p] |= act
    if is_fitted(lv.sphere):   # strong Dirichlet: no DoF on the box boundary
        m[0], m[-1], m[:, 0], m[:, -1], m[:, :, 0], m[:, :, -1] = (False,) * 6
    return m


def ghost_faces3(lv):
    """(axis, i, j, k): face between cell (i,j,k) and its + neighbour along axis."""
    out = []
    n = lv.n
    for k in range(n):
        for j in range(n):
            for i in range(n):
                for axis in range(3):
                    i2, j2, k2 = i + (axis == 0), j + (axis == 1), k + (axis == 2)
                    t1, t2 = lv.ctype(i, j, k), lv.ctype(i2, j2, k2)
                    if t1 != OUTSIDE and t2 != OUTSIDE and (t1 == CUT or t2 == CUT):
                        out.append((axis, i, j, k))
    return out


# ---- quadrature (reading R12) ----------------------------------------------

def _breaks(lo, hi, pts):
    return sorted(set(b for b in [lo, hi] + pts if lo <= b <= hi))


def cut_cell_rules3(lo, hi, sph, n):
    """Volume rule on T ∩ Omega and surface rule on Gamma ∩ T for a box
    [lo, hi] and the sphere: Saye's height-function recursion with the roots
    in closed form.
      1. height axis h = argmax_d |centre_d - c_d| (ties to the larger d);
         base axes = the other two; among them the inner axis v is chosen by
         the same rule, the outer axis is u.
      2. the base integrand is smooth away from the circles (in the (u, v)
         plane, centred at (c_u, c_v)) of radius r (silhouette) and
         sqrt(r^2 - (face_h - c_h)^2) for the two faces normal to h.  The outer
         interval [u_lo, u_hi] is split where a circle meets v = v_lo or
         v = v_hi and at c_u +- R; at each outer Gauss node the inner interval
         is split where a circle meets the line.
      3. at each base node the inside part of the height line is the single
         interval [max(lo_h, c_h - S), min(hi_h, c_h + S)], S = sqrt(r^2 -
         rho^2), integrated with an n-point Gauss rule; the sphere points
         c_h +- S strictly inside (lo_h, hi_h) are surface points with
         weight w_u w_v r / S and outward normal (x - c) / r.
    Returns (vol_pts (m,3), vol_w, surf_pts (k,3), surf_w, normals (k,3))."""
    c = np.array([sph.cx, sph.cy, sph.cz])
    r = sph.r
    r2 = r * r
    lo = [float(v) for v in lo]
    hi = [float(v) for v in hi]
    xc = [0.5 * (lo[d] + hi[d]) for d in range(3)]
    dist = [abs(xc[d] - c[d]) for d in range(3)]
    hax = max(range(3), key=lambda d: (dist[d], d))
    base = [d for d in range(3) if d != hax]
    vax = max(base, key=lambda d: (dist[d], d))
    uax = base[0] if base[1] == vax else base[1]
    radii2 = [r2]
    for face in (lo[hax], hi[hax]):
        dd = face - c[hax]
        D = r2 - dd * dd
        if D > 0.0:
            radii2.append(D)
    g, w = gauss_legendre(n)
    ubr = []
    for R2 in radii2:
        for vf in (lo[vax], hi[vax]):
            dv = vf - c[vax]
            D = R2 - dv * dv
            if D > 0.0:
                q = math.sqrt(D)
                ubr += [c[uax] - q, c[uax] + q]
        R = math.sqrt(R2)
        ubr += [c[uax] - R, c[uax] + R]
    ub = _breaks(lo[uax], hi[uax], ubr)
    vp, vw, spts, sw, sn = [], [], [], [], []
    for ua, ubb in zip(ub[:-1], ub[1:]):
        if not ubb > ua:
            continue
        for gi, wi in zip(g, w):
            u = ua + (ubb - ua) * gi
            wu = wi * (ubb - ua)
            du = u - c[uax]
            vbr = []
            for R2 in radii2:
                D = R2 - du * du
                if D > 0.0:
                    q = math.sqrt(D)
                    vbr += [c[vax] - q, c[vax] + q]
            vb = _breaks(lo[vax], hi[vax], vbr)
            for va, vbb in zip(vb[:-1], vb[1:]):
                if not vbb > va:
                    continue
                for gj, wj in zip(g, w):
                    v = va + (vbb - va) * gj
                    wuv = wu * (wj * (vbb - va))
                    dv = v - c[vax]
                    D = r2 - (du * du + dv * dv)
                    if not D > 0.0:
                        continue
                    S = math.sqrt(D)
                    hl = max(lo[hax], c[hax] - S)
                    hh = min(hi[hax], c[hax] + S)
                    pt = [0.0, 0.0, 0.0]
                    pt[uax], pt[vax] = u, v
                    if hh > hl:
                        for gk, wk in zip(g, w):
                            pt[hax] = hl + (hh - hl) * gk
                            vp.append(tuple(pt))
                            vw.append(wuv * (wk * (hh - hl)))
                    for sv in (c[hax] - S, c[hax] + S):
                        if lo[hax] < sv < hi[hax]:
                            pt[hax] = sv
                            spts.append(tuple(pt))
                            sw.append(wuv * r / S)
                            sn.append(tuple((np.array(pt) - c) / r))
    as3 = lambda a: np.array(a, dtype=np.float64).reshape(-1, 3)
    return as3(vp), np.array(vw), as3(spts), np.array(sw), as3(sn)


def tensor_gauss3(lo, hi, n):
    g, w = gauss_legendre(n)
    axes = [lo[d] + (hi[d] - lo[d]) * g for d in range(3)]
    W = [w * (hi[d] - lo[d]) for d in range(3)]
    Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    WW = W[2][:, None, None] * W[1][None, :, None] * W[0][None, None, :]
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1), WW.ravel()


# ---- assembly --------------------------------------------------------------

def cell_dofs3(lv, i, j, k):
    p, nl = lv.p, lv.nl
    ids = []
    for kz in range(p + 1):
        for ky in range(p + 1):
            for kx in range(p + 1):
                ids.append(lv.dof_index[((k * p + kz) * nl + (j * p + ky)) * nl + (i * p + kx)])
    return np.array(ids, dtype=np.int64)


def eval_basis3(lv, i, j, k, pts):
    """values and physical gradients of the (p+1)^3 basis, local index
    (kz (p+1) + ky) (p+1) + kx"""
    p, h = lv.p, lv.h
    o = lv.lo(i, j, k)
    xi = [(pts[:, d] - o[d]) / h for d in range(3)]
    B = [basis_1d(p, xi[d]) for d in range(3)]
    D = [basis_1d(p, xi[d], 1) / h for d in range(3)]
    def t(a, b_, c_):
        return (c_[:, None, None, :] * b_[None, :, None, :] * a[None, None, :, :]).reshape((p + 1) ** 3, -1)
    v = t(B[0], B[1], B[2])
    return v, t(D[0], B[1], B[2]), t(B[0], D[1], B[2]), t(B[0], B[1], D[2])


def cell_matrix3(lv, i, j, k, prm):
    ct = lv.cell_type[k, j, i]
    lo = lv.lo(i, j, k)
    hi = lv.hi(i, j, k)
    if ct == INSIDE:
        vp, vw = tensor_gauss3(lo, hi, prm.n_q)
        sp_ = np.zeros((0, 3)); sw = np.zeros(0); sn = np.zeros((0, 3))
    else:
        vp, vw, sp_, sw, sn = cut_cell_rules3(lo, hi, lv.sphere, prm.n_q)
    nb = (lv.p + 1) ** 3
    E = np.zeros((nb, nb))
    if len(vw):
        _, gx, gy, gz = eval_basis3(lv, i, j, k, vp)
        E += (gx * vw) @ gx.T + (gy * vw) @ gy.T + (gz * vw) @ gz.T
    if len(sw):
        v, sx, sy, sz = eval_basis3(lv, i, j, k, sp_)
        dn = sx * sn[:, 0] + sy * sn[:, 1] + sz * sn[:, 2]
        E += -((v * sw) @ dn.T) - ((dn * sw) @ v.T) + (prm.gamma_D / lv.h) * ((v * sw) @ v.T)
    return E


def ghost_face_matrix3(lv, axis, i, j, k, prm):
    """g_l on one face: sum_k gamma_k h^(2k+sigma)/(k!)^2 ([[d_n^k u]],
    [[d_n^k v]])_F with a (p+1)^2 Gauss rule on the full face (P l.104-108)."""
    p, h = lv.p, lv.h
    c2 = (i + (axis == 0), j + (axis == 1), k + (axis == 2))
    g, w = gauss_legendre(p + 1)
    t1, t2 = [d for d in range(3) if d != axis]
    W = np.outer(w * h, w * h).ravel()   # [q1 (t1), q2 (t2)] -> t1 slow
    d1 = np.concatenate([cell_dofs3(lv, i, j, k), cell_dofs3(lv, *c2)])
    nb = (p + 1) ** 3
    M = np.zeros((2 * nb, 2 * nb))
    for kk in range(1, p + 1):
        J = np.zeros((2 * nb, len(W)))
        for side, xiv in ((0, 1.0), (1, 0.0)):
            dn = basis_1d(p, [xiv], kk)[:, 0] / h ** kk
            b1 = basis_1d(p, g)    # tangential values at Gauss points
            for kz in range(p + 1):
                for ky in range(p + 1):
                    for kx in range(p + 1):
                        idx = (kz * (p + 1) + ky) * (p + 1) + kx
                        kd = (kx, ky, kz)
                        val = dn[kd[axis]] * np.outer(b1[kd[t1]], b1[kd[t2]]).ravel()
                        J[side * nb + idx] = val if side == 0 else -val
        coef = prm.gamma_k[kk - 1] * h ** (2 * kk + prm.sigma) / float(factorial(kk)) ** 2
        M += coef * ((J * W) @ J.T)
    return d1, M


def assemble_matrix3(lv, prm, with_ghost=True, with_cells=True):
    prm = prm.resolved(lv.p)
    rows, cols, vals = [], [], []
    n = lv.n
    inside_E = None
    for k in range(n):
        for j in range(n):
            for i in range(n):
                ct = lv.cell_type[k, j, i]
                if ct == OUTSIDE or not with_cells:
                    continue
                if ct == INSIDE:
                    if inside_E is None:
                        inside_E = cell_matrix3(lv, i, j, k, prm)
                    E = inside_E
                else:
                    E = cell_matrix3(lv, i, j, k, prm)
                d = cell_dofs3(lv, i, j, k)
                rows.append(np.repeat(d, d.size)); cols.append(np.tile(d, d.size)); vals.append(E.ravel())
    if with_ghost:
        for axis, i, j, k in ghost_faces3(lv):
            d, M = ghost_face_matrix3(lv, axis, i, j, k, prm)
            rows.append(np.repeat(d, d.size)); cols.append(np.tile(d, d.size)); vals.append(M.ravel())
    R, C, V = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    keep = (R >= 0) & (C >= 0)   # nodes without a DoF (fitted boundary: u = 0 strongly) drop out
    A = sp.coo_matrix((V[keep], (R[keep], C[keep])), shape=(lv.n_dofs, lv.n_dofs)).tocsr()
    A.sum_duplicates()
    return A


# ---- patches ---------------------------------------------------------------

def vertex_patch3(lv, I, J, K):
    """3D analogue of oracle.geometry.vertex_patch (readings R3, R4): patch at
    every vertex of an active cell, interior set = DoF nodes whose active
    support lies in the patch; Cartesian iff the 8 cells are Inside and none
    of the 24 face neighbours of the 2x2x2 block is Cut; colour = (I mod 2) +
    2 (J mod 2) + 4 (K mod 2)."""
    p, nl = lv.p, lv.nl
    block = [(i, j, k) for k in (K - 1, K) for j in (J - 1, J) for i in (I - 1, I)]
    cells = [c for c in block if lv.active(*c)]
    if not cells:
        return None
    if is_fitted(lv.sphere) and not (0 < I < lv.n and 0 < J < lv.n and 0 < K < lv.n):
        return None   # vertices contained in the open box (P l.143)
    pt = Patch()
    pt.I, pt.J = I, J
    pt.K = K
    pt.cells = cells
    cs = set(cells)
    interior = []
    for c in range(max(0, p * (K - 1)), min(nl - 1, p * (K + 1)) + 1):
        for b in range(max(0, p * (J - 1)), min(nl - 1, p * (J + 1)) + 1):
            for a in range(max(0, p * (I - 1)), min(nl - 1, p * (I + 1)) + 1):
                if not lv.dof_mask[c, b, a]:
                    continue
                if set(lv.node_support(a, b, c)) <= cs:
                    interior.append(int(lv.dof_index[(c * nl + b) * nl + a]))
    pt.interior = np.array(interior, dtype=np.int64)
    all_inside = len(cells) == 8 and all(lv.ctype(*c) == INSIDE for c in cells)
    nbrs = []
    for axis in range(3):
        for side in (-2, 1):
            for s1 in (-1, 0):
                for s2 in (-1, 0):
                    o = [I, J, K]
                    off = [0, 0, 0]
                    off[axis] = side
                    t = [d for d in range(3) if d != axis]
                    off[t[0]] = s1
                    off[t[1]] = s2
                    nbrs.append((o[0] + off[0], o[1] + off[1], o[2] + off[2]))
    touches = any(lv.ctype(*c) == CUT for c in nbrs)
    pt.kind = CARTESIAN if (all_inside and not touches) else CUTPATCH
    pt.colour = (I % 2) + 2 * (J % 2) + 4 * (K % 2)
    return pt


def build_patches3(lv):
    out = []
    for K in range(lv.n + 1):
        for J in range(lv.n + 1):
            for I in range(lv.n + 1):
                pt = vertex_patch3(lv, I, J, K)
                if pt is not None:
                    out.append(pt)
    return out


# ---- transfer --------------------------------------------------------------

def prolongation_matrix3(coarse, fine):
    """P[j, i] = phi^c_i(x_j) (P l.130-133), as in oracle.transfer."""
    p = fine.p
    xi = gauss_lobatto_nodes(p)
    rows, cols, vals = [], [], []
    nlf, nlc = fine.nl, coarse.nl
    for jf, node in enumerate(fine.dof_nodes):
        c, rem = divmod(int(node), nlf * nlf)
        b, a = divmod(rem, nlf)
        i_f, j_f, k_f = fine.node_support(a, b, c)[0]
        loc = (a - i_f * p, b - j_f * p, c - k_f * p)
        C = (i_f // 2, j_f // 2, k_f // 2)
        xs = [((f % 2) + xi[l]) / 2.0 for f, l in zip((i_f, j_f, k_f), loc)]
        bx, by, bz = [basis_1d(p, [v])[:, 0] for v in xs]
        for nz in range(p + 1):
            for ny in range(p + 1):
                for nx in range(p + 1):
                    wgt = bx[nx] * by[ny] * bz[nz]
                    ic = coarse.dof_index[((C[2] * p + nz) * nlc + C[1] * p + ny) * nlc + C[0] * p + nx]
                    if wgt != 0.0 and ic >= 0:   # (ic < 0: fitted boundary node, coefficient 0)
                        rows.append(jf); cols.append(int(ic)); vals.append(wgt)
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine.n_dofs, coarse.n_dofs))
