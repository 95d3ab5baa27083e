"""Background mesh hierarchy, cell classification, ghost faces, vertex patches
and their colouring.

PAPER.md l.65-69 (nested Cartesian meshes M_0 ⊏ ... ⊏ M_L; M_{l,Omega} cells
with nonempty intersection with Omega; M_{l,Gamma} cells cut by Gamma),
l.96-101 (ghost faces F_G), l.141-156 (vertex patches), l.179 (colouring),
l.187 (interior vs cut patches), l.217 (experimental setup).

Conventions: cell (i, j) is
[x0 + i h, x0 + (i+1) h] x [y0 + j h, y0 + (j+1) h], arrays are indexed
[j, i] (y-major).  Lattice node (a, b), 0 <= a, b <= n p, sits at
x0 + (a div p + xi_{a mod p}) h with xi the Gauss-Lobatto nodes.

Test infrastructure only (see oracle/__init__.py).
"""
from dataclasses import dataclass

import numpy as np

OUTSIDE, INSIDE, CUT = 0, 1, 2


@dataclass(frozen=True)
class Circle:
    """Analytic level set phi(x) = |x - c| - r ("analytic
    level set function with exact zero level on the perimeter")."""
    cx: float
    cy: float
    r: float


@dataclass(frozen=True)
class FittedBox:
    """Fitted domain: Omega = the open background box itself (its boundary on
    mesh lines), homogeneous Dirichlet condition imposed strongly (nodes on
    the box boundary carry no DoF).  The paper's "Square" baseline (PAPER.md
    Table 1 l.219-238, Fig. 2 square curves l.388-399) and BASELINE.json
    configs[4]'s fitted cube: every cell is Inside, there are no cut cells,
    ghost faces or Nitsche terms, and patches sit at the vertices contained
    in Omega (P l.143 read literally: the interior vertices), all Cartesian.
    Used for 2D and 3D levels."""


def is_fitted(dom):
    return isinstance(dom, FittedBox)


class Level:
    """One level M_l of the nested Cartesian hierarchy with its geometry."""

    def __init__(self, x0, y0, length, n, circle, p):
        self.x0, self.y0, self.length, self.n, self.p = float(x0), float(y0), float(length), int(n), int(p)
        self.circle = circle
        self.h = self.length / self.n           # R1: h = L / n, fp64 division
        self.nl = self.n * self.p + 1           # lattice nodes per side
        self.dim = 2
        self.n_colours = 4
        self.cell_type = classify_cells(self)
        self.dof_mask = node_mask(self)
        self.dof_index = -np.ones(self.nl * self.nl, dtype=np.int64)
        flat = np.flatnonzero(self.dof_mask.ravel())
        self.dof_index[flat] = np.arange(flat.size)   # lexicographic (b-major, a-minor)
        self.dof_nodes = flat
        self.n_dofs = flat.size

    def cell_bounds(self, i, j):
        h = self.h
        return (self.x0 + i * h, self.x0 + (i + 1) * h, self.y0 + j * h, self.y0 + (j + 1) * h)

    def active(self, i, j):
        return 0 <= i < self.n and 0 <= j < self.n and self.cell_type[j, i] != OUTSIDE

    def ctype(self, i, j):
        if 0 <= i < self.n and 0 <= j < self.n:
            return int(self.cell_type[j, i])
        return OUTSIDE

    def node_cells_1d(self, a):
        """Cells (1D indices) whose closure contains lattice line a."""
        p, n = self.p, self.n
        if a % p == 0:
            return [c for c in (a // p - 1, a // p) if 0 <= c < n]
        return [a // p]

    def node_support(self, a, b):
        """Active cells containing lattice node (a, b): the support of its
        basis function."""
        return [(i, j) for j in self.node_cells_1d(b) for i in self.node_cells_1d(a) if self.active(i, j)]


def classify_cells(lv):
    """Inside / Cut / Outside per cell.  Reading R2: exact
    fp64 test on the squared distance from the circle centre to the closed
    cell box: Outside iff min-dist^2 >= r^2 (tangential touch is Outside),
    Inside iff max-dist^2 <= r^2, Cut otherwise.  Cell bounds are
    x0 + i*h and x0 + (i+1)*h (product rounded, then sum)."""
    c = lv.circle
    n = lv.n
    if is_fitted(c):
        return np.full((n, n), INSIDE, dtype=np.int8)
    r2 = c.r * c.r
    idx = np.arange(n, dtype=np.float64)
    xl, xh = lv.x0 + idx * lv.h, lv.x0 + (idx + 1.0) * lv.h
    yl, yh = lv.y0 + idx * lv.h, lv.y0 + (idx + 1.0) * lv.h
    qx = np.minimum(np.maximum(c.cx, xl), xh) - c.cx
    qy = np.minimum(np.maximum(c.cy, yl), yh) - c.cy
    fx = np.maximum(np.abs(xl - c.cx), np.abs(xh - c.cx))
    fy = np.maximum(np.abs(yl - c.cy), np.abs(yh - c.cy))
    dmin2 = qx[None, :] * qx[None, :] + qy[:, None] * qy[:, None]     # [j, i]
    dmax2 = fx[None, :] * fx[None, :] + fy[:, None] * fy[:, None]
    out = np.full((n, n), CUT, dtype=np.int8)
    out[dmax2 <= r2] = INSIDE
    out[dmin2 >= r2] = OUTSIDE
    return out


def node_mask(lv):
    """Lattice nodes that carry a DoF: nodes of active cells (PAPER.md l.121:
    "only basis functions associated to the cells in Omega_l are part of this
    basis")."""
    p, n = lv.p, lv.n
    act = lv.cell_type != OUTSIDE
    m = np.zeros((lv.nl, lv.nl), dtype=bool)
    for ky in range(p + 1):
        for kx in range(p + 1):
            m[ky:ky + n * p:p, kx:kx + n * p:p] |= act
    if is_fitted(lv.circle):   # strong Dirichlet: no DoF on the box boundary
        m[0, :] = m[-1, :] = m[:, 0] = m[:, -1] = False
    return m


def ghost_faces(lv):
    """F_G = faces F(T1,T2), T1,T2 active, T1 or T2 cut.
    Returned as (axis, i, j): axis 0 = face between (i,j) and (i+1,j),
    axis 1 = face between (i,j) and (i,j+1)."""
    out = []
    n = lv.n
    for j in range(n):
        for i in range(n):
            for axis, (i2, j2) in ((0, (i + 1, j)), (1, (i, j + 1))):
                if lv.active(i, j) and lv.active(i2, j2) and (lv.ctype(i, j) == CUT or lv.ctype(i2, j2) == CUT):
                    out.append((axis, i, j))
    return out


class Patch:
    __slots__ = ("I", "J", "K", "cells", "kind", "colour", "interior")


CARTESIAN, CUTPATCH = 0, 1


def vertex_patch(lv, I, J, vertices="active"):
    """The patch of vertex (I, J) or None (see build_patches)."""
    p = lv.p
    block = [(i, j) for j in (J - 1, J) for i in (I - 1, I)]
    cells = [c for c in block if lv.active(*c)]
    if not cells:
        return None
    if is_fitted(lv.circle) and not (0 < I < lv.n and 0 < J < lv.n):
        return None   # vertices contained in the open box (P l.143)
    if vertices == "inside":
        X = lv.x0 + I * lv.h - lv.circle.cx
        Y = lv.y0 + J * lv.h - lv.circle.cy
        if not X * X + Y * Y < lv.circle.r * lv.circle.r:
            return None
    pt = Patch()
    pt.I, pt.J, pt.cells = I, J, cells
    cellset = set(cells)
    interior = []
    for b in range(max(0, p * (J - 1)), min(lv.nl - 1, p * (J + 1)) + 1):
        for a in range(max(0, p * (I - 1)), min(lv.nl - 1, p * (I + 1)) + 1):
            if not lv.dof_mask[b, a]:
                continue
            if set(lv.node_support(a, b)) <= cellset:
                interior.append(int(lv.dof_index[b * lv.nl + a]))
    pt.interior = np.array(interior, dtype=np.int64)
    all_inside = len(cells) == 4 and all(lv.ctype(*c) == INSIDE for c in cells)
    nbrs = [(I - 2, J - 1), (I - 2, J), (I + 1, J - 1), (I + 1, J),
            (I - 1, J - 2), (I, J - 2), (I - 1, J + 1), (I, J + 1)]
    touches_ghost = any(lv.ctype(*c) == CUT for c in nbrs)
    pt.kind = CARTESIAN if (all_inside and not touches_ghost) else CUTPATCH
    pt.colour = (I % 2) + 2 * (J % 2)
    return pt


def build_patches(lv, vertices="active"):
    """Vertex patches with interior DoF sets, kind and colour.

    PAPER.md l.141-156: the patch of vertex X_j is the set of cells having X_j
    as a vertex; V_{l,j} are the functions of V_l with support on the patch.
    Reading R3: every vertex of an active cell carries a patch made
    of its active cells, so that the patches cover Omega_l (l.141 "covering of
    Omega, here actually Omega_l"); for vertices inside Omega this is exactly
    the paper's patch.  Interior set = DoF nodes whose support (active cells
    containing the node) lies in the patch.
    Reading R4: a patch is Cartesian (tensor-product local problem, PAPER.md
    l.187, l.192) iff its four cells are Inside and no ghost face touches them,
    i.e. none of the 8 face neighbours of the 2x2 block is Cut; all others are
    cut patches (l.193).
    Colouring (l.179): colour = (I mod 2) + 2 (J mod 2); Cartesian and cut
    patches are listed separately (l.195-212).  Order: J-major, I-minor."""
    patches = []
    for J in range(lv.n + 1):
        for I in range(lv.n + 1):
            pt = vertex_patch(lv, I, J, vertices)
            if pt is not None:
                patches.append(pt)
    return patches


def hierarchy(x0, y0, length, n0, n_levels, circle, p):
    """Levels l = 0..L with n_l = n0 2^l cells per side (PAPER.md l.65-69,
    l.217: each cell of M_{l-1} is the union of four cells of M_l)."""
    return [Level(x0, y0, length, n0 * 2 ** l, circle, p) for l in range(n_levels)]
