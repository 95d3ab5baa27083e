"""Vertex-patch smoother, V-cycle, CG and GMRES.

PAPER.md l.156-164 (local solver Q^T A_j^{-1} Q (A x - b)), l.165-178
(multiplicative vertex-patch smoother), l.179 (colouring: patches of one
colour are independent), l.181 (inconsistent treatment: ghost-penalty
coupling between patches of one colour is ignored), l.195-212 (partitioned
smoother: Cartesian patches, then n_c sweeps over cut patches), l.124
(V-cycle, exact coarse solve), l.217 (one pre- and one post-smoothing step).

The local matrices A_j are the principal submatrices of the assembled A_l at
the patch interior DoFs (l.156: "obtained by selecting the corresponding rows
and columns from the matrix A_l") and are inverted densely (numpy.linalg.inv);
the oracle does not use fast diagonalisation.

Test infrastructure only (see oracle/__init__.py).
"""
import math

import numpy as np

from .assemble import Params, assemble_matrix
from .geometry import CARTESIAN, CUTPATCH, Circle, build_patches, hierarchy
from .transfer import prolongation_matrix


LOCAL_READINGS = ("principal", "patch", "patch_matrix", "no_ghost")


def _boundary_ghost_rows(lv, prm, patches):
    """Per patch: the rows (at the interior set I) of the ghost-face terms on
    faces F(T1, T2) with exactly one of T1, T2 in the patch -- the coupling
    "through ghost penalties between neighboring vertex patches" of PAPER.md
    l.181 -- as a sparse (|I| x n_dofs) matrix.  Only for the sensitivity
    study of the local-solver readings (R9 / "Q2/Q3 iteration
    counts"); the default reading does not use it."""
    import scipy.sparse as sp
    from .assemble import ghost_face_matrix
    from .geometry import ghost_faces
    prm = prm.resolved(lv.p)
    by_cell = {}
    faces = []
    for axis, i, j in ghost_faces(lv):
        c2 = (i + 1, j) if axis == 0 else (i, j + 1)
        d, M = ghost_face_matrix(lv, axis, i, j, prm)
        faces.append(((i, j), c2, d, M))
        by_cell.setdefault((i, j), []).append(len(faces) - 1)
        by_cell.setdefault(c2, []).append(len(faces) - 1)
    out = []
    for pt in patches:
        cells = set(pt.cells)
        fids = {f for c in cells for f in by_cell.get(c, ())}
        pos = {int(g): r for r, g in enumerate(pt.interior)}
        rows, cols, vals = [], [], []
        for f in fids:
            c1, c2, d, M = faces[f]
            if (c1 in cells) == (c2 in cells):
                continue                      # interior face of the patch (or none)
            for a, ga in enumerate(d):
                r = pos.get(int(ga))
                if r is None:
                    continue
                rows.extend([r] * d.size); cols.extend(d.tolist()); vals.extend(M[a].tolist())
        out.append(sp.csr_matrix((vals, (rows, cols)), shape=(pt.interior.size, lv.n_dofs)))
    return out


class LevelData:
    """One level with A_l, its vertex patches and local solvers.

    `local` selects the reading of the local problem of PAPER.md l.156-164 /
    l.181 (R9, R10): "principal" (default) -- A_j = rows/columns of
    A_l at the interior set and the residual of the global A_l;
    "patch" -- A_j and the residual rows both from the patch-local operator
    (patch cells and the ghost faces between two patch cells; the ghost faces
    on the patch boundary are dropped); "patch_matrix" -- only A_j patch-local;
    "no_ghost" -- A_j without any ghost term.  The non-default readings exist
    for the iteration-count sensitivity study (scripts/oracle_sensitivity.py)
    and are 2D only."""

    def __init__(self, lv, prm, vertices="active", local="principal"):
        self.lv = lv
        if local not in LOCAL_READINGS:
            raise ValueError(local)
        self.local = local
        if getattr(lv, "dim", 2) == 3:
            from .dim3 import assemble_matrix3, build_patches3
            self.A = assemble_matrix3(lv, prm)
            self.patches = build_patches3(lv)
            if local != "principal":
                raise ValueError("local readings other than 'principal' are 2D only")
        else:
            self.A = assemble_matrix(lv, prm)
            self.patches = build_patches(lv, vertices)
        self.nc = lv.n_colours
        self.groups = {(k, c): [] for k in (CARTESIAN, CUTPATCH) for c in range(self.nc)}
        self.inv = []
        self.bnd = _boundary_ghost_rows(lv, prm, self.patches) if local in ("patch", "patch_matrix") else None
        A_ng = assemble_matrix(lv, prm, with_ghost=False) if local == "no_ghost" else None
        for idx, pt in enumerate(self.patches):
            self.groups[(pt.kind, pt.colour)].append(idx)
        # A_j[r, c] = A_l[I_r, I_c] (l.156), gathered for all patches of one
        # interior size at once (scipy element lookup), inverted as a stack
        Asel = (A_ng if A_ng is not None else self.A).tocsr()
        self.inv = [None] * len(self.patches)
        by_m = {}
        for idx, pt in enumerate(self.patches):
            by_m.setdefault(pt.interior.size, []).append(idx)
        for m, idxs in by_m.items():
            if m == 0:
                for idx in idxs:
                    self.inv[idx] = np.zeros((0, 0))
                continue
            Is = np.stack([self.patches[idx].interior for idx in idxs])          # (k, m)
            rows = np.repeat(Is, m, axis=1).ravel()                               # I_r, r-major
            cols = np.tile(Is, (1, m)).ravel()                                    # I_c
            Aj = np.asarray(Asel[rows, cols]).reshape(len(idxs), m, m)
            if self.bnd is not None:
                Aj = Aj - np.stack([self.bnd[idx][:, self.patches[idx].interior].toarray() for idx in idxs])
            inv = np.linalg.inv(Aj)
            for q, idx in enumerate(idxs):
                self.inv[idx] = inv[q]

    def colour_step(self, x, b, kind, colour):
        """One colour of the multiplicative smoother: the residual b - A x is
        taken at the start of the colour and every patch of the colour is
        corrected from it."""
        r = b - self.A @ x
        for idx in self.groups[(kind, colour)]:
            I = self.patches[idx].interior
            if I.size:
                rI = r[I]
                if self.local == "patch":
                    rI = rI + self.bnd[idx] @ x
                x[I] += self.inv[idx] @ rI

    def smooth(self, x, b, n_c, reverse=False):
        """S(x, b) of eq. (smoother-split): Cartesian
        colours 0..3, then n_c sweeps over cut colours 0..3.  reverse=True
        applies the steps in the opposite order (the adjoint sweep, used as
        post-smoother; reading R9)."""
        seq = [(CARTESIAN, c) for c in range(self.nc)] + [(CUTPATCH, c) for _ in range(n_c) for c in range(self.nc)]
        if reverse:
            seq = seq[::-1]
        for kind, c in seq:
            self.colour_step(x, b, kind, c)
        return x


class Hierarchy:
    """Levels 0..L of PAPER.md l.65-69 with operators, patches and transfers."""

    def __init__(self, x0, y0, length, n0, n_levels, circle, p, prm=None, n_c=2, symmetric=True, vertices="active",
                 levels=None, local="principal"):
        self.prm = prm if prm is not None else Params()
        self.p = p
        self.n_c = n_c
        self.symmetric = symmetric
        if levels is None:
            levels = hierarchy(x0, y0, length, n0, n_levels, circle, p)
        self.levels = [LevelData(lv, self.prm, vertices, local) for lv in levels]
        if getattr(levels[0], "dim", 2) == 3:
            from .dim3 import prolongation_matrix3 as prolong
        else:
            prolong = prolongation_matrix
        self.P = [None] + [prolong(self.levels[l - 1].lv, self.levels[l].lv) for l in range(1, len(levels))]
        A0 = self.levels[0].A.toarray()
        self.A0inv = np.linalg.inv(A0)

    @property
    def fine(self):
        return self.levels[-1]

    def vcycle(self, l, x, b):
        """V-cycle (one pre- and one post-smoothing step,
        l.217; exact solve on level 0)."""
        if l == 0:
            x[:] = self.A0inv @ b
            return x
        ld = self.levels[l]
        ld.smooth(x, b, self.n_c)
        r = b - ld.A @ x
        bc = self.P[l].T @ r
        xc = np.zeros_like(bc)
        self.vcycle(l - 1, xc, bc)
        x += self.P[l] @ xc
        ld.smooth(x, b, self.n_c, reverse=self.symmetric)
        return x

    def precondition(self, r):
        """One V-cycle with zero initial guess (a fixed linear operator)."""
        return self.vcycle(len(self.levels) - 1, np.zeros_like(r), r)

    def solve_cg(self, b, tol=1e-8, max_it=500):
        """Preconditioned CG with the V-cycle; stop when ||r||/||r_0|| <= tol
        (BASELINE.json north_star "CG+MG").  Returns x, iterations, history."""
        A = self.fine.A
        x = np.zeros_like(b)
        r = b.copy()
        r0 = np.linalg.norm(r)
        hist = [r0]
        if r0 == 0.0:
            return x, 0, hist
        z = self.precondition(r)
        p = z.copy()
        rho = r @ z
        it = 0
        while it < max_it:
            q = A @ p
            alpha = rho / (p @ q)
            x += alpha * p
            r -= alpha * q
            it += 1
            rn = np.linalg.norm(r)
            hist.append(rn)
            if rn <= tol * r0:
                break
            z = self.precondition(r)
            rho_new = r @ z
            p = z + (rho_new / rho) * p
            rho = rho_new
        return x, it, hist

    def solve_gmres(self, b, tol=1e-9, max_it=500, left=False):
        """Full (non-restarted) GMRES with modified Gram-Schmidt (PAPER.md
        Table 1 caption: "Multigrid preconditioner for GMRES solver, iteration
        counts to reduce residual by 10^-9").  Right preconditioning (the
        default) measures the true residual ||b - A x||; left=True solves
        M A x = M b and measures the preconditioned residual ||M (b - A x)||
        (the paper does not say which; sensitivity study only)."""
        A = self.fine.A
        n = b.size
        r0 = self.precondition(b) if left else b
        beta = np.linalg.norm(r0)
        hist = [beta]
        if beta == 0.0:
            return np.zeros(n), 0, hist
        V = [r0 / beta]
        Z = []
        H = np.zeros((max_it + 1, max_it))
        g = np.zeros(max_it + 1); g[0] = beta
        cs, sn = np.zeros(max_it), np.zeros(max_it)
        it = 0
        for k in range(max_it):
            if left:
                z = V[k]
                w = self.precondition(A @ z)
            else:
                z = self.precondition(V[k])
                w = A @ z
            Z.append(z)
            for i in range(k + 1):
                H[i, k] = w @ V[i]
                w = w - H[i, k] * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = math.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            it = k + 1
            hist.append(abs(g[k + 1]))
            if abs(g[k + 1]) <= tol * beta:
                break
            V.append(w / (np.linalg.norm(w) if np.linalg.norm(w) > 0 else 1.0))
        y = np.linalg.solve(np.triu(H[:it, :it]), g[:it])
        x = sum(y[i] * Z[i] for i in range(it))
        return x, it, hist

    def solve_vcycle(self, b, tol=1e-9, max_it=500):
        """Stationary V-cycle iteration x <- x + V(b - A x) (Table 3
        caption); divergence (||r|| > 10 ||r_0||) is reported as it = None."""
        A = self.fine.A
        x = np.zeros_like(b)
        r0 = np.linalg.norm(b)
        hist = [r0]
        for it in range(1, max_it + 1):
            x += self.precondition(b - A @ x)
            rn = np.linalg.norm(b - A @ x)
            hist.append(rn)
            if rn <= tol * r0:
                return x, it, hist
            if rn > 10 * r0 or not np.isfinite(rn):
                return x, None, hist
        return x, max_it, hist


def fractional_iterations(n_it, r_final, r_0):
    """n_frac = n_it * (-8) / log10(||r_n|| / ||r_0||)."""
    return n_it * (-8.0) / math.log10(r_final / r_0)


def from_workload(w, prm=None, **kw):
    """Hierarchy for a workloads.Workload description (2D circle or 3D sphere,
    or the fitted box, oracle.geometry.FittedBox)."""
    from .geometry import FittedBox
    fitted = getattr(w, "domain", "cut") == "fitted"
    if getattr(w, "dim", 2) == 3:
        from .dim3 import Level3, Sphere
        dom = FittedBox() if fitted else Sphere(w.cx, w.cy, w.cz, w.r)
        levels = [Level3(w.x0, w.y0, w.z0, w.length, w.n_coarse * 2 ** l, dom, w.p) for l in range(w.n_levels)]
        return Hierarchy(None, None, None, None, None, None, w.p, prm=prm, n_c=w.n_c, levels=levels, **kw)
    dom = FittedBox() if fitted else Circle(w.cx, w.cy, w.r)
    return Hierarchy(w.x0, w.y0, w.length, w.n_coarse, w.n_levels, dom, w.p, prm=prm, n_c=w.n_c, **kw)
