"""Oracle pins for the fitted domain (oracle.geometry.FittedBox): the paper's
"Square" baseline (Table 1 l.219-238, Fig. 2 square data
l.388-399) and BASELINE.json configs[4]'s fitted cube."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads
from oracle.assemble import Params, assemble_matrix, assemble_rhs, l2_error
from oracle.geometry import CARTESIAN, FittedBox, Level
from oracle.solver import from_workload

# Fig. 2 square data (l.388-399, "standardcutfemp"): DoFs and GMRES iterations
# per row; the DoF count includes the (constrained) boundary nodes:
# (n p + 1)^2 with n = 2^(l-1) cells for Q1 and 2^(l-2) for Q2 / Q3
FIG2_SQUARE = [  # (dof_q1, it_q1, dof_q2, it_q2, dof_q3, it_q3)
    (81, 5, 81, 4, 169, 3), (289, 6, 289, 4, 625, 3), (1089, 6, 1089, 4, 2401, 3), (4225, 6, 4225, 4, 9409, 3),
    (16641, 5, 16641, 4, 37249, 3), (66049, 5, 66049, 4, 148225, 3), (263169, 5, 263169, 4, 591361, 3),
    (1050625, 5, 1050625, 4, 2362369, 3), (4198401, 5, 4198401, 4, 9443329, 3)]


def square(p, n):
    return Level(0.0, 0.0, 1.0, n, FittedBox(), p)


@pytest.mark.parametrize("row", range(len(FIG2_SQUARE)))
def test_fig2_square_dof_counts(row):
    # row r is level l = r + 4: 2^(l-1) Q1 cells, 2^(l-2) Q2 / Q3 cells per side
    l = row + 4
    for p, n, dof in ((1, 2 ** (l - 1), FIG2_SQUARE[row][0]), (2, 2 ** (l - 2), FIG2_SQUARE[row][2]),
                      (3, 2 ** (l - 2), FIG2_SQUARE[row][4])):
        assert (n * p + 1) ** 2 == dof
        if n * p <= 256:
            lv = square(p, n)
            assert lv.n_dofs == (n * p - 1) ** 2   # the free DoFs (boundary eliminated)


@pytest.mark.parametrize("L", [6, 7])
def test_table1_square_gmres_counts(L):
    # Table 1 square block (GMRES + MG, 1e-9): Q1 5, Q2 4, Q3 3 at every L;
    # Fig. 2's data gives 6 for Q1 at l = 5..7.  Oracle within 1.
    for p, paper in ((1, 5), (2, 4), (3, 3)):
        nf = 2 ** (L - 1) if p == 1 else 2 ** (L - 2)
        w = workloads.fitted("sq", 2, int(np.log2(nf)), p, x0=0.0, length=1.0, tol=1e-9)
        h = from_workload(w, symmetric=False)
        b = np.random.default_rng(7).standard_normal(h.fine.lv.n_dofs)
        it = h.solve_gmres(b, 1e-9, 100)[1]
        assert abs(it - paper) <= 1, (p, it, paper)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_fitted_patches_are_interior_vertices_and_cartesian(p):
    # P l.143 literal: patches at the vertices contained in the open box, all
    # with tensor structure and the full (2p-1)^2 interior; they cover every DoF
    w = workloads.fitted("sq", 2, 3, p)
    ld = from_workload(w).fine
    lv = ld.lv
    assert {(pt.I, pt.J) for pt in ld.patches} == {(I, J) for I in range(1, lv.n) for J in range(1, lv.n)}
    assert all(pt.kind == CARTESIAN and pt.interior.size == (2 * p - 1) ** 2 for pt in ld.patches)
    cover = np.zeros(lv.n_dofs, dtype=bool)
    for pt in ld.patches:
        cover[pt.interior] = True
    assert cover.all()


def test_fitted_q1_stencil_and_spd():
    lv = square(1, 8)
    A = assemble_matrix(lv, Params()).toarray()
    assert np.allclose(np.diag(A), 8.0 / 3.0) and np.abs(A - A.T).max() < 1e-14
    assert np.linalg.eigvalsh(A).min() > 0


@pytest.mark.parametrize("p,ns", [(1, (8, 16, 32)), (2, (4, 8, 16)), (3, (4, 8, 16))])
def test_fitted_manufactured_solution_rate(p, ns):
    # u* = sin(pi x) sin(pi y) on the unit square, u* = 0 on the boundary:
    # optimal O(h^(p+1)) L2 convergence
    ex = lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y)
    f = lambda x, y: 2 * np.pi ** 2 * ex(x, y)
    errs = []
    for n in ns:
        lv = square(p, n)
        A = assemble_matrix(lv, Params())
        b = assemble_rhs(lv, Params(), f, lambda x, y: 0.0 * x)
        errs.append(l2_error(lv, spla.spsolve(A.tocsc(), b), ex, p + 3))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates[-1] > p + 1 - 0.25, (errs, rates)


def test_fitted_cube_3d():
    # 3D: (n p - 1)^3 free DoFs, 27-DoF Cartesian patches at the interior
    # vertices, CG + V-cycle converges
    w = workloads.fitted("cube", 2, 3, 2, dim=3)
    h = from_workload(w)
    lv = h.fine.lv
    assert lv.n_dofs == (lv.n * 2 - 1) ** 3
    assert len(h.fine.patches) == (lv.n - 1) ** 3
    assert all(pt.kind == CARTESIAN and pt.interior.size == 27 for pt in h.fine.patches)
    b = np.random.default_rng(3).standard_normal(lv.n_dofs)
    x, it, hist = h.solve_cg(b, 1e-8)
    assert hist[-1] <= 1e-8 * hist[0] and it <= 10
