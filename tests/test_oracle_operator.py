"""Oracle pins for A_l = a_l + g_l and the rhs."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.assemble import Params, assemble_matrix, assemble_rhs, l2_error
from oracle.geometry import CUT, INSIDE, Circle, Level, ghost_faces
from oracle.quadrature import cut_cell_rules

C1 = Circle(0.0, 0.0, 1.0)


def paper_level(n, p):
    return Level(-1.105, -1.105, 2.21, n, C1, p)


def interp(lv, fn):
    """Nodal interpolant on the DoF nodes (lattice positions)."""
    from oracle.fe import gauss_lobatto_nodes
    xi = gauss_lobatto_nodes(lv.p)
    b, a = np.divmod(lv.dof_nodes, lv.nl)
    def pos(k, o):
        c = np.minimum(k // lv.p, lv.n - 1)
        return o + (c + xi[k - c * lv.p]) * lv.h
    return fn(pos(a, lv.x0), pos(b, lv.y0))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_symmetric_positive_definite(p):
    lv = paper_level(8, p)
    A = assemble_matrix(lv, Params()).toarray()
    assert np.abs(A - A.T).max() <= 1e-12 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0


def test_q1_interior_stencil():
    # 4 Inside cells, no ghost face nearby: the Q1 Laplacian stencil 8/3, -1/3
    lv = paper_level(16, 1)
    A = assemble_matrix(lv, Params()).tocsr()
    a = b = 8  # the vertex at the origin
    i = lv.dof_index[b * lv.nl + a]
    row = A.getrow(i).toarray().ravel()
    assert abs(row[i] - 8.0 / 3.0) < 1e-14
    nb = [lv.dof_index[(b + db) * lv.nl + a + da] for db in (-1, 0, 1) for da in (-1, 0, 1) if (da, db) != (0, 0)]
    assert np.allclose(row[nb], -1.0 / 3.0, atol=1e-14)
    assert np.count_nonzero(np.abs(row) > 1e-15) == 9


@pytest.mark.parametrize("p", [1, 2, 3])
def test_constant_function_sees_only_nitsche_penalty(p):
    # A(1, phi_i) = -(1, d_n phi_i)_Gamma + gamma_D/h (1, phi_i)_Gamma; summing
    # over i (partition of unity): gamma_D/h |Gamma| with |Gamma| = sum of the
    # surface weights (and -> 2 pi).
    lv = paper_level(32, p)
    prm = Params().resolved(p)
    A = assemble_matrix(lv, prm)
    y = A @ np.ones(lv.n_dofs)
    arc = 0.0
    for j, i in zip(*np.nonzero(lv.cell_type == CUT)):
        arc += cut_cell_rules(*lv.cell_bounds(i, j), C1, prm.n_q)[3].sum()
    assert abs(y.sum() - prm.gamma_D / lv.h * arc) < 1e-10 * abs(y.sum())
    assert abs(arc - 2 * math.pi) < 1e-5
    # rows whose support is away from Gamma vanish (bulk and ghost terms)
    assert np.abs(y).max() > 0


@pytest.mark.parametrize("p", [1, 2, 3])
def test_ghost_penalty_consistency(p):
    # g_l vanishes on global polynomials of degree <= p (jumps of derivatives
    # of a smooth function are zero) and is positive semidefinite
    lv = paper_level(16, p)
    G = assemble_matrix(lv, Params(), with_cells=False)
    for fn in (lambda x, y: x ** p + 0.3 * x * y - y, lambda x, y: (x - 0.2) ** p * 1.0 + y ** p):
        u = interp(lv, fn)
        assert np.abs(G @ u).max() <= 1e-10 * max(1.0, np.abs(G).max() * np.abs(u).max())
    x = np.random.default_rng(1).standard_normal(lv.n_dofs)
    assert x @ (G @ x) >= 0
    assert np.linalg.eigvalsh(G.toarray()).min() > -1e-12 * np.abs(G).max()


@pytest.mark.parametrize("sigma", [-1, 1])
def test_ghost_single_line_kink_closed_form(sigma):
    # u = |x - x_F| (exact in Q1): [[d_x u]] = -2 on faces of the line x = x_F,
    # so g(u,u) = gamma_1 h^(2+sigma) * 4 * h per ghost face on that line
    lv = paper_level(16, 1)
    xF = lv.x0 + 6 * lv.h
    G = assemble_matrix(lv, Params(gamma_k=[0.1], sigma=sigma), with_cells=False)
    u = interp(lv, lambda x, y: np.abs(x - xF))
    nf = sum(1 for (axis, i, j) in ghost_faces(lv) if axis == 0 and i == 5)
    assert nf > 0
    expect = nf * 0.1 * lv.h ** (2 + sigma) * 4 * lv.h
    assert abs(u @ (G @ u) - expect) < 1e-12 * expect


@pytest.mark.parametrize("sigma", [-1, 1])
@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("p,k", [(2, 1), (2, 2), (3, 1), (3, 2), (3, 3)])
def test_ghost_kink_closed_form_each_order(p, k, axis, sigma):
    # u = s^(k-1)|s|, s = x - x_F (or y - y_F), is piecewise a polynomial of
    # degree k <= p on each side of the mesh line x = x_F (exact in Q_p), C^(k-1)
    # across it, and its k-th normal derivative jumps by 2 k!.  So only the
    # order-k term of g_l sees it:
    #   g(u,u) = gamma_k h^(2k+sigma)/(k!)^2 (2 k!)^2 |F| = 4 gamma_k h^(2k+sigma) h
    # per ghost face on that line.  Distinct gamma_1..gamma_p catch an index
    # slip; both sigma catch a wrong h power; k = 2, 3 catch (k!)^2 vs k!.
    lv = paper_level(16, p)
    gam = [0.1, 0.23, 0.37][:p]
    G = assemble_matrix(lv, Params(gamma_k=gam, sigma=sigma), with_cells=False)
    line = 6
    if axis == 0:
        xF = lv.x0 + line * lv.h
        u = interp(lv, lambda x, y: (x - xF) ** (k - 1) * np.abs(x - xF))
    else:
        yF = lv.y0 + line * lv.h
        u = interp(lv, lambda x, y: (y - yF) ** (k - 1) * np.abs(y - yF))
    nf = sum(1 for (ax, i, j) in ghost_faces(lv) if ax == axis and (i if axis == 0 else j) == line - 1)
    assert nf > 0
    expect = nf * 4.0 * gam[k - 1] * lv.h ** (2 * k + sigma) * lv.h
    # rounding: the face terms away from the line cancel in G u; bound by the
    # absolute quadratic form (|u|^T |G| |u| is ~1e3 x expect at k = 3)
    scale = np.abs(u) @ (abs(G) @ np.abs(u))
    assert abs(u @ (G @ u) - expect) < 1e-13 * scale + 1e-12 * expect, (u @ (G @ u), expect, scale)
    assert abs(u @ (G @ u) - expect) < 1e-6 * expect


@pytest.mark.parametrize("p,ns", [(1, (16, 32, 64)), (2, (8, 16, 32)), (3, (8, 16, 32))])
def test_manufactured_solution_rate(p, ns):
    # optimal O(h^(p+1)) L2 convergence (BASELINE.json north_star) for
    # u* = sin(pi x) sin(pi y), f = 2 pi^2 u*, g = u*|_Gamma on the unit circle
    ex = lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y)
    f = lambda x, y: 2 * np.pi ** 2 * ex(x, y)
    errs = []
    for n in ns:
        lv = paper_level(n, p)
        A = assemble_matrix(lv, Params())
        b = assemble_rhs(lv, Params(), f, ex)
        u = spla.spsolve(A.tocsc(), b)
        errs.append(l2_error(lv, u, ex, p + 3))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates[-1] > p + 1 - 0.25, (errs, rates)
