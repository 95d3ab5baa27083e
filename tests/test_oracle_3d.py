"""Oracle pins for the 3D (sphere) version: closed forms, invariants,
manufactured solution (BASELINE.json configs[2..4]; same method as PAPER.md
with d = 3)."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads
from oracle.assemble import Params
from oracle.dim3 import (CARTESIAN, CUT, CUTPATCH, INSIDE, Level3, Sphere, assemble_matrix3, build_patches3,
                         cell_dofs3, cut_cell_rules3, eval_basis3, ghost_faces3, prolongation_matrix3,
                         tensor_gauss3)
from oracle.fe import gauss_lobatto_nodes
from oracle.solver import from_workload

S1 = Sphere(0.0, 0.0, 0.0, 1.0)


def lev(n, p, sph=S1):
    return Level3(-1.105, -1.105, -1.105, 2.21, n, sph, p)


def interp3(lv, fn):
    xi = gauss_lobatto_nodes(lv.p)
    c, rem = np.divmod(lv.dof_nodes, lv.nl * lv.nl)
    b, a = np.divmod(rem, lv.nl)
    def pos(k, o):
        cc = np.minimum(k // lv.p, lv.n - 1)
        return o + (cc + xi[k - cc * lv.p]) * lv.h
    return fn(pos(a, lv.x0), pos(b, lv.y0), pos(c, lv.z0))


def test_spherical_cap_closed_form():
    # box [0.5,1.5] x [-1.5,1.5]^2 cuts the cap x >= 0.5 of the unit sphere:
    # volume pi h^2 (3 r - h) / 3, area 2 pi r h with h = 0.5
    errs = []
    for n in (6, 12):
        vp, vw, sp, sw, sn = cut_cell_rules3([0.5, -1.5, -1.5], [1.5, 1.5, 1.5], S1, n)
        errs.append((abs(vw.sum() - math.pi * 0.25 * 2.5 / 3), abs(sw.sum() - math.pi)))
        assert np.allclose(np.linalg.norm(sp, axis=1), 1.0, atol=1e-14)
        assert np.allclose(np.linalg.norm(sn, axis=1), 1.0, atol=1e-14)
    assert errs[1][0] < errs[0][0] and errs[1][1] < errs[0][1]
    assert errs[1][0] < 1e-5 and errs[1][1] < 2e-3   # algebraic: the base region has sqrt-type edges


@pytest.mark.parametrize("n,tol", [(16, 2e-5), (32, 1e-7)])
def test_global_volume_and_area(n, tol):
    lv = lev(n, 2)
    vol = float((lv.cell_type == INSIDE).sum()) * lv.h ** 3
    area = 0.0
    for k, j, i in zip(*np.nonzero(lv.cell_type == CUT)):
        lo = lv.lo(i, j, k)
        vp, vw, sp, sw, sn = cut_cell_rules3(lo, lv.hi(i, j, k), S1, 3)
        vol += vw.sum()
        area += sw.sum()
    assert abs(vol - 4 * math.pi / 3) < tol
    assert abs(area - 4 * math.pi) < 20 * tol


def test_tensor_gauss3_exactness():
    pts, w = tensor_gauss3(np.zeros(3), np.ones(3), 3)
    assert abs(w @ (pts[:, 0] ** 5 * pts[:, 1] ** 4 * pts[:, 2] ** 3) - 1 / 120) < 1e-15


def test_classification_and_ghost_faces_brute_force():
    sph = Sphere(0.013, -0.021, 0.007, 0.61)
    lv = Level3(-1.0, -1.0, -1.0, 2.0, 8, sph, 1)
    s = np.linspace(0, 1, 17)
    for k in range(lv.n):
        for j in range(lv.n):
            for i in range(lv.n):
                lo = lv.lo(i, j, k)
                X, Y, Z = np.meshgrid(lo[0] + lv.h * s, lo[1] + lv.h * s, lo[2] + lv.h * s)
                d2 = (X - sph.cx) ** 2 + (Y - sph.cy) ** 2 + (Z - sph.cz) ** 2
                t = lv.cell_type[k, j, i]
                if t == INSIDE:
                    assert d2.max() <= sph.r ** 2 + 1e-12
                elif t == CUT:
                    assert d2.min() < sph.r ** 2 < d2.max()
    ref = set()
    for k in range(lv.n):
        for j in range(lv.n):
            for i in range(lv.n):
                for ax in range(3):
                    c2 = (i + (ax == 0), j + (ax == 1), k + (ax == 2))
                    t1, t2 = lv.ctype(i, j, k), lv.ctype(*c2)
                    if t1 and t2 and CUT in (t1, t2):
                        ref.add((ax, i, j, k))
    assert set(ghost_faces3(lv)) == ref


@pytest.mark.parametrize("p", [1, 2])
def test_patches_cover_and_colour(p):
    lv = lev(8, p)
    pts = build_patches3(lv)
    cov = np.zeros(lv.n_dofs, dtype=int)
    for pt in pts:
        cov[pt.interior] += 1
        if pt.kind == CARTESIAN:
            assert pt.interior.size == (2 * p - 1) ** 3
    assert cov.min() >= 1
    for kind in (CARTESIAN, CUTPATCH):
        for c in range(8):
            grp = [pt for pt in pts if pt.kind == kind and pt.colour == c]
            cells = [cl for pt in grp for cl in pt.cells]
            assert len(cells) == len(set(cells))


def test_q1_stencil_3d():
    # 27-point Q1 Laplacian at an interior vertex: 8h/3, edges -h/6, corners -h/12, faces 0
    lv = lev(8, 1)
    A = assemble_matrix3(lv, Params()).tocsr()
    a = 4
    i = lv.dof_index[(a * lv.nl + a) * lv.nl + a]
    row = A.getrow(i).toarray().ravel()
    h = lv.h
    assert abs(row[i] - 8 * h / 3) < 1e-14
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                nz = abs(dx) + abs(dy) + abs(dz)
                if nz == 0:
                    continue
                j = lv.dof_index[((a + dz) * lv.nl + a + dy) * lv.nl + a + dx]
                expect = {1: 0.0, 2: -h / 6, 3: -h / 12}[nz]
                assert abs(row[j] - expect) < 1e-14


@pytest.mark.parametrize("p", [1, 2])
def test_spd_symmetry_constant_and_ghost_consistency(p):
    lv = lev(8, p)
    prm = Params().resolved(p)
    A = assemble_matrix3(lv, prm)
    Ad = A.toarray()
    assert np.abs(Ad - Ad.T).max() < 1e-12 * np.abs(Ad).max()
    assert np.linalg.eigvalsh(Ad).min() > 0
    area = 0.0
    for k, j, i in zip(*np.nonzero(lv.cell_type == CUT)):
        lo = lv.lo(i, j, k)
        area += cut_cell_rules3(lo, lv.hi(i, j, k), S1, prm.n_q)[3].sum()
    y = A @ np.ones(lv.n_dofs)
    assert abs(y.sum() - prm.gamma_D / lv.h * area) < 1e-10 * abs(y.sum())
    G = assemble_matrix3(lv, prm, with_cells=False)
    u = interp3(lv, lambda x, yy, z: x ** p - 0.3 * yy * z + z ** p)
    assert np.abs(G @ u).max() < 1e-10 * max(1.0, np.abs(G).max())
    v = np.random.default_rng(0).standard_normal(lv.n_dofs)
    assert v @ (G @ v) >= 0


def test_prolongation_reproduces_polynomials_3d():
    for p in (1, 2):
        c, f = lev(4, p), lev(8, p)
        P = prolongation_matrix3(c, f)
        q = lambda x, y, z: x ** p * y - z ** p + 0.5 * x * y * z + 1.0
        assert np.allclose(P @ interp3(c, q), interp3(f, q), atol=1e-12)


@pytest.mark.parametrize("p,ns", [(1, (8, 16, 32)), (2, (4, 8, 16))])
def test_manufactured_solution_rate_3d(p, ns):
    from oracle.dim3 import cell_matrix3
    ex = lambda x, y, z: np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    errs = []
    for n in ns:
        lv = lev(n, p)
        prm = Params().resolved(p)
        A = assemble_matrix3(lv, prm)
        b = np.zeros(lv.n_dofs)
        err_pts = []
        for k in range(n):
            for j in range(n):
                for i in range(n):
                    ct = lv.cell_type[k, j, i]
                    if ct == 0:
                        continue
                    lo = lv.lo(i, j, k)
                    if ct == INSIDE:
                        vp, vw = tensor_gauss3(lo, lv.hi(i, j, k), p + 1)
                        sp_ = np.zeros((0, 3)); sw = np.zeros(0); sn = np.zeros((0, 3))
                    else:
                        vp, vw, sp_, sw, sn = cut_cell_rules3(lo, lv.hi(i, j, k), S1, p + 1)
                    d = cell_dofs3(lv, i, j, k)
                    if len(vw):
                        v, *_ = eval_basis3(lv, i, j, k, vp)
                        b[d] += v @ (vw * 3 * np.pi ** 2 * ex(*vp.T))
                    if len(sw):
                        v, gx, gy, gz = eval_basis3(lv, i, j, k, sp_)
                        dn = gx * sn[:, 0] + gy * sn[:, 1] + gz * sn[:, 2]
                        gv = sw * ex(*sp_.T)
                        b[d] += -(dn @ gv) + (prm.gamma_D / lv.h) * (v @ gv)
                    err_pts.append((i, j, k, ct))
        u = spla.spsolve(A.tocsc(), b)
        e2 = 0.0
        for i, j, k, ct in err_pts:
            lo = lv.lo(i, j, k)
            if ct == INSIDE:
                vp, vw = tensor_gauss3(lo, lv.hi(i, j, k), p + 3)
            else:
                vp, vw, *_ = cut_cell_rules3(lo, lv.hi(i, j, k), S1, p + 3)
            if len(vw):
                v, *_ = eval_basis3(lv, i, j, k, vp)
                e2 += float(np.sum(vw * (u[cell_dofs3(lv, i, j, k)] @ v - ex(*vp.T)) ** 2))
        errs.append(math.sqrt(e2))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates[-1] > p + 1 - 0.3, (errs, rates)


def test_smoother_and_vcycle_3d():
    w = workloads.sphere("t3", 2, 3, 1)
    h = from_workload(w)
    ld = h.fine
    x = np.random.default_rng(1).standard_normal(ld.lv.n_dofs)
    b = ld.A @ x
    y = x.copy()
    ld.smooth(y, b, 2)
    assert np.allclose(y, x, atol=1e-12)
    v, u = np.random.default_rng(2).standard_normal((2, ld.lv.n_dofs))
    assert abs(v @ h.precondition(u) - u @ h.precondition(v)) < 1e-10 * abs(v @ h.precondition(u))
    xs, it, hist = h.solve_cg(v, 1e-8)
    assert hist[-1] <= 1e-8 * hist[0] and it < 15
