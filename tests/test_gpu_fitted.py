"""Fitted-box mode (cutfem_params.domain = 1; BASELINE.json configs[4]'s
fitted cube, the paper's "Square" baseline) vs the oracle's FittedBox through
the C ABI: structure bit-exact (all cells Inside, no DoF on the box boundary,
Cartesian patches at exactly the interior vertices, no cut patch), operator,
smoothing steps forward / reverse and the fused Cartesian sweep to 1e-10,
V-cycle to 1e-9 (R14), identical CG iteration counts; NaN on the
boundary nodes of the inputs never reaches a DoF."""
import functools

import numpy as np
import pytest

import workloads
from gpu_util import KIND, compact, rel_err
from oracle.solver import from_workload

pytestmark = pytest.mark.gpu
TOL = 1e-10

CASES = [
    workloads.fitted("square-Q1-32", 2, 5, 1),
    workloads.fitted("square-Q2-32", 2, 5, 2),
    workloads.fitted("square-Q3-16", 2, 4, 3),
    workloads.fitted("square-Q2-48", 3, 5, 2),            # non-power-of-two coarse mesh (as CONFIG4_SQUARE)
    workloads.fitted("cube-Q1-16", 2, 4, 1, dim=3),
    workloads.fitted("cube-Q2-12", 3, 3, 2, dim=3),       # 3 x 2^2 (as CONFIG4_CUBE)
]
IDS = [w.name for w in CASES]


@functools.lru_cache(maxsize=8)
def oracle(w, symmetric=True):
    return from_workload(w, symmetric=symmetric)


def gpu(w, **kw):
    from paper_2508_11608_b200 import cutfem
    return cutfem.Problem.from_workload(w, **kw)


def vid(w, pt, n1):
    return (pt.K * n1 + pt.J) * n1 + pt.I if w.dim == 3 else pt.J * n1 + pt.I


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_fitted_structure(w):
    o, g = oracle(w), gpu(w)
    nc = 8 if w.dim == 3 else 4
    for l, ld in enumerate(o.levels):
        lv = ld.lv
        assert np.array_equal(g.cell_types(l), lv.cell_type)
        assert np.array_equal(g.dof_mask(l), lv.dof_mask)
        assert g.level_info(l).n_dofs == lv.n_dofs == (lv.n * w.p - 1) ** w.dim
        n1 = lv.n + 1
        for c in range(nc):
            ref = [vid(w, pt, n1) for pt in ld.patches if pt.kind == KIND[0] and pt.colour == c]
            assert np.array_equal(g.patches(l, 0, c), np.array(ref, dtype=np.int32)), (l, c)
            assert len(g.patches(l, 1, c)) == 0


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_fitted_operator_smoother(w):
    o, g = oracle(w), gpu(w)
    for l in range(1, w.n_levels):
        ld = o.levels[l]
        lv = ld.lv
        xl, bl = workloads.lattice_vector(w, 60 + l, l), workloads.lattice_vector(w, 80 + l, l)
        y = g.zeros(l)
        g.apply_operator(l, g.to_device(xl, l), y)    # boundary entries of x are nonzero: ignored
        assert rel_err(compact(lv, g.to_host(y, l)), ld.A @ compact(lv, xl)) < TOL
        for rev in (False, True):
            x = g.to_device(xl, l)
            g.smooth(l, x, g.to_device(bl, l), rev)
            xo = ld.smooth(compact(lv, xl).copy(), compact(lv, bl), w.n_c, reverse=rev)
            assert rel_err(compact(lv, g.to_host(x, l)), xo) < TOL, (l, rev)
            out = g.to_host(x, l)
            assert np.all(out[~lv.dof_mask.ravel()] == 0.0)   # non-DoF entries are 0 on output


@pytest.mark.parametrize("w", [c for c in CASES if c.dim == 2], ids=[c.name for c in CASES if c.dim == 2])
def test_fitted_cartesian_sweep_kind2(w):
    # the fused Cartesian sweep (the whole smoothing step in fitted mode)
    o, g = oracle(w), gpu(w)
    L = w.n_levels - 1
    ld = o.fine
    xl, bl = workloads.lattice_vector(w, 5), workloads.lattice_vector(w, 6)
    for rev in (0, 1):
        x = g.to_device(xl)
        g.colour_step(L, 2, rev, x, g.to_device(bl))
        xo = compact(ld.lv, xl).copy()
        for c in (3, 2, 1, 0) if rev else (0, 1, 2, 3):
            ld.colour_step(xo, compact(ld.lv, bl), KIND[0], c)
        assert rel_err(compact(ld.lv, g.to_host(x)), xo) < TOL


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_fitted_vcycle_cg(w):
    o, g = oracle(w), gpu(w)
    lf = o.fine.lv
    bl = workloads.lattice_vector(w, 7)
    x = g.zeros()
    g.vcycle(x, g.to_device(bl))
    assert rel_err(compact(lf, g.to_host(x)), o.precondition(compact(lf, bl))) < 10 * TOL
    xs = g.zeros()
    it, rel = g.solve_cg_mg(xs, g.to_device(bl), tol=1e-8, max_it=100)
    xo, ito, _ = o.solve_cg(compact(lf, bl), 1e-8, 100)
    assert it == ito and rel <= 1e-8
    assert rel_err(compact(lf, g.to_host(xs)), xo) < 1e-7


def test_fitted_nan_on_boundary_ignored():
    w = CASES[1]
    o, g = oracle(w), gpu(w)
    ld = o.fine
    lv = ld.lv
    L = w.n_levels - 1
    xl, bl = workloads.lattice_vector(w, 8), workloads.lattice_vector(w, 9)
    xn = xl.copy()
    xn[~lv.dof_mask.ravel()] = np.nan
    x = g.to_device(xn)
    g.smooth(L, x, g.to_device(bl))
    xo = ld.smooth(compact(lv, xl).copy(), compact(lv, bl), w.n_c)
    assert rel_err(compact(lv, g.to_host(x)), xo) < TOL
    y = g.zeros()
    g.apply_operator(L, g.to_device(xn), y)
    assert rel_err(compact(lv, g.to_host(y)), ld.A @ compact(lv, xl)) < TOL


def test_config4_square_fullsize():
    # BASELINE configs[4] (2D analogue, the bench line): 384^2 cells, Q2,
    # 588 289 DoFs: one smoothing step and the CG count vs the oracle
    w = workloads.CONFIG4_SQUARE
    o, g = oracle(w), gpu(w)
    ld = o.fine
    lv = ld.lv
    L = w.n_levels - 1
    assert lv.n_dofs == 767 ** 2
    xl, bl = workloads.lattice_vector(w, 31), workloads.lattice_vector(w, 32)
    x = g.to_device(xl)
    g.smooth(L, x, g.to_device(bl))
    xo = ld.smooth(compact(lv, xl).copy(), compact(lv, bl), w.n_c)
    assert rel_err(compact(lv, g.to_host(x)), xo) < TOL
    xs = g.zeros()
    it, rel = g.solve_cg_mg(xs, g.to_device(bl), tol=w.tol, max_it=100)
    _, ito, _ = o.solve_cg(compact(lv, bl), w.tol, 100)
    assert it == ito
