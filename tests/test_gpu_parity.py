"""CUDA path vs oracle, element by element, through the C ABI (PAPER.md
l.81-212).  Structure (classification, DoF mask, patch lists, colours,
interior sets) must agree bit-exactly; operator, colour steps, smoother,
transfer and V-cycle to a relative 1e-10 (BASELINE.json north_star); CG
iteration counts must be identical."""
import numpy as np
import pytest

import workloads
from gpu_util import KIND, compact, expand, gpu, lattice_random, oracle, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-10

CASES = [
    workloads.CONFIG0,
    workloads.paper_level(1, 7),   # 64 x 64 Q1, several Cartesian tiles + ragged tail
    workloads.paper_level(2, 7),   # 32 x 32 Q2
    workloads.paper_level(3, 6),   # 16 x 16 Q3
    workloads.Workload("offcentre-Q2", -0.5, -0.5, 1.0, 3, 4, 0.0137, -0.0211, 0.3071, 2),
    workloads.Workload("offcentre-Q4", -0.5, -0.5, 1.0, 2, 3, 0.0137, -0.0211, 0.3071, 4),
]
IDS = [w.name for w in CASES]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_structure_bit_exact(w, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    for l, ld in enumerate(o.levels):
        lv = ld.lv
        assert np.array_equal(g.cell_types(l), lv.cell_type)
        assert np.array_equal(g.dof_mask(l), lv.dof_mask)
        info = g.level_info(l)
        assert info.n_dofs == lv.n_dofs
        for kind in (0, 1):
            for c in range(4):
                ref = [pt.I + (lv.n + 1) * pt.J for pt in ld.patches if pt.kind == KIND[kind] and pt.colour == c]
                assert np.array_equal(g.patches(l, kind, c), np.array(ref, dtype=np.int32)), (l, kind, c)
        off, nodes = g.cut_interior(l)
        ref = [lv.dof_nodes[pt.interior] for c in range(4) for pt in ld.patches
               if pt.kind == KIND[1] and pt.colour == c]
        assert len(off) == len(ref) + 1
        for k, r in enumerate(ref):
            assert np.array_equal(nodes[off[k]:off[k + 1]], r), (l, k)


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_operator_parity(w, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    for l, ld in enumerate(o.levels):
        xl = lattice_random(w, 10 + l, l)
        x = g.to_device(xl, l)
        y = g.zeros(l)
        g.apply_operator(l, x, y)
        yg = g.to_host(y, l)
        yo = ld.A @ compact(ld.lv, xl)
        assert rel_err(compact(ld.lv, yg), yo) < TOL, (l, rel_err(compact(ld.lv, yg), yo))
        # inactive entries are written as zero
        assert np.all(yg[~ld.lv.dof_mask.ravel()] == 0.0)


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_colour_steps_parity(w, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    l = len(o.levels) - 1
    ld = o.levels[l]
    xl, bl = lattice_random(w, 1, l), lattice_random(w, 2, l)
    for kind in (0, 1):
        for c in range(4):
            x = g.to_device(xl, l)
            b = g.to_device(bl, l)
            g.colour_step(l, kind, c, x, b)
            xo = compact(ld.lv, xl).copy()
            ld.colour_step(xo, compact(ld.lv, bl), KIND[kind], c)
            assert rel_err(compact(ld.lv, g.to_host(x, l)), xo) < TOL, (kind, c)


@pytest.mark.parametrize("w", CASES, ids=IDS)
@pytest.mark.parametrize("reverse", [False, True])
def test_smoother_parity(w, reverse, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    for l in range(1, len(o.levels)):
        ld = o.levels[l]
        xl, bl = lattice_random(w, 3, l), lattice_random(w, 4, l)
        x = g.to_device(xl, l)
        b = g.to_device(bl, l)
        g.smooth(l, x, b, reverse)
        xo = compact(ld.lv, xl).copy()
        ld.smooth(xo, compact(ld.lv, bl), w.n_c, reverse=reverse)
        assert rel_err(compact(ld.lv, g.to_host(x, l)), xo) < TOL, l


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_transfer_parity(w, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    for l in range(1, len(o.levels)):
        c, f = o.levels[l - 1].lv, o.levels[l].lv
        xc = lattice_random(w, 5, l - 1)
        xf = lattice_random(w, 6, l)
        dxf = g.to_device(xf * f.dof_mask.ravel(), l)
        g.prolongate_add(l, g.to_device(xc, l - 1), dxf)
        ref = compact(f, xf) + o.P[l] @ compact(c, xc)
        assert rel_err(compact(f, g.to_host(dxf, l)), ref) < TOL
        bc = g.zeros(l - 1)
        g.restrict(l, g.to_device(xf * f.dof_mask.ravel(), l), bc)
        ref = o.P[l].T @ compact(f, xf)
        assert rel_err(compact(c, g.to_host(bc, l - 1)), ref) < TOL


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_vcycle_parity(w, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    lf = o.fine.lv
    bl = lattice_random(w, 7, None)
    x = g.zeros()
    g.vcycle(x, g.to_device(bl))
    ref = o.precondition(compact(lf, bl))
    # a V-cycle composes 2 (L-1) smoothing steps (each within TOL), transfers and
    # the exact coarse inverse; rounding differences of the local and coarse
    # inverses (Q4 local matrices have condition numbers ~1e6) compound, so the
    # composite bound is 10 TOL
    assert rel_err(compact(lf, g.to_host(x)), ref) < 10 * TOL


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_cg_iterations_identical(w, torch_cuda):
    o = oracle(w)
    g = gpu(w)
    lf = o.fine.lv
    bl = lattice_random(w, 8, None)
    x = g.zeros()
    it, rel = g.solve_cg_mg(x, g.to_device(bl), tol=1e-8, max_it=200)
    xo, ito, hist = o.solve_cg(compact(lf, bl), 1e-8, 200)
    assert it == ito
    assert rel <= 1e-8
    assert rel_err(compact(lf, g.to_host(x)), xo) < 1e-7


def test_host_pointer_entry_points(torch_cuda):
    w = workloads.CONFIG0
    o = oracle(w)
    g = gpu(w)
    lf = o.fine.lv
    nl, ld = g.lattice_shape()
    bl = lattice_random(w, 9, None)
    bh = np.zeros((nl, ld)); bh[:, :nl] = bl.reshape(nl, nl)
    xh = np.zeros((nl, ld))
    it, rel = g.solve_cg_mg_host(xh.ravel(), bh.ravel(), 1e-8, 200)
    xo, ito, _ = o.solve_cg(compact(lf, bl), 1e-8, 200)
    assert it == ito
    assert rel_err(compact(lf, xh[:, :nl].ravel()), xo) < 1e-7
    xs = np.zeros((nl, ld)); xs[:, :nl] = lattice_random(w, 11, None).reshape(nl, nl)
    x0 = xs[:, :nl].ravel().copy()
    g.smooth_host(len(o.levels) - 1, xs.ravel(), bh.ravel())
    ref = compact(lf, x0).copy()
    o.fine.smooth(ref, compact(lf, bl), w.n_c)
    assert rel_err(compact(lf, xs[:, :nl].ravel()), ref) < TOL


@pytest.mark.parametrize("w", [CASES[0], CASES[2], CASES[4]], ids=[IDS[0], IDS[2], IDS[4]])
def test_runtime_quadrature_mode_parity(w, torch_cuda):
    # cut_mode 1: the cut-cell bulk + Nitsche terms are evaluated by quadrature
    # on the fly (warp reductions) instead of precomputed element matrices
    o = oracle(w)
    g = gpu(w, cut_mode=1)
    l = len(o.levels) - 1
    ld = o.levels[l]
    xl, bl = lattice_random(w, 12, l), lattice_random(w, 13, l)
    y = g.zeros(l)
    g.apply_operator(l, g.to_device(xl, l), y)
    assert rel_err(compact(ld.lv, g.to_host(y, l)), ld.A @ compact(ld.lv, xl)) < TOL
    x = g.to_device(xl, l)
    g.smooth(l, x, g.to_device(bl, l))
    xo = compact(ld.lv, xl).copy()
    ld.smooth(xo, compact(ld.lv, bl), w.n_c)
    assert rel_err(compact(ld.lv, g.to_host(x, l)), xo) < TOL


@pytest.mark.parametrize("w", [workloads.paper_level(2, 8), workloads.CONFIG0], ids=["paper-Q2-L8", "config0"])
def test_non_dof_entries_ignored(w, torch_cuda):
    """include/cutfem_mg.h: entries of nodes without a DoF are ignored on input
    (NaN there must not reach any DoF: operator, smoothing steps, V-cycle,
    CG), written as 0 by the output vectors (operator, CG) and left untouched
    by the in-place updates (smoothing step, V-cycle)"""
    g = gpu(w)
    mask = g.dof_mask().ravel()
    xl, bl = lattice_random(w, 91, None), lattice_random(w, 92, None)
    xn, bn = xl.copy(), bl.copy()
    xn[~mask] = np.nan
    bn[~mask] = np.nan
    L = w.n_levels - 1
    outs = []
    for xv, bv in ((xl, bl), (xn, bn)):
        x = g.to_device(xv)
        b = g.to_device(bv)
        y = g.zeros()
        g.apply_operator(L, x, y)
        g.smooth(L, x, b)
        g.smooth(L, x, b, True)
        g.vcycle(x, b)
        xs = g.zeros()
        it, _ = g.solve_cg_mg(xs, b, tol=1e-8)
        outs.append((g.to_host(y), g.to_host(x), g.to_host(xs), it))
    for k, (a, b_) in enumerate(zip(outs[0][:3], outs[1][:3])):
        assert np.all(np.isfinite(b_[mask]))
        np.testing.assert_array_equal(a[mask], b_[mask])
        if k == 1:   # in place: untouched
            assert np.all(np.isnan(b_[~mask]))
        else:
            assert np.all(b_[~mask] == 0.0)
    assert outs[0][3] == outs[1][3]
