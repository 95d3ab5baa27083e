"""Parity of the alternative code paths and parameter edge cases (CUDA vs
oracle): fast-diagonalisation Cartesian sweep (CUTFEM_MMA=0), separate
colour kernels (CUTFEM_FUSED=0), scatter-kernel cut steps
(CUTFEM_PINGPONG=0), no PDL, n_c = 1, forward post-smoother (symmetric = 0),
sigma = +1, a circle that barely cuts the box cells, degree 3 and 4."""
import os

import numpy as np
import pytest

import workloads
from gpu_util import compact, lattice_random, rel_err
from oracle.assemble import Params
from oracle.solver import from_workload

pytestmark = pytest.mark.gpu
TOL = 1e-10
W = workloads.paper_level(2, 7)


def run_smoother(w, env=None, oracle_kw=None, **gkw):
    from paper_2508_11608_b200 import cutfem
    saved = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        g = cutfem.Problem.from_workload(w, **gkw)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    o = from_workload(w, **(oracle_kw or {}))
    l = len(o.levels) - 1
    ld = o.levels[l]
    xl, bl = lattice_random(w, 60, l), lattice_random(w, 61, l)
    y = g.zeros(l)
    g.apply_operator(l, g.to_device(xl, l), y)
    assert rel_err(compact(ld.lv, g.to_host(y, l)), ld.A @ compact(ld.lv, xl)) < TOL
    for rev in (False, True):
        x = g.to_device(xl, l)
        g.smooth(l, x, g.to_device(bl, l), rev)
        xo = compact(ld.lv, xl).copy()
        ld.smooth(xo, compact(ld.lv, bl), w.n_c, reverse=rev)
        assert rel_err(compact(ld.lv, g.to_host(x, l)), xo) < TOL, rev
    return g, o


@pytest.mark.parametrize("env", [{"CUTFEM_MMA": "0"}, {"CUTFEM_FUSED": "0"}, {"CUTFEM_PINGPONG": "0"},
                                 {"CUTFEM_PDL": "0"}, {"CUTFEM_TMA": "0"}, {"CUTFEM_CTACUT": "0"},
                                 {"CUTFEM_TILEAPPLY": "0"}, {"CUTFEM_CART_SPLIT": "1"},
                                 {"CUTFEM_CART_SPLIT": "1", "CUTFEM_TMA": "0"},
                                 {"CUTFEM_CART_SPLIT": "1", "CUTFEM_MMA": "0"}, {"CUTFEM_TC32_MIN_N": "32"},
                                 {"CUTFEM_TC32_MIN_N": "32", "CUTFEM_CART_SPLIT": "1"}, {"CUTFEM_CUTMAP": "0"},
                                 {"CUTFEM_TC32_MIN_N": "32", "CUTFEM_TCX": "24"},
                                 {"CUTFEM_TC32_MIN_N": "32", "CUTFEM_TCX": "16", "CUTFEM_CART_SPLIT": "1"}],
                         ids=["fd", "separate", "no-pingpong", "no-pdl", "no-tma", "warp-per-cut-patch", "node-apply",
                              "cart-split-tma", "cart-per-colour-mma", "cart-per-colour-fd", "tile32", "tile32-split",
                              "cut-step-matrix-free", "tile24x32", "tile16x32-split"])
def test_alternative_paths(env):
    run_smoother(W, env=env)


def test_nc1_and_forward_postsmoother_cg_gmres_free():
    w = workloads.paper_level(1, 7, n_c=1)
    g, o = run_smoother(w)
    # forward post-smoother: V-cycle parity (not symmetric, so no CG)
    from paper_2508_11608_b200 import cutfem
    g2 = cutfem.Problem.from_workload(w, symmetric=0)
    o2 = from_workload(w, symmetric=False)
    bl = lattice_random(w, 62, None)
    x = g2.zeros()
    g2.vcycle(x, g2.to_device(bl))
    lf = o2.fine.lv
    assert rel_err(compact(lf, g2.to_host(x)), o2.precondition(compact(lf, bl))) < 10 * TOL


def test_sigma_plus_one_and_gamma():
    w = workloads.paper_level(2, 6)
    prm = Params(sigma=1, gamma_k=[0.05, 0.15], gamma_D=20.0)
    from paper_2508_11608_b200 import cutfem
    g = cutfem.Problem.from_workload(w, sigma=1, gamma_k=(0.05, 0.15), gamma_D=20.0)
    o = from_workload(w, prm=prm)
    l = len(o.levels) - 1
    ld = o.levels[l]
    xl = lattice_random(w, 63, l)
    y = g.zeros(l)
    g.apply_operator(l, g.to_device(xl, l), y)
    assert rel_err(compact(ld.lv, g.to_host(y, l)), ld.A @ compact(ld.lv, xl)) < TOL
    bl = lattice_random(w, 64, None)
    x = g.zeros()
    it, rel = g.solve_cg_mg(x, g.to_device(bl), tol=1e-8)
    xo, ito, _ = o.solve_cg(compact(o.fine.lv, bl), 1e-8)
    assert it == ito


@pytest.mark.parametrize("w", [
    workloads.Workload("tangent-ish", -1.0, -1.0, 2.0, 2, 5, 0.0, 0.0, 0.50001, 2),   # circle hugging cell faces
    workloads.Workload("tiny-cuts", -1.0, -1.0, 2.0, 2, 5, 0.0312, 0.0, 0.7501, 1),
    workloads.Workload("Q3", -1.105, -1.105, 2.21, 2, 5, 0.0, 0.0, 1.0, 3),
    workloads.Workload("Q4", -1.105, -1.105, 2.21, 2, 4, 0.0, 0.0, 1.0, 4),
    # the circle passes exactly through mesh vertices (fp64-exact ties: cells
    # touching it in one point are Outside, R2) on every level
    workloads.Workload("vertex-touch", -1.0, -1.0, 2.0, 2, 5, 0.0, 0.0, 0.5, 2),
    # a domain inside one coarse cell: no Cartesian patch on the coarse levels
    workloads.Workload("small-domain", -0.5, -0.5, 1.0, 2, 5, 0.1, 0.07, 0.12, 2),
], ids=["tangent-ish", "tiny-cuts", "Q3", "Q4", "vertex-touch", "small-domain"])
def test_edge_geometries_and_degrees(w):
    g, o = run_smoother(w)
    bl = lattice_random(w, 65, None)
    x = g.zeros()
    it, rel = g.solve_cg_mg(x, g.to_device(bl), tol=1e-8, max_it=200)
    xo, ito, _ = o.solve_cg(compact(o.fine.lv, bl), 1e-8, 200)
    assert it == ito and rel <= 1e-8


def test_cart_split_equals_inplace_fullsize():
    """config1 (512^2, Q2): the two-launch Cartesian sweep through the shadow
    buffer (used when the tiles are not co-resident) gives bit-identical
    smoothing steps to the in-place cooperative sweep"""
    from paper_2508_11608_b200 import cutfem
    import torch
    w = workloads.CONFIG1
    L = w.n_levels - 1
    xl, bl = lattice_random(w, 70, L), lattice_random(w, 71, L)
    outs = []
    for split in ("0", "1"):
        os.environ["CUTFEM_CART_SPLIT"] = split
        try:
            g = cutfem.Problem.from_workload(w)
        finally:
            os.environ.pop("CUTFEM_CART_SPLIT", None)
        x = g.to_device(xl)
        b = g.to_device(bl)
        for rev in (False, True, False):
            g.smooth(L, x, b, rev)
        torch.cuda.synchronize()
        outs.append(g.to_host(x))
        g.close()
    np.testing.assert_array_equal(outs[0], outs[1])


def test_domain_missing_the_box_fails_loudly():
    # no active cell on some level: setup reports a geometry error (no silent
    # empty problem)
    from paper_2508_11608_b200 import cutfem
    w = workloads.Workload("outside", -0.5, -0.5, 1.0, 2, 3, 5.0, 5.0, 0.3, 1)
    with pytest.raises(cutfem.CutfemError, match="no DoF"):
        cutfem.Problem.from_workload(w)
