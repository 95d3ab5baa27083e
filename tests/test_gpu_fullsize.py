"""Parity at BASELINE.json's full size (configs[1]: circle, Q2, 512x512,
680065 DoFs) in the configuration bench.py times, against the oracle's whole
hierarchy built in this session (~2 min of CPU): structure bit-exact on the
finest level, the operator, the fused Cartesian sweep (k_cart_fused_tma, the
benched kernel) and the cut sweeps (k_cut_step7) forward and reverse, whole
smoothing steps forward and reverse, one V-cycle, all element by element, and
the CG iteration count identical; plus sampled single colour steps."""
import functools

import numpy as np
import pytest

import workloads
from gpu_util import KIND, compact, rel_err
from oracle.assemble import Params, assemble_matrix
from oracle.geometry import CARTESIAN, CUTPATCH, Circle, Level, vertex_patch
from oracle.solver import from_workload

pytestmark = pytest.mark.gpu

W = workloads.CONFIG1
TOL = 1e-10


@functools.lru_cache(maxsize=1)
def oracle_hierarchy():
    return from_workload(W)


def oracle_level():
    h = oracle_hierarchy()
    return h.fine.lv, h.fine.A


@functools.lru_cache(maxsize=1)
def gpu():
    from paper_2508_11608_b200 import cutfem
    return cutfem.Problem.from_workload(W)


def sample_vertices(lv, k, seed):
    rng = np.random.default_rng(seed)
    verts = set(map(tuple, rng.integers(0, lv.n + 1, size=(k, 2))))
    # plus every vertex of a band around the circle (where cut patches live)
    s = np.arange(lv.n + 1) * lv.h + lv.x0
    X, Y = np.meshgrid(s, s, indexing="ij")
    band = np.argwhere(np.abs(np.hypot(X, Y) - W.r) < 3 * lv.h)
    verts |= set(map(tuple, band[rng.permutation(len(band))[:k]]))
    return sorted(verts)


def test_structure_fullsize():
    lv, _ = oracle_level()
    g = gpu()
    L = W.n_levels - 1
    assert np.array_equal(g.cell_types(L), lv.cell_type)
    assert np.array_equal(g.dof_mask(L), lv.dof_mask)
    assert g.level_info(L).n_dofs == lv.n_dofs == 680065
    lists = {(k, c): set(g.patches(L, k, c).tolist()) for k in (0, 1) for c in range(4)}
    off, nodes = g.cut_interior(L)
    cut_order = [v for c in range(4) for v in g.patches(L, 1, c).tolist()]
    pos = {v: i for i, v in enumerate(cut_order)}
    for I, J in sample_vertices(lv, 1500, 0):
        pt = vertex_patch(lv, I, J)
        v = I + (lv.n + 1) * J
        found = [key for key, s in lists.items() if v in s]
        if pt is None:
            assert not found
            continue
        assert found == [({v2: k for k, v2 in KIND.items()}[pt.kind], pt.colour)]
        if pt.kind == CUTPATCH:
            k = pos[v]
            assert np.array_equal(nodes[off[k]:off[k + 1]], lv.dof_nodes[pt.interior])


def test_operator_fullsize():
    lv, A = oracle_level()
    g = gpu()
    L = W.n_levels - 1
    xl = workloads.lattice_vector(W, 21)
    y = g.zeros()
    g.apply_operator(L, g.to_device(xl), y)
    assert rel_err(compact(lv, g.to_host(y)), A @ compact(lv, xl)) < TOL


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("colour", [0, 1, 2, 3])
def test_colour_step_fullsize_sampled(kind, colour):
    lv, A = oracle_level()
    g = gpu()
    L = W.n_levels - 1
    xl, bl = workloads.lattice_vector(W, 22), workloads.lattice_vector(W, 23)
    x = g.to_device(xl)
    g.colour_step(L, kind, colour, x, g.to_device(bl))
    xg = compact(lv, g.to_host(x))
    x0, b0 = compact(lv, xl), compact(lv, bl)
    r = b0 - A @ x0
    verts = g.patches(L, kind, colour)
    rng = np.random.default_rng(100 + 10 * kind + colour)
    touched = np.zeros(lv.n_dofs, dtype=bool)
    for v in verts[rng.permutation(len(verts))[:300]]:
        pt = vertex_patch(lv, int(v) % (lv.n + 1), int(v) // (lv.n + 1))
        I = pt.interior
        z = np.linalg.solve(A[I][:, I].toarray(), r[I])
        assert rel_err(xg[I], x0[I] + z) < TOL
    # nodes outside every patch interior of this step are untouched
    for v in verts:
        pt = vertex_patch(lv, int(v) % (lv.n + 1), int(v) // (lv.n + 1)) if kind == 1 else None
        if pt is not None:
            touched[pt.interior] = True
    if kind == 1:
        assert np.array_equal(xg[~touched], x0[~touched])


def test_smoother_fixed_point_fullsize():
    # S(x*, A x*) = x* (the local corrections vanish when the residual does)
    lv, A = oracle_level()
    g = gpu()
    L = W.n_levels - 1
    xs = compact(lv, workloads.lattice_vector(W, 24))
    b = np.zeros(lv.nl * lv.nl)
    b[lv.dof_nodes] = A @ xs
    xl = np.zeros(lv.nl * lv.nl)
    xl[lv.dof_nodes] = xs
    x = g.to_device(xl)
    g.smooth(L, x, g.to_device(b))
    assert rel_err(compact(lv, g.to_host(x)), xs) < 1e-9


def test_cg_fullsize_true_residual():
    lv, A = oracle_level()
    g = gpu()
    bl = workloads.lattice_vector(W, 25)
    x = g.zeros()
    it, rel = g.solve_cg_mg(x, g.to_device(bl), tol=W.tol, max_it=100)
    b = compact(lv, bl)
    res = np.linalg.norm(b - A @ compact(lv, g.to_host(x))) / np.linalg.norm(b)
    assert rel <= W.tol and res <= 1.01 * W.tol and it <= 12


def _inputs(seed_x, seed_b):
    lv, _ = oracle_level()
    xl, bl = workloads.lattice_vector(W, seed_x), workloads.lattice_vector(W, seed_b)
    return xl, bl, compact(lv, xl), compact(lv, bl)


@pytest.mark.parametrize("reverse", [0, 1])
def test_cartesian_sweep_fullsize(reverse):
    # colour_step kind 2 = the fused Cartesian sweep of the bench (k_cart_fused_tma,
    # all four colours in one launch) vs the oracle's four Cartesian colour steps
    h = oracle_hierarchy()
    g = gpu()
    L = W.n_levels - 1
    xl, bl, x0, b0 = _inputs(41, 42)
    x = g.to_device(xl)
    g.colour_step(L, 2, reverse, x, g.to_device(bl))
    xo = x0.copy()
    for c in (3, 2, 1, 0) if reverse else (0, 1, 2, 3):
        h.fine.colour_step(xo, b0, CARTESIAN, c)
    assert rel_err(compact(h.fine.lv, g.to_host(x)), xo) < TOL


@pytest.mark.parametrize("reverse", [0, 1])
def test_cut_sweeps_fullsize(reverse):
    # colour_step kind 3 = the n_c sweeps over the cut colours (k_cut_step7 chain)
    h = oracle_hierarchy()
    g = gpu()
    L = W.n_levels - 1
    xl, bl, x0, b0 = _inputs(43, 44)
    x = g.to_device(xl)
    g.colour_step(L, 3, reverse, x, g.to_device(bl))
    xo = x0.copy()
    seq = [c for _ in range(W.n_c) for c in range(4)]
    for c in seq[::-1] if reverse else seq:
        h.fine.colour_step(xo, b0, CUTPATCH, c)
    assert rel_err(compact(h.fine.lv, g.to_host(x)), xo) < TOL


@pytest.mark.parametrize("reverse", [0, 1])
def test_smooth_fullsize_vs_oracle(reverse):
    # the benched call: one smoothing step S(x, b) on the 512^2 level
    h = oracle_hierarchy()
    g = gpu()
    L = W.n_levels - 1
    xl, bl, x0, b0 = _inputs(31, 32)
    x = g.to_device(xl)
    g.smooth(L, x, g.to_device(bl), bool(reverse))
    xo = h.fine.smooth(x0.copy(), b0, W.n_c, reverse=bool(reverse))
    assert rel_err(compact(h.fine.lv, g.to_host(x)), xo) < TOL


def test_vcycle_fullsize_vs_oracle():
    # one V-cycle from x = 0: 2 (L-1) smoothing steps, transfers and the exact
    # coarse solve; tolerance 10 x TOL (R14)
    h = oracle_hierarchy()
    g = gpu()
    _, bl, _, b0 = _inputs(31, 32)
    x = g.zeros()
    g.vcycle(x, g.to_device(bl))
    assert rel_err(compact(h.fine.lv, g.to_host(x)), h.precondition(b0)) < 10 * TOL


def test_cg_fullsize_iterations_equal_oracle():
    # north_star: identical CG iteration counts at full size
    h = oracle_hierarchy()
    g = gpu()
    _, bl, _, b0 = _inputs(31, 32)
    x = g.zeros()
    it, rel = g.solve_cg_mg(x, g.to_device(bl), tol=W.tol, max_it=100)
    xo, ito, hist = h.solve_cg(b0, W.tol)
    assert it == ito, (it, ito)
    assert rel <= W.tol and hist[-1] <= W.tol * hist[0]
    assert rel_err(compact(h.fine.lv, g.to_host(x)), xo) < 1e-7
