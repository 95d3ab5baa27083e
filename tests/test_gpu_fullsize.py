"""Parity at BASELINE.json's full size (configs[1]: circle, Q2, 512x512,
680065 DoFs) in the configuration bench.py times: structure bit-exact on the
finest level (whole arrays, patch kinds on sampled vertices), the operator
element by element, every colour step on sampled patches (the oracle computes
those patches one by one), and properties of the smoothing step and the CG
solve that hold at any size."""
import functools

import numpy as np
import pytest

import workloads
from gpu_util import KIND, compact, rel_err
from oracle.assemble import Params, assemble_matrix
from oracle.geometry import CUTPATCH, Circle, Level, vertex_patch

pytestmark = pytest.mark.gpu

W = workloads.CONFIG1
TOL = 1e-10


@functools.lru_cache(maxsize=1)
def oracle_level():
    lv = Level(W.x0, W.y0, W.length, W.n_fine, Circle(W.cx, W.cy, W.r), W.p)
    return lv, assemble_matrix(lv, Params())


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
