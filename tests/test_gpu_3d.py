"""CUDA 3D (sphere) path vs the 3D oracle through the C ABI: structure
bit-exact, operator / colour steps / smoothing steps / transfer to 1e-10,
V-cycle to 1e-9, identical CG iteration counts; Q1, Q2 and Q3."""
import functools

import numpy as np
import pytest

import workloads
from gpu_util import KIND, rel_err
from oracle.solver import from_workload

pytestmark = pytest.mark.gpu
TOL = 1e-10

CASES = [
    workloads.sphere("sphere-Q1-16", 2, 4, 1),
    workloads.sphere("sphere-Q2-8", 2, 3, 2),
    workloads.sphere("offc-Q2-8", 2, 3, 2, x0=-0.5, length=1.0, c=(0.0137, -0.0211, 0.0093), r=0.3071),
    workloads.sphere("sphere-Q3-8", 2, 3, 3),    # Q3 (configs[3]'s degree): m up to 189 > 160 (global-memory inverse)
]
IDS = [w.name for w in CASES]


@functools.lru_cache(maxsize=4)
def oracle(w):
    return from_workload(w)


def gpu(w, **kw):
    from paper_2508_11608_b200 import cutfem
    return cutfem.Problem.from_workload(w, **kw)


def rnd(w, seed, level):
    return workloads.lattice_vector(w, seed, level)


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_structure_3d(w):
    o, g = oracle(w), gpu(w)
    for l, ld in enumerate(o.levels):
        lv = ld.lv
        assert np.array_equal(g.cell_types(l), lv.cell_type)
        assert np.array_equal(g.dof_mask(l), lv.dof_mask)
        n1 = lv.n + 1
        for kind in (0, 1):
            for c in range(8):
                ref = [(pt.K * n1 + pt.J) * n1 + pt.I for pt in ld.patches if pt.kind == KIND[kind] and pt.colour == c]
                assert np.array_equal(g.patches(l, kind, c), np.array(ref, dtype=np.int32)), (l, kind, c)
        off, nodes = g.cut_interior(l)
        ref = [lv.dof_nodes[pt.interior] for c in range(8) for pt in ld.patches if pt.kind == KIND[1] and pt.colour == c]
        for k, r in enumerate(ref):
            assert np.array_equal(nodes[off[k]:off[k + 1]], r)


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_operator_3d(w):
    o, g = oracle(w), gpu(w)
    for l, ld in enumerate(o.levels):
        xl = rnd(w, 30 + l, l)
        y = g.zeros(l)
        g.apply_operator(l, g.to_device(xl, l), y)
        assert rel_err(g.to_host(y, l)[ld.lv.dof_nodes], ld.A @ xl[ld.lv.dof_nodes]) < TOL, l


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_colour_steps_and_smoother_3d(w):
    o, g = oracle(w), gpu(w)
    l = len(o.levels) - 1
    ld = o.levels[l]
    dn = ld.lv.dof_nodes
    xl, bl = rnd(w, 40, l), rnd(w, 41, l)
    for kind in (0, 1):
        for c in range(8):
            x = g.to_device(xl, l)
            g.colour_step(l, kind, c, x, g.to_device(bl, l))
            xo = xl[dn].copy()
            ld.colour_step(xo, bl[dn], KIND[kind], c)
            assert rel_err(g.to_host(x, l)[dn], xo) < TOL, (kind, c)
    for rev in (False, True):
        x = g.to_device(xl, l)
        g.smooth(l, x, g.to_device(bl, l), rev)
        xo = xl[dn].copy()
        ld.smooth(xo, bl[dn], w.n_c, reverse=rev)
        assert rel_err(g.to_host(x, l)[dn], xo) < TOL


@pytest.mark.parametrize("w", CASES, ids=IDS)
def test_transfer_vcycle_cg_3d(w):
    o, g = oracle(w), gpu(w)
    for l in range(1, len(o.levels)):
        c, f = o.levels[l - 1].lv, o.levels[l].lv
        xc, xf = rnd(w, 50, l - 1), rnd(w, 51, l) * f.dof_mask.ravel()
        d = g.to_device(xf, l)
        g.prolongate_add(l, g.to_device(xc, l - 1), d)
        assert rel_err(g.to_host(d, l)[f.dof_nodes], xf[f.dof_nodes] + o.P[l] @ xc[c.dof_nodes]) < TOL
        bc = g.zeros(l - 1)
        g.restrict(l, g.to_device(xf, l), bc)
        assert rel_err(g.to_host(bc, l - 1)[c.dof_nodes], o.P[l].T @ xf[f.dof_nodes]) < TOL
    lf = o.fine.lv
    bl = rnd(w, 52, None)
    x = g.zeros()
    g.vcycle(x, g.to_device(bl))
    assert rel_err(g.to_host(x)[lf.dof_nodes], o.precondition(bl[lf.dof_nodes])) < 10 * TOL
    x = g.zeros()
    it, rel = g.solve_cg_mg(x, g.to_device(bl), tol=1e-8, max_it=100)
    xo, ito, _ = o.solve_cg(bl[lf.dof_nodes], 1e-8, 100)
    assert it == ito and rel <= 1e-8
    assert rel_err(g.to_host(x)[lf.dof_nodes], xo) < 1e-7


@pytest.mark.parametrize("env,wi", [({"CUTFEM_CUT3": "2"}, 2), ({"CUTFEM_TMA": "0"}, 2), ({"CUTFEM_CUT3": "1"}, 2),
                                    ({"CUTFEM_SYM_PACKED": "1"}, 2), ({"CUTFEM_SYM_PACKED": "1"}, 3),
                                    ({"CUTFEM_SYM_PACKED": "1", "CUTFEM_CUT3": "2"}, 2)],
                         ids=["cut3-v2", "cut3-no-tma", "cut3-v1", "sym-packed-q2", "sym-packed-q3", "sym-packed-v2"])
def test_alternative_cut_kernels_3d(env, wi, monkeypatch):
    # alternative 3D cut kernels and the packed symmetric local inverses (the
    # storage large 3D Q3 problems switch to) vs the oracle's colour steps
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = CASES[wi]
    o, g = oracle(w), gpu(w)
    l = len(o.levels) - 1
    ld = o.levels[l]
    dn = ld.lv.dof_nodes
    xl, bl = rnd(w, 42, l), rnd(w, 43, l)
    for c in range(8):
        x = g.to_device(xl, l)
        g.colour_step(l, 1, c, x, g.to_device(bl, l))
        xo = xl[dn].copy()
        ld.colour_step(xo, bl[dn], KIND[1], c)
        assert rel_err(g.to_host(x, l)[dn], xo) < TOL, c


def test_sphere64_fullsize_vs_oracle_goldens():
    # 3D at 64^3 (Q2, 910 701 DoFs; the multi-wave level of config2's
    # hierarchy, TMA cut-patch windows): forward / reverse smoothing step,
    # V-cycle and CG count vs the oracle's outputs written by
    # scripts/make_fullsize_goldens.py (oracle only) on a fixed subset of DoFs
    # (every DoF within 3 h of the sphere + every 11th other one)
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "fullsize_sphere64.npz"))
    w = workloads.sphere("sphere-Q2-64^3", 2, 6, 2)
    assert str(d["workload"]) == w.name
    g = gpu(w)
    L = w.n_levels - 1
    assert g.level_info(L).n_dofs == int(d["n_dofs"])
    nodes = np.flatnonzero(g.dof_mask(L).ravel())[d["idx"]]
    xl, bl = rnd(w, 31, None), rnd(w, 32, None)
    for rev, key in ((False, "y_fwd"), (True, "y_rev")):
        x = g.to_device(xl)
        g.smooth(L, x, g.to_device(bl), rev)
        assert rel_err(g.to_host(x)[nodes], d[key]) < TOL, key
    v = g.zeros()
    g.vcycle(v, g.to_device(bl))
    assert rel_err(g.to_host(v)[nodes], d["v"]) < 10 * TOL
    xs = g.zeros()
    it, rel = g.solve_cg_mg(xs, g.to_device(bl), tol=float(d["tol"]), max_it=100)
    assert it == int(d["cg_it"]) and rel <= float(d["tol"])


def test_sphere_q3_16_smoother_vcycle_cg():
    # Q3 at 16^3 (63 001 DoFs, 2310 cut patches, interiors up to 183 DoFs):
    # smoothing steps forward / reverse, V-cycle, identical CG count
    w = workloads.sphere("sphere-Q3-16", 2, 4, 3)
    o, g = oracle(w), gpu(w)
    L = w.n_levels - 1
    lv = o.fine.lv
    xl, bl = rnd(w, 41, None), rnd(w, 42, None)
    for rev in (False, True):
        x = g.to_device(xl)
        g.smooth(L, x, g.to_device(bl), rev)
        xo = o.fine.smooth(xl[lv.dof_nodes].copy(), bl[lv.dof_nodes], w.n_c, reverse=rev)
        assert rel_err(g.to_host(x)[lv.dof_nodes], xo) < TOL, rev
    v = g.zeros()
    g.vcycle(v, g.to_device(bl))
    assert rel_err(g.to_host(v)[lv.dof_nodes], o.precondition(bl[lv.dof_nodes])) < 10 * TOL
    xs = g.zeros()
    it, rel = g.solve_cg_mg(xs, g.to_device(bl), tol=1e-8, max_it=100)
    _, ito, _ = o.solve_cg(bl[lv.dof_nodes], 1e-8, 100)
    assert it == ito and rel <= 1e-8
