"""The one-launch cut sweep (k_cut_sweep, csrc/sweep.cuh) against the
launch-per-colour-step chain (k_cut_step7, CUTFEM_SWEEP=0) and the oracle.

The sweep runs, per CTA, the backward dependency cone of the nodes it owns
with k_cut_step7's per-patch arithmetic, so every smoothing step must be
BIT-IDENTICAL to the step chain (same maps, same inputs per patch); both are
compared with the oracle's coloured smoother (P eq. smoother-split
l.196-210, R9) at the north_star tolerance.  Cases: Q1-Q3, n_c = 1 and 2, an
off-centre circle (ragged cut pattern), forced CTA counts (1: no redundancy;
odd counts: ownership boundaries everywhere), NaN in non-DoF entries, and
config1 at full size (the benched call)."""
import os

import numpy as np
import pytest

import workloads
from gpu_util import compact, lattice_random, oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10

OFFC = workloads.Workload("offcentre-Q2", -1.105, -1.105, 2.21, 2, 6, 0.0137, -0.0211, 0.9071, 2)


def dofs(g, l):
    return np.flatnonzero(g.dof_mask(l).ravel())


def problem(w, env):
    from paper_2508_11608_b200 import cutfem
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return cutfem.Problem.from_workload(w)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def smooth_pair(g, h, w, l, rev, seed=70, nan=False):
    nl = workloads.lattice_nodes(w, l)
    xl, bl = lattice_random(w, seed, l), lattice_random(w, seed + 1, l)
    if nan:   # non-DoF entries may hold anything (include/cutfem_mg.h)
        mask = np.zeros(nl * nl, bool)
        mask[dofs(g, l)] = True
        xl = np.where(mask, xl, np.nan)
        bl = np.where(mask, bl, np.nan)
    out = []
    for q in (g, h):
        x = q.to_device(xl, l)
        q.smooth(l, x, q.to_device(bl, l), rev)
        out.append(q.to_host(x, l))
    return xl, bl, out[0], out[1]


@pytest.mark.parametrize("w", [workloads.paper_level(1, 7), workloads.paper_level(2, 7),
                               workloads.paper_level(3, 7), workloads.paper_level(2, 7, n_c=1),
                               workloads.paper_level(2, 7, n_c=4), OFFC, workloads.CONFIG0],
                         ids=["Q1", "Q2", "Q3", "Q2-nc1", "Q2-nc4", "offcentre", "config0"])
def test_sweep_bitidentical_every_level(w):
    g = problem(w, {})
    h = problem(w, {"CUTFEM_SWEEP": "0"})
    built = 0
    for l in range(w.n_levels):
        info = g.level_info(l)
        built += info.sweep_ctas[0] > 0
        assert h.level_info(l).sweep_ctas[0] == 0
        for rev in (False, True):
            _, _, a, b = smooth_pair(g, h, w, l, rev)
            dn = dofs(g, l)
            assert np.array_equal(a[dn], b[dn]), (l, rev)
    assert built >= w.n_levels - 2   # every level with cut patches runs the one-launch sweep


@pytest.mark.parametrize("ng", ["1", "3", "7", "148"])
def test_sweep_forced_cta_counts_vs_oracle(ng):
    w = workloads.paper_level(2, 7)
    g = problem(w, {"CUTFEM_SWEEP_NG": ng})
    h = problem(w, {"CUTFEM_SWEEP": "0"})
    o = oracle(w)
    l = w.n_levels - 1
    ld = o.levels[l]
    assert 0 < g.level_info(l).sweep_ctas[0] <= int(ng)
    for rev in (False, True):
        xl, bl, a, b = smooth_pair(g, h, w, l, rev, seed=80)
        dn = dofs(g, l)
        assert np.array_equal(a[dn], b[dn]), rev
        xo = compact(ld.lv, xl).copy()
        ld.smooth(xo, compact(ld.lv, bl), w.n_c, reverse=rev)
        assert rel_err(compact(ld.lv, a), xo) < TOL, rev


def test_sweep_nan_outside_dofs():
    w = workloads.paper_level(2, 7)
    g = problem(w, {})
    h = problem(w, {"CUTFEM_SWEEP": "0"})
    l = w.n_levels - 1
    for rev in (False, True):
        xl, _, a, b = smooth_pair(g, h, w, l, rev, nan=True)
        dn = dofs(g, l)
        assert np.isfinite(a[dn]).all() and np.array_equal(a[dn], b[dn])
        off = np.ones(a.size, bool)
        off[dn] = False
        assert np.isnan(a[off]).all()   # non-DoF entries unchanged


def test_sweep_vcycle_and_cg_identical():
    w = workloads.paper_level(2, 8)
    g = problem(w, {})
    h = problem(w, {"CUTFEM_SWEEP": "0"})
    bl = lattice_random(w, 90, None)
    xs = []
    for q in (g, h):
        x = q.zeros()
        q.vcycle(x, q.to_device(bl))
        xs.append(q.to_host(x))
    dn = dofs(g, -1)
    assert np.array_equal(xs[0][dn], xs[1][dn])
    its = []
    for q in (g, h):
        x = q.zeros()
        it, _ = q.solve_cg_mg(x, q.to_device(bl), tol=1e-8)
        its.append(it)
    assert its[0] == its[1]


def test_sweep_config1_fullsize_bitidentical():
    w = workloads.CONFIG1
    g = problem(w, {})
    h = problem(w, {"CUTFEM_SWEEP": "0"})
    l = w.n_levels - 1
    info = g.level_info(l)
    assert info.sweep_ctas[0] > 1 and info.sweep_ctas[1] > 1
    assert 1.0 <= info.sweep_redundancy[0] < 4.0
    for rev in (False, True):
        _, _, a, b = smooth_pair(g, h, w, l, rev, seed=95)
        dn = dofs(g, l)
        assert np.array_equal(a[dn], b[dn]), rev


@pytest.mark.parametrize("world", [2, 4])
def test_sweep_partitioned_bitexact(world):
    """Slab partition (in-process ranks on one GPU): the wide-halo levels run
    the one-launch sweep over each rank's owned rows, on its share of the SMs,
    bit-identical to one rank."""
    from test_gpu_slab import owned, run_ranks
    import torch
    w = workloads.paper_level(2, 9)   # 128^2 finest
    L = w.n_levels - 1
    x0 = workloads.lattice_vector(w, 21)
    b0 = workloads.lattice_vector(w, 22)
    g1 = problem(w, {})
    x1 = g1.to_device(x0)
    for rev in (False, True):
        g1.smooth(L, x1, g1.to_device(b0), reverse=rev)
    torch.cuda.synchronize()

    def fn(r, g, s):
        x = g.to_device(x0)
        b = g.to_device(b0)
        for rev in (False, True):
            g.smooth(L, x, b, reverse=rev, stream=s.cuda_stream)
        return x

    xs, gs = run_ranks(w, world, fn)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    ref = x1.cpu().numpy().reshape(-1, g1.lattice_shape(L)[1])[:, :g1.lattice_shape(L)[0]]
    for g, x in zip(gs, xs):
        info = g.level_info(L)
        assert g.partition_info(L)["part"] and 0 < info.sweep_ctas[0] <= nsm // world
        r0, r1, a = owned(g, x, L)
        np.testing.assert_array_equal(a, ref[r0:r1])


def test_smooth_host_pinned_spans():
    """cutfem_smooth_host with pinned host vectors moves only the DoF span of
    every lattice row (k_copy_spans): same DoF results as the device call,
    non-DoF host entries untouched (NaN stays NaN), the span kernels launched."""
    import torch
    from paper_2508_11608_b200 import cutfem
    w = workloads.paper_level(2, 8)
    g = problem(w, {})
    L = w.n_levels - 1
    nl, ld = g.lattice_shape(L)
    mask = np.zeros((nl, ld), bool)
    mask[:, :nl] = g.dof_mask(L)
    xl = np.zeros((nl, ld))
    bl = np.zeros((nl, ld))
    xl[:, :nl] = workloads.lattice_vector(w, 31, L).reshape(nl, nl)
    bl[:, :nl] = workloads.lattice_vector(w, 32, L).reshape(nl, nl)
    xl[~mask] = np.nan
    bl[~mask] = np.nan
    xh = torch.from_numpy(xl.ravel().copy()).pin_memory()
    bh = torch.from_numpy(bl.ravel().copy()).pin_memory()
    x = g.to_device(np.nan_to_num(xl[:, :nl]).ravel(), L)
    g.smooth(L, x, g.to_device(np.nan_to_num(bl[:, :nl]).ravel(), L), False)
    ref = x.cpu().numpy().reshape(nl, ld)
    l0 = cutfem.launch_count()
    g.smooth_host(L, xh.numpy(), bh.numpy())
    assert cutfem.launch_count() - l0 >= 2 + 2   # the span copies (x and b in, x out) ran with the step
    out = xh.numpy().reshape(nl, ld)
    assert np.array_equal(out[mask], ref[mask])
    assert np.isnan(out[~mask]).all()
    info = g.level_info(L)
    assert int(mask.sum()) <= info.host_span_doubles < nl * ld
