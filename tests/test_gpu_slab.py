"""Slab partition of the background mesh (north_star:
slabs with a halo exchange per colour sweep and per residual) on one GPU.

W ranks run as W host threads of this process, each with its own problem
handle and CUDA stream, joined by the in-process communicator
(cutfem_comm_local_create): the decomposition (row ownership, work-list
filtering, halo schedule, replicated coarse levels, distributed dot products)
is the code under test; only the transport differs from the NCCL endpoint.

Every node of a partitioned smoothing step / V-cycle is computed from the same
inputs in the same order as on one rank, so the owned rows must agree
BIT-EXACTLY with the single-rank path (itself parity-tested against the
oracle); CG sums its dot products per rank, so its iterates agree to rounding
and its iteration counts exactly.
"""
import os
import threading

import numpy as np
import pytest

import workloads
from workloads import Workload

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

# section-4 circle (R1) at 128^2 (Q2, Q3) / 256^2 (Q1); an off-centre circle for ragged cut patterns
W_Q2 = workloads.paper_level(2, 9)                 # 2 .. 128 cells per side
W_Q1 = workloads.paper_level(1, 9)                 # 2 .. 256
W_Q3 = workloads.paper_level(3, 9)
W_OFF = Workload("offcentre-Q2-256", -1.105, -1.105, 2.21, 2, 8, 0.0137, -0.0211, 0.9071, 2)
W_FIT = workloads.fitted("square-Q2-256", 2, 8, 2)   # configs[4] 2D analogue: fitted box, no cut patch


def _cutfem():
    from paper_2508_11608_b200 import cutfem
    return cutfem


def run_ranks(w, world, fn, timeout=300, env=None, pre=None):
    """fn(rank, problem, stream) on `world` threads; returns the per-rank results.
    pre(problem): work on the unpartitioned problem before partition()."""
    cutfem = _cutfem()
    comms = cutfem.Comm.local(world)
    gs = []
    for c in comms:
        g = with_env(env, lambda: cutfem.Problem.from_workload(w))
        if pre is not None:
            pre(g)
            torch.cuda.synchronize()
        g.partition(c)
        gs.append(g)
    torch.cuda.synchronize()
    out, errs = [None] * world, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, gs[r], s)
            s.synchronize()
        except BaseException as e:  # noqa: BLE001  (re-raised below)
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a rank hung (halo exchange mismatch)"
    if errs:
        raise errs[0]
    torch.cuda.synchronize()
    return out, gs


def with_env(env, fn):
    saved = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return fn()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def owned(g, v, level=-1):
    info = g.partition_info(level)
    nl, ld = g.lattice_shape(level)
    a = v.detach().cpu().numpy().reshape(-1, ld)[:, :nl]
    return info["r0"], info["r1"], a[info["r0"]:info["r1"]]


def single(w):
    return _cutfem().Problem.from_workload(w)


@pytest.mark.parametrize("w,world", [(W_Q2, 2), (W_Q2, 4), (W_Q1, 2), (W_Q1, 8), (W_Q3, 2)])
def test_partition_layout(w, world):
    """owned rows tile the lattice; valid rows = owned + HALO cells; the levels
    below the first non-partitionable one are replicated"""
    _, gs = run_ranks(w, world, lambda r, g, s: None)
    for level in range(w.n_levels):
        infos = [g.partition_info(level) for g in gs]
        nl, _ = gs[0].lattice_shape(level)
        parts = {i["part"] for i in infos}
        assert len(parts) == 1
        if infos[0]["part"]:
            assert infos[0]["r0"] == 0 and infos[-1]["r1"] == nl
            for a, b in zip(infos, infos[1:]):
                assert a["r1"] == b["r0"]
            s = (infos[0]["r1"] - infos[0]["r0"]) // w.p       # slab thickness in cells
            for i in infos:
                # only slabs thick enough for the wide halo (12 n_c cells) are partitioned
                assert i["halo"] == 12 * w.n_c and s >= 12 * w.n_c + 1
                h = i["halo"]
                assert i["v0"] == max(0, i["r0"] - h * w.p) and i["v1"] == min(nl, i["r1"] + h * w.p + 1)
        else:
            assert all(i["r0"] == 0 and i["r1"] == nl for i in infos)
    top = [g.partition_info(-1)["part"] for g in gs]
    assert all(top), "the finest level must be partitioned in these cases"
    # monotone: partitioned levels form a suffix of the hierarchy
    flags = [gs[0].partition_info(l)["part"] for l in range(w.n_levels)]
    assert flags == sorted(flags)


def test_smooth_before_partition():
    """smoothing steps on the unpartitioned problem (in-place cooperative
    Cartesian sweep: its grid-barrier counter advances by the full tile count),
    then partition() (fewer tiles per rank) and partitioned steps: still
    bit-exact, no hang (the counter restarts for the new grid)"""
    w, world = W_Q2, 2
    L = w.n_levels - 1
    x0, b0 = workloads.lattice_vector(w, 13), workloads.lattice_vector(w, 14)

    def pre(g):
        x, b = g.to_device(x0), g.to_device(b0)
        for rev in (False, True, False):
            g.smooth(L, x, b, reverse=rev)

    g1 = single(w)
    x1 = g1.to_device(x0)
    for _ in range(2):
        g1.smooth(L, x1, g1.to_device(b0))
    torch.cuda.synchronize()

    def fn(r, g, s):
        x, b = g.to_device(x0), g.to_device(b0)
        for _ in range(2):
            g.smooth(L, x, b, stream=s.cuda_stream)
        return x

    xs, gs = run_ranks(w, world, fn, pre=pre, timeout=120)
    ref = x1.cpu().numpy().reshape(-1, g1.lattice_shape(L)[1])[:, :g1.lattice_shape(L)[0]]
    for g, x in zip(gs, xs):
        r0, r1, a = owned(g, x, L)
        np.testing.assert_array_equal(a, ref[r0:r1])


TC32 = {"CUTFEM_TC32_MIN_N": "128"}   # 32-cell fused tiles on the 128^2 / 256^2 levels
SPLIT = {"CUTFEM_CART_SPLIT": "1"}    # two-launch Cartesian sweep through the shadow buffer
NARROW = {"CUTFEM_WIDE_HALO": "0"}    # one exchange per cut step everywhere


@pytest.mark.parametrize("w,world,env", [(W_Q2, 2, None), (W_Q2, 4, None), (W_Q1, 2, None), (W_Q1, 8, None),
                                         (W_FIT, 2, None), (W_FIT, 4, None),
                                         (W_Q3, 2, None), (W_OFF, 4, None), (W_Q2, 2, TC32), (W_OFF, 4, TC32),
                                         (W_Q2, 4, SPLIT), (W_Q2, 2, NARROW), (W_OFF, 4, NARROW)])
@pytest.mark.parametrize("reverse", [0, 1])
def test_smooth_bitexact(w, world, env, reverse):
    L = w.n_levels - 1
    x0 = workloads.lattice_vector(w, 11)
    b0 = workloads.lattice_vector(w, 12)
    g1 = with_env(env, lambda: single(w))
    x1 = g1.to_device(x0)
    for _ in range(2):
        g1.smooth(L, x1, g1.to_device(b0), reverse=bool(reverse))
    torch.cuda.synchronize()

    def fn(r, g, s):
        x = g.to_device(x0)
        b = g.to_device(b0)
        for _ in range(2):
            g.smooth(L, x, b, reverse=bool(reverse), stream=s.cuda_stream)
        return x

    xs, gs = run_ranks(w, world, fn, env=env)
    ref = x1.cpu().numpy().reshape(-1, g1.lattice_shape(L)[1])[:, :g1.lattice_shape(L)[0]]
    for g, x in zip(gs, xs):
        r0, r1, a = owned(g, x, L)
        np.testing.assert_array_equal(a, ref[r0:r1])


@pytest.mark.parametrize("w,world", [(W_Q2, 2), (W_Q2, 4), (W_Q1, 8), (W_Q3, 2), (W_OFF, 2)])
def test_operator_bitexact(w, world):
    L = w.n_levels - 1
    x0 = workloads.lattice_vector(w, 21)
    g1 = single(w)
    y1 = g1.zeros()
    g1.apply_operator(L, g1.to_device(x0), y1)
    torch.cuda.synchronize()

    def fn(r, g, s):
        y = g.zeros()
        g.apply_operator(L, g.to_device(x0), y, stream=s.cuda_stream)
        return y

    ys, gs = run_ranks(w, world, fn)
    nl, ld = g1.lattice_shape(L)
    ref = y1.cpu().numpy().reshape(-1, ld)[:, :nl]
    for g, y in zip(gs, ys):
        r0, r1, a = owned(g, y, L)
        np.testing.assert_array_equal(a, ref[r0:r1])


@pytest.mark.parametrize("w,world,env", [(W_Q2, 2, None), (W_Q2, 4, None), (W_Q1, 2, None), (W_Q1, 8, None),
                                         (W_FIT, 2, None), (W_FIT, 4, None),
                                         (W_Q3, 2, None), (W_OFF, 4, None), (W_OFF, 2, TC32), (W_OFF, 4, NARROW)])
def test_vcycle_bitexact(w, world, env):
    b0 = workloads.lattice_vector(w, 31)
    x0 = workloads.lattice_vector(w, 32)
    g1 = with_env(env, lambda: single(w))
    x1 = g1.to_device(x0)
    g1.vcycle(x1, g1.to_device(b0))
    torch.cuda.synchronize()

    def fn(r, g, s):
        x = g.to_device(x0)
        g.vcycle(x, g.to_device(b0), stream=s.cuda_stream)
        return x

    xs, gs = run_ranks(w, world, fn, env=env)
    nl, ld = g1.lattice_shape(-1)
    ref = x1.cpu().numpy().reshape(-1, ld)[:, :nl]
    for g, x in zip(gs, xs):
        r0, r1, a = owned(g, x)
        np.testing.assert_array_equal(a, ref[r0:r1])


@pytest.mark.parametrize("w,world", [(W_Q2, 2), (W_Q2, 4), (W_Q1, 8), (W_OFF, 4)])
def test_cg_iterations(w, world):
    """identical iteration counts; solution within rounding of the single-rank
    solve (the dot products are summed per rank first)"""
    b0 = workloads.lattice_vector(w, 41)
    g1 = single(w)
    xs1 = g1.zeros()
    it1, rel1 = g1.solve_cg_mg(xs1, g1.to_device(b0), tol=1e-9)
    torch.cuda.synchronize()

    def fn(r, g, s):
        x = g.zeros()
        it, rel = g.solve_cg_mg(x, g.to_device(b0), tol=1e-9, stream=s.cuda_stream)
        return x, it, rel

    res, gs = run_ranks(w, world, fn)
    nl, ld = g1.lattice_shape(-1)
    ref = xs1.cpu().numpy().reshape(-1, ld)[:, :nl]
    scale = np.abs(ref).max()
    for g, (x, it, rel) in zip(gs, res):
        assert it == it1
        assert abs(rel - rel1) <= 1e-6 * max(rel1, 1e-300) + 1e-14
        r0, r1, a = owned(g, x)
        assert np.abs(a - ref[r0:r1]).max() <= 1e-10 * scale


def test_halo_exchange_rows():
    """after an exchange, every rank's halo rows equal the owners' rows"""
    w, world = W_Q2, 4
    L = w.n_levels - 1

    def fn(r, g, s):
        nl, ld = g.lattice_shape(L)
        v = torch.full((nl * ld,), -1.0, dtype=torch.float64, device="cuda")   # (level halo: wide here)
        info = g.partition_info(L)
        rows = torch.arange(nl, dtype=torch.float64, device="cuda").repeat_interleave(ld)
        lo, hi = info["r0"] * ld, info["r1"] * ld
        v[lo:hi] = rows[lo:hi] + 1000.0 * r
        g.halo_exchange(L, v, stream=s.cuda_stream)
        return v

    vs, gs = run_ranks(w, world, fn)
    infos = [g.partition_info(L) for g in gs]
    nl, ld = gs[0].lattice_shape(L)
    for r, (g, v) in enumerate(zip(gs, vs)):
        a = v.cpu().numpy().reshape(nl, ld)
        i = infos[r]
        for row in range(i["v0"], i["v1"]):
            owner = next(q for q, j in enumerate(infos) if j["r0"] <= row < j["r1"])
            assert a[row, 0] == row + 1000.0 * owner, (r, row)


@pytest.mark.parametrize("transport", ["nccl", "local"])
def test_world1_transports(transport):
    """a one-rank partition (every tile-aligned level "partitioned" into one
    slab, no peers) through the NCCL endpoint (dlopen, ncclCommInitRank,
    ncclAllReduce on the stream) and the in-process one: bit-identical smoothing
    step and V-cycle, identical CG iterations"""
    cutfem = _cutfem()
    w = W_OFF
    L = w.n_levels - 1
    if transport == "nccl":
        comm = cutfem.Comm.nccl(cutfem.Comm.nccl_unique_id(), 0, 1)
    else:
        comm = cutfem.Comm.local(1)[0]
    g = cutfem.Problem.from_workload(w)
    g.partition(comm)
    assert g.partition_info(L)["part"] == 1
    g1 = single(w)
    x0, b0 = workloads.lattice_vector(w, 51), workloads.lattice_vector(w, 52)
    outs = []
    for h in (g1, g):
        x = h.to_device(x0)
        b = h.to_device(b0)
        h.smooth(L, x, b)
        h.vcycle(x, b)
        xs = h.zeros()
        it, _ = h.solve_cg_mg(xs, b, tol=1e-9)
        torch.cuda.synchronize()
        outs.append((h.to_host(x), it, h.to_host(xs)))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
    assert np.abs(outs[0][2] - outs[1][2]).max() <= 1e-10 * np.abs(outs[0][2]).max()


# ---- 3D: slabs of z-planes (narrow halo, one exchange per colour step) ----
S3_Q2 = workloads.sphere("sphere-Q2-32", 2, 5, 2)                      # 2 .. 32 cells per side
S3_Q1 = workloads.sphere("sphere-Q1-32-off", 2, 5, 1, c=(0.031, -0.017, 0.023), r=0.93)
S3_Q3 = workloads.sphere("sphere-Q3-16", 2, 4, 3)        # configs[3] degree
C3_Q2 = workloads.fitted("cube-Q2-24", 3, 4, 2, dim=3)   # configs[4] fitted cube


def _rows3(g, v, level=-1):
    """(planes, nl*ld) view of a 3D lattice vector and the rank's owned planes"""
    info = g.partition_info(level)
    nl, ld = g.lattice_shape(level)
    a = v.detach().cpu().numpy().reshape(nl, nl, ld)[:, :, :nl]
    return a[info["r0"]:info["r1"]], info


@pytest.mark.parametrize("w,world", [(S3_Q2, 2), (S3_Q2, 4), (S3_Q1, 2), (S3_Q3, 2), (C3_Q2, 2)])
def test_3d_partition_bitexact(w, world):
    """3D smoothing steps (forward, reverse), operator and V-cycle on the owned
    planes bit-exact vs one rank; CG iteration counts identical"""
    L = w.n_levels - 1
    x0, b0 = workloads.lattice_vector(w, 61), workloads.lattice_vector(w, 62)
    g1 = single(w)
    ref = {}
    x = g1.to_device(x0)
    b = g1.to_device(b0)
    g1.smooth(L, x, b)
    g1.smooth(L, x, b, reverse=True)
    ref["smooth"] = x.clone()
    y = g1.zeros()
    g1.apply_operator(L, g1.to_device(x0), y)
    ref["apply"] = y
    xv = g1.to_device(x0)
    g1.vcycle(xv, b)
    ref["vcycle"] = xv
    xs = g1.zeros()
    ref["cg"] = g1.solve_cg_mg(xs, b, tol=1e-9)
    ref["cg_x"] = xs
    torch.cuda.synchronize()

    def fn(r, g, s):
        st = s.cuda_stream
        out = {}
        x = g.to_device(x0)
        b = g.to_device(b0)
        g.smooth(L, x, b, stream=st)
        g.smooth(L, x, b, reverse=True, stream=st)
        out["smooth"] = x
        y = g.zeros()
        g.apply_operator(L, g.to_device(x0), y, stream=st)
        out["apply"] = y
        xv = g.to_device(x0)
        g.vcycle(xv, b, stream=st)
        out["vcycle"] = xv
        xs = g.zeros()
        out["cg"] = g.solve_cg_mg(xs, b, tol=1e-9, stream=st)
        out["cg_x"] = xs
        return out

    outs, gs = run_ranks(w, world, fn)
    assert gs[0].partition_info(L)["part"] == 1
    for g, o in zip(gs, outs):
        for key in ("smooth", "apply", "vcycle"):
            a, info = _rows3(g, o[key])
            full = ref[key].cpu().numpy().reshape(a.shape[1], a.shape[1], -1)[:, :, :a.shape[2]]
            np.testing.assert_array_equal(a, full[info["r0"]:info["r1"]], err_msg=key)
        assert o["cg"][0] == ref["cg"][0]
        a, info = _rows3(g, o["cg_x"])
        r = ref["cg_x"].cpu().numpy().reshape(a.shape[1], a.shape[1], -1)[info["r0"]:info["r1"], :, :a.shape[2]]
        assert np.abs(a - r).max() <= 1e-10 * np.abs(ref["cg_x"].cpu().numpy()).max()


@pytest.mark.parametrize("world", [2, 4])
def test_fullsize_config1_partition(world):
    """config1 (512^2, Q2: 24 x 32-cell Cartesian tiles, wide-halo cut sweeps,
    the bench's launch configuration) split into `world` slabs: the smoothing
    step pair and a V-cycle bit-exact on every rank's rows, CG iterations equal"""
    w = workloads.CONFIG1
    L = w.n_levels - 1
    x0, b0 = workloads.lattice_vector(w, 1), workloads.lattice_vector(w, 2)
    g1 = single(w)
    x = g1.to_device(x0)
    b = g1.to_device(b0)
    g1.smooth(L, x, b)
    g1.smooth(L, x, b, reverse=True)
    g1.vcycle(x, b)
    xs = g1.zeros()
    it1, _ = g1.solve_cg_mg(xs, b, tol=1e-8)
    torch.cuda.synchronize()
    nl, ld = g1.lattice_shape(L)
    ref = x.cpu().numpy().reshape(nl, ld)[:, :nl]
    refcg = xs.cpu().numpy().reshape(nl, ld)[:, :nl]
    g1.close()

    def fn(r, g, s):
        st = s.cuda_stream
        x = g.to_device(x0)
        b = g.to_device(b0)
        g.smooth(L, x, b, stream=st)
        g.smooth(L, x, b, reverse=True, stream=st)
        g.vcycle(x, b, stream=st)
        xs = g.zeros()
        it, _ = g.solve_cg_mg(xs, b, tol=1e-8, stream=st)
        return x, xs, it

    res, gs = run_ranks(w, world, fn, timeout=600)
    assert gs[0].partition_info(L)["halo"] == 24
    for g, (x, xs, it) in zip(gs, res):
        r0, r1, a = owned(g, x, L)
        np.testing.assert_array_equal(a, ref[r0:r1])
        assert it == it1
        _, _, c = owned(g, xs, L)
        assert np.abs(c - refcg[r0:r1]).max() <= 1e-10 * np.abs(refcg).max()


def test_partition_errors():
    """a second partition is refused (ERR_STATE) and leaves the problem usable;
    slab plans that do not divide are refused (ERR_ARG)"""
    cutfem = _cutfem()
    w = W_Q2
    g = cutfem.Problem.from_workload(w)
    g.partition(cutfem.Comm.local(1)[0])
    extra = cutfem.Comm.local(1)[0]
    with pytest.raises(cutfem.CutfemError, match="already partitioned"):
        g.partition(extra)
    x = g.to_device(workloads.lattice_vector(w, 3))
    b = g.to_device(workloads.lattice_vector(w, 4))
    g.smooth(-1, x, b)
    torch.cuda.synchronize()
    assert np.all(np.isfinite(g.to_host(x)))
    with pytest.raises(cutfem.CutfemError):
        cutfem.slab_plan(100, 2, 3, 0, 4)
    with pytest.raises(cutfem.CutfemError):
        cutfem.slab_plan(16, 2, 4, 0, 4)
