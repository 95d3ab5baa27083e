"""The slab partition over REAL GPUs with the NCCL transport (DESIGN.md
"Multi-GPU"): world = min(2, device_count) processes, one per GPU, joined by
torch.distributed (nccl) for the id broadcast; the halo exchanges run inside
libcutfem_mg.so over ncclSend/ncclRecv.  The owned rows of smoothing steps and
of a V-cycle must agree BIT-EXACTLY with one rank, and CG iteration counts
must be identical (test_gpu_slab.py checks the same decomposition with the
in-process transport on one GPU).  Skips on a one-GPU box."""
import os
import socket

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

W = workloads.paper_level(2, 9)   # section-4 circle, Q2, 2 .. 128 cells per side


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _single():
    """reference results of one rank on cuda:0 (lattice arrays)"""
    from paper_2508_11608_b200 import cutfem
    torch.cuda.set_device(0)
    g = cutfem.Problem.from_workload(W)
    L = W.n_levels - 1
    x0, b0 = workloads.lattice_vector(W, 51), workloads.lattice_vector(W, 52)
    x, b = g.to_device(x0), g.to_device(b0)
    for rev in (False, True):
        g.smooth(L, x, b, rev)
    v = g.zeros()
    g.vcycle(v, b)
    xs = g.zeros()
    it, rel = g.solve_cg_mg(xs, b, tol=W.tol, max_it=100)
    torch.cuda.synchronize()
    out = {"smooth": g.to_host(x), "vcycle": g.to_host(v), "cg_it": it}
    g.close()
    return out


def _rank(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch.distributed as dist
        from paper_2508_11608_b200 import cutfem
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        g = cutfem.Problem.from_workload(W)
        g.partition(cutfem.Comm.nccl_from_torch(dist))
        L = W.n_levels - 1
        x0, b0 = workloads.lattice_vector(W, 51), workloads.lattice_vector(W, 52)
        x, b = g.to_device(x0), g.to_device(b0)
        for rev in (False, True):
            g.smooth(L, x, b, rev)
        v = g.zeros()
        g.vcycle(v, b)
        xs = g.zeros()
        it, rel = g.solve_cg_mg(xs, b, tol=W.tol, max_it=100)
        torch.cuda.synchronize()
        info = g.partition_info(L)
        q.put((rank, info["r0"], info["r1"], g.to_host(x), g.to_host(v), it))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001  (reported to the parent)
        q.put((rank, "error", repr(e)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (NCCL ranks on distinct devices)")
def test_nccl_partition_bitexact_vs_one_rank():
    import torch.multiprocessing as mp
    world = min(2, torch.cuda.device_count())
    ref = _single()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(60)
    for r in res:
        assert r[1] != "error", r
    nl = W.n_fine * W.p + 1
    for rank, r0, r1, x, v, it in res:
        xa, va = x.reshape(nl, nl), v.reshape(nl, nl)
        xr, vr = ref["smooth"].reshape(nl, nl), ref["vcycle"].reshape(nl, nl)
        np.testing.assert_array_equal(xa[r0:r1], xr[r0:r1])
        np.testing.assert_array_equal(va[r0:r1], vr[r0:r1])
        assert it == ref["cg_it"]
