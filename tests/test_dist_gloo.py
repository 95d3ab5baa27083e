"""world_size-2 gloo tests (CPU) of the multi-process bench plumbing."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_11608_b200.dist import (broadcast_nccl_id, max_over_ranks, rank_env, replica_throughput,
                                         strong_throughput)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = rank_env()
    t = max_over_ranks(10.0 + 5.0 * rank, dist)        # rank 1 is slower
    v = replica_throughput(1000, 4, w, t)
    dist.barrier()
    q.put((r, w, lr, t, v))
    dist.destroy_process_group()


def test_max_over_ranks_and_throughput_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[:3] for r in res] == [(0, 2, 0), (1, 2, 1)]
    for r in res:
        assert r[3] == 15.0                          # max over ranks
        assert r[4] == pytest.approx(1000 * 4 * 2 / 15e-3)


def test_single_process_identity():
    assert max_over_ranks(3.5) == 3.5
    assert replica_throughput(10, 2, 1, 1.0) == pytest.approx(2e4)


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_11608_b200 import cutfem
    uid = broadcast_nccl_id(dist, cutfem.Comm.nccl_unique_id)
    t = strong_throughput(680065, 10, max_over_ranks(2.0 + rank, dist))
    dist.barrier()
    q.put((rank, uid, t))
    dist.destroy_process_group()


def test_nccl_id_broadcast_world2():
    """the slab partition's NCCL endpoint: rank 0's unique id (cutfem_comm_nccl_unique_id,
    128 bytes) reaches every rank; strong-scaling throughput uses the max time"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert len(res[0][1]) == 128 and res[0][1] == res[1][1]
    assert res[0][2] == res[1][2] == pytest.approx(680065 * 10 / 3e-3)


def _halo_worker(rank, world, port, q, n, p, halo):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_11608_b200 import cutfem
    plan = cutfem.slab_plan(n, p, world, rank, halo)
    nl, ld = n * p + 1, 6
    ref = torch.arange(nl * ld, dtype=torch.float64).reshape(nl, ld)
    v = torch.full((nl, ld), float("nan"), dtype=torch.float64)
    v[plan["r0"]:plan["r1"]] = ref[plan["r0"]:plan["r1"]]
    # the same transfers the library runs with ncclSend / ncclRecv, here over gloo
    reqs, bufs = [], []
    for x in plan["xfers"]:
        reqs.append(dist.isend(v[x["send_off"]:x["send_off"] + x["send_n"]].contiguous(), x["peer"]))
        buf = torch.empty((x["recv_n"], ld), dtype=torch.float64)
        bufs.append((x, buf))
        reqs.append(dist.irecv(buf, x["peer"]))
    for r in reqs:
        r.wait()
    for x, buf in bufs:
        v[x["recv_off"]:x["recv_off"] + x["recv_n"]] = buf
    ok_valid = bool(torch.equal(v[plan["v0"]:plan["v1"]], ref[plan["v0"]:plan["v1"]]))
    outside = torch.cat([v[:plan["v0"]], v[plan["v1"]:]])
    ok_out = bool(torch.isnan(outside).all()) if outside.numel() else True
    dist.barrier()
    q.put((rank, plan["r0"], plan["r1"], ok_valid, ok_out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,p,halo", [(2, 64, 2, 4), (3, 96, 2, 24), (4, 128, 1, 4)])
def test_slab_halo_exchange_gloo(world, n, p, halo):
    """the partition's slab plan (cutfem_slab_plan, the code partition() uses)
    driven over a world_size > 1 gloo group: owned rows tile the lattice and
    after one exchange every rank holds the owners' values on exactly its
    valid rows"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q, n, p, halo)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res[0][1] == 0 and res[-1][2] == n * p + 1
    assert all(a[2] == b[1] for a, b in zip(res, res[1:]))
    assert all(r[3] and r[4] for r in res)
