"""Multi-process plumbing of bench.py (torch.distributed): rank environment,
max-over-ranks device time, whole-job throughput, and the NCCL communicator
endpoint of the slab partition (its unique id broadcast over the torch process
group; the halo exchanges themselves run inside libcutfem_mg.so, DESIGN.md
"Multi-GPU")."""
import os


def rank_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value, dist=None, device="cpu"):
    """max of a float over all ranks (identity without a process group)."""
    if dist is None or not dist.is_initialized():
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(units_per_rank, steps, world, max_ms):
    """whole-job units/s: every rank processes units_per_rank per step."""
    return units_per_rank * steps * world / (max_ms * 1e-3)


def strong_throughput(global_units, steps, max_ms):
    """whole-job units/s when the ranks share one problem of global_units per step."""
    return global_units * steps / (max_ms * 1e-3)


def broadcast_nccl_id(dist, make_id):
    """rank 0's NCCL unique id (bytes from make_id()) on every rank of the group."""
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
