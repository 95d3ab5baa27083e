"""Multi-process plumbing of bench.py (torch.distributed): rank environment,
max-over-ranks device time, whole-job throughput.  Round 1 runs one
independent replica of the problem per GPU (no data-path collective); the
slab decomposition with halo exchange is the next row."""
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
