"""Batch-shard host logic for multi-GPU runs (PAPER.md:809-812
"DP forces every GPU to load the layer").

Each rank owns an independent context on its own GPU, streams every layer over its
own host link and decodes its own slice of the global batch; there is no
collective on the hot path.  torch.distributed is used only for plumbing: a
barrier around the timed region and the max-over-ranks of the device times.
"""
from __future__ import annotations


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of the sequences rank `rank` decodes.  Uneven batches give the
    first (global_batch % world) ranks one extra sequence."""
    if world <= 0 or not 0 <= rank < world or global_batch < world:
        raise ValueError("need 0 <= rank < world <= global_batch")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank float (device-timed seconds) across the process group."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    if dev == "cuda":
        dev = f"cuda:{torch.cuda.current_device()}"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def aggregate_throughput(per_rank_sequences: int, world: int, steps: int, max_seconds: float) -> float:
    """Whole-job decode tokens/s: all ranks' tokens over the slowest rank's time."""
    return per_rank_sequences * world * steps / max_seconds
