"""Batch sharding across the GPUs of one box.

Inference is embarrassingly parallel over images: rank r of W owns images
[r*B, (r+1)*B) of the global batch (for synthetic data: elements
[(r*B)*CHW, ...) of the SeededStream), weights are replicated, and no
collective runs on the data path.  The only collectives are bookkeeping:
the max-over-ranks step time, and the optional final gather of the logits
to rank 0 (NCCL on GPUs, gloo in the CPU tests).

Two ways to run N GPUs: one process per GPU (torchrun; bench.py, this module
for the bookkeeping) or one process for all of them (api.MultiEngine,
xlf_multi_*: a native host worker thread + stream per device).  Both shard
with the same rule (xlf_shard).
"""
from __future__ import annotations


def shard(rank: int, world: int, per_rank: int):
    """(first_image, count) of `rank` -- weak scaling, fixed images per rank:
    the library's shard rule (xlf_shard, the MultiEngine's) over world*per_rank images."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad shard request")
    from .api import shard_range
    return shard_range(world * per_rank, world, rank)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(t):
    """Gathers equally shaped per-rank tensors to rank 0 (concatenated along
    dim 0, rank order); other ranks get None.  Off the timed hot path."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t.contiguous())
    return torch.cat(parts, 0) if dist.get_rank() == 0 else None
