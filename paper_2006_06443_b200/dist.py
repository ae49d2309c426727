"""Multi-GPU plumbing of the data-parallel hot path.

The compressed layer shards by image: every rank holds the same weights (one
`lrs_conv_create` per device) and evaluates its own contiguous slice of the
batch; there is no collective on the data path.  torch.distributed (NCCL on
the GPUs, gloo in the CPU tests) carries only the barrier, the max-over-ranks
timing reduction and the optional verification gather of Y.
"""
from __future__ import annotations

from typing import Tuple


def shard_range(global_batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous images [start, end) of `rank`; the first global_batch % world
    ranks take one extra image, so the shards tile the batch exactly."""
    if world < 1 or not 0 <= rank < world or global_batch < 0:
        raise ValueError(f"bad shard request: batch {global_batch}, rank {rank}, world {world}")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank scalar (the slowest rank's time) over the process group."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_shards(y_local, global_batch: int, group=None):
    """Verification only (outside any timed region): gather every rank's Y
    shard [n_r, ...] into the full [global_batch, ...] tensor on every rank.
    Shards may differ by one image (shard_range), so each is padded to the
    largest before the collective and trimmed after."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return y_local
    sizes = [shard_range(global_batch, r, world) for r in range(world)]
    most = max(e - s for s, e in sizes)
    pad = torch.zeros((most,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    pad[: y_local.shape[0]] = y_local
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([o[: e - s] for o, (s, e) in zip(out, sizes)], dim=0)


def allreduce_grads(tensors, group=None) -> None:
    """The one exchange of the backward pass: data-parallel fine-tuning
    sums each parameter gradient over the ranks' image shards (weight gradients are sums over
    images).  In place, SUM, one all-reduce per tensor (NCCL on the GPUs, gloo in the tests)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    for t in tensors:
        if t is not None and t.numel():
            dist.all_reduce(t, group=group)
