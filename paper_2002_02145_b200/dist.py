"""Minibatch sharding across GPUs.

The reference's only parallelism is the OpenMP annotation over `img`
(include/nestrank/presets.hpp:125); the conv nest has no order-constraining dependences and
every image writes a disjoint output slab, so a layer is split across the GPUs of one box by
image range with no collective on the hot path. Rank r of W takes images
[floor(r*N/W), floor((r+1)*N/W)). Collectives appear only after timing: a max over ranks of
the step time, and a gather of the output shards to rank 0 for verification.
"""
from __future__ import annotations


def image_range(rank: int, world: int, n_img: int) -> tuple[int, int]:
    """(img_begin, img_count) of this rank's shard."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    b0 = rank * n_img // world
    b1 = (rank + 1) * n_img // world
    return b0, b1 - b0


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_shards(local, n_img: int, per_image: int):
    """All-gather variable-size image shards (flat tensors of count*per_image elements) and
    return the full [n_img*per_image] tensor on every rank (NCCL on GPU, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    counts = [image_range(r, world, n_img)[1] for r in range(world)]
    cmax = max(counts)
    buf = torch.zeros(cmax * per_image, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.cat([parts[r][: counts[r] * per_image] for r in range(world)])
