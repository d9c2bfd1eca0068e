"""Batch-sharded end-to-end inference across the GPUs of one box (cfg4 b64
sharded 8x8).

One process per GPU. Every rank builds the same plan (graph, tuned layouts
and weights replicated) for its batch shard, runs it on its own device with
no collective on the data path, and the logits come back in one gather at the
end (64x1000 fp32 = 256 KB). Shards are contiguous and balanced: rank r of W
owns images [start, start + count) with the remainder spread over the first
ranks, so the gathered rows are in global batch order.
"""
from typing import Callable, Tuple


def batch_shard(global_batch: int, rank: int, world: int) -> Tuple[int, int]:
    """(start, count) of `rank`'s contiguous shard of the global batch."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(global_batch, world)
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


def gather_rows(local, global_batch: int, rank: int, world: int):
    """All ranks' row blocks concatenated in global batch order (a single
    all_gather of fixed-size padded blocks; the padding is dropped)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    width = local.shape[1]
    cap = -(-global_batch // world)
    buf = torch.zeros((cap, width), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    rows = []
    for r in range(world):
        _, cnt = batch_shard(global_batch, r, world)
        rows.append(parts[r][:cnt])
    return torch.cat(rows, 0)


def run_sharded(forward: Callable, x_global, rank: int, world: int):
    """Run `forward` (batch -> [batch, classes]) on this rank's shard of
    x_global and gather the full logits on every rank."""
    n = x_global.shape[0]
    start, count = batch_shard(n, rank, world)
    local = forward(x_global[start:start + count])
    return gather_rows(local, n, rank, world)
