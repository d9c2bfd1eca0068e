"""Batch-sharded inference plumbing (SURVEY.md §8e, cfg4 b64 sharded 8x8):
balanced contiguous shards and an in-order gather, checked with world size 2
(gloo, CPU) against the unsharded forward."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_12415_b200 import shard


@pytest.mark.parametrize("n,world", [(64, 8), (64, 3), (7, 4), (1, 2), (0, 2)])
def test_batch_shard_partitions(n, world):
    spans = [shard.batch_shard(n, r, world) for r in range(world)]
    assert sum(c for _, c in spans) == n
    pos = 0
    for s, c in spans:
        assert s == pos
        pos += c
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _forward(x):
    # stand-in for the plan: a fixed per-image function
    w = torch.arange(12, dtype=torch.float32).view(3, 4)
    return x.view(x.shape[0], -1)[:, :3] @ w


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    x = torch.randn(n, 3, 2, 2)
    out = shard.run_sharded(_forward, x, rank, world)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [64, 5])
def test_sharded_gather_matches_unsharded(n):
    torch.manual_seed(0)
    x = torch.randn(n, 3, 2, 2)
    ref = _forward(x)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, o in outs:
        assert torch.equal(o, ref)
