"""Multi-process (gloo, world size 2, CPU) coverage of the sharded tuner path
(SURVEY.md §8e): each rank measures its own candidates, results are
gathered and committed in candidate-index order with the reference's
first-index-wins tie rule (tuner.cpp:180-189)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_12415_b200 import ir, tuner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_measure(graph, cand, inputs=None, **kw):
    """Deterministic stand-in for the GPU measurement (no device here):
    cost depends only on the layout factors; one point is 'illegal'."""
    f = cand.factors[0]
    if f == (128, 64, 128):
        return tuner.Result(cand, None, "EUNSUPPORTED")
    cost = 1000.0 / (f[0] * f[2]) ** 0.5 + f[1] * 1e-3
    if f[2] == 512 and f[0] == 256:
        cost = 0.5  # tie partner below
    if f[2] == 256 and f[0] == 512:
        cost = 0.5
    return tuner.Result(cand, cost)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = ir.gemm(1024, 1024, 1024)
    cands = tuner.gemm_candidates(1024, 1024, 1024)
    results, best_i, secs, n_local = tuner.sweep_distributed(g, cands, measure_fn=fake_measure)
    q.put((rank, [r.cost_us for r in results], best_i, n_local))
    dist.destroy_process_group()


def test_sharded_sweep_matches_serial():
    g = ir.gemm(1024, 1024, 1024)
    cands = tuner.gemm_candidates(1024, 1024, 1024)
    serial, best_serial, _, n = tuner.sweep_distributed(g, cands, measure_fn=fake_measure)
    assert n == len(cands)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    costs0, costs1 = out[0][1], out[1][1]
    assert costs0 == costs1 == [r.cost_us for r in serial]      # same committed history
    assert out[0][2] == out[1][2] == best_serial                  # same winner on every rank
    assert out[0][3] + out[1][3] == len(cands)                    # shards partition the stream
    assert abs(out[0][3] - out[1][3]) <= 1
    # first-index-wins tie rule
    ties = [i for i, c in enumerate(costs0) if c == 0.5]
    assert best_serial == ties[0]
    assert None in costs0  # the illegal candidate stays rejected, not dropped
