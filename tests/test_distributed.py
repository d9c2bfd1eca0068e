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


def faulty_measure_rank1(graph, cand, inputs=None, **kw):
    """Rank 1's device 'fails' on its third measurement (a CUDA fault is any
    non-legality exception); rank 0 stays healthy."""
    faulty_measure_rank1.calls = getattr(faulty_measure_rank1, "calls", 0) + 1
    if dist.get_rank() == 1 and faulty_measure_rank1.calls == 3:
        raise RuntimeError("[3] CUDA error: an illegal memory access was encountered")
    return fake_measure(graph, cand, inputs)


def always_faulty(graph, cand, inputs=None, **kw):
    raise RuntimeError("[3] device lost")


def _fault_worker(rank, world, port, q, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = ir.gemm(1024, 1024, 1024)
    cands = tuner.gemm_candidates(1024, 1024, 1024)[:40]
    try:
        if mode == "one":
            results, best_i, _, n_local = tuner.sweep_distributed(g, cands, measure_fn=faulty_measure_rank1)
            q.put((rank, "ok", [r.cost_us for r in results], best_i, n_local))
        elif mode == "all":
            tuner.sweep_distributed(g, cands, measure_fn=always_faulty)
            q.put((rank, "no-raise", None, None, None))
        else:  # measure_top with predictions
            pred = [float((i * 7) % 13) for i in range(len(cands))]
            idx, res, best = tuner.measure_top(g, cands, predicted=pred, top_k=8, measure_fn=fake_measure)
            q.put((rank, "top", idx, [r.cost_us for r in res], best))
    except tuner.DeviceFault as e:
        q.put((rank, "fault", str(e)[:80], None, None))
    dist.destroy_process_group()


def _run2(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fault_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_device_fault_requeues_on_healthy_rank():
    # Rank 1 fails mid-sweep: its unmeasured candidates (and the one that
    # faulted) are re-dealt to rank 0; the committed history equals the
    # fault-free serial run on both ranks, and neither rank hangs.
    g = ir.gemm(1024, 1024, 1024)
    cands = tuner.gemm_candidates(1024, 1024, 1024)[:40]
    serial, best_serial, _, _ = tuner.sweep_distributed(g, cands, measure_fn=fake_measure)
    out = _run2("one")
    assert [o[1] for o in out] == ["ok", "ok"]
    assert out[0][2] == out[1][2] == [r.cost_us for r in serial]
    assert out[0][3] == out[1][3] == best_serial
    assert out[0][4] > out[1][4]  # rank 0 picked up rank 1's share


def test_all_ranks_faulty_raises_everywhere():
    out = _run2("all")
    assert [o[1] for o in out] == ["fault", "fault"]


def test_measure_top_dispatches_topk_in_prediction_order():
    # tuner.cpp:243-274: stable-sort by prediction, measure top_k, strict-<
    # best in that order; the k measurements are split across the ranks.
    g = ir.gemm(1024, 1024, 1024)
    cands = tuner.gemm_candidates(1024, 1024, 1024)[:40]
    pred = [float((i * 7) % 13) for i in range(len(cands))]
    idx_s, res_s, best_s = tuner.measure_top(g, cands, predicted=pred, top_k=8, measure_fn=fake_measure)
    assert idx_s == sorted(range(len(cands)), key=lambda i: pred[i])[:8]
    out = _run2("top")
    for o in out:
        assert o[1] == "top" and o[2] == idx_s and o[3] == [r.cost_us for r in res_s] and o[4] == best_s
