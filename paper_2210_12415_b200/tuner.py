"""GPU-measured candidate search: the tuner's measure seam on B200.

The reference tuner lowers each candidate and scores it with simulate_cache
(proj/src/tuner.cpp:165-191); measure_top measures at most top_k candidates
serially (tuner.cpp:243-274). Here a candidate (layout factors per complex
node + decoded loop points) becomes a GPU plan and is scored by
Plan.measure (median device microseconds). Candidates the kernels cannot
legalise raise LfError(EUNSUPPORTED) and are rejected, exactly like the
reference rejects candidates whose lowering throws (tuner.cpp:169-174).
The PPO/surrogate search policy of the reference is out of scope
(SURVEY.md §2); this module provides the candidate streams and the
measurement, and shards candidates across GPUs (one process per GPU) with
no collective on the data path.
"""
import itertools
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import _abi, runtime
from .ir import Graph, is_complex_op


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


@dataclass
class Candidate:
    factors: Dict[int, Tuple[int, ...]]          # complex node -> template factors
    scheds: List = field(default_factory=list)   # lfgpu_sched entries
    label: str = ""


@dataclass
class Result:
    candidate: Candidate
    cost_us: Optional[float]   # None: rejected (not legal on tensor cores)
    error: str = ""


def seqs_for(graph: Graph, cand: Candidate):
    seqs = {}
    for node, f in cand.factors.items():
        seqs.update(runtime.decode_layout(graph, node, list(f)))
    return seqs


def measure(graph: Graph, cand: Candidate, inputs=None, flags=_abi.PLAN_REQUIRE_TC,
            warmup=2, reps=5, flush_l2=True, ctx=None):
    """One tuner measurement (the simulate_cache call at tuner.cpp:178)."""
    try:
        p = runtime.Plan(graph, seqs_for(graph, cand), cand.scheds,
                         flags | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
    except runtime.LfError as e:
        if e.code in (_abi.EUNSUPPORTED, _abi.EINVAL, _abi.ERANGE):
            return Result(cand, None, str(e))
        raise
    try:
        if inputs:
            for tid, v in inputs.items():
                p.set_input_device(tid, v)
        c = p.measure(warmup=warmup, reps=reps, flush_l2=flush_l2)
        return Result(cand, c.cost)
    finally:
        p.close()


def sweep(graph: Graph, cands, inputs=None, shard=(0, 1), **kw):
    """Measure every candidate of this rank's shard; returns (results, seconds)."""
    rank, world = shard
    t0 = time.perf_counter()
    res = [measure(graph, c, inputs, **kw) for i, c in enumerate(cands) if i % world == rank]
    return res, time.perf_counter() - t0


def best(results):
    ok = [r for r in results if r.cost_us is not None]
    return min(ok, key=lambda r: r.cost_us) if ok else None


class DeviceFault(RuntimeError):
    """A measurement failed for a reason other than candidate legality
    (CUDA fault, lost device): the rank stops measuring and its remaining
    candidates are re-queued on the healthy ranks."""


def _safe_measure(fn, graph, cand, inputs, kw):
    """(cost_us, error, fault) for one candidate; never raises, so every rank
    reaches the collective even when its device fails (a raise between
    collectives would leave the other ranks blocked in all_gather)."""
    try:
        r = fn(graph, cand, inputs, **kw)
        return r.cost_us, r.error, False
    except Exception as e:  # noqa: BLE001 - turned into a fault record
        return None, f"{type(e).__name__}: {e}", True


def sweep_distributed(graph: Graph, cands, inputs=None, measure_fn=None, max_rounds=4, **kw):
    """One process per GPU: each rank measures candidates i with
    i % world == rank (no collective on the data path), then the (index,
    cost) pairs are all-gathered and committed in candidate-index order, so
    the winner is the reference's: strictly lowest cost, first index on ties
    (tuner.cpp:180-189).

    Fault handling: a rank whose measurement raises anything
    but a legality rejection marks itself failed, stops measuring, and its
    unmeasured candidates are dealt again, round-robin, over the ranks still
    healthy (up to `max_rounds` rounds). Every rank joins every gather, so a
    failing device never blocks the others. Returns (results in index
    order, best index, local seconds, local count); raises DeviceFault when
    no healthy rank is left with candidates pending."""
    import torch.distributed as dist
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
    fn = measure_fn or measure
    t0 = time.perf_counter()
    done = {}                      # index -> (cost, error)
    healthy = list(range(world))
    pending = list(range(len(cands)))
    me_ok = True
    nloc = 0
    faults = []
    for _ in range(max_rounds):
        if not pending:
            break
        if not healthy:
            raise DeviceFault("every rank failed; unmeasured candidates: %d (%s)" % (
                len(pending), "; ".join(faults)[:300]))
        mine = []
        if me_ok and rank in healthy:
            slot = healthy.index(rank)
            for k, i in enumerate(pending):
                if k % len(healthy) != slot:
                    continue
                if not me_ok:  # device failed earlier in this round: leave the rest
                    break
                cost, err, fault = _safe_measure(fn, graph, cands[i], inputs, kw)
                nloc += 1
                if fault:
                    me_ok = False
                    mine.append((i, None, err, True))
                else:
                    mine.append((i, cost, err, False))
        if world > 1:
            gathered = [None] * world
            dist.all_gather_object(gathered, (rank, me_ok, mine))
        else:
            gathered = [(rank, me_ok, mine)]
        for r, ok, part in gathered:
            if not ok and r in healthy:
                healthy.remove(r)
            for i, cost, err, fault in part:
                if fault:
                    faults.append(f"rank {r}: {err}")
                else:
                    done[i] = (cost, err)
        pending = [i for i in range(len(cands)) if i not in done]
    if pending:
        raise DeviceFault("candidates left unmeasured after %d rounds: %d (%s)" % (
            max_rounds, len(pending), "; ".join(faults)[:300]))
    secs = time.perf_counter() - t0
    results = [Result(cands[i], done[i][0], done[i][1]) for i in range(len(cands))]
    best_i, best_c = -1, float("inf")
    for i, r in enumerate(results):
        if r.cost_us is not None and r.cost_us < best_c:
            best_i, best_c = i, r.cost_us
    return results, best_i, secs, nloc


def measure_top(graph: Graph, cands, predicted=None, top_k=8, inputs=None, **kw):
    """The reference's measure_top (tuner.cpp:243-274) with the top-k
    measurements of one call dispatched across the GPUs of the job.

    Candidates are ranked by `predicted` cost (the surrogate's prediction,
    stable sort, tuner.cpp:250-258) when given, else kept in index order; the
    first `top_k` are measured, one GPU each (sweep_distributed), and the
    results are committed in rank order with the strict-< best rule, so the
    bookkeeping is identical to the serial loop. Returns (measured indices,
    their results, best index or -1)."""
    idx = list(range(len(cands)))
    if predicted is not None:
        idx.sort(key=lambda i: predicted[i])  # list.sort is stable
    idx = idx[:top_k]
    res, _, _, _ = sweep_distributed(graph, [cands[i] for i in idx], inputs, **kw)
    best_i, best_c = -1, float("inf")
    for k, r in zip(idx, res):
        if r.cost_us is not None and r.cost_us < best_c:
            best_i, best_c = k, r.cost_us
    return idx, res, best_i


# --- candidate streams -------------------------------------------------------

def gemm_candidates(M, K, N, node=0):
    """GMM template points (m_t, k_t, n_t) with tensor-core-friendly bricks,
    crossed with the innermost loop tile (which picks the UMMA N width)."""
    out = []
    for mt in [d for d in divisors(M) if d >= 128 or d == M]:
        for kt in [d for d in divisors(K) if d % 64 == 0]:
            for nt in [d for d in divisors(N) if d % 64 == 0]:
                for tl in (64, 128, 256):
                    if tl > nt and nt != N:
                        continue
                    # order: 0 = split-K by heuristic, 1 = no split (lfgpu_sched docs)
                    for order in (0, 1):
                        out.append(Candidate({node: (mt, kt, nt)},
                                             [runtime.sched(node, tile_last=tl, order=order)],
                                             f"m_t={mt} k_t={kt} n_t={nt} tile={tl} order={order}"))
    return out


def conv_candidates(graph: Graph, node, fuse=0):
    """C2D template points (h_t, w_t, o_t, i_t, i'_t, o'_t) whose bricks map
    onto 128-row UMMA tiles: 32..128 output pixels per tile, channel bricks
    that are multiples of 16 (SURVEY.md §7 hard part 1)."""
    n = graph.nodes[node]
    y = graph.tensor(n.output)
    x = graph.tensor(n.inputs[0])
    _, O, Ho, Wo = y.extents
    I = x.extents[1]
    out = []
    for ht in divisors(Ho):
        for wt in divisors(Wo):
            if wt > 128:
                continue
            rows = min(ht, 128 // wt) * wt
            if rows < 32:
                continue
            for ot in [d for d in divisors(O) if d % 16 == 0 and d <= 256]:
                for it in [d for d in divisors(I) if d % 16 == 0 and d < I and d <= 64]:
                    for o2 in sorted({ot, 16, O}):
                        if O % o2 or o2 % 16:
                            continue
                        out.append(Candidate({node: (ht, wt, ot, it, it, o2)},
                                             [runtime.sched(node, fuse=fuse)],
                                             f"h_t={ht} w_t={wt} o_t={ot} i_t={it} o'={o2}"))
                        # channels-as-rows orientation (schedule unroll=2) for
                        # wide channel tiles on small spatial tiles
                        if ot % 128 == 0 and o2 % 64 == 0 and ht * wt <= 256:
                            out.append(Candidate({node: (ht, wt, ot, it, it, o2)},
                                                 [runtime.sched(node, fuse=fuse, unroll=2)],
                                                 f"h_t={ht} w_t={wt} o_t={ot} i_t={it} o'={o2} trans"))
    return out
