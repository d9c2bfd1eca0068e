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


def sweep_distributed(graph: Graph, cands, inputs=None, measure_fn=None, **kw):
    """One process per GPU: each rank measures candidates i with
    i % world == rank (no collective on the data path), then the (index,
    cost) pairs are all-gathered and committed in candidate-index order, so
    the winner is the reference's: strictly lowest cost, first index on ties
    (tuner.cpp:180-189). Returns (results in index order, best index,
    local seconds, local count)."""
    import torch.distributed as dist
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
    fn = measure_fn or measure
    t0 = time.perf_counter()
    local = [(i, fn(graph, c, inputs, **kw)) for i, c in enumerate(cands) if i % world == rank]
    secs = time.perf_counter() - t0
    mine = [(i, r.cost_us, r.error) for i, r in local]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
    else:
        gathered = [mine]
    merged = {}
    for part in gathered:
        for i, cost, err in part:
            merged[i] = Result(cands[i], cost, err)
    results = [merged[i] for i in range(len(cands))]
    best_i, best_c = -1, float("inf")
    for i, r in enumerate(results):
        if r.cost_us is not None and r.cost_us < best_c:
            best_i, best_c = i, r.cost_us
    return results, best_i, secs, len(local)


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
