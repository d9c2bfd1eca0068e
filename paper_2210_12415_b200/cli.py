"""The reference's front door (proj/src/cli.cpp:53-173, proj/include/
layoutforge/cli.hpp) on the GPU backend:

  python -m paper_2210_12415_b200.cli compile --graph G [--plan P] [--sched S]
         --out DIR [--seed N] [--backend gpu] [--exact]
  python -m paper_2210_12415_b200.cli tune --graph G --out REPORT [--budget N]
         [--seed N] [--cache C] [--backend gpu]
  python -m paper_2210_12415_b200.cli bench --graph G --plan P [--plan P ...]
         --out TABLE [--budget N] [--backend gpu]

Same files (json_io.py restates json_io.cpp), same exit codes: 0 success,
2 invalid input (lf::Error), 3 oracle mismatch.

compile: the graph with its plan's assignments and conversions
(insert_conversions, propagation.cpp:265-313) and loop schedules runs on the
GPU on the reference's random_inputs(seed) (bit-identical, lfgpu_random_inputs)
— tensor cores where the layouts allow, or the reference's arithmetic with
--exact — and is checked against the GPU's evaluation of the same graph on
logical layouts in fp64-accumulating mode (the reference_eval of cli.cpp:74-82
moved to the device) with the reference's rule (cli.cpp:30-49: int32 exact,
float 1e-5 relative). Writes DIR/plan.txt (the kernel of every node) and
DIR/verdict.json ({"oracle", "max_rel_diff", "seed"}).

tune: the GPU-measured candidate search (tuner.py; the reference's PPO
policy is the CPU search side, out of this backend's scope) over each complex
node's template layouts x loop points, within --budget measurements; writes
the reference's report keys (json_io.cpp:303-323).

bench: each plan file's layouts with a loop-point sweep per complex node
(the reference's loop-only stage, cli.cpp:128-173), rows sorted by cost.
"""
import argparse
import os
import sys
import time

import numpy as np

from . import _abi, ir, json_io, runtime, tuner

EXIT_OK, EXIT_INVALID, EXIT_MISMATCH = 0, 2, 3


def load_graph(path):
    g = json_io.graph_from_json(json_io.load_json_file(path))
    return json_io.infer_shapes(g)


def oracle_matches(g, ref, got):
    """cli.cpp:30-49: int32 exact, float 1e-5 relative, scale max(1,|a|,|b|)."""
    ok, worst = True, 0.0
    for tid, r in ref.items():
        if tid not in got:
            continue
        a, b = np.asarray(r, dtype=np.float64), np.asarray(got[tid], dtype=np.float64)
        if a.size != b.size:
            return False, float("inf")
        d = np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
        w = float(d.max()) if d.size else 0.0
        worst = max(worst, w)
        if w > (0.0 if g.tensor(tid).dtype == ir.I32 else 1e-5):
            ok = False
    return ok, worst


def _fail(msg):
    sys.stderr.write(f"error: {msg}\n")
    return EXIT_INVALID


def cmd_compile(a):
    try:
        g0 = load_graph(a.graph)
        asg, convs = ({}, [])
        if a.plan:
            asg, convs = json_io.plan_from_json(json_io.load_json_file(a.plan), g0)
        g, asg, _ = json_io.insert_conversions(g0, asg, convs)
        scheds = json_io.schedules_from_json(json_io.load_json_file(a.sched), g) if a.sched else []
    except (json_io.WireError, KeyError, TypeError) as e:
        return _fail(e)
    try:
        inputs = runtime.random_inputs(g0, a.seed)
        flags = _abi.PLAN_EXACT if a.exact else _abi.PLAN_DEFAULT
        p = runtime.Plan(g, asg, scheds, flags | _abi.PLAN_KEEP_ALL)
        for tid, v in inputs.items():
            p.set_input(tid, v)
        p.run()
        got = {n.output: p.get_output(n.output) for n in g.nodes if n.output in {m.output for m in g0.nodes}}
        ref = runtime.interpret(g0, {}, [], inputs, flags=_abi.PLAN_EXACT)
        os.makedirs(a.out, exist_ok=True)
        with open(os.path.join(a.out, "plan.txt"), "w") as f:
            for i, n in enumerate(g.nodes):
                f.write(f"{i:3d} {ir.OP_NAMES[n.kind]:13s} {n.output:24s} {p.node_kernel(i)}\n")
        p.close()
    except (runtime.LfError, json_io.WireError, ValueError) as e:
        return _fail(e)
    ok, worst = oracle_matches(g0, ref, got)
    json_io.write_json_file(os.path.join(a.out, "verdict.json"),
                            {"oracle": "pass" if ok else "fail", "max_rel_diff": worst, "seed": a.seed,
                             "backend": "gpu", "mode": "exact" if a.exact else "tensor_cores"})
    print(f"program: {a.out}/plan.txt")
    print(f"oracle: {'pass' if ok else 'fail'} (max rel diff {worst:g})")
    return EXIT_OK if ok else EXIT_MISMATCH


def _device_inputs(g, seed):
    import torch
    return {k: torch.tensor(v, dtype=torch.float32, device="cuda").view(g.tensor(k).extents)
            for k, v in runtime.random_inputs(g, seed).items()}


def _candidates(g, node):
    nd = g.nodes[node]
    if nd.kind == ir.GMM:
        a, b = g.tensor(nd.inputs[0]), g.tensor(nd.inputs[1])
        return tuner.gemm_candidates(a.extents[0], a.extents[1], b.extents[1], node)
    if nd.kind == ir.C2D:
        fuse = 1 if any(ir.is_elementwise_op(g.nodes[c].kind) for c in g.consumers_of(nd.output)) else 0
        return tuner.conv_candidates(g, node, fuse)
    return []


def _search(g, node_cands, budget, inputs, base=None):
    """Greedy over complex nodes in order: each node's candidates measured
    with the other nodes at their current choice, within `budget` total
    measurements; returns (choice per node, best result, history)."""
    choice = dict(base or {})
    history, best_r, used = [], None, 0
    for node, cands in node_cands:
        per = max(1, (budget - used) // max(1, sum(1 for n, _ in node_cands if n not in choice) or 1))
        stride = max(1, len(cands) // per)
        node_best = None
        for c in cands[::stride][:per]:
            merged = tuner.Candidate(dict(), [], c.label)
            for n2, c2 in choice.items():
                if n2 != node:
                    merged.factors.update(c2.factors)
                    merged.scheds += c2.scheds
            merged.factors.update(c.factors)
            merged.scheds += c.scheds
            r = tuner.measure(g, merged, inputs, flags=0)
            used += 1
            if r.cost_us is None:
                continue
            history.append(("gpu", r.cost_us))
            if node_best is None or r.cost_us < node_best[1].cost_us:
                node_best = (c, r)
        if node_best:
            choice[node] = node_best[0]
            best_r = node_best[1]
    return choice, best_r, history, used


def cmd_tune(a):
    try:
        g = load_graph(a.graph)
        if a.cache:
            json_io.cache_config_from_json(json_io.load_json_file(a.cache))
    except (json_io.WireError, KeyError, TypeError) as e:
        return _fail(e)
    try:
        inputs = _device_inputs(g, a.seed)
        nodes = [(i, _candidates(g, i)) for i, n in enumerate(g.nodes) if ir.is_complex_op(n.kind)]
        nodes = [(i, c) for i, c in nodes if c]
        t0 = time.perf_counter()
        choice, best, history, used = _search(g, nodes, a.budget, inputs)
        if best is None:
            return _fail("no legal candidate")
        merged = tuner.Candidate({}, [])
        for c in choice.values():
            merged.factors.update(c.factors)
            merged.scheds += c.scheds
        asg = tuner.seqs_for(g, merged)
        p = runtime.Plan(g, asg, merged.scheds, _abi.PLAN_CUDA_GRAPH)
        for k, v in inputs.items():
            p.set_input_device(k, v)
        c = p.measure(warmup=3, reps=7, flush_l2=True)
        p.close()
        rep = json_io.tune_report(asg, merged.scheds, g, c.cost, json_io.counters_to_json(c), history, a.seed, used)
        rep["seconds"] = round(time.perf_counter() - t0, 3)
        json_io.write_json_file(a.out, rep)
    except (runtime.LfError, json_io.WireError, ValueError) as e:
        return _fail(e)
    print(f"best_cost: {c.cost}")
    print(f"counters: insts={c.kernels} l1_loads={c.bytes_moved} l1_misses=0 l1_stores={c.tc_nodes}")
    print(f"report: {a.out}")
    return EXIT_OK


def cmd_bench(a):
    try:
        g = load_graph(a.graph)
        plans = []
        for path in a.plan:
            pj = json_io.load_json_file(path)
            asg, convs = json_io.plan_from_json(pj, g)
            plans.append((pj.get("name", path), asg, convs))
    except (json_io.WireError, KeyError, TypeError) as e:
        return _fail(e)
    rows = []
    try:
        inputs = _device_inputs(g, a.seed)
        for name, asg, convs in plans:
            g2, asg2, _ = json_io.insert_conversions(g, asg, convs)
            best = None
            used = 0
            for ni, n in enumerate(g2.nodes):
                if not ir.is_complex_op(n.kind):
                    continue
                for tl in (1, 64, 128, 256):
                    for order in (0, 1):
                        if used >= a.budget:
                            break
                        sc = [runtime.sched(ni, tile_last=tl, order=order, fuse=1)]
                        try:
                            p = runtime.Plan(g2, asg2, sc, _abi.PLAN_CUDA_GRAPH)
                        except runtime.LfError:
                            continue
                        for k, v in inputs.items():
                            p.set_input_device(k, v)
                        c = p.measure(warmup=2, reps=5, flush_l2=True)
                        p.close()
                        used += 1
                        if best is None or c.cost < best.cost:
                            best = c
            if best is None:  # no complex node: the plan as given
                p = runtime.Plan(g2, asg2, [], _abi.PLAN_CUDA_GRAPH)
                for k, v in inputs.items():
                    p.set_input_device(k, v)
                best = p.measure(warmup=2, reps=5, flush_l2=True)
                p.close()
            rows.append((name, best))
    except (runtime.LfError, json_io.WireError, ValueError) as e:
        return _fail(e)
    rows.sort(key=lambda r: r[1].cost)  # stable, like std::stable_sort
    table = []
    for name, c in rows:
        jr = json_io.counters_to_json(c)
        jr["name"] = name
        jr["cost"] = c.cost
        table.append(jr)
    json_io.write_json_file(a.out, {"budget": a.budget, "rows": table, "backend": "gpu"})
    for name, c in rows:
        print(f"{name}: cost={c.cost} misses=0")
    return EXIT_OK


def main(argv=None):
    ap = argparse.ArgumentParser(prog="layoutforge-gpu")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("compile")
    c.add_argument("--graph", required=True)
    c.add_argument("--plan", default="")
    c.add_argument("--sched", default="")
    c.add_argument("--out", required=True)
    c.add_argument("--seed", type=int, default=42)
    c.add_argument("--exact", action="store_true", help="the reference's arithmetic (fp64 accumulation)")
    t = sub.add_parser("tune")
    t.add_argument("--graph", required=True)
    t.add_argument("--out", required=True)
    t.add_argument("--cache", default="")
    t.add_argument("--budget", type=int, default=64)
    t.add_argument("--seed", type=int, default=42)
    b = sub.add_parser("bench")
    b.add_argument("--graph", required=True)
    b.add_argument("--plan", action="append", required=True)
    b.add_argument("--out", required=True)
    b.add_argument("--budget", type=int, default=64)
    b.add_argument("--seed", type=int, default=0)
    for p in (c, t, b):
        p.add_argument("--backend", default="gpu", choices=["gpu"],
                       help="gpu: this B200 backend (the simulator backend is the reference's own CLI)")
    a = ap.parse_args(argv)
    return {"compile": cmd_compile, "tune": cmd_tune, "bench": cmd_bench}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
