"""Wire formats of the reference (proj/src/json_io.cpp:56-329), restated for
the GPU backend's front door (cli.py): graphs, 1-based layout primitive
sequences, propagation plans with conversions, loop schedules, cache
configs, counters and tune reports — same keys, same 1-based dims, same
error messages, so files written by either tool read in the other.

Plus the pieces of the reference's graph loading the CLI needs:
`insert_conversions` (propagation.cpp:265-313: one `<id>__cv<k>`
LayoutConvert per conversion, spliced in before its consumer) and a shape
check. GPU schedules: a loop point is carried as the decoded parameter set
(`lfgpu_sched`) under a "gpu" key next to the reference's
loop primitives; primitives alone are mapped back to those parameters
(`sched_from_prims`).
"""
import json
from typing import Dict, List, Optional, Tuple

from . import _abi, ir, runtime
from .layout import LayoutPrimitive, fuse, padding, reorder, split, store_at, unfold


class WireError(ValueError):
    """lf::Error raised while reading a wire format (the CLI's exit code 2)."""


_KINDS = {v: k for k, v in ir.OP_NAMES.items()}
_ROLES = {"input": ir.INPUT, "constant": ir.CONSTANT, "intermediate": ir.INTERMEDIATE, "output": ir.OUTPUT}
_ROLE_NAMES = {v: k for k, v in _ROLES.items()}


# ---- graphs (json_io.cpp:56-106) -------------------------------------------

def graph_from_json(j) -> ir.Graph:
    if not isinstance(j, dict) or "tensors" not in j or "nodes" not in j:
        raise WireError("graph JSON must contain 'tensors' and 'nodes'")
    g = ir.Graph()
    for t in j["tensors"]:
        dims = [(d["name"], int(d.get("extent", 0))) for d in t["dims"]]
        dtype = ir.I32 if t.get("dtype", "float32") == "int32" else ir.F32
        role = t.get("role", "intermediate")
        if role not in _ROLES:
            raise WireError(f"unknown tensor role '{role}'")
        g.tensors.append(ir.TensorDecl(t["id"], dims, _ROLES[role], dtype))
    for n in j["nodes"]:
        kind = n["kind"]
        if kind not in _KINDS:
            raise WireError(f"unknown operator kind '{kind}'")
        attrs = {k: int(v) for k, v in n.get("attrs", {}).items()}
        g.nodes.append(ir.OperatorNode(_KINDS[kind], list(n["inputs"]), n["output"], attrs))
    return g


def graph_to_json(g: ir.Graph):
    return {
        "tensors": [{"id": t.id, "dims": [{"name": nm, "extent": e} for nm, e in t.dims],
                     "dtype": "int32" if t.dtype == ir.I32 else "float32", "role": _ROLE_NAMES[t.role]}
                    for t in g.tensors],
        "nodes": [{"kind": ir.OP_NAMES[n.kind], "attrs": dict(sorted(n.attrs.items())), "inputs": list(n.inputs),
                   "output": n.output} for n in g.nodes]}


# ---- layout primitive sequences, 1-based dims (json_io.cpp:108-185) --------

def seq_from_json(j) -> List[LayoutPrimitive]:
    seq = []
    for p in j:
        op = p.get("op")
        if op == "split":
            seq.append(split(int(p["dim"]) - 1, [int(f) for f in p["factors"]]))
        elif op == "reorder":
            seq.append(reorder([int(x) - 1 for x in p["perm"]]))
        elif op == "fuse":
            dims = [int(x) for x in p["dims"]]
            if any(b != a + 1 for a, b in zip(dims, dims[1:])):
                raise WireError("fuse: dims must be contiguous")
            seq.append(fuse(dims[0] - 1, len(dims)))
        elif op == "unfold":
            seq.append(unfold(int(p["dim"]) - 1, int(p["tile"]), int(p["stride"])))
        elif op == "pad":
            seq.append(padding(int(p["dim"]) - 1, int(p["size"])))
        elif op == "store_at":
            seq.append(store_at(p["target"], int(p["dim"]) - 1))
        else:
            raise WireError(f"unknown layout primitive '{op}'")
    return seq


def seq_to_json(seq) -> list:
    out = []
    for p in seq:
        k = p.kind
        if k == _abi.SPLIT:
            out.append({"op": "split", "dim": p.dim + 1, "factors": list(p.factors)})
        elif k == _abi.REORDER:
            out.append({"op": "reorder", "perm": [x + 1 for x in p.perm]})
        elif k == _abi.FUSE:
            out.append({"op": "fuse", "dims": [p.dim + 1 + i for i in range(p.span)]})
        elif k == _abi.UNFOLD:
            out.append({"op": "unfold", "dim": p.dim + 1, "tile": p.tile, "stride": p.stride})
        elif k == _abi.PAD:
            out.append({"op": "pad", "dim": p.dim + 1, "size": p.pad})
        elif k == _abi.STORE_AT:
            out.append({"op": "store_at", "target": p.target, "dim": p.dim + 1})
        else:
            raise WireError("inverse primitives are not serialized")
    return out


# ---- propagation plans (json_io.cpp:187-215) -------------------------------

def plan_from_json(j, g: ir.Graph):
    """(assignments {tensor: seq}, conversions [(tensor, consumer node, seq)])."""
    assignments = {t: seq_from_json(s) for t, s in j.get("assignments", {}).items()}
    conversions = []
    for c in j.get("conversions", []):
        tensor, consumer_out = c["edge"][0], c["edge"][1]
        idx = g.producer_of(consumer_out) if isinstance(consumer_out, str) else int(consumer_out)
        if idx < 0:
            raise WireError(f"schedule references unknown node output '{consumer_out}'")
        conversions.append((tensor, idx, seq_from_json(c["seq"])))
    return assignments, conversions


def plan_to_json(assignments, conversions=(), g: Optional[ir.Graph] = None):
    return {"assignments": {t: seq_to_json(s) for t, s in sorted(assignments.items())},
            "conversions": [{"edge": [t, g.nodes[c].output if g else c], "seq": seq_to_json(s)}
                            for t, c, s in conversions]}


def insert_conversions(g: ir.Graph, assignments, conversions):
    """propagation.cpp:265-313: conversions sorted (stably) by consumer, each
    a new tensor `<id>__cv<k>` produced by a LayoutConvert spliced in right
    before its consumer, whose input is rewired. Returns (graph, assignments,
    node_map original -> new index)."""
    out = ir.Graph(list(g.tensors), [])
    asg = dict(assignments)
    convs = sorted(conversions, key=lambda c: c[1])
    pending, rewires = [], {}
    for k, (tensor, consumer, seq) in enumerate(convs):
        src = g.tensor(tensor)
        tid = f"{tensor}__cv{k}"
        out.tensors.append(ir.TensorDecl(tid, list(src.dims), ir.INTERMEDIATE, src.dtype))
        pending.append([consumer, ir.OperatorNode(ir.LAYOUT_CONVERT, [tensor], tid)])
        rewires.setdefault(consumer, []).append((tensor, tid))
        asg[tid] = seq
    node_map = []
    for i, n in enumerate(g.nodes):
        for pc in pending:
            if pc[0] == i:
                out.nodes.append(pc[1])
                pc[0] = -2
        ins = list(n.inputs)
        for frm, to in rewires.get(i, []):
            ins = [to if x == frm else x for x in ins]
        node_map.append(len(out.nodes))
        out.nodes.append(ir.OperatorNode(n.kind, ins, n.output, dict(n.attrs)))
    return out, asg, node_map


# ---- loop schedules (json_io.cpp:217-275) ----------------------------------

_SCHED_KEYS = ("tile_last", "tile_second", "order", "vectorize", "parallel", "unroll", "fuse")


def sched_from_prims(node, prims):
    """A loop point's decoded parameters from the reference's primitives
    (decode_loop_point, space.cpp:509-589, run backwards): the splits are
    emitted second-innermost first, then innermost; `order` is the number of
    spatial loops after the last reduction of the reorder (reductions are the
    kernel's K loop: names starting with 'r'); annotations and fuse_consumer
    map one to one."""
    kw = dict(tile_last=1, tile_second=1, order=0, vectorize=0, parallel=0, unroll=0, fuse=0)
    splits = [p for p in prims if p.get("op") == "split"]
    if len(splits) == 1:
        kw["tile_last"] = int(splits[0]["factor"])
    elif len(splits) >= 2:
        kw["tile_second"], kw["tile_last"] = int(splits[0]["factor"]), int(splits[-1]["factor"])
    for p in prims:
        op = p.get("op")
        if op == "reorder":
            order = list(p["order"])
            red = [i for i, v in enumerate(order) if v.startswith("r")]
            if red:
                kw["order"] = min(2, len(order) - 1 - red[-1])
        elif op == "annotate":
            ann = p["ann"]
            if ann not in ("vectorize", "parallel", "unroll"):
                raise WireError(f"unknown annotation '{ann}'")
            kw[ann] = 1
        elif op == "fuse_consumer":
            kw["fuse"] = 1
        elif op != "split":
            raise WireError(f"unknown loop primitive '{op}'")
    return runtime.sched(node, **kw)


def schedules_from_json(j, g: ir.Graph):
    out = []
    for s in j:
        if "output" in s:
            node = g.producer_of(s["output"])
            if node < 0:
                raise WireError(f"schedule references unknown node output '{s['output']}'")
        else:
            node = int(s["node"])
        if "gpu" in s:
            out.append(runtime.sched(node, **{k: int(s["gpu"].get(k, 1 if k.startswith("tile") else 0))
                                             for k in _SCHED_KEYS}))
        else:
            out.append(sched_from_prims(node, s.get("prims", [])))
    return out


def schedules_to_json(scheds, g: ir.Graph):
    return [{"output": g.nodes[s.node].output, "prims": [],
             "gpu": {k: int(getattr(s, k)) for k in _SCHED_KEYS}} for s in scheds]


# ---- cache config, counters, reports (json_io.cpp:277-329) -----------------

def cache_config_from_json(j):
    """Accepted for file compatibility (the simulator's knobs); the GPU
    backend measures the device, so only validation happens here."""
    c = {"line_elems": 16, "num_lines": 512, "prefetch_lines": 2, "weights": [1.0, 1.0, 8.0, 1.0],
         "vector_lanes": 8, "parallel_threads": 8}
    c.update({k: j[k] for k in c if k in j})
    if "weights" in j and len(j["weights"]) != 4:
        raise WireError("cache config: weights must have 4 entries")
    if c["line_elems"] < 1 or c["num_lines"] < 1 or c["prefetch_lines"] < 1:
        raise WireError("cache config: line_elems, num_lines, prefetch_lines must be positive")
    return c


def counters_to_json(c):
    """lf::ProfileCounters as the GPU measure backend fills it:
    insts = kernel launches, l1_loads = algorithmic bytes, l1_misses = 0,
    l1_stores = tensor-core nodes, cost = median device microseconds."""
    return {"insts": int(c.kernels), "l1_loads": int(c.bytes_moved), "l1_misses": 0,
            "l1_stores": int(c.tc_nodes), "cost": float(c.cost)}


def tune_report(assignments, scheds, g: ir.Graph, best_cost, counters, history, seed, measurements):
    return {"plan": plan_to_json(assignments), "schedules": schedules_to_json(scheds, g),
            "best_cost": best_cost, "counters": counters,
            "history": [{"step": i + 1, "stage": st, "cost": c} for i, (st, c) in enumerate(history)],
            "seed": seed, "sim_calls": measurements, "rebuilds": {"joint": 0, "loop_only": 0},
            "backend": "gpu"}


def load_json_file(path):
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise WireError(f"cannot open '{path}'")
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise WireError(f"invalid JSON in '{path}': {e}")


def write_json_file(path, j):
    with open(path, "w") as f:
        json.dump(j, f, indent=2)
        f.write("\n")


# ---- shapes (ir.cpp:175-264, the subset the CLI needs) ----------------------

def infer_shapes(g: ir.Graph) -> ir.Graph:
    """Fill zero extents of node outputs from their inputs (ir.cpp:175-264):
    C2D / DEP / MaxPool windows, Padding, GMM, element-wise, pools and the
    encoder extension. Declared extents are checked, not overwritten."""
    ext = {t.id: list(t.extents) for t in g.tensors}

    def dims_of(tid):
        return ext[tid]

    for n in g.nodes:
        a = dims_of(n.inputs[0])
        b = dims_of(n.inputs[1]) if len(n.inputs) > 1 else None
        k = n.kind
        if k == ir.C2D:
            v = n.attr("stride", 1)
            shape = [a[0], b[0], (a[2] - b[2]) // v + 1, (a[3] - b[3]) // v + 1]
        elif k == ir.DEP:
            v = n.attr("stride", 1)
            shape = [a[0], a[1], (a[2] - b[1]) // v + 1, (a[3] - b[2]) // v + 1]
        elif k == ir.MAXPOOL:
            w, v = n.attr("window", 1), n.attr("stride", 1)
            shape = [a[0], a[1], (a[2] - w) // v + 1, (a[3] - w) // v + 1]
        elif k == ir.PADDING:
            p = n.attr("pad", 0)
            shape = [a[0], a[1], a[2] + 2 * p, a[3] + 2 * p]
        elif k == ir.GMM:
            shape = [a[0], b[1]]
        elif k == ir.GLOBAL_AVGPOOL:
            shape = [a[0], a[1]]
        elif k == ir.BMM_QK:
            shape = [n.attr("heads", 1), a[0], b[0]]
        elif k == ir.BMM_PV:
            dh = n.attr("head_dim", 0)
            shape = [a[1], n.attr("heads", 1) * dh if dh else b[1]]
        else:  # element-wise, LayoutConvert, Softmax, LayerNorm
            shape = list(a)
        out = g.tensor(n.output)
        cur = ext[n.output]
        if all(e == 0 for e in cur):
            ext[n.output] = shape
        elif cur != shape:
            raise WireError(f"shape mismatch for '{n.output}': declared {cur}, inferred {shape}")
        del out
    for t in g.tensors:
        if any(e <= 0 for e in ext[t.id]):
            raise WireError(f"tensor '{t.id}' has no extent (not produced by any node)")
    return ir.Graph([ir.TensorDecl(t.id, [(nm, e) for (nm, _), e in zip(t.dims, ext[t.id])], t.role, t.dtype)
                     for t in g.tensors], list(g.nodes))
