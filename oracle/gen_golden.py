"""Generate tests/golden/*.json from the reference build (oracle/_ref/libref.so).

TEST INFRASTRUCTURE ONLY. Run here (where /root/reference exists):
    make -C oracle && python oracle/gen_golden.py
The fixtures let the GPU box (no /root/reference) check parity: seeded
inputs, materializations, reference_eval outputs, decoded template layouts
and planner contexts, each recorded as FNV-1a(fp32) checksums (and full
values for the tiny known-answer cases).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as O  # noqa: E402
from paper_2210_12415_b200 import ir  # noqa: E402
from paper_2210_12415_b200.layout import fuse, padding, reorder, split, unfold  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def seq_json(seq):
    return [{"kind": p.kind, "dim": p.dim, "factors": p.factors, "perm": p.perm, "span": p.span,
             "tile": p.tile, "stride": p.stride, "pad": p.pad, "target": p.target} for p in seq]


def stats(v):
    v = np.asarray(v, dtype=np.float64)
    return {"n": int(v.size), "sum": float(v.sum()), "sumsq": float((v * v).sum()),
            "fnv": O.fnv1a(v), "head": [float(x) for x in v[:4]]}


# Materialization cases: (logical extents, sequence). Cover every primitive
# the reference materializes (interp.cpp:181-264) plus the template layouts.
MATERIALIZE = [
    ("nchwc16", [1, 64, 56, 56], [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])]),
    ("nchwc4_b2", [2, 8, 5, 7], [split(1, [2, 4]), reorder([0, 1, 3, 4, 2])]),
    ("unfold_kat", [5], [unfold(0, 3, 2)]),
    ("unfold_overhang", [6], [unfold(0, 3, 2)]),
    ("unfold_2d", [1, 3, 10, 10], [unfold(2, 6, 4), unfold(4, 6, 4), reorder([0, 2, 4, 1, 3, 5])]),
    ("pad", [2, 3, 4], [padding(1, 2)]),
    ("fuse_split", [2, 3, 3, 8], [fuse(1, 3), split(1, [2, 4, 9]), reorder([0, 1, 3, 2])]),
    ("pad_split", [3, 14], [padding(1, 2), split(1, [4, 4])]),
    ("cfg1_xp_tiled", [1, 64, 58, 58],
     [unfold(3, 16, 14), unfold(2, 6, 4), split(1, [4, 16]), reorder([0, 3, 5, 1, 4, 6, 2])]),
    ("gemm_a_bricks", [256, 192], [split(1, [3, 64]), split(0, [2, 128]), reorder([0, 2, 1, 3])]),
    ("gemm_b_mmajor", [192, 256], [split(0, [3, 64]), reorder([0, 2, 1])]),
    ("reorder_3d", [4, 5, 6], [reorder([2, 0, 1])]),
]


def materialize_cases():
    out = []
    for idx, (name, ext, seq) in enumerate(MATERIALIZE):
        rng = np.random.default_rng(7 + idx)
        src = np.round(rng.uniform(-1, 1, int(np.prod(ext))) * 64) / 64
        if name == "unfold_kat":
            src = np.array([1, 2, 3, 4, 5], dtype=np.float64)
        if name == "unfold_overhang":
            src = np.arange(1, 7, dtype=np.float64)
        got = O.materialize(ext, seq, src, lib="ref")
        case = {"name": name, "extents": ext, "seq": seq_json(seq), "src_seed": 7 + idx,
                "src": stats(src), "phys": O.derive(ext, seq), "out": stats(got)}
        if got.size <= 64:
            case["src_values"] = [float(x) for x in src]
            case["values"] = [float(x) for x in got]
        out.append(case)
    return out


GRAPHS = {
    "cfg1_pad_conv": lambda: ir.pad_conv(1, 64, 64, 56, 3, 1, 1),
    "cfg2_gemm1024": lambda: ir.gemm(1024, 1024, 1024),
    "conv_chain_s": lambda: ir.conv_chain(1, 2, 4, 6, 3, 1, 1),
    "conv_chain_i32": lambda: ir.conv_chain(1, 2, 3, 6, 3, 1, 1, dtype=ir.I32),
    "gmm_chain": lambda: ir.gmm_chain(8, 4, 8),
    "dep_chain": lambda: ir.dep_chain(1, 4, 6, 3, 1, 1),
    "bare_conv_s2": lambda: ir.bare_conv(1, 3, 5, 11, 3, 2),
}


def eval_cases():
    out = []
    for name, mk in GRAPHS.items():
        g = mk()
        bufs = O.random_inputs(g, 42, lib="ref")
        inputs = {t.id: stats(bufs[i]) for i, t in enumerate(g.tensors)
                  if t.role in (ir.INPUT, ir.CONSTANT)}
        O.reference_eval(g, bufs, lib="ref")
        outputs = {n.output: stats(bufs[g.tensor_index(n.output)]) for n in g.nodes}
        out.append({"graph": name, "seed": 42, "inputs": inputs, "outputs": outputs})
    return out


DECODE = [
    ("cfg1_pad_conv", 1, [4, 14, 16, 16, 16, 16], 1),
    ("cfg1_pad_conv", 1, [56, 56, 64, 64, 64, 64], 1),
    ("cfg1_pad_conv", 1, [8, 8, 32, 64, 64, 32], 1),
    ("cfg1_pad_conv", 1, [4, 28, 16, 64, 32, 16, 2, 7, 4], 2),
    ("cfg2_gemm1024", 0, [128, 64, 256], 1),
    ("cfg2_gemm1024", 0, [128, 1024, 64], 1),
    ("cfg2_gemm1024", 0, [1024, 64, 1024], 1),
    ("cfg2_gemm1024", 0, [128, 1024, 1024], 1),
    ("dep_chain", 1, [2, 3, 2, 4, 2], 1),
    ("bare_conv_s2", 0, [1, 5, 5, 3, 1, 5], 1),
]


def decode_cases():
    out = []
    for name, node, factors, levels in DECODE:
        g = GRAPHS[name]()
        seqs = O.ref_decode_layout(g, node, factors, levels)
        out.append({"graph": name, "node": node, "factors": factors, "levels": levels,
                    "seqs": {k: seq_json(v) for k, v in sorted(seqs.items())}})
    return out


def template_cases():
    out = []
    for name, node, levels in [("cfg1_pad_conv", 1, 1), ("cfg1_pad_conv", 1, 2),
                               ("cfg2_gemm1024", 0, 1), ("dep_chain", 1, 1)]:
        g = GRAPHS[name]()
        ext, nd = O.ref_layout_template(g, node, levels)
        out.append({"graph": name, "node": node, "levels": levels, "extents": ext,
                    "ndivisors": nd})
    return out


def interpret_cases():
    """Reference interpret(lower(...)) under template layouts (test_executor.cpp:148-159)."""
    out = []
    g = ir.conv_chain(1, 2, 4, 6, 3, 1, 1)
    seqs = {"conv": [split(1, [2, 2]), reorder([0, 1, 3, 4, 2])],
            "xp": [unfold(2, 5, 3), unfold(4, 5, 3), reorder([0, 2, 4, 1, 3, 5])],
            "ker": [split(0, [2, 2]), reorder([0, 2, 3, 4, 1])]}
    bufs = O.random_inputs(g, 5, lib="ref")
    rc = O.ref_interpret(g, seqs, [], bufs)
    assert rc == 0
    out.append({"graph": "conv_chain_s", "seed": 5,
                "seqs": {k: seq_json(v) for k, v in seqs.items()},
                "outputs": {n.output: stats(bufs[g.tensor_index(n.output)]) for n in g.nodes}})
    return out


def graph_json(g):
    return {"tensors": [{"id": x.id, "dims": [[n, e] for n, e in x.dims], "role": x.role,
                         "dtype": x.dtype} for x in g.tensors],
            "nodes": [{"kind": n.kind, "inputs": list(n.inputs), "output": n.output,
                       "attrs": dict(n.attrs)} for n in g.nodes]}


def two_convs(with_padding=False, h=8, ci=2, co=4):
    """test_propagation.cpp:22-46: two back-to-back C2Ds (optionally with a
    Padding between them)."""
    T, O_ = ir.TensorDecl, ir.OperatorNode
    g = ir.Graph()
    h1 = h - 2
    g.tensors = [T("x", [("N", 1), ("I", ci), ("H", h), ("W", h)], ir.INPUT),
                 T("k1", [("O", co), ("I", ci), ("KH", 3), ("KW", 3)], ir.CONSTANT),
                 T("k2", [("O", co), ("I", co), ("KH", 3), ("KW", 3)], ir.CONSTANT),
                 T("c1", [("N", 1), ("O", co), ("H", h1), ("W", h1)], ir.INTERMEDIATE)]
    if with_padding:
        g.tensors.append(T("c1p", [("N", 1), ("O", co), ("H", h1 + 2), ("W", h1 + 2)], ir.INTERMEDIATE))
        g.tensors.append(T("c2", [("N", 1), ("O", co), ("H", h1), ("W", h1)], ir.OUTPUT))
        g.nodes = [O_(ir.C2D, ["x", "k1"], "c1", {"stride": 1}), O_(ir.PADDING, ["c1"], "c1p", {"pad": 1}),
                   O_(ir.C2D, ["c1p", "k2"], "c2", {"stride": 1})]
    else:
        g.tensors.append(T("c2", [("N", 1), ("O", co), ("H", h1 - 2), ("W", h1 - 2)], ir.OUTPUT))
        g.nodes = [O_(ir.C2D, ["x", "k1"], "c1", {"stride": 1}), O_(ir.C2D, ["c1", "k2"], "c2", {"stride": 1})]
    return g


def with_convert(g, tid, dst_seq, src_seq):
    """The graph insert_conversions (propagation.cpp:265-313) builds for one
    conflicting edge: `tid` keeps src_seq, a LayoutConvert writes
    `<tid>__cv0` in dst_seq for its (last) consumer."""
    import copy
    g2 = copy.deepcopy(g)
    cv = tid + "__cv0"
    src = g2.tensor(tid)
    g2.tensors.append(ir.TensorDecl(cv, list(src.dims), ir.INTERMEDIATE, src.dtype))  # appended, as the reference does
    cons = [i for i, n in enumerate(g2.nodes) if tid in n.inputs][-1]
    g2.nodes[cons].inputs = [cv if x == tid else x for x in g2.nodes[cons].inputs]
    g2.nodes.insert(cons, ir.OperatorNode(ir.LAYOUT_CONVERT, [tid], cv))
    return g2, {tid: src_seq, cv: dst_seq}


def plan_context_cases():
    """LayoutConvert graphs: from the reference planner (claim_operator per
    complex op on decoded template layouts + insert_conversions), and the
    explicit conflicting edge of test_propagation.cpp:140-161 / 187-210,
    each with the reference interpret's outputs; plus the unfold-overhang
    destination for which the reference interpret throws out-of-range
    (interp.cpp:352-359)."""
    out = []
    # (h_t, w_t, o_t, i_t, i'_t, o'_t) per C2D, topological order (space.cpp:60-68)
    planner_cases = [("two_convs", False, 8, [2, 3, 2, 2, 2, 2, 2, 4, 2, 2, 4, 2]),
                     ("two_convs", False, 8, [6, 6, 4, 1, 1, 4, 4, 2, 2, 4, 2, 2]),
                     ("two_convs_pad", True, 8, [3, 2, 2, 2, 2, 2, 2, 3, 4, 4, 2, 4]),
                     ("two_convs", False, 10, [4, 2, 2, 2, 2, 4, 3, 3, 4, 2, 4, 4])]
    for name, pad, h, factors in planner_cases:
        g = two_convs(pad, h)
        g2, seqs = O.ref_plan_context(g, factors)
        n_cv = sum(n.kind == ir.LAYOUT_CONVERT for n in g2.nodes)
        bufs = O.random_inputs(g2, 31, lib="ref")
        rc = O.ref_interpret(g2, seqs, [], bufs)
        assert rc == 0, O.ref().ref_last_error()
        out.append({"name": f"{name}_h{h}", "source": "ref_plan_context", "factors": factors,
                    "graph": graph_json(g2), "seqs": {k: seq_json(v) for k, v in sorted(seqs.items())},
                    "converts": n_cv, "seed": 31, "throws": False,
                    "outputs": {n.output: stats(bufs[g2.tensor_index(n.output)]) for n in g2.nodes}})
    base = two_convs(False, 8)
    src = [split(1, [2, 2]), reorder([0, 1, 3, 4, 2])]
    g2, seqs = with_convert(base, "c1", [unfold(2, 4, 2), unfold(4, 4, 2), reorder([0, 2, 4, 1, 3, 5])], src)
    bufs = O.random_inputs(g2, 31, lib="ref")
    assert O.ref_interpret(g2, seqs, [], bufs) == 0, O.ref().ref_last_error()
    out.append({"name": "explicit_unfold", "source": "test_propagation.cpp:140-210", "graph": graph_json(g2),
                "seqs": {k: seq_json(v) for k, v in sorted(seqs.items())}, "converts": 1, "seed": 31,
                "throws": False,
                "outputs": {n.output: stats(bufs[g2.tensor_index(n.output)]) for n in g2.nodes}})
    # Unfold overhang in a LayoutConvert destination ((D-B) % S != 0): the
    # nest reads the source past its end. Run in a child process: the
    # reference build either throws out-of-range (interp.cpp:352-359) or
    # dies; both are recorded as the reference's outcome.
    for name, gg, sq in overhang_graphs():
        out.append({"name": name, "source": "interp.cpp:352-359 (A7 edge case)", "graph": graph_json(gg),
                    "seqs": {k: seq_json(v) for k, v in sorted(sq.items())}, "converts": 1, "seed": 31,
                    "throws": True, "reference_outcome": reference_outcome(name)})
    return out


def overhang_graphs():
    g = ir.Graph()
    d = [("N", 1), ("C", 4), ("H", 6), ("W", 6)]
    g.tensors = [ir.TensorDecl("x", d, ir.INPUT), ir.TensorDecl("y", d, ir.OUTPUT)]
    g.nodes = [ir.OperatorNode(ir.LAYOUT_CONVERT, ["x"], "y")]
    g2, s2 = with_convert(two_convs(False, 8), "c1",
                          [unfold(2, 3, 2), unfold(4, 3, 2), reorder([0, 2, 4, 1, 3, 5])],
                          [split(1, [2, 2]), reorder([0, 1, 3, 4, 2])])
    return [("convert_overhang_h", g, {"y": [unfold(2, 3, 2)]}),
            ("explicit_overhang", g2, s2)]


def reference_outcome(name):
    import subprocess
    code = ("import sys; sys.path[:0]=%r; import gen_golden as G, oracle_lib as O\n"
            "g, s = [(gg, sq) for n, gg, sq in G.overhang_graphs() if n == %r][0]\n"
            "b = O.random_inputs(g, 31, lib='ref'); rc = O.ref_interpret(g, s, [], b)\n"
            "print('rc=%%d %%s' %% (rc, O.ref().ref_last_error().decode()))") % (
        [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")], name)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    if r.returncode < 0:
        return "reference process died (signal %d) inside interpret" % -r.returncode
    return r.stdout.strip().splitlines()[-1] if r.stdout.strip() else "rc=%d" % r.returncode


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libref.so missing: run `make -C oracle` where "
                         "/root/reference exists")
    os.makedirs(OUT, exist_ok=True)
    data = {
        "generator": "oracle/gen_golden.py over oracle/_ref/libref.so (reference sources "
                     "compiled unmodified)",
        "checksum": "FNV-1a 64 over little-endian fp32 bytes, buffer order",
        "materialize": materialize_cases(),
        "reference_eval": eval_cases(),
        "decode_layout": decode_cases(),
        "layout_template": template_cases(),
        "interpret": interpret_cases(),
        "plan_context": plan_context_cases(),
    }
    with open(os.path.join(OUT, "reference_golden.json"), "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "reference_golden.json"))


if __name__ == "__main__":
    main()
