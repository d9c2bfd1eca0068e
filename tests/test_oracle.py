"""The oracle (oracle/lf_oracle.c) pinned against the reference.

Two anchors: the golden vectors generated from the
compiled reference (tests/golden/reference_golden.json, oracle/gen_golden.py)
and — where /root/reference was built here — direct cross-checks against
oracle/_ref/libref.so on fresh random cases.
"""
import numpy as np
import pytest

import oracle_lib as O
from paper_2210_12415_b200 import ir
from paper_2210_12415_b200.layout import LayoutPrimitive, fuse, padding, reorder, split, store_at, unfold

GRAPHS = {
    "cfg1_pad_conv": lambda: ir.pad_conv(1, 64, 64, 56, 3, 1, 1),
    "cfg2_gemm1024": lambda: ir.gemm(1024, 1024, 1024),
    "conv_chain_s": lambda: ir.conv_chain(1, 2, 4, 6, 3, 1, 1),
    "conv_chain_i32": lambda: ir.conv_chain(1, 2, 3, 6, 3, 1, 1, dtype=ir.I32),
    "gmm_chain": lambda: ir.gmm_chain(8, 4, 8),
    "dep_chain": lambda: ir.dep_chain(1, 4, 6, 3, 1, 1),
    "bare_conv_s2": lambda: ir.bare_conv(1, 3, 5, 11, 3, 2),
}


def seq_from(js):
    return [LayoutPrimitive(kind=p["kind"], dim=p["dim"], factors=p["factors"], perm=p["perm"],
                            span=p["span"], tile=p["tile"], stride=p["stride"], pad=p["pad"],
                            target=p["target"]) for p in js]


def src_for(case):
    if "src_values" in case:
        return np.array(case["src_values"])
    rng = np.random.default_rng(case["src_seed"])
    return np.round(rng.uniform(-1, 1, int(np.prod(case["extents"]))) * 64) / 64


def test_unfold_known_answer():
    # acceptance.cpp:291-305: {1,2,3,4,5} unfolds (B=3, S=2) to {1,2,3,3,4,5}.
    got = O.materialize([5], [unfold(0, 3, 2)], np.arange(1, 6, dtype=np.float64))
    assert list(got) == [1, 2, 3, 3, 4, 5]


def test_golden_materialize(golden):
    for case in golden["materialize"]:
        seq = seq_from(case["seq"])
        src = src_for(case)
        assert O.fnv1a(src) == case["src"]["fnv"], case["name"]
        assert O.derive(case["extents"], seq) == case["phys"], case["name"]
        got = O.materialize(case["extents"], seq, src)
        assert O.fnv1a(got) == case["out"]["fnv"], case["name"]
        if "values" in case:
            assert [float(x) for x in got] == case["values"], case["name"]


def test_golden_reference_eval(golden):
    for case in golden["reference_eval"]:
        g = GRAPHS[case["graph"]]()
        bufs = O.random_inputs(g, case["seed"])
        for tid, st in case["inputs"].items():
            b = bufs[g.tensor_index(tid)]
            assert O.fnv1a(b) == st["fnv"], (case["graph"], tid)
            assert float(b.sum()) == st["sum"]
        O.reference_eval(g, bufs)
        for tid, st in case["outputs"].items():
            b = bufs[g.tensor_index(tid)]
            assert O.fnv1a(b) == st["fnv"], (case["graph"], tid)


def test_cfg1_known_values():
    # first inputs / outputs of cfg1 at seed 42.
    g = GRAPHS["cfg1_pad_conv"]()
    bufs = O.random_inputs(g, 42)
    assert list(bufs[0][:3]) == [0.515625, 0.28125, 0.5]
    assert float(bufs[0].sum()) == -69.375
    assert float(bufs[1].sum()) == 204.546875
    O.reference_eval(g, bufs)
    y = bufs[3]
    assert abs(y[0] - -10.821) < 1e-3 and abs(y[1] - -3.83545) < 1e-4
    assert abs(float(y.sum()) - 2107.810547) < 1e-5


def test_to_logical_inverts_materialize():
    rng = np.random.default_rng(3)
    for ext, seq in [([2, 8, 5, 7], [split(1, [2, 4]), reorder([0, 1, 3, 4, 2])]),
                     ([1, 3, 10, 10], [unfold(2, 6, 4), unfold(4, 6, 4),
                                       reorder([0, 2, 4, 1, 3, 5])]),
                     ([2, 3, 3, 8], [fuse(1, 3), split(1, [2, 4, 9]), reorder([0, 1, 3, 2])])]:
        x = rng.standard_normal(int(np.prod(ext)))
        phys = O.materialize(ext, seq, x)
        assert np.array_equal(O.to_logical(ext, seq, phys), x)


def test_padding_nest_zero_overhang():
    # The Padding nest writes 0 outside the interior and in unfold overhang
    # (lower.cpp:228-238), where materialization would clamp.
    x = np.arange(1, 1 + 1 * 1 * 4 * 4, dtype=np.float64)
    dst = [unfold(2, 3, 2)]  # Hp = 6 -> tiles 3, last tile covers 4..6 (overhang 1)
    rc, got = O.padding_nest([1, 1, 4, 4], 1, [], dst, x)
    assert rc == 0
    got = got.reshape(3, 3, 6)
    assert np.all(got[2, 2, :] == 0)  # row 6 does not exist
    xp = np.zeros((6, 6))
    xp[1:5, 1:5] = x.reshape(4, 4)
    assert np.array_equal(got[0], xp[0:3])
    assert np.array_equal(got[1], xp[2:5])


@pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) absent")
class TestAgainstReference:
    def test_random_inputs_bitwise(self):
        for g in [GRAPHS["cfg1_pad_conv"](), GRAPHS["conv_chain_i32"](), ir.gmm_chain(5, 7, 3)]:
            for seed in (0, 1, 42, 12345):
                a = O.random_inputs(g, seed)
                b = O.random_inputs(g, seed, lib="ref")
                for i in range(len(a)):
                    assert np.array_equal(a[i], b[i])

    def test_reference_store_at_rules(self):
        """Pins the store_at semantics the GPU plan mirrors (lower.cpp:32-82):
        an accepted attachment leaves values unchanged (test_executor.cpp:
        196-201); rejected ones carry the messages test_gpu_plan.py expects."""
        g = ir.gmm_chain(256, 128, 256)
        ok = [{"bias": [store_at("b", 0)]},
              {"b": [split(1, [2, 128]), reorder([1, 0, 2])], "bias": [store_at("b", 0)]}]
        bad = [({"a": [store_at("b", 0)]}, "store_at on non-constant tensor 'a'"),
               ({"bias": [store_at("b", 0), split(0, [2, 128])]},
                "store_at must be the final primitive"),
               ({"bias": [split(0, [4, 64]), store_at("b", 0)]},
                "store_at: source must match target with one dim removed"),
               ({"bias": [store_at("nope", 0)]}, "store_at target"),
               ({"bias": [store_at("b", 2)]}, "store_at: dim out of range"),
               ({"bias": [store_at("b", 0)], "b": [split(0, [2, 64])]}, "dim K has extent 129")]
        want = O.random_inputs(g, 8)
        O.reference_eval(g, want)
        for seqs in ok:
            bufs = O.random_inputs(g, 8)
            assert O.ref_interpret(g, seqs, [], bufs) == 0, O.ref().ref_last_error()
            y = g.tensor_index("y")
            assert np.array_equal(bufs[y], want[y])
        for seqs, msg in bad:
            assert O.ref_interpret(g, seqs, [], O.random_inputs(g, 8)) != 0
            assert msg in O.ref().ref_last_error().decode(), O.ref().ref_last_error()

    def test_materialize_fuzz(self):
        rng = np.random.default_rng(11)
        n = 0
        while n < 150:
            rank = int(rng.integers(1, 4))
            ext = [int(rng.integers(1, 7)) for _ in range(rank)]
            seq, cur = [], list(ext)
            for _ in range(int(rng.integers(1, 4))):
                k = int(rng.integers(0, 5))
                d = int(rng.integers(0, len(cur)))
                if k == 0 and cur[d] > 1:
                    divs = [f for f in range(1, cur[d] + 1) if cur[d] % f == 0]
                    f = int(rng.choice(divs))
                    p = split(d, [cur[d] // f, f])
                elif k == 1:
                    p = reorder(list(rng.permutation(len(cur))))
                elif k == 2 and len(cur) > 1 and d + 1 < len(cur):
                    p = fuse(d, 2)
                elif k == 3:
                    b = int(rng.integers(1, cur[d] + 1))
                    s = int(rng.integers(1, b + 1))
                    p = unfold(d, b, s)
                else:
                    p = padding(d, int(rng.integers(0, 3)))
                try:
                    cur = O.derive(cur, [p])
                except ValueError:
                    continue
                seq.append(p)
            x = rng.integers(-64, 64, int(np.prod(ext))) / 64.0
            a = O.materialize(ext, seq, x)
            b = O.materialize(ext, seq, x, lib="ref")
            assert np.array_equal(a, b), (ext, seq)
            n += 1

    def test_reference_eval_micrographs(self):
        for g in [ir.conv_chain(2, 3, 4, 7, 3, 2, 1), ir.dep_chain(1, 3, 7, 3, 2, 1),
                  ir.gmm_chain(6, 5, 4), ir.bare_conv(1, 2, 3, 9, 3, 1)]:
            a = O.random_inputs(g, 9)
            b = [x.copy() for x in a]
            O.reference_eval(g, a)
            O.reference_eval(g, b, lib="ref")
            for i in range(len(a)):
                assert np.array_equal(a[i], b[i])

    def test_padding_nest_matches_interpret(self):
        # The reference interpret of Padding on an unfolded output layout,
        # converted back to logical, equals the oracle's nest -> to_logical.
        g = ir.Graph()
        g.tensors = [ir.TensorDecl("x", [("N", 1), ("C", 2), ("H", 5), ("W", 5)], ir.INPUT),
                     ir.TensorDecl("xp", [("N", 1), ("C", 2), ("H", 7), ("W", 7)], ir.OUTPUT)]
        g.nodes = [ir.OperatorNode(ir.PADDING, ["x"], "xp", {"pad": 1})]
        seqs = {"xp": [unfold(2, 3, 2), unfold(4, 5, 3), reorder([0, 2, 4, 1, 3, 5])]}
        bufs = O.random_inputs(g, 4, lib="ref")
        x = bufs[0].copy()
        assert O.ref_interpret(g, seqs, [], bufs) == 0
        rc, phys = O.padding_nest([1, 2, 5, 5], 1, [], seqs["xp"], x)
        assert rc == 0
        assert np.array_equal(O.to_logical([1, 2, 7, 7], seqs["xp"], phys), bufs[1])


def test_oracle_matches_reference_planner_graphs(golden):
    # LayoutConvert graphs from the reference planner (oracle/gen_golden.py
    # plan_context): the oracle's reference_eval reproduces the reference
    # interpret's logical outputs (a LayoutConvert is the identity on
    # logical values, interp.cpp:166-169).
    from test_gpu_parity import _graph_from
    n = 0
    for c in golden["plan_context"]:
        if c["throws"]:
            assert "signal" in c["reference_outcome"] or "out-of-range" in c["reference_outcome"]
            continue
        g = _graph_from(c["graph"])
        bufs = O.random_inputs(g, c["seed"])
        O.reference_eval(g, bufs)
        for tid, st in c["outputs"].items():
            assert O.fnv1a(bufs[g.tensor_index(tid)]) == st["fnv"], (c["name"], tid)
            n += 1
    assert n >= 10


# ---- BERT-encoder op-set extension (lfgpu.h LFGPU_OP_GELU .. BMM_PV): the
# reference has no such ops (ir.hpp:42), so the oracle's restatement is
# checked against an independent numpy formulation of lfgpu.h's semantics.
def _run_oracle(g, seed=5):
    bufs = O.random_inputs(g, seed)
    O.reference_eval(g, bufs)
    return {t.id: bufs[i] for i, t in enumerate(g.tensors)}


def _graph(tensors, nodes):
    g = ir.Graph()
    g.tensors = [ir.TensorDecl(tid, dims, role) for tid, dims, role in tensors]
    g.nodes = [ir.OperatorNode(*n) for n in nodes]
    return g


def test_oracle_encoder_ops_match_numpy():
    import math
    T, H, Dh = 6, 2, 4
    D = H * Dh
    g = _graph([("q", [("M", T), ("N", D)], ir.INPUT), ("k", [("M", T), ("N", D)], ir.INPUT),
                ("v", [("M", T), ("N", D)], ir.INPUT), ("gb", [("P", 2), ("N", D)], ir.CONSTANT),
                ("s", [("H", H), ("M", T), ("T", T)], ir.INTERMEDIATE),
                ("p", [("H", H), ("M", T), ("T", T)], ir.INTERMEDIATE),
                ("c", [("M", T), ("N", D)], ir.INTERMEDIATE), ("n", [("M", T), ("N", D)], ir.INTERMEDIATE),
                ("y", [("M", T), ("N", D)], ir.OUTPUT)],
               [(ir.BMM_QK, ["q", "k"], "s", {"heads": H}), (ir.SOFTMAX, ["s"], "p"),
                (ir.BMM_PV, ["p", "v"], "c", {"heads": H}), (ir.LAYERNORM, ["c", "gb"], "n", {"eps_exp": 5}),
                (ir.GELU, ["n"], "y")])
    b = _run_oracle(g)
    q, k, v = (b[x].reshape(T, H, Dh) for x in "qkv")
    s = np.einsum("ihd,jhd->hij", q, k)
    assert np.allclose(b["s"].reshape(H, T, T), s, rtol=1e-13, atol=1e-13)
    e = np.exp(s - s.max(-1, keepdims=True))
    p = e / e.sum(-1, keepdims=True)
    assert np.allclose(b["p"].reshape(H, T, T), p, rtol=1e-13, atol=1e-13)
    c = np.einsum("hij,jhd->ihd", p, v).reshape(T, D)
    assert np.allclose(b["c"].reshape(T, D), c, rtol=1e-13, atol=1e-13)
    gb = b["gb"].reshape(2, D)
    mu, var = c.mean(-1, keepdims=True), c.var(-1, keepdims=True)
    n = (c - mu) / np.sqrt(var + 1e-5) * gb[0] + gb[1]
    assert np.allclose(b["n"].reshape(T, D), n, rtol=1e-12, atol=1e-12)
    y = 0.5 * n * (1.0 + np.vectorize(math.erf)(n / math.sqrt(2.0)))
    assert np.allclose(b["y"].reshape(T, D), y, rtol=1e-12, atol=1e-12)


def test_oracle_packed_qkv_slices_match_numpy():
    """BmmQK / BmmPV on column slices of one packed [T, 3*H*Dh] operand
    (a_col0 / b_col0 / head_dim) equal the unpacked ops on the slices."""
    T, H, Dh = 5, 2, 4
    D = H * Dh
    g = _graph([("qkv", [("M", T), ("N", 3 * D)], ir.INPUT),
                ("s", [("H", H), ("M", T), ("T", T)], ir.INTERMEDIATE),
                ("c", [("M", T), ("N", D)], ir.OUTPUT)],
               [(ir.BMM_QK, ["qkv", "qkv"], "s", {"heads": H, "a_col0": 0, "b_col0": D, "head_dim": Dh}),
                (ir.BMM_PV, ["s", "qkv"], "c", {"heads": H, "b_col0": 2 * D, "head_dim": Dh})])
    b = _run_oracle(g)
    x = b["qkv"].reshape(T, 3 * D)
    q, k, v = (x[:, i * D:(i + 1) * D].reshape(T, H, Dh) for i in range(3))
    s = np.einsum("ihd,jhd->hij", q, k)
    assert np.allclose(b["s"].reshape(H, T, T), s, rtol=1e-13, atol=1e-13)
    c = np.einsum("hij,jhd->ihd", s, v).reshape(T, D)
    assert np.allclose(b["c"].reshape(T, D), c, rtol=1e-13, atol=1e-13)
    # out-of-range slices are rejected (the planner's EINVAL, lf_runtime.cpp)
    g.nodes[0].attrs["b_col0"] = 2 * D + 1
    with pytest.raises(Exception):
        _run_oracle(g)
