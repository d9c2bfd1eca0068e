"""Whole-graph execution on the GPU (interpret / plans / measure) against the
oracle's reference_eval, and the tcgen05 contractions on tuned layouts.

Tolerances (proj/src/cli.cpp:30-49): int32 exact; float
1e-5 relative with scale max(1,|a|,|b|). Contractions whose operands are the
reference's k/64 inputs are bit-exact on tensor cores (bf16 products are
exact, fp32 partial sums stay exact for K <= 4096), so those are checked
with ==.
"""
import numpy as np
import pytest

import oracle_lib as O
from paper_2210_12415_b200 import _abi, ir, runtime
from paper_2210_12415_b200.layout import reorder, split, store_at, unfold

pytestmark = pytest.mark.gpu


def oracle_outputs(g, seed):
    bufs = O.random_inputs(g, seed)
    inputs = {t.id: bufs[i].copy() for i, t in enumerate(g.tensors)
              if t.role in (ir.INPUT, ir.CONSTANT)}
    O.reference_eval(g, bufs)
    ref = {n.output: bufs[g.tensor_index(n.output)] for n in g.nodes}
    return inputs, ref


def tol_of(g, tid):
    return 0.0 if g.tensor(tid).dtype == ir.I32 else 1e-5


def check(g, got, ref, exact=False):
    for tid, want in ref.items():
        d = O.max_rel_diff(got[tid], want)
        assert d <= (0.0 if exact else tol_of(g, tid)), (tid, d)


def test_interpret_template_layouts_golden(golden):
    # test_executor.cpp:148-159 via the reference's own interpret output.
    case = golden["interpret"][0]
    g = ir.conv_chain(1, 2, 4, 6, 3, 1, 1)
    from test_oracle import seq_from
    seqs = {k: seq_from(v) for k, v in case["seqs"].items()}
    bufs = O.random_inputs(g, case["seed"])
    inputs = {t.id: bufs[i] for i, t in enumerate(g.tensors) if t.role in (ir.INPUT, ir.CONSTANT)}
    got = runtime.interpret(g, seqs, [], inputs, flags=_abi.PLAN_EXACT)
    for tid, st in case["outputs"].items():
        assert O.fnv1a(got[tid]) == st["fnv"], tid


MICRO = [
    lambda: ir.conv_chain(1, 2, 4, 6, 3, 1, 1),
    lambda: ir.conv_chain(2, 3, 5, 8, 3, 2, 1),
    lambda: ir.conv_chain(1, 2, 3, 6, 3, 1, 1, dtype=ir.I32),
    lambda: ir.dep_chain(1, 4, 6, 3, 1, 1),
    lambda: ir.gmm_chain(8, 4, 8),
    lambda: ir.bare_conv(1, 3, 5, 11, 3, 2),
]


@pytest.mark.parametrize("flags", [_abi.PLAN_EXACT, _abi.PLAN_DEFAULT, _abi.PLAN_TENSOR_CORES])
def test_interpret_micrographs_identity(flags):
    # PLAN_DEFAULT in lfgpu_interpret means reference semantics (EXACT);
    # PLAN_TENSOR_CORES opts into the tcgen05 paths where they are legal.
    for mk in MICRO:
        g = mk()
        inputs, ref = oracle_outputs(g, 17)
        got = runtime.interpret(g, {}, [], inputs, flags=flags)
        check(g, got, ref)


def test_interpret_fuzz_template_layouts():
    # test_executor.cpp:413-440: random template layouts through decode_layout.
    rng = np.random.default_rng(23)
    for it in range(60):
        which = it % 3
        if which == 0:
            g = ir.conv_chain(1, 1 + int(rng.integers(0, 3)), 2 + int(rng.integers(0, 3)),
                              4 + 2 * int(rng.integers(0, 3)), 3, 1 + int(rng.integers(0, 2)), 1)
        elif which == 1:
            g = ir.dep_chain(1, 2 + int(rng.integers(0, 3)), 6, 3, 1, 1)
        else:
            g = ir.gmm_chain(4 + 4 * int(rng.integers(0, 2)), 4, 4 + 4 * int(rng.integers(0, 2)))
        seqs = {}
        for node, n in enumerate(g.nodes):
            if not ir.is_complex_op(n.kind):
                continue
            t = runtime.layout_template(g, node)
            factors = []
            for _, e in t:
                divs = [d for d in range(1, e + 1) if e % d == 0]
                factors.append(int(rng.choice(divs)))
            seqs.update(runtime.decode_layout(g, node, factors))
        inputs, ref = oracle_outputs(g, 1000 + it)
        got = runtime.interpret(g, seqs, [], inputs, flags=_abi.PLAN_EXACT)
        check(g, got, ref)


def gemm_case(M, K, N, factors):
    g = ir.gemm(M, K, N)
    seqs = runtime.decode_layout(g, 0, factors) if factors else {}
    inputs, ref = oracle_outputs(g, 42)
    return g, seqs, inputs, ref


@pytest.mark.parametrize("factors", [(128, 64, 128), (128, 64, 256), (256, 128, 64),
                                     (128, 512, 64), None, (64, 64, 64)])
def test_umma_gemm_bitexact(factors):
    M = K = N = 512
    g, seqs, inputs, ref = gemm_case(M, K, N, factors)
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    assert p.node_kernel(0).startswith("umma_gemm"), p.node_kernel(0)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("c")
    assert np.array_equal(got, ref["c"]), np.abs(got - ref["c"]).max()


def test_umma_gemm_cfg2_1024():
    g, seqs, inputs, ref = gemm_case(1024, 1024, 1024, (128, 64, 128))
    got = runtime.interpret(g, seqs, [runtime.sched(0, tile_last=64)], inputs, flags=_abi.PLAN_TENSOR_CORES)
    assert np.array_equal(got["c"], ref["c"])


def test_umma_gemm_mn_major_a_and_k_major_b():
    # m-only split: A becomes (M/m_t) K m_t (M-contiguous); k-only split on B
    # gives (K/k_t) N k_t (K-contiguous B).
    g = ir.gemm(256, 256, 256)
    seqs = {"a": [split(0, [2, 128]), reorder([0, 2, 1])],
            "b": [split(0, [4, 64]), reorder([0, 2, 1])]}
    inputs, ref = oracle_outputs(g, 3)
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("c"), ref["c"])


# (h_t, w_t, o_t, i_t, i'_t, o'_t). i_t < I keeps the channel brick innermost
# (space.cpp:322-337), which the K-major A operand needs.
CONV_FACTORS = [
    (4, 28, 16, 32, 32, 16),   # 112 rows, KC=32 (64 B swizzle), o'=16 (32 B)
    (4, 14, 16, 16, 16, 16),   # SURVEY's example point: 56 rows, KC=16
    (8, 8, 32, 32, 32, 32),    # 64 rows
    (2, 56, 64, 32, 32, 64),   # untiled W outside the H tile: (w, h) row order
    (4, 28, 32, 16, 32, 32),   # i_t != i'_t: KC = gcd = 16
]


@pytest.mark.parametrize("factors", CONV_FACTORS)
def test_umma_conv_cfg1_bitexact(factors):
    g = ir.pad_conv(1, 64, 64, 56, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(factors))
    inputs, ref = oracle_outputs(g, 42)
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    assert p.node_kernel(1).startswith("umma_conv"), p.node_kernel(1)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("xp"), ref["xp"])
    y = p.get_output("y")
    assert np.array_equal(y, ref["y"]), np.abs(y - ref["y"]).max()


def test_umma_conv_stride2_batch():
    g = ir.pad_conv(2, 64, 64, 28, 3, 2, 1)  # Ho = 14, untiled W
    seqs = runtime.decode_layout(g, 1, [7, 14, 32, 32, 32, 32])
    inputs, ref = oracle_outputs(g, 4)
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("y"), ref["y"])


def test_fused_epilogue_conv_chain():
    # Padding -> C2D -> BiasAdd -> ReLU with the C2D schedule's fuse flag:
    # bias and relu run in the tcgen05 epilogue (lower.cpp:566-608).
    g = ir.conv_chain(1, 64, 64, 56, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, [4, 28, 16, 32, 32, 16])
    for t in ("biased", "y"):
        seqs[t] = seqs["conv"]
    inputs, ref = oracle_outputs(g, 42)
    p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1)], flags=_abi.PLAN_REQUIRE_TC)
    assert p.node_kernel(2) == "fused" and p.node_kernel(3) == "fused"
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("y"), ref["y"])
    with pytest.raises(runtime.LfError):
        p.get_output("conv")  # fused away, never materialized


def test_require_tc_rejects_illegal_layout():
    g = ir.pad_conv(1, 3, 8, 10, 3, 1, 1)
    with pytest.raises(runtime.LfError) as e:
        runtime.Plan(g, {}, [], flags=_abi.PLAN_REQUIRE_TC)
    assert e.value.code == _abi.EUNSUPPORTED


def test_measure_reports_device_time():
    g = ir.pad_conv(1, 64, 64, 56, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, [4, 28, 16, 32, 32, 16])
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_CUDA_GRAPH)
    inputs, _ = oracle_outputs(g, 42)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    c = p.measure(warmup=3, reps=20, flush_l2=True)
    assert c.cost > 0 and c.min_us <= c.cost and c.kernels == 2 and c.tc_nodes == 1
    assert c.flops == 2 * 64 * 64 * 56 * 56 * 9


# Epilogue variants of the tcgen05 kernel: the TMA-store epilogue (schedule
# `vectorize`=1), split-K with the distributed column-slice reduction
# (`order`), fused bias/ReLU chains, on GEMM and on the halo C2D path.
@pytest.mark.parametrize("factors,tile,order,vec", [
    ((128, 64, 256), 64, 1, 1), ((128, 64, 256), 128, 0, 1), ((128, 64, 256), 256, 0, 1),
    ((256, 128, 128), 128, 2, 0), ((128, 64, 128), 64, 0, 1)])
@pytest.mark.parametrize("one_cta", [1, 0])
def test_umma_gemm_epilogue_variants(factors, tile, order, vec, one_cta, monkeypatch):
    # one_cta=1 pins the 1-CTA kernel (its TMA-store / split-K epilogues);
    # one_cta=0 lets the planner take the CTA-pair kernel (k_pair.cu).
    if one_cta:
        monkeypatch.setenv("LFGPU_NO_PAIR", "1")
    M = K = N = 512
    g = ir.gmm_chain(M, K, N)
    seqs = runtime.decode_layout(g, 0, list(factors))
    seqs["biased"] = seqs["c"]
    seqs["y"] = seqs["c"]
    inputs, ref = oracle_outputs(g, 11)
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=tile, order=order, vectorize=vec, fuse=1)],
                     flags=_abi.PLAN_REQUIRE_TC)
    k = p.node_kernel(0)
    assert k.startswith("umma_gemm"), k
    # An N-major B half needs >= 64 columns: tile 64 stays on the 1-CTA kernel.
    assert ("gemm-pair" in k) == (not one_cta and tile >= 128), k
    if vec and one_cta:
        assert "store=2" in k, k
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("y")
    assert np.array_equal(got, ref["y"]), np.abs(got - ref["y"]).max()


@pytest.mark.parametrize("f,vec", [((8, 14, 64, 32, 32, 64), 1), ((7, 14, 32, 32, 32, 32), 1),
                                   ((14, 14, 64, 64, 64, 64), 0), ((28, 28, 64, 32, 32, 64), 1),
                                   ((28, 28, 32, 32, 32, 32), 1)])
def test_halo_conv_tma_store(f, vec):
    n, c, h = (1, 64, 56) if f[0] != 14 else (1, 256, 14)
    g = ir.pad_conv(n, c, 64 if c == 64 else c, h, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(f))
    inputs, ref = oracle_outputs(g, 5)
    p = runtime.Plan(g, seqs, [runtime.sched(1, vectorize=vec)], flags=_abi.PLAN_REQUIRE_TC)
    k = p.node_kernel(1)
    assert "conv-halo" in k, k
    if f[1] == 28 and vec:  # w-innermost output: transposed TMA-store box (112-byte rows)
        assert "store=2" in k, k
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("y")
    assert np.array_equal(got, ref["y"]), np.abs(got - ref["y"]).max()


def test_transposed_tma_store_fused_chain():
    """Padding -> C2D -> BiasAdd -> ReLU with a w-innermost output: the
    fused chain runs before the transposed TMA-store staging."""
    g = ir.conv_chain(2, 64, 64, 56, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, [28, 28, 64, 32, 32, 64])
    for t in ("biased", "y"):
        seqs[t] = seqs["conv"]
    inputs, ref = oracle_outputs(g, 21)
    p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1, vectorize=1)], flags=_abi.PLAN_REQUIRE_TC)
    assert "store=2" in p.node_kernel(1), p.node_kernel(1)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("y"), ref["y"])


@pytest.mark.parametrize("shape,f", [((1, 512, 512, 7), (7, 7, 128, 64, 64, 128)),
                                     ((1, 64, 128, 7), (7, 7, 128, 32, 32, 128)),
                                     ((1, 128, 128, 14), (14, 14, 128, 64, 64, 128))])
def test_halo_conv_channels_as_rows(shape, f):
    """Schedule unroll=2: output channels are the 128 UMMA rows and the
    tile's pixels the N columns (weights = A, shifted input tile = B)."""
    n, c, o, h = shape
    g = ir.pad_conv(n, c, o, h, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(f))
    inputs, ref = oracle_outputs(g, 9)
    p = runtime.Plan(g, seqs, [runtime.sched(1, unroll=2)], flags=_abi.PLAN_REQUIRE_TC)
    assert "conv-halo-trans" in p.node_kernel(1), p.node_kernel(1)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("y")
    assert np.array_equal(got, ref["y"]), np.abs(got - ref["y"]).max()


def _store_at_cases(g):
    t = runtime.decode_layout(g, 0, [128, 64, 128])
    return {
        "plain": {"bias": [store_at("b", 0)]},
        "b_split_n": {"a": t["a"], "c": t["c"], "b": [split(1, [2, 128]), reorder([1, 0, 2])],
                      "bias": [store_at("b", 0)]},
    }


@pytest.mark.parametrize("case", ["plain", "b_split_n"])
@pytest.mark.parametrize("fuse", [0, 1])
def test_store_at_gmm_bias(case, fuse):
    """test_executor.cpp:196-201 at tensor-core size: bias store_at-attached
    to the weights runs like the unfused graph (lower.cpp:32-82 folds it
    offline; the attachment co-locates storage, values are unchanged)."""
    g = ir.gmm_chain(256, 128, 256)
    seqs = _store_at_cases(g)[case]
    inputs, ref = oracle_outputs(g, 8)
    p = runtime.Plan(g, seqs, [runtime.sched(0, fuse=fuse)], flags=_abi.PLAN_REQUIRE_TC)
    assert p.node_kernel(0).startswith("umma_gemm"), p.node_kernel(0)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("y"), ref["y"])


@pytest.mark.parametrize("seqs,msg", [
    # messages are the reference's own (checked against oracle/_ref in
    # test_oracle.py::test_reference_store_at_rules)
    ({"a": [store_at("b", 0)]}, "store_at on non-constant tensor 'a'"),
    ({"bias": [store_at("b", 0), split(0, [2, 128])]}, "store_at must be the final primitive"),
    ({"bias": [split(0, [4, 64]), store_at("b", 0)]},
     "store_at: source must match target with one dim removed"),
    ({"bias": [store_at("nope", 0)]}, "store_at target"),
    ({"bias": [store_at("b", 2)]}, "store_at: dim out of range"),
    ({"bias": [store_at("b", 0)], "b": [split(0, [2, 64])]}, "dim K has extent 129"),
])
def test_store_at_rules(seqs, msg):
    g = ir.gmm_chain(256, 128, 256)
    with pytest.raises(runtime.LfError) as e:
        runtime.Plan(g, seqs, [])
    assert e.value.code == _abi.EINVAL and msg in str(e.value), str(e.value)


@pytest.mark.parametrize("shape,f,fuse", [
    ((2, 64, 28, 3, 1), None, 0),                    # logical NCHW: W is the fast dim
    ((2, 64, 28, 3, 1), (7, 14, 32, 32, 32), 1),     # channel bricks, ReLU fused
    ((1, 96, 27, 5, 2), (7, 7, 32, 32, 32), 1),      # 5x5 stride 2 (14x14 output)
    ((1, 96, 27, 3, 2), (7, 7, 32, 32, 32), 1),      # 3x3 stride 2: rolling-window kernel, V = 2
    ((2, 64, 30, 3, 1), (10, 15, 32, 32, 32), 0),    # 3x3: row blocks of 8 over 30 rows (ragged)
    ((1, 32, 14, 7, 1), (14, 14, 16, 16, 16), 0),    # 7x7
    ((1, 48, 10, 4, 1), None, 1),                    # even window: the generic-K path
])
def test_dep_direct(shape, f, fuse):
    """K6: DEP (interp.cpp:90-108) on its template layouts (space.cpp:76-90)
    through the per-dim offset tables, against reference_eval."""
    n, c, h, k, s = shape
    g = ir.dep_chain(n, c, h, k, s, k // 2)
    seqs = {}
    if f is not None:
        # Every parametrized point is a legal template point: a decode
        # failure is a regression, not a skip.
        seqs = runtime.decode_layout(g, 1, list(f))
        seqs["y"] = seqs["conv"]
    inputs, ref = oracle_outputs(g, 13)
    p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=fuse)])
    assert p.node_kernel(1).startswith("dep_direct"), p.node_kernel(1)
    # K = 3 channel-brick points run the rolling-window variant of dep_direct4
    if f is not None and c % 4 == 0 and f[4] % 4 == 0:
        assert p.node_kernel(1) == "dep_direct4", p.node_kernel(1)
    if fuse:
        assert p.node_kernel(2) == "fused"
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("y")
    assert np.array_equal(got, ref["y"]), O.max_rel_diff(got, ref["y"])


def _dep_residual_graph(n, c, h):
    """Padding -> DEP 3x3 -> BiasAdd -> EwAdd(skip) -> ReLU: every epilogue
    kind the K6 kernel fuses (bias per channel, residual in the output
    layout, ReLU)."""
    g = ir.Graph()
    d4 = [("N", n), ("C", c), ("H", h), ("W", h)]
    g.tensors = [
        ir.TensorDecl("x", d4, ir.INPUT),
        ir.TensorDecl("ker", [("C", c), ("KH", 3), ("KW", 3)], ir.CONSTANT),
        ir.TensorDecl("bias", [("C", c)], ir.CONSTANT),
        ir.TensorDecl("skip", d4, ir.INPUT),
        ir.TensorDecl("xp", [("N", n), ("C", c), ("H", h + 2), ("W", h + 2)], ir.INTERMEDIATE),
        ir.TensorDecl("conv", d4, ir.INTERMEDIATE),
        ir.TensorDecl("biased", d4, ir.INTERMEDIATE),
        ir.TensorDecl("summed", d4, ir.INTERMEDIATE),
        ir.TensorDecl("y", d4, ir.OUTPUT),
    ]
    g.nodes = [
        ir.OperatorNode(ir.PADDING, ["x"], "xp", {"pad": 1}),
        ir.OperatorNode(ir.DEP, ["xp", "ker"], "conv", {"stride": 1}),
        ir.OperatorNode(ir.BIASADD, ["conv", "bias"], "biased"),
        ir.OperatorNode(ir.EWADD, ["biased", "skip"], "summed"),
        ir.OperatorNode(ir.RELU, ["summed"], "y"),
    ]
    return g


@pytest.mark.parametrize("brick", [None, 16])
def test_dep_direct_fused_bias_residual(brick):
    g = _dep_residual_graph(2, 64, 28)
    seqs = {}
    if brick:
        seqs = runtime.decode_layout(g, 1, [14, 14, brick, brick, brick])
        for t in ("biased", "summed", "y", "skip"):
            seqs[t] = seqs["conv"]
    inputs, ref = oracle_outputs(g, 29)
    p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1)])
    assert p.node_kernel(1).startswith("dep_direct"), p.node_kernel(1)
    assert all(p.node_kernel(i) == "fused" for i in (2, 3, 4)), [p.node_kernel(i) for i in range(5)]
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("y"), ref["y"])


@pytest.mark.parametrize("knobs", [{}, {"LFGPU_NO_EPI_ALIAS": "1"}, {"LFGPU_DUAL_MMA": "1"},
                                   {"LFGPU_DUAL_MMA": "0"}, {"LFGPU_NO_EPI_ALIAS": "1", "LFGPU_DUAL_MMA": "1"},
                                   {"LFGPU_DUAL_MMA": "2"}])
@pytest.mark.parametrize("case", ["conv", "gemm"])
def test_umma_epilogue_alias_and_dual_issuer_parity(case, knobs, monkeypatch):
    """The 1-CTA kernel's epilogue-in-ring aliasing (default when each CTA
    gets at most one unit) and the two-MMA-issuer path give bit-identical
    results to the plain variants."""
    monkeypatch.setenv("LFGPU_NO_PAIR", "1")
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    if case == "conv":
        g = ir.pad_conv(2, 64, 64, 56, 3, 1, 1)
        seqs = runtime.decode_layout(g, 1, [28, 28, 64, 32, 32, 64])
        node = 1
    else:
        g = ir.gemm(512, 512, 1024)
        seqs = runtime.decode_layout(g, 0, [128, 64, 128])
        node = 0
    inputs, ref = oracle_outputs(g, 31)
    p = runtime.Plan(g, seqs, [runtime.sched(node, tile_last=64 if case == "gemm" else 1)],
                     flags=_abi.PLAN_REQUIRE_TC)
    k = p.node_kernel(node)
    if knobs.get("LFGPU_DUAL_MMA") == "1":
        assert " dual" in k, k
    if knobs.get("LFGPU_DUAL_MMA") == "2":  # split issue: two issuers, two accumulators per unit
        assert " split-issue" in k, k
    if knobs.get("LFGPU_NO_EPI_ALIAS") == "1":
        assert "epi-in-ring" not in k, k
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    out = g.nodes[-1].output
    assert np.array_equal(p.get_output(out), ref[out])


def test_run_on_user_stream_joins_async_set_input():
    """set_input_device(wait=False) enqueues the K1 conversion on the plan's
    stream; run(stream=user) must wait for it and get_output must wait for
    the run (both races)."""
    torch = pytest.importorskip("torch")
    g = ir.gemm(512, 512, 512)
    seqs = runtime.decode_layout(g, 0, [256, 64, 256])
    inputs, ref = oracle_outputs(g, 41)
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    user = torch.cuda.Stream()
    ps = torch.cuda.ExternalStream(p.stream)
    for rep in range(3):
        # inputs scaled by (rep + 1): stale operands would give the previous
        # rep's product (k/64 values doubled / tripled stay exact)
        a = torch.tensor(inputs["a"] * (rep + 1), dtype=torch.float32, device="cuda").view(512, 512)
        b = torch.tensor(inputs["b"], dtype=torch.float32, device="cuda").view(512, 512)
        torch.cuda.synchronize()
        with torch.cuda.stream(ps):
            torch.cuda._sleep(1_000_000)  # delay the async conversions on the plan's stream
        p.set_input_device("a", a, wait=False)
        p.set_input_device("b", b, wait=False)
        p.run(stream=user.cuda_stream)
        got = p.get_output("c")
        assert np.array_equal(got, ref["c"] * (rep + 1)), rep


def test_set_input_device_waits_for_producer_stream():
    """The plan's stream is non-blocking: a device input still being
    written on torch's default stream (a delayed producer) must be read only
    after its producer, and one produced on a side stream after that stream
    (found by the bench's 4096^3 check reading a freshly generated operand)."""
    torch = pytest.importorskip("torch")
    n = 1024
    g = ir.gemm(n, n, n)
    seqs = runtime.decode_layout(g, 0, [256, 64, 256])
    p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    side = torch.cuda.Stream()
    for rep, stream in enumerate([None, side, None]):
        torch.cuda.synchronize()
        ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.default_stream())
        with ctx:
            torch.cuda._sleep(2_000_000)  # the producer is still pending when set_input_device runs
            a = torch.randint(-64, 65, (n, n), generator=gen, device="cuda").float() / 64
            b = torch.randint(-64, 65, (n, n), generator=gen, device="cuda").float() / 64
            p.set_input_device("a", a, wait=(rep != 2))
            p.set_input_device("b", b, wait=(rep != 2))
        p.run()
        got = torch.tensor(p.get_output("c"), device="cuda").view(n, n)
        assert torch.equal(got, a.double() @ b.double()), rep


# Loop-point parameters the GPU lowering maps to kernel structure
# (space.cpp:483-589 -> DESIGN.md §4.4): tile_second picks the GEMM M tile
# (128: 1-CTA kernel, else the CTA pair) and caps the C2D rows per UMMA tile;
# parallel picks the pair kernel's tile rasterization and the 1-CTA kernel's
# unit dealing (contiguous chunks vs cyclic). Every variant is bit-exact.
@pytest.mark.parametrize("ts,par", [(1, 0), (1, 1), (128, 0), (128, 1), (256, 1)])
def test_gemm_loop_point_tile_second_parallel(ts, par):
    g, seqs, inputs, ref = gemm_case(512, 1024, 1024, (256, 64, 128))
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=128, tile_second=ts, parallel=par)],
                     flags=_abi.PLAN_REQUIRE_TC)
    k = p.node_kernel(0)
    assert ("gemm-pair" in k) == (ts != 128), k
    if ts != 128:
        assert ("raster=rows" if par else "raster=group8") in k, k
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("c")
    assert np.array_equal(got, ref["c"]), np.abs(got - ref["c"]).max()


@pytest.mark.parametrize("factors,ts,rows", [((28, 2, 32, 32, 32, 32), 1, "28x"), ((28, 2, 32, 32, 32, 32), 7, "7x"),
                                             ((28, 2, 32, 32, 32, 32), 4, "4x"), ((8, 8, 32, 32, 32, 32), 3, "2x")])
@pytest.mark.parametrize("par", [0, 1])
def test_conv_loop_point_tile_second_parallel(factors, ts, rows, par):
    g = ir.pad_conv(1, 64, 64, 56, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(factors))
    inputs, ref = oracle_outputs(g, 42)
    p = runtime.Plan(g, seqs, [runtime.sched(1, tile_second=ts, parallel=par)], flags=_abi.PLAN_REQUIRE_TC)
    k = p.node_kernel(1)
    assert f"rows={rows}" in k, k
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    y = p.get_output("y")
    assert np.array_equal(y, ref["y"]), np.abs(y - ref["y"]).max()


# Split-K over DSMEM in the 1-CTA kernel (k_umma.cu, one unit per CTA: the S
# splits of a tile are one cluster) against the workspace protocol and the
# oracle, for the BERT-size GEMMs it serves (M = 128), MN- and K-major B.
@pytest.mark.parametrize("K,N,f,bk", [(768, 768, (128, 64, 64), 0), (3072, 768, (128, 64, 64), 0),
                                      (768, 768, (128, 128, 128), 1), (3072, 768, (128, 128, 128), 1),
                                      (768, 768, (128, 128, 128), 0)])
@pytest.mark.parametrize("knob", [{}, {"LFGPU_NO_XSPLIT": "1"}])
def test_split_k_dsmem_exchange(K, N, f, bk, knob, monkeypatch):
    for k, v in knob.items():
        monkeypatch.setenv(k, v)
    g, seqs, inputs, ref = gemm_case(128, K, N, f)
    if bk:
        seqs["b"] = [split(0, [K // 64, 64]), reorder([0, 2, 1])]
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=f[2])], flags=_abi.PLAN_REQUIRE_TC)
    assert "splits=1 " not in p.node_kernel(0), p.node_kernel(0)
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    got = p.get_output("c")
    assert np.array_equal(got, ref["c"]), np.abs(got - ref["c"]).max()


@pytest.mark.parametrize("kcs", ["64", "128", "256"])
@pytest.mark.parametrize("layout", ["tuned", "a_mn", "b_k", "kouter_rows"])
def test_gemm_multi_slab_stages(layout, kcs, monkeypatch):
    """K per stage of the 1-CTA GEMM: 64, 128 or 256 (several 64-wide K
    slabs per TMA box, one UMMA group per slab) on K-major and MN-major A
    and B, and on column-brick activations [K/64][M][64]; bit-exact against
    the oracle whatever the stage depth."""
    monkeypatch.setenv("LFGPU_NO_PAIR", "1")
    monkeypatch.setenv("LFGPU_GEMM_KCS", kcs)
    M, K, N = 256, 1024, 512
    g = ir.gemm(M, K, N)
    if layout == "tuned":
        seqs = runtime.decode_layout(g, 0, [128, 64, 64])
    elif layout == "a_mn":  # A [K/64][M/64][64 k][64 m]: MN-major A
        seqs = runtime.decode_layout(g, 0, [128, 64, 64])
        seqs["a"] = [split(0, [M // 64, 64]), split(2, [K // 64, 64]), reorder([2, 0, 3, 1])]
    elif layout == "b_k":  # B [N/64][K/64][64 n][64 k]: K-major B
        seqs = runtime.decode_layout(g, 0, [128, 64, 64])
        seqs["b"] = [split(0, [K // 64, 64]), split(2, [N // 64, 64]), reorder([2, 0, 3, 1])]
    else:  # A as column bricks over full rows, C the same
        seqs = runtime.decode_layout(g, 0, [128, 64, 64])
        seqs["a"] = [split(1, [K // 64, 64]), reorder([1, 0, 2])]
        seqs["c"] = [split(1, [N // 64, 64]), reorder([1, 0, 2])]
    inputs, ref = oracle_outputs(g, 37)
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=64, tile_second=128)], flags=_abi.PLAN_REQUIRE_TC)
    k = p.node_kernel(0)
    assert k.startswith("umma_gemm") and "KC=" in k, k
    assert int(k.split("KC=")[1].split(" ")[0]) == int(kcs), k
    for tid, v in inputs.items():
        p.set_input(tid, v)
    p.run()
    assert np.array_equal(p.get_output("c"), ref["c"]), k
