"""cfg4 pieces on the GPU: conversions between two different C2D templates
(source-table digit maps), the pool ops, the direct small-I conv, and
ResNet-18 end to end.

Tolerances: conversions, pools and single k/64 contractions are bit-exact
against the oracle. The ResNet-18 logits go through 20 chained convs whose
activations are stored / fed to tcgen05 in bf16 (SURVEY.md §8c "chained
fp32 graphs"): they are checked (a) against a float64 reference that applies
the same bf16 rounding to tensor-core operands, max_rel_diff <= 1e-4, and
(b) against the exact float64 forward, max_rel_diff <= 2e-3 (the stated
bf16-activation tolerance of this path).
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle_lib as O
from paper_2210_12415_b200 import _abi, ir, runtime, workloads
from paper_2210_12415_b200.layout import reorder, split

from paper_2210_12415_b200 import e2e as R  # noqa: E402

pytestmark = pytest.mark.gpu

# (in extents, y template factors of the producer, xp template factors of the consumer)
TEMPLATE_PAIRS = [
    ((1, 64, 56, 56), (8, 7, 32, 32, 32, 32), (7, 7, 32, 32, 32, 32)),
    ((2, 64, 28, 28), (2, 28, 32, 64, 64, 16), (14, 4, 64, 16, 16, 64)),
    ((1, 128, 14, 14), (7, 7, 16, 64, 64, 16), (7, 14, 32, 32, 32, 32)),
]


def test_padding_between_templates_is_exact():
    rng = np.random.default_rng(3)
    for ext, fy, fx in TEMPLATE_PAIRS:
        n, c, h, _ = ext
        g = ir.pad_conv(n, c, c, h, 3, 1, 1)
        y_seq = runtime.decode_layout(g, 1, list(fy))["y"]
        xp_seq = runtime.decode_layout(g, 1, list(fx))["xp"]
        x = rng.integers(-64, 65, int(np.prod(ext))) / 64.0
        xs = O.materialize(list(ext), y_seq, x)   # source in the producer's output layout
        rc, want = O.padding_nest(list(ext), 1, y_seq, xp_seq, xs)
        assert rc == 0
        for dt in (torch.float32, torch.bfloat16):
            src = torch.tensor(xs, dtype=torch.float32, device="cuda")
            dst = torch.full((want.size,), float("nan"), dtype=dt, device="cuda")
            runtime.pad_convert(src, [("N", n), ("C", c), ("H", h), ("W", h)], 1, y_seq, xp_seq,
                                dst)
            torch.cuda.synchronize()
            assert np.array_equal(dst.double().cpu().numpy(), want), (ext, fy, fx, dt)


def pool_graph(n, c, h):
    g = ir.Graph()
    g.tensors = [
        ir.TensorDecl("x", [("N", n), ("C", c), ("H", h), ("W", h)], ir.INPUT),
        ir.TensorDecl("xp", [("N", n), ("C", c), ("H", h + 2), ("W", h + 2)]),
        ir.TensorDecl("mp", [("N", n), ("C", c), ("H", h // 2), ("W", h // 2)]),
        ir.TensorDecl("y", [("N", n), ("C", c)], ir.OUTPUT),
    ]
    g.nodes = [
        ir.OperatorNode(ir.PADDING, ["x"], "xp", {"pad": 1}),
        ir.OperatorNode(ir.MAXPOOL, ["xp"], "mp", {"window": 3, "stride": 2}),
        ir.OperatorNode(ir.GLOBAL_AVGPOOL, ["mp"], "y"),
    ]
    return g


@pytest.mark.parametrize("layouts", [
    {},
    {"x": [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])],
     "mp": [split(1, [4, 16]), split(3, [2, 7]), reorder([0, 1, 3, 4, 5, 2])]},
])
def test_pools_match_oracle(layouts):
    g = pool_graph(2, 64, 28)
    bufs = O.random_inputs(g, 42)
    ins = {"x": bufs[0].copy()}
    O.reference_eval(g, bufs)
    out = runtime.interpret(g, layouts, [], ins)
    assert np.array_equal(out["mp"], bufs[g.tensor_index("mp")])       # max: exact
    assert O.max_rel_diff(out["y"], bufs[g.tensor_index("y")]) <= 1e-6


@pytest.mark.parametrize("path,hw", [("im2col_umma", 64), ("c2d_direct", 64), ("im2col_umma", 224)])
def test_direct_stem_conv_fused_exact(path, hw, monkeypatch):
    # 3-channel 7x7 stride-2 conv (the ResNet stem) + BiasAdd + ReLU: k/64
    # inputs make fp32 (and bf16-operand) accumulation exact, so both the
    # im2col + tcgen05 path and the CUDA-core direct kernel must match.
    if path == "c2d_direct":
        monkeypatch.setenv("LFGPU_NO_IM2COL", "1")
    # hw=224: 112-pixel output rows, one per GEMM tile (rows-per-tile < 128)
    g = ir.conv_chain(2 if hw == 64 else 1, 3, 64, hw, 7, 2, 3)
    bufs = O.random_inputs(g, 42)
    ins = {t.id: bufs[i].copy() for i, t in enumerate(g.tensors) if t.role in (ir.INPUT, ir.CONSTANT)}
    O.reference_eval(g, bufs)
    p = runtime.Plan(g, {}, [runtime.sched(1, fuse=1)])
    assert p.node_kernel(1).startswith(path), p.node_kernel(1)
    if path == "im2col_umma":  # the Padding is read through by im2col (zero outside x)
        assert p.node_kernel(0) == "fused"
        with pytest.raises(runtime.LfError):
            p.get_output("xp")
    assert p.node_kernel(2) == "fused" and p.node_kernel(3) == "fused"
    for k, v in ins.items():
        p.set_input(k, v)
    p.run()
    assert np.array_equal(p.get_output("y"), bufs[g.tensor_index("y")])


@pytest.mark.parametrize("shape,factors,force", [
    ((1, 512, 512, 7, 3, 1, 1), (7, 7, 16, 64, 64, 16), None),     # auto split-K (deep K, 32 tiles)
    ((1, 64, 64, 56, 3, 1, 1), (4, 28, 16, 32, 32, 16), "3"),      # forced, uneven stage ranges
    ((2, 256, 256, 14, 3, 1, 1), (14, 14, 32, 64, 64, 32), "5"),
])
def test_splitk_conv_exact(shape, factors, force, monkeypatch):
    if force:
        monkeypatch.setenv("LFGPU_SPLITK", force)
    n, ci, co, h, k, s, p = shape
    g = ir.pad_conv(n, ci, co, h, k, s, p)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    x = R.k64((n, ci, h, h), gen)
    w = R.k64((co, ci, k, k), gen)
    plan = runtime.Plan(g, runtime.decode_layout(g, 1, list(factors)), [runtime.sched(1)],
                        _abi.PLAN_REQUIRE_TC)
    plan.set_input_device("x", x)
    plan.set_input_device("ker", w)
    for _ in range(3):  # re-launches exercise the re-armed arrival counters
        plan.run()
    y = torch.tensor(plan.get_output("y"), device="cuda")
    ref = torch.nn.functional.conv2d(x.double(), w.double(), stride=s, padding=p).flatten()
    assert torch.equal(y, ref)


def test_splitk_fused_epilogue():
    # bias + ReLU applied once, by the last CTA of each tile
    g = ir.conv_chain(1, 256, 256, 14, 3, 1, 1)
    bufs = O.random_inputs(g, 42)
    ins = {t.id: bufs[i].copy() for i, t in enumerate(g.tensors) if t.role in (ir.INPUT, ir.CONSTANT)}
    O.reference_eval(g, bufs)
    seqs = runtime.decode_layout(g, 1, [7, 7, 16, 64, 64, 16])
    seqs = workloads.propagate_elementwise(g, seqs)
    p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1)], _abi.PLAN_REQUIRE_TC)
    assert "umma" in p.node_kernel(1) and p.node_kernel(3) == "fused"
    for k, v in ins.items():
        p.set_input(k, v)
    p.run()
    p.run()
    assert np.array_equal(p.get_output("y"), bufs[g.tensor_index("y")])


FIXED_FACTORS_B1 = {
    # a residual-consistent assignment (stage output bricks shared by the
    # second convs and the downsample conv), used so the test needs no tuning
    "s1b1_a": (8, 7, 32, 32, 32, 32), "s1b1_b": (8, 7, 32, 32, 32, 32),
    "s1b2_a": (8, 7, 32, 32, 32, 32), "s1b2_b": (8, 7, 32, 32, 32, 32),
    "s2b1_ds": (28, 28, 32, 64, 64, 32), "s2b1_a": (28, 2, 16, 32, 32, 16),
    "s2b1_b": (28, 28, 32, 64, 64, 32), "s2b2_a": (28, 28, 32, 64, 64, 32),
    "s2b2_b": (28, 28, 32, 64, 64, 32),
    "s3b1_ds": (14, 14, 16, 64, 64, 16), "s3b1_a": (7, 7, 32, 64, 64, 32),
    "s3b1_b": (14, 14, 16, 64, 64, 16), "s3b2_a": (14, 14, 16, 64, 64, 16),
    "s3b2_b": (14, 14, 16, 64, 64, 16),
    "s4b1_ds": (7, 7, 16, 64, 64, 16), "s4b1_a": (7, 7, 16, 64, 64, 16),
    "s4b1_b": (7, 7, 16, 64, 64, 16), "s4b2_a": (7, 7, 16, 64, 64, 16),
    "s4b2_b": (7, 7, 16, 64, 64, 16),
}


def test_resnet18_b1_logits():
    gen = torch.Generator(device="cuda")
    gen.manual_seed(42)
    g, convs, plan = R.build_resnet18(1, FIXED_FACTORS_B1)
    kinds = [plan.node_kernel(i) for i in range(len(g.nodes))]
    tc = frozenset(i for i, k in enumerate(kinds) if k.startswith("umma"))
    assert len(tc) >= 17, kinds                # every conv but the stem on tcgen05
    assert kinds[convs[0]["node"]].startswith("im2col_umma")  # the stem: im2col operand + tcgen05
    assert "ix_copy" not in kinds                # template-to-template Paddings are digit maps
    ins = R.make_inputs(g, gen)
    for k, x in ins.items():
        plan.set_input_device(k, x)
    plan.run()
    out = torch.tensor(plan.get_output("logits"), device="cuda").view(1, -1)
    emu = R.reference(g, ins, tc, emulate=True)["logits"]
    ex = R.reference(g, ins)["logits"]
    assert R.max_rel(out, emu) <= 1e-4
    assert R.max_rel(out, ex) <= 2e-3


def _two_conv_graph(n=1, c=64, h=56):
    """conv -> BiasAdd -> ReLU -> Padding -> conv: the edge a ResNet basic
    block has between its two 3x3 convs."""
    b = workloads.Builder()
    nchw = lambda tid, cc, hh, role=ir.INTERMEDIATE: b.t(tid, [("N", n), ("C", cc), ("H", hh), ("W", hh)], role)
    x = nchw("x", c, h, ir.INPUT)
    xp = nchw("xp", c, h + 2)
    b.op(ir.PADDING, [x], xp, pad=1)
    w1 = b.t("w1", [("O", c), ("I", c), ("KH", 3), ("KW", 3)], ir.CONSTANT)
    b1 = b.t("b1", [("O", c)], ir.CONSTANT)
    y1 = nchw("y1", c, h)
    b.op(ir.C2D, [xp, w1], y1, stride=1)
    yb = nchw("yb", c, h)
    b.op(ir.BIASADD, [y1, b1], yb)
    yr = nchw("yr", c, h)
    b.op(ir.RELU, [yb], yr)
    yp = nchw("yp", c, h + 2)
    b.op(ir.PADDING, [yr], yp, pad=1)
    w2 = b.t("w2", [("O", c), ("I", c), ("KH", 3), ("KW", 3)], ir.CONSTANT)
    y2 = nchw("y2", c, h, ir.OUTPUT)
    b.op(ir.C2D, [yp, w2], y2, stride=1)
    return b.g


@pytest.mark.parametrize("f1,f2", [((8, 14, 64, 32, 32, 64), (8, 14, 64, 32, 32, 64)),
                                   ((7, 14, 32, 32, 32, 32), (4, 28, 64, 32, 32, 64)),
                                   ((14, 14, 64, 16, 16, 64), (8, 8, 32, 32, 32, 32))])
def test_padding_absorbed_into_producer_epilogue(f1, f2, monkeypatch):
    """The Padding between two tensor-core convs is written by the first
    conv's epilogue straight into the second conv's padded, unfolded bf16
    layout (no conversion kernel), bit-identical to the separate K2 step."""
    g = _two_conv_graph()
    seqs = {}
    seqs.update(runtime.decode_layout(g, 1, list(f1)))
    seqs.update(runtime.decode_layout(g, 5, list(f2)))
    seqs = workloads.propagate_elementwise(g, seqs)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    ins = {"x": R.k64((1, 64, 56, 56), gen), "w1": R.k64((64, 64, 3, 3), gen, 1 / 8),
           "b1": R.k64((64,), gen, 1 / 8), "w2": R.k64((64, 64, 3, 3), gen, 1 / 8)}
    outs = []
    for absorb in (True, False):
        if absorb:
            monkeypatch.delenv("LFGPU_NO_PAD_ABSORB", raising=False)
        else:
            monkeypatch.setenv("LFGPU_NO_PAD_ABSORB", "1")
        p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1), runtime.sched(5)], _abi.PLAN_REQUIRE_TC)
        kinds = [p.node_kernel(i) for i in range(len(g.nodes))]
        assert (kinds[4] == "fused") == absorb, kinds
        for k, v in ins.items():
            p.set_input_device(k, v)
        p.run()
        outs.append(p.get_output("y2"))
    assert np.array_equal(outs[0], outs[1])
    ref = torch.nn.functional.conv2d(
        torch.relu(torch.nn.functional.conv2d(ins["x"].double(), ins["w1"].double(), padding=1)
                   + ins["b1"].double().view(1, -1, 1, 1)).bfloat16().double(),
        ins["w2"].double(), padding=1).flatten().cpu().numpy()
    assert np.max(np.abs(outs[0] - ref) / np.maximum(1, np.abs(ref))) < 1e-4


@pytest.mark.parametrize("layouts", [
    {},
    {"x": [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])],
     "mp": [split(1, [4, 16]), split(3, [2, 7]), reorder([0, 1, 3, 4, 5, 2])]},
])
def test_pool_kernels_fp32(layouts):
    """k_small.cu's table-driven MaxPool / GlobalAvgPool (the default plans;
    the exact mode keeps the generic kernels): max exact, mean within 1e-6."""
    g = pool_graph(2, 64, 28)
    bufs = O.random_inputs(g, 43)
    ins = {"x": bufs[0].copy()}
    O.reference_eval(g, bufs)
    for flags in (_abi.PLAN_KEEP_ALL, _abi.PLAN_DEFAULT):
        p = runtime.Plan(g, layouts, [], flags=flags)
        # without KEEP_ALL the Padding is absorbed into the MaxPool's reads
        pad_kind = "fused" if flags == _abi.PLAN_DEFAULT else p.node_kernel(0)
        assert [p.node_kernel(i) for i in range(3)] == [pad_kind, "maxpool", "global_avgpool"]
        p.set_input("x", ins["x"])
        p.run()
        assert np.array_equal(p.get_output("mp"), bufs[g.tensor_index("mp")])
        assert O.max_rel_diff(p.get_output("y"), bufs[g.tensor_index("y")]) <= 1e-6
    # zero padding takes part in the max: all-negative inputs give 0 on the border
    p.set_input("x", -np.abs(ins["x"]) - 1.0)
    p.run()
    mp = p.get_output("mp").reshape(2, 64, 14, 14) if not layouts else None
    if mp is not None:
        assert (mp[:, :, 0, :] == 0).all() and (mp[:, :, 1:, 1:] < 0).all()


@pytest.mark.parametrize("m,fuse", [(1, 1), (4, 1), (1, 0), (16, 1)])
def test_gemv_classifier_fused(m, fuse):
    """The small-M GMM (batch-1 classifier) with BiasAdd + ReLU fused: fp32
    sums of k/64 products are exact, so == the oracle."""
    K, N = 512, 1000
    g = ir.Graph()
    g.tensors = [ir.TensorDecl("a", [("M", m), ("K", K)], ir.INPUT),
                 ir.TensorDecl("w", [("K", K), ("N", N)], ir.CONSTANT),
                 ir.TensorDecl("bias", [("N", N)], ir.CONSTANT),
                 ir.TensorDecl("c", [("M", m), ("N", N)], ir.INTERMEDIATE),
                 ir.TensorDecl("cb", [("M", m), ("N", N)], ir.INTERMEDIATE),
                 ir.TensorDecl("y", [("M", m), ("N", N)], ir.OUTPUT)]
    g.nodes = [ir.OperatorNode(ir.GMM, ["a", "w"], "c"), ir.OperatorNode(ir.BIASADD, ["c", "bias"], "cb"),
               ir.OperatorNode(ir.RELU, ["cb"], "y")]
    bufs = O.random_inputs(g, 44)
    ins = {t: bufs[g.tensor_index(t)].copy() for t in ("a", "w", "bias")}
    O.reference_eval(g, bufs)
    p = runtime.Plan(g, {}, [runtime.sched(0, fuse=fuse)])
    kinds = [p.node_kernel(i) for i in range(3)]
    assert kinds[0] == "gemv" and (kinds[1:] == ["fused", "fused"]) == bool(fuse), kinds
    for k, v in ins.items():
        p.set_input(k, v)
    p.run()
    assert np.array_equal(p.get_output("y"), bufs[g.tensor_index("y")])


@pytest.mark.parametrize("window,stride,pad", [(3, 2, 1), (2, 2, 0), (3, 1, 1)])
def test_maxpool_window_stride_absorbed_padding(window, stride, pad):
    """k_small.cu MaxPool over window / stride variants, reading through an
    absorbed Padding when there is one: == the oracle (max is exact)."""
    n, c, h = 2, 32, 17
    hp = h + 2 * pad
    ho = (hp - window) // stride + 1
    g = ir.Graph()
    g.tensors = [ir.TensorDecl("x", [("N", n), ("C", c), ("H", h), ("W", h)], ir.INPUT),
                 ir.TensorDecl("xp", [("N", n), ("C", c), ("H", hp), ("W", hp)]),
                 ir.TensorDecl("y", [("N", n), ("C", c), ("H", ho), ("W", ho)], ir.OUTPUT)]
    g.nodes = [ir.OperatorNode(ir.PADDING, ["x"], "xp", {"pad": pad}),
               ir.OperatorNode(ir.MAXPOOL, ["xp"], "y", {"window": window, "stride": stride})]
    bufs = O.random_inputs(g, 45)
    x = bufs[0].copy()
    O.reference_eval(g, bufs)
    p = runtime.Plan(g, {}, [])
    assert p.node_kernel(1) == "maxpool" and p.node_kernel(0) == "fused"
    p.set_input("x", x)
    p.run()
    assert np.array_equal(p.get_output("y"), bufs[g.tensor_index("y")])


def test_gemv_residual_and_blocked_layouts():
    """GEMV with a residual EwAdd fused, on a blocked weight layout and a
    blocked output / residual layout: exact (k/64 products)."""
    m, K, N = 2, 256, 1000  # N not a multiple of 16: no tensor-core tile, the GEMV path
    g = ir.Graph()
    g.tensors = [ir.TensorDecl("a", [("M", m), ("K", K)], ir.INPUT),
                 ir.TensorDecl("w", [("K", K), ("N", N)], ir.CONSTANT),
                 ir.TensorDecl("r", [("M", m), ("N", N)], ir.INPUT),
                 ir.TensorDecl("c", [("M", m), ("N", N)], ir.INTERMEDIATE),
                 ir.TensorDecl("y", [("M", m), ("N", N)], ir.OUTPUT)]
    g.nodes = [ir.OperatorNode(ir.GMM, ["a", "w"], "c"), ir.OperatorNode(ir.EWADD, ["c", "r"], "y")]
    seqs = {"w": [split(1, [N // 40, 40]), reorder([1, 0, 2])],
            "c": [split(1, [N // 125, 125]), reorder([1, 0, 2])]}
    seqs["y"] = seqs["r"] = seqs["c"]
    bufs = O.random_inputs(g, 46)
    ins = {t: bufs[g.tensor_index(t)].copy() for t in ("a", "w", "r")}
    O.reference_eval(g, bufs)
    p = runtime.Plan(g, seqs, [runtime.sched(0, fuse=1)])
    assert [p.node_kernel(i) for i in range(2)] == ["gemv", "fused"]
    for k, v in ins.items():
        p.set_input(k, v)
    p.run()
    assert np.array_equal(p.get_output("y"), bufs[g.tensor_index("y")])
