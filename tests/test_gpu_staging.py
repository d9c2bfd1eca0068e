"""Host-buffer staging of the drop-in entry points (lfgpu_plan_set_input /
lfgpu_plan_get_output, the reference's BufferMap of doubles): float tensors
are narrowed to f32 / bf16 on the host and widened back there, so the link
carries 4 or 2 bytes per element instead of 8. The host conversions restate
the device's (cvt.rn.f32.f64, then cvt.rn.bf16.f32): the stored values must
be bit-identical to staging the doubles and converting on the device
(LFGPU_STAGE_F64=1), on the values where rounding is delicate."""
import os

import numpy as np
import pytest

from paper_2210_12415_b200 import _abi, ir, runtime

pytestmark = pytest.mark.gpu


def _tricky(n, seed=3):
    rng = np.random.default_rng(seed)
    f = rng.standard_normal(n // 4).astype(np.float32)
    up = np.nextafter(f, np.float32(np.inf))
    mid = (f.astype(np.float64) + up.astype(np.float64)) / 2  # exact f32 ties
    b = (rng.integers(0, 1 << 31, n // 4, dtype=np.uint32) & 0xFFFF0000) | 0x8000  # exact bf16 ties
    with np.errstate(invalid="ignore"):
        bt = b.view(np.float32).astype(np.float64)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-320, -1e-40, 3.4e38, 3.39e38, 1e39,
                        np.finfo(np.float32).max, np.finfo(np.float32).tiny / 3])
    m = n - 2 * (n // 4) - special.size
    scales = 10.0 ** rng.uniform(-46, 39, m)  # f32 subnormals .. beyond the bf16 / f32 range
    wide = rng.standard_normal(m) * scales
    v = np.concatenate([mid, bt, wide, special])
    rng.shuffle(v)
    return v


def _plans_both_ways(g, vals, outs, seqs=None, scheds=()):
    res = []
    for mode in ("narrow", "f64"):
        if mode == "f64":
            os.environ["LFGPU_STAGE_F64"] = "1"
        try:
            p = runtime.Plan(g, dict(seqs or {}), list(scheds), flags=_abi.PLAN_KEEP_ALL)
            for k, v in vals.items():
                p.set_input(k, v)
            p.run()
            res.append({t: p.get_output(t) for t in outs})
            p.close()
        finally:
            os.environ.pop("LFGPU_STAGE_F64", None)
    return res


def _same(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_narrowed_staging_bit_identical_f32_and_bf16():
    n = 4096
    # x feeds a GEMM (bf16 operand copy) and an EwAdd (f32 copy): both storages
    g = ir.Graph()
    g.tensors = [ir.TensorDecl("x", [("M", 64), ("K", 64)], ir.INPUT),
                 ir.TensorDecl("w", [("K", 64), ("N", 64)], ir.CONSTANT),
                 ir.TensorDecl("z", [("M", 64), ("K", 64)], ir.INPUT),
                 ir.TensorDecl("c", [("M", 64), ("N", 64)], ir.OUTPUT),
                 ir.TensorDecl("s", [("M", 64), ("K", 64)], ir.OUTPUT)]
    g.nodes = [ir.OperatorNode(ir.GMM, ["x", "w"], "c"), ir.OperatorNode(ir.EWADD, ["x", "z"], "s")]
    x = _tricky(n)
    vals = {"x": x, "w": np.full(n, 0.5), "z": np.zeros(n)}
    seqs = runtime.decode_layout(g, 0, [64, 64, 64])
    a, b = _plans_both_ways(g, vals, ["x", "s"], seqs, [runtime.sched(0, tile_last=64)])
    for t in ("x", "s"):
        nan_a, nan_b = np.isnan(a[t]), np.isnan(b[t])
        assert np.array_equal(nan_a, nan_b), t
        assert _same(a[t][~nan_a], b[t][~nan_a]), t
    # the stored f32 values are float32(x): exact widening back
    keep = ~np.isnan(x)
    with np.errstate(over="ignore"):
        assert np.array_equal(a["x"][keep], x[keep].astype(np.float32).astype(np.float64))


def test_narrowed_staging_bf16_only_operand():
    # a GEMM-only input is stored as bf16 alone: the host narrows straight
    # to bf16 (through float, as the device does)
    g = ir.gemm(64, 64, 64)
    x = _tricky(64 * 64, seed=4)
    vals = {"a": x, "b": np.ones(64 * 64) / 64}
    seqs = runtime.decode_layout(g, 0, [64, 64, 64])
    a, b = _plans_both_ways(g, vals, ["a", "c"], seqs, [runtime.sched(0, tile_last=64)])
    for t in ("a", "c"):
        nan_a = np.isnan(a[t])
        assert np.array_equal(nan_a, np.isnan(b[t])), t
        assert _same(a[t][~nan_a], b[t][~nan_a]), t


def test_narrowed_staging_kernels():
    """Both staging storages are really exercised: x has an f32 and a bf16
    copy, the GEMM-only operand a bf16 copy alone."""
    g = ir.gemm(64, 64, 64)
    seqs = runtime.decode_layout(g, 0, [64, 64, 64])
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=64)], flags=_abi.PLAN_KEEP_ALL)
    assert p.node_kernel(0).startswith("umma_gemm")
    assert p.buffer("a")[1] == _abi.ELEM_BF16
    p.close()


def test_int32_tensors_keep_f64_staging():
    """int32 tensors are not narrowed on the host (their conversion is the
    device's truncating cvt): an int32 graph through set_input / get_output
    matches the oracle exactly."""
    g = ir.conv_chain(1, 2, 3, 6, 3, 1, 1, dtype=ir.I32)
    import oracle_lib as O
    bufs = O.random_inputs(g, 47)
    ins = {t.id: bufs[i].copy() for i, t in enumerate(g.tensors) if t.role in (ir.INPUT, ir.CONSTANT)}
    O.reference_eval(g, bufs)
    out = runtime.interpret(g, {}, [], ins, flags=_abi.PLAN_EXACT)
    last = g.nodes[-1].output
    assert np.array_equal(out[last], bufs[g.tensor_index(last)])
