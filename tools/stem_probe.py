"""ResNet stem (Padding -> C2D 3->64 7x7 s2 -> BiasAdd -> ReLU) at batch 64
and 1 through im2col + tcgen05 GEMM, L2 flushed: whole-plan time with the
tiled im2col and the flat one (LFGPU_IM2COL_FLAT=1) (diagnostics)."""
import os
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, workloads, runtime, e2e  # noqa: E402

for nb in (64, 1):
    b = workloads.Builder()
    x = b.t("x", [("N", nb), ("C", 3), ("H", 224), ("W", 224)], ir.INPUT)
    xp = b.t("xp", [("N", nb), ("C", 3), ("H", 230), ("W", 230)])
    b.op(ir.PADDING, [x], xp, pad=3)
    w = b.t("stem_w", [("O", 64), ("I", 3), ("KH", 7), ("KW", 7)], ir.CONSTANT)
    y = b.t("y", [("N", nb), ("C", 64), ("H", 112), ("W", 112)])
    b.op(ir.C2D, [xp, w], y, stride=2)
    bias = b.t("stem_b", [("O", 64)], ir.CONSTANT)
    yb = b.t("yb", [("N", nb), ("C", 64), ("H", 112), ("W", 112)])
    b.op(ir.BIASADD, [y, bias], yb)
    yr = b.t("yr", [("N", nb), ("C", 64), ("H", 112), ("W", 112)], ir.OUTPUT)
    b.op(ir.RELU, [yb], yr)
    g = b.g
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    ins = e2e.make_inputs(g, gen)
    outs = {}
    for mode in ("tiles", "flat"):
        if mode == "flat":
            os.environ["LFGPU_IM2COL_FLAT"] = "1"
        p = runtime.Plan(g, {}, [runtime.sched(1, fuse=1)], _abi.PLAN_DEFAULT)
        for k, v in ins.items():
            p.set_input_device(k, v)
        p.run()
        outs[mode] = p.get_output("yr")
        m = p.measure(warmup=3, reps=10, flush_l2=True)
        print(f"b{nb} {mode}: {m.cost:.1f} us  {p.node_kernel(1)[:60]}", flush=True)
        p.close()
        os.environ.pop("LFGPU_IM2COL_FLAT", None)
    print("identical:", (outs["tiles"] == outs["flat"]).all())
