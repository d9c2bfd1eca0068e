"""K6 depthwise 3x3 over 16x256x56x56 (padded input 58x58) on channel-brick
layouts, DEP node alone, L2-flushed and warm, with HBM bytes / time
(diagnostics). LFGPU_DEP_ROWS selects output rows per thread."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

for f in ((56, 28, 32, 32, 32), (56, 56, 64, 64, 64), (28, 28, 16, 16, 16)):
    gc = ir.dep_chain(16, 256, 56, 3, 1, 1)
    sq = runtime.decode_layout(gc, 1, list(f))
    g = ir.Graph()
    g.tensors = [ir.TensorDecl("xp", [("N", 16), ("C", 256), ("H", 58), ("W", 58)], ir.INPUT),
                 ir.TensorDecl("ker", [("C", 256), ("KH", 3), ("KW", 3)], ir.CONSTANT),
                 ir.TensorDecl("conv", [("N", 16), ("C", 256), ("H", 56), ("W", 56)], ir.OUTPUT)]
    g.nodes = [ir.OperatorNode(ir.DEP, ["xp", "ker"], "conv", {"stride": 1})]
    seqs = {k: sq[k] for k in ("xp", "ker", "conv") if k in sq}
    p = runtime.Plan(g, seqs, [runtime.sched(0)])
    x = (torch.randint(-64, 65, (16, 256, 58, 58), device="cuda").float() / 64)
    w = (torch.randint(-64, 65, (256, 3, 3), device="cuda").float() / 64)
    p.set_input_device("xp", x)
    p.set_input_device("ker", w)
    p.run()
    got = torch.tensor(p.get_output("conv"), device="cuda").view(16, 256, 56, 56)
    ref = torch.nn.functional.conv2d(x.double(), w.double().view(256, 1, 3, 3), groups=256).float()
    cold = p.measure(warmup=3, reps=10, flush_l2=True).cost
    warm = p.measure(warmup=3, reps=10, flush_l2=False).cost
    byts = 16 * 256 * (58 * 58 + 56 * 56) * 4
    print(f"f={f} {p.node_kernel(0)}: cold {cold:.2f} us ({byts / cold / 1e3:.0f} GB/s) warm {warm:.2f} us"
          f" exact={torch.equal(got, ref)}", flush=True)
    p.close()
