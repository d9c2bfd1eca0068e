"""Stem C2D (3->64, 7x7 s2): im2col + tcgen05 vs the CUDA-core direct kernel.
Diagnostics only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

for nb in (1, 16, 64):
    g = ir.pad_conv(nb, 3, 64, 224, 7, 2, 3)
    p = runtime.Plan(g, {}, [runtime.sched(1)], _abi.PLAN_CUDA_GRAPH)
    p.set_input_device("x", torch.randn(nb, 3, 224, 224, device="cuda"))
    p.set_input_device("ker", torch.randn(64, 3, 7, 7, device="cuda"))
    c = p.measure()
    print(nb, [p.node_kernel(i)[:60] for i in range(len(g.nodes))], f"{c.cost:.1f} us")
