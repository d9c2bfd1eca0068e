"""ResNet-18 b1 plan: kernel per node and the tcgen05 chain timeline (diagnostics)."""
import ctypes as C
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e, ir, runtime, workloads  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(1)
fac = workloads.tune_resnet18(1, lambda sub: e2e.make_inputs(sub, gen))
g, convs, p = e2e.build_resnet18(1, fac)
for k, x in e2e.make_inputs(g, gen).items():
    p.set_input_device(k, x)
m = p.measure(warmup=3, reps=5, flush_l2=False)
print("latency warm us", round(m.cost, 1), "launches", m.kernels)
for i, nd in enumerate(g.nodes):
    k = p.node_kernel(i)
    if k != "fused":
        print(i, ir.OP_NAMES[nd.kind], nd.output, k[:110])
