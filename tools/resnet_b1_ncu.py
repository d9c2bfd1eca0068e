"""ResNet-18 b1 plan, run 3 times with direct launches (for ncu launch lists)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e, workloads  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(1)
fac = workloads.tune_resnet18(1, lambda sub: e2e.make_inputs(sub, gen))
g, convs, p = e2e.build_resnet18(1, fac, flags=0)
for k, x in e2e.make_inputs(g, gen).items():
    p.set_input_device(k, x)
for _ in range(3):
    p.run()
torch.cuda.synchronize()
