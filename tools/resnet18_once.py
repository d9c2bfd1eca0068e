"""One untuned-or-tuned ResNet-18 plan replay for launch-list profiling."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import resnet18_run as R  # noqa: E402
from paper_2210_12415_b200 import workloads  # noqa: E402

n = int(os.environ.get("BATCH", "1"))
gen = torch.Generator(device="cuda")
gen.manual_seed(42)
factors = workloads.tune_resnet18(n, lambda sub: R.make_inputs(sub, gen))
g, convs, plan = R.build(n, factors)
ins = R.make_inputs(g, gen)
for k, x in ins.items():
    plan.set_input_device(k, x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
plan.run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
for i in range(len(g.nodes)):
    print(i, g.nodes[i].output, plan.node_kernel(i)[:60])
