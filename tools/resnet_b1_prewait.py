"""ResNet-18 b1: one tuning, then the same plan with and without the pre-wait
weight loads (diagnostics)."""
import os
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e, workloads  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(1)
fac = workloads.tune_resnet18(1, lambda sub: e2e.make_inputs(sub, gen))
for rep in range(2):
    for off in ("0", "1"):
        if off == "1":
            os.environ["LFGPU_NO_W_PREWAIT"] = "1"
        else:
            os.environ.pop("LFGPU_NO_W_PREWAIT", None)
        g, _, p = e2e.build_resnet18(1, fac)
        for k, x in e2e.make_inputs(g, gen).items():
            p.set_input_device(k, x)
        m = p.measure(warmup=3, reps=9, flush_l2=False)
        mc = p.measure(warmup=3, reps=9, flush_l2=True)
        print("prewait" if off == "0" else "no-prewait", "warm %.1f cold %.1f us" % (m.cost, mc.cost), m.kernels)
        p.close()
