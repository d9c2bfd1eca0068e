"""A/B of a plan-build environment switch on ResNet-18 b1 with one set of
tuned conv layouts (diagnostics): python tools/resnet_ab.py VAR[=VALUE] ..."""
import os
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e, workloads  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(1)
fac = workloads.tune_resnet18(1, lambda sub: e2e.make_inputs(sub, gen))
switches = sys.argv[1:] or ["LFGPU_NO_PAD_ABSORB=1"]
res = {}
for rep in range(3):
    for sw in [None] + switches:
        if sw:
            k, _, v = sw.partition("=")
            os.environ[k] = v or "1"
        g, convs, p = e2e.build_resnet18(1, fac)
        for k2, x in e2e.make_inputs(g, gen).items():
            p.set_input_device(k2, x)
        m = p.measure(warmup=3, reps=7, flush_l2=False)
        res.setdefault(sw or "default", []).append((round(m.cost, 1), int(m.kernels)))
        p.close()
        if sw:
            os.environ.pop(sw.partition("=")[0], None)
for k, v in res.items():
    print(k, v)
