"""Build a cfg4/cfg5 plan and run it a few times (for ncu launch lists).
  python tools/plan_once.py bert|r18 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi  # noqa: E402

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
if which == "bert":
    import bert_run as B
    g, gmms, plan = B.build(12, 64, 0, flags=_abi.PLAN_DEFAULT)
    ins = B.make_inputs(g, gen)
else:
    import resnet18_run as R
    import test_gpu_resnet as T  # fixed b1 factors
    g, convs, plan = R.build(1, T.FIXED_FACTORS_B1)
    ins = R.make_inputs(g, gen)
for k, x in ins.items():
    plan.set_input_device(k, x)
torch.cuda.synchronize()
for _ in range(reps):
    plan.run()
torch.cuda.synchronize()
print("ok", len(g.nodes))
