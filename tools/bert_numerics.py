"""12-layer BERT chain: max rel diff vs the bf16-emulating fp64 model for
split-K on/off and PDL on/off (diagnostics)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
from paper_2210_12415_b200 import _abi
from paper_2210_12415_b200.e2e import build_bert as _bb, make_bert_inputs as _mb  # noqa: E402
class B:  # noqa: E302
    build = staticmethod(_bb)
    make_inputs = staticmethod(_mb)
from paper_2210_12415_b200.e2e import max_rel, reference  # noqa: E402
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for order in (0, 1):
    g, gmms, plan = B.build(layers, 64, order, flags=_abi.PLAN_DEFAULT)
    gen = torch.Generator(device="cuda"); gen.manual_seed(42)
    ins = B.make_inputs(g, gen)
    for k, x in ins.items():
        plan.set_input_device(k, x)
    plan.run()
    out = torch.tensor(plan.get_output("out"), device="cuda").view(128, 768)
    emu = reference(g, ins, frozenset(gmms), emulate=True)
    e = emu["out"]
    # per-layer drift
    drift = []
    for l in range(layers):
        tid = f"l{l + 1}_h" if l < layers - 1 else "out"
        try:
            got = torch.tensor(plan.get_output(tid), device="cuda").view(128, 768)
            drift.append(f"{max_rel(got, emu[tid]):.1e}")
        except Exception:
            drift.append("-")
    print(f"order={order} PDL={os.environ.get('LFGPU_PDL', '1')}: out max_rel {max_rel(out, e):.3g} |out| {float(e.abs().max()):.3g}; per layer: {' '.join(drift)}", flush=True)
