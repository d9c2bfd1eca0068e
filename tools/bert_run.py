"""cfg5 CLI: sweep brick widths, build, check and time the BERT-base GEMM
chain (paper_2210_12415_b200.e2e).  python tools/bert_run.py [--layers 12] [--t 64]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import runtime, workloads  # noqa: E402
from paper_2210_12415_b200.e2e import build_bert as build, make_bert_inputs as make_inputs, max_rel, reference  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--t", type=int, nargs="*", default=[64, 128, 256])
    a = ap.parse_args()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(42)
    best = None
    for t in a.t:
        for order in (0, 1):
            try:
                g, gmms, plan = build(a.layers, t, order)
            except runtime.LfError as e:
                print(f"t={t} order={order}: {e}")
                continue
            m = plan.measure(warmup=5, reps=30, flush_l2=True)
            fl = workloads.BERT_FLOPS_PER_LAYER * a.layers
            print(f"t={t} order={order}: {m.cost:.1f} us ({m.kernels} launches) "
                  f"{fl / (m.cost * 1e-6) / 1e12:.1f} TFLOP/s | {plan.node_kernel(gmms[0])}", flush=True)
            if best is None or m.cost < best[0]:
                best = (m.cost, t, order)
            plan.close()
    _, t, order = best
    g, gmms, plan = build(a.layers, t, order)
    ins = make_inputs(g, gen)
    for k, x in ins.items():
        plan.set_input_device(k, x)
    plan.run()
    out = torch.tensor(plan.get_output("out"), device="cuda").view(128, 768)
    kinds = [plan.node_kernel(i) for i in range(len(g.nodes))]
    tc = frozenset(i for i, k in enumerate(kinds) if k.startswith("umma"))
    emu = reference(g, ins, tc, emulate=True)["out"]
    ex = reference(g, ins)["out"]
    print(f"best t={t} order={order}: {best[0]:.1f} us; out max_rel_diff vs bf16-emulating fp64 ref "
          f"{max_rel(out, emu):.3g}, vs exact fp64 ref {max_rel(out, ex):.3g}")
