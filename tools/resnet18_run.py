"""cfg4 CLI: tune, build, check and time ResNet-18 inference
(paper_2210_12415_b200.e2e).  python tools/resnet18_run.py [--batch 1] [--no-tune]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import workloads  # noqa: E402
from paper_2210_12415_b200.e2e import build_resnet18 as build, make_inputs, max_rel, reference  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-tune", action="store_true")
    a = ap.parse_args()
    n = a.batch
    gen = torch.Generator(device="cuda")
    gen.manual_seed(42)
    t0 = time.perf_counter()
    if a.no_tune:
        factors = {}
    else:
        factors = workloads.tune_resnet18(
            n, lambda sub: make_inputs(sub, gen), log=lambda s: print("  " + s, flush=True))
    print(f"tuning {time.perf_counter() - t0:.1f} s", flush=True)
    g, convs, plan = build(n, factors)
    ins = make_inputs(g, gen)
    for k, x in ins.items():
        plan.set_input_device(k, x)
    plan.run()
    out = torch.tensor(plan.get_output("logits"), device="cuda").view(n, -1)
    kinds = [plan.node_kernel(i) for i in range(len(g.nodes))]
    tc = frozenset(i for i, k in enumerate(kinds) if k.startswith("umma"))
    from collections import Counter
    print("kernels:", dict(Counter(kinds)))
    emu = reference(g, ins, tc, emulate=True)["logits"]
    ex = reference(g, ins)["logits"]
    print(f"logits max_rel_diff vs bf16-emulating fp64 ref: {max_rel(out, emu):.3g}; "
          f"vs exact fp64 ref: {max_rel(out, ex):.3g}; |logits| max {float(ex.abs().max()):.3g}")
    m = plan.measure(warmup=5, reps=30, flush_l2=True)
    print(f"batch {n}: {m.cost:.1f} us per inference step ({m.kernels} launches), "
          f"{3.628e9 * n / (m.cost * 1e-6) / 1e12:.2f} TFLOP/s")
