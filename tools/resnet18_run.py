"""cfg4: ResNet-18 inference through one whole-graph plan.

Tunes per-conv layouts (workloads.tune_resnet18), builds the plan (fused
epilogues, CUDA graph), checks the logits against float64 torch references
(exact, and emulating the plan's numerics: bf16 operands on tensor-core
convs, fp32 storage), and times the plan.
  python tools/resnet18_run.py [--batch 1] [--no-tune]
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime, workloads  # noqa: E402


def k64(shape, gen, scale=1.0):
    return torch.randint(-64, 65, shape, generator=gen, device="cuda").float() / 64 * scale


def make_inputs(g, gen):
    """k/64 values; conv / FC weights scaled by a power of two ~ 1/sqrt(fan_in)
    so activations stay O(1) and every weight stays exact in bf16."""
    out = {}
    for t in g.tensors:
        if t.role not in (ir.INPUT, ir.CONSTANT):
            continue
        shape = t.extents
        if t.id.endswith("_w"):
            fan_in = math.prod(shape[1:]) if len(shape) == 4 else shape[0]
            out[t.id] = k64(shape, gen, 2.0 ** -round(math.log2(math.sqrt(fan_in))))
        elif t.id.endswith("_b"):
            out[t.id] = k64(shape, gen, 1.0 / 8)
        else:
            out[t.id] = k64(shape, gen)
    return out


def reference(g, ins, tc_nodes=frozenset(), emulate=False):
    """Float64 forward of the graph; with emulate, tensor-core contraction
    operands are rounded to bf16 and node outputs to fp32."""
    v = {k: x.double() for k, x in ins.items()}

    def rb(x):
        return x.bfloat16().double() if emulate else x

    def rf(x):
        return x.float().double() if emulate else x

    for i, nd in enumerate(g.nodes):
        a = [v[t] for t in nd.inputs]
        if nd.kind == ir.PADDING:
            p = nd.attr("pad", 0)
            r = F.pad(a[0], (p, p, p, p))
        elif nd.kind == ir.LAYOUT_CONVERT:
            r = a[0]
        elif nd.kind == ir.C2D:
            tc = i in tc_nodes
            r = rf(F.conv2d(rb(a[0]) if tc else a[0], rb(a[1]) if tc else a[1],
                            stride=nd.attr("stride", 1)))
        elif nd.kind == ir.GMM:
            tc = i in tc_nodes
            r = rf((rb(a[0]) if tc else a[0]) @ (rb(a[1]) if tc else a[1]))
        elif nd.kind == ir.BIASADD:
            r = rf(a[0] + (a[1].view(1, -1, 1, 1) if a[0].dim() == 4 else a[1].view(1, -1)))
        elif nd.kind == ir.EWADD:
            r = rf(a[0] + a[1])
        elif nd.kind == ir.RELU:
            r = a[0].clamp_min(0)
        elif nd.kind == ir.MAXPOOL:
            r = F.max_pool2d(a[0], nd.attr("window", 1), nd.attr("stride", 1))
        elif nd.kind == ir.GLOBAL_AVGPOOL:
            r = rf(a[0].mean(dim=(2, 3)))
        else:
            raise ValueError(nd.kind)
        v[nd.output] = r
    return v


def max_rel(a, b):
    s = torch.maximum(torch.ones_like(a), torch.maximum(a.abs(), b.abs()))
    return float(((a - b).abs() / s).max())


def build(n, factors, ctx=None):
    g, convs = workloads.resnet18(n)
    seqs = workloads.resnet18_seqs(g, convs, factors)
    scheds = [runtime.sched(c["node"], fuse=1) for c in convs]
    gi = len(g.nodes) - 2  # the FC GMM
    scheds.append(runtime.sched(gi, fuse=1))
    plan = runtime.Plan(g, seqs, scheds, _abi.PLAN_CUDA_GRAPH, ctx=ctx)
    return g, convs, plan


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
