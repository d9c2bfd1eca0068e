"""cfg3: tune + verify + time every ResNet-50 conv shape on the GPU.

For each shape: GPU-measured sweep over the C2D template candidates
(tuner.conv_candidates), then the winner is verified against a float64
torch conv on the device (exact when I*KH*KW <= 4096, else 1e-5 relative,
SURVEY.md §8c) and timed (graph and C2D kernel alone).
  python tools/cfg3_sweep.py [--batch 1] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, runtime, tuner, workloads  # noqa: E402


def k64(shape):
    return torch.randint(-64, 65, shape, device="cuda").float() / 64


def run_shape(name, nb, ci, co, h, k, s, p, verbose=True):
    g, node = workloads.conv_graph(nb, ci, co, h, k, s, p)
    x = k64((nb, ci, h, h))
    w = k64((co, ci, k, k))
    ins = {"x": x, "ker": w}
    cands = tuner.conv_candidates(g, node)
    t0 = time.perf_counter()
    res, _ = tuner.sweep(g, cands, ins, warmup=1, reps=3)
    ts = time.perf_counter() - t0
    br = tuner.best(res)
    flops = workloads.conv_flops(nb, ci, co, h, k, s, p)
    if br is not None:
        plan = runtime.Plan(g, tuner.seqs_for(g, br.candidate), br.candidate.scheds,
                            _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH)
        label = br.candidate.label
    else:
        plan = runtime.Plan(g, {}, [runtime.sched(node)], _abi.PLAN_CUDA_GRAPH)
        label = "logical layout (no tensor-core candidate)"
    for tid, v in ins.items():
        plan.set_input_device(tid, v)
    plan.run()
    y = torch.tensor(plan.get_output("y"), device="cuda")
    ref = torch.nn.functional.conv2d(x.double(), w.double(), stride=s, padding=p).flatten()
    if ci * k * k <= 4096:
        ok = bool(torch.equal(y, ref))
        err = float((y - ref).abs().max())
    else:
        sc = torch.maximum(torch.ones_like(ref), torch.maximum(y.abs(), ref.abs()))
        err = float(((y - ref).abs() / sc).max())
        ok = err <= 1e-5
    m = plan.measure(warmup=3, reps=20, flush_l2=True)
    kern = " | ".join(plan.node_kernel(i) for i in range(len(g.nodes)))
    plan.close()
    row = {"shape": name, "batch": nb, "gflop": round(flops / 1e9, 4), "layout": label,
           "candidates": len(res), "legal": sum(r.cost_us is not None for r in res),
           "tune_s": round(ts, 2), "us": round(m.cost, 3),
           "tflops": round(flops / (m.cost * 1e-6) / 1e12, 2), "exact_or_tol": ok,
           "max_err": err, "kernels": kern}
    if verbose:
        print(f"{name:20s} b{nb:<3d} {row['us']:9.2f} us {row['tflops']:8.2f} TF/s "
              f"ok={ok} err={err:.2g} legal={row['legal']}/{row['candidates']} {label}", flush=True)
    return row


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1])
    ap.add_argument("--json", default=None)
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    rows = []
    for nb in a.batch:
        for sh in workloads.RESNET50_CONVS:
            if a.only and a.only not in sh[0]:
                continue
            try:
                rows.append(run_shape(sh[0], nb, *sh[1:]))
            except Exception as e:  # report and continue: this is a survey tool
                print(f"{sh[0]:20s} b{nb}: FAILED {type(e).__name__}: {e}", flush=True)
                rows.append({"shape": sh[0], "batch": nb, "error": str(e)})
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)
