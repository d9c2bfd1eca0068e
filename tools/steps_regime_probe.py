"""Per-launch time of the cfg2 bench plan back to back over R rotating
replicas for K timed steps (bench.time_plan_rotating), R x K grid — checks
that the headline regime does not depend on the step count (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402

f = tuple(int(x) for x in (sys.argv[1:4] or (256, 64, 128)))
g = ir.gemm(1024, 1024, 1024)
c = tuner.Candidate({0: f}, [runtime.sched(0, tile_last=64, order=1)])
A = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
B = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
ctx = runtime.context(0)
for R in (16, 32):
    reps = []
    for _ in range(R):
        p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
        p.set_input_device("a", A)
        p.set_input_device("b", B)
        reps.append(p)
    for K in (8, 20, 64, 200):
        for W in (5, 16):
            ms, wall = bench.time_plan_rotating(torch, reps, K, W, 1)
            print(f"R={R} K={K} W={W}: {ms / K * 1e3:.3f} us/launch (wall {wall * 1e3:.2f} ms) | {reps[0].node_kernel(0)[:60]}", flush=True)
    for p in reps:
        p.close()
