"""Where the cfg2 sustained floor comes from (diagnostics): our plan back
to back with R = 1/2/4/8/32 rotating replicas, burst (no pre-roll) and
sustained (pre-roll), and torch.matmul (cuBLAS bf16) in the same two
regimes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402

g = ir.gemm(1024, 1024, 1024)
c = tuner.Candidate({0: (512, 64, 256)}, [runtime.sched(0, tile_last=64, order=1)])
A = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
B = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
ctx = runtime.context(0)
for R in [int(x) for x in os.environ.get("FLOOR_R", "1 2 4 8 32").split()]:
    reps = []
    for _ in range(R):
        p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
        p.set_input_device("a", A)
        p.set_input_device("b", B)
        reps.append(p)
    for pre in (False, True):
        ms, _ = bench.time_plan_rotating(torch, reps, 64, 8, 1, preroll=pre)
        print(f"ours R={R} {'sustained' if pre else 'burst'}: {ms / 64 * 1e3:.3f} us/launch | {reps[0].node_kernel(0)[60:]}", flush=True)
    for p in reps:
        p.close()
ab, bb = A.to(torch.bfloat16), B.to(torch.bfloat16)
for R in (1, 32):
    xs = [(ab.clone(), bb.clone()) for _ in range(R)]
    fns = [(lambda x=x: torch.matmul(x[0], x[1])) for x in xs]
    burst = bench.time_rotating_fn(torch, fns, 20, 3)
    # sustained: 64 untimed calls right before the timed ones
    long = bench.time_rotating_fn(torch, fns, 200, 3)
    print(f"cuBLAS R={R}: 20 steps {burst:.3f} us/call, 200 steps {long:.3f} us/call", flush=True)
