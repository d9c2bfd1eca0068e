"""Breakdown of the drop-in host-buffer step (diagnostics): wall time of
lfgpu_plan_set_input (a, b), run, get_output (c) for the cfg2 GEMM plan,
median over reps, with the narrowed staging and with LFGPU_STAGE_F64."""
import os
import sys
import time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

M = K = N = 1024
g = ir.gemm(M, K, N)
seqs = runtime.decode_layout(g, 0, [128, 64, 64])
rng = np.random.default_rng(0)
a = rng.integers(-64, 65, M * K) / 64.0
b = rng.integers(-64, 65, K * N) / 64.0
c = np.empty(M * N)
for mode in ("narrow", "f64"):
    if mode == "f64":
        os.environ["LFGPU_STAGE_F64"] = "1"
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=64)], _abi.PLAN_DEFAULT)
    ts = {"set_a": [], "set_b": [], "run": [], "get_c": [], "step": []}
    for it in range(30):
        t0 = time.perf_counter(); p.set_input("a", a); t1 = time.perf_counter()
        p.set_input("b", b); t2 = time.perf_counter()
        p.run(); torch.cuda.synchronize(); t3 = time.perf_counter()
        p.get_output("c", out=c); t4 = time.perf_counter()
        if it >= 5:
            for k, v in zip(ts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
                ts[k].append(v * 1e3)
    print(mode, {k: round(float(np.median(v)), 4) for k, v in ts.items()}, "ms", flush=True)
    p.close()
    os.environ.pop("LFGPU_STAGE_F64", None)
print("threads", os.cpu_count())
