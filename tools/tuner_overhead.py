"""Where a tuner measurement's time goes (diagnostics): plan build, input
conversion, device measurement, teardown — cfg2 and cfg1 candidates."""
import sys
import time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402

ctx = runtime.context(0)
for name, g, cands, ins in [
    ("cfg2", ir.gemm(1024, 1024, 1024), tuner.gemm_candidates(1024, 1024, 1024),
     {"a": torch.rand(1024, 1024, device="cuda"), "b": torch.rand(1024, 1024, device="cuda")}),
    ("cfg1", ir.pad_conv(1, 64, 64, 56, 3, 1, 1), None,
     {"x": torch.rand(1, 64, 56, 56, device="cuda"), "ker": torch.rand(64, 64, 3, 3, device="cuda")})]:
    if cands is None:
        cands = tuner.conv_candidates(g, 1)
    cands = cands[:60]
    tb = ti = tm = tc = 0.0
    for warm in (True, False):
        for c in cands[:5] if warm else cands:
            t0 = time.perf_counter()
            try:
                p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_CUDA_GRAPH, ctx=ctx)
            except runtime.LfError:
                continue
            t1 = time.perf_counter()
            for k, v in ins.items():
                p.set_input_device(k, v)
            t2 = time.perf_counter()
            m = p.measure(warmup=2, reps=5, flush_l2=True)
            t3 = time.perf_counter()
            p.close()
            t4 = time.perf_counter()
            if not warm:
                tb += t1 - t0; ti += t2 - t1; tm += t3 - t2; tc += t4 - t3
    n = len(cands)
    print(f"{name}: per candidate ms: build {tb / n * 1e3:.2f} inputs {ti / n * 1e3:.2f} "
          f"measure {tm / n * 1e3:.2f} close {tc / n * 1e3:.2f} -> {n / (tb + ti + tm + tc):.1f} cand/s")
