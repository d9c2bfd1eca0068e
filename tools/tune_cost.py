import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2210_12415_b200 import _abi, ir, runtime, tuner
g = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
x = torch.randint(-64, 65, (16, 64, 56, 56), device="cuda").float() / 64
w = torch.randint(-64, 65, (64, 64, 3, 3), device="cuda").float() / 64
cands = tuner.conv_candidates(g, 1)[:60]
tb = tm = ts = 0
for c in cands:
    t0 = time.perf_counter()
    try:
        p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH)
    except runtime.LfError:
        continue
    t1 = time.perf_counter()
    p.set_input_device("x", x); p.set_input_device("ker", w)
    t2 = time.perf_counter()
    p.measure(warmup=2, reps=5, flush_l2=True)
    t3 = time.perf_counter()
    p.close()
    tb += t1 - t0; ts += t2 - t1; tm += t3 - t2
print(f"per candidate: build {tb/len(cands)*1e3:.2f} ms, set_input {ts/len(cands)*1e3:.2f} ms, measure {tm/len(cands)*1e3:.2f} ms")

g2 = ir.gemm(1024, 1024, 1024)
A = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
cands2 = tuner.gemm_candidates(1024, 1024, 1024)[:120]
for label in ("first", "second", "third with 512MB torch buffer", "fourth"):
    if label.startswith("third"):
        flush = torch.zeros(128 << 20, device="cuda")
    if label == "fourth":
        del flush
        torch.cuda.empty_cache()
    res, secs = tuner.sweep(g2, cands2, {"a": A, "b": A}, warmup=2, reps=5)
    print(f"gemm sweep ({label}): {len(cands2) / secs:.1f} candidates/s", flush=True)
