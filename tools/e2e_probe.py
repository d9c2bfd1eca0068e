import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2210_12415_b200 import _abi, ir, runtime
sys.argv = ["x"]
import bench
g = ir.gemm(1024, 1024, 1024)
seqs = runtime.decode_layout(g, 0, [256, 64, 256])
p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=128)], flags=_abi.PLAN_REQUIRE_TC)
A = (torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64)
B = (torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64)
dt, ok = bench.e2e_capi(p, A, B, 1024, 1024, 1024, 20)
print("e2e ms", dt * 1e3, ok, "TF/s", 2 * 1024**3 / dt / 1e12)
a = A.double().cpu().numpy().ravel().copy()
t0 = time.perf_counter()
for _ in range(20): p.set_input("a", a)
print("set_input ms", (time.perf_counter() - t0) / 20 * 1e3)
c = np.empty(1024 * 1024)
t0 = time.perf_counter()
for _ in range(20): p.get_output("c", out=c)
print("get_output ms", (time.perf_counter() - t0) / 20 * 1e3)
