"""K per stage of the 1-CTA GEMM (LFGPU_GEMM_KCS = 64 / 128 / 256) on cfg2's
tuned brick layouts (diagnostics): per-launch time back to back (warm) and
cold, and the kernel summary."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for kcs in ("64", "128", "256"):
        env = dict(os.environ, LFGPU_GEMM_KCS=kcs)
        subprocess.run([sys.executable, __file__, "run"], env=env, check=False)
    sys.exit(0)

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

M = K = N = 1024
g = ir.gemm(M, K, N)
a = torch.randint(-64, 65, (M, K), device="cuda").float() / 64
b = torch.randint(-64, 65, (K, N), device="cuda").float() / 64
for fac, tl, order in (((128, 64, 64), 64, 0), ((128, 64, 64), 64, 1), ((128, 64, 128), 128, 0), ((128, 64, 128), 128, 1)):
    seqs = runtime.decode_layout(g, 0, list(fac))
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=tl, tile_second=128, order=order)], _abi.PLAN_REQUIRE_TC)
    p.set_input_device("a", a)
    p.set_input_device("b", b)
    p.run()
    ok = torch.equal(torch.tensor(p.get_output("c"), device="cuda").view(M, N), a @ b)
    warm = p.measure(warmup=3, reps=20, flush_l2=False).cost
    cold = p.measure(warmup=3, reps=20, flush_l2=True).cost
    print(f"KCS={os.environ.get('LFGPU_GEMM_KCS')} fac={fac} order={order}: warm {warm:.2f} us cold {cold:.2f} us exact={ok} | {p.node_kernel(0)}", flush=True)
    p.close()
