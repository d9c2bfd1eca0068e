"""Per-CTA unit cadence of the stem GEMM at batch 64 (1-CTA tcgen05 kernel,
~48 tiles per CTA) from the kernel's debug stamps (diagnostics)."""
import ctypes as C
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, workloads, runtime, e2e  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
b = workloads.Builder()
x = b.t("x", [("N", nb), ("C", 3), ("H", 224), ("W", 224)], ir.INPUT)
xp = b.t("xp", [("N", nb), ("C", 3), ("H", 230), ("W", 230)])
b.op(ir.PADDING, [x], xp, pad=3)
w = b.t("stem_w", [("O", 64), ("I", 3), ("KH", 7), ("KW", 7)], ir.CONSTANT)
y = b.t("y", [("N", nb), ("C", 64), ("H", 112), ("W", 112)])
b.op(ir.C2D, [xp, w], y, stride=2)
if "nobias" in sys.argv:
    yr = b.t("yr", [("N", nb), ("C", 64), ("H", 112), ("W", 112)], ir.OUTPUT)
    b.op(ir.RELU, [y], yr)
else:
    bias = b.t("stem_b", [("O", 64)], ir.CONSTANT)
    yb = b.t("yb", [("N", nb), ("C", 64), ("H", 112), ("W", 112)])
    b.op(ir.BIASADD, [y, bias], yb)
    yr = b.t("yr", [("N", nb), ("C", 64), ("H", 112), ("W", 112)], ir.OUTPUT)
    b.op(ir.RELU, [yb], yr)
g = b.g
gen = torch.Generator(device="cuda")
gen.manual_seed(3)
p = runtime.Plan(g, {}, [runtime.sched(1, fuse=1)], 0)
for k, v in e2e.make_inputs(g, gen).items():
    p.set_input_device(k, v)
p.run()
torch.cuda.synchronize()
print(p.node_kernel(1))
buf = torch.zeros(32 * 4096, dtype=torch.int64, device="cuda")
runtime.lib().lfgpu_debug_umma_trace(C.c_void_p(buf.data_ptr()))
p.run()
torch.cuda.synchronize()
runtime.lib().lfgpu_debug_umma_trace(None)
t = buf.view(-1, 32).cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
r = (t - t0) / 1e3
print("CTAs", len(t))
for name, col in (("entry", 0), ("setup", 1), ("tma_done", 2), ("first_full", 3), ("acc0_ready", 5), ("epi_done", 6)):
    print(f"{name:10s} med {np.median(r[:, col]):8.2f} max {r[:, col].max():8.2f}")
for i in range(4):
    print(f"unit {i}: epi start med {np.median(r[:, 8 + i]):7.2f}  end med {np.median(r[:, 12 + i]):7.2f}")
if (t[:, 24] > 0).all():
    rr = lambda k: np.median((t[:, k] - t[:, 8]) / 1e3)
    print("mode-2 unit-0 chunk0 (us after epi start): waited %.2f ld %.2f staged %.2f barred %.2f | chunk1 waited %.2f"
          % (rr(24), rr(25), rr(26), rr(27), rr(29)))
ck = [np.median((t[:, 20 + k] - t[:, 8]) / 1e3) for k in range(8) if (t[:, 20 + k] > 0).all()]
print("unit-0 chunk ends (us after epi start):", " ".join(f"{v:.2f}" for v in ck))
