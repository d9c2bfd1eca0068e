"""Timeline of the tcgen05 launches of a chained plan (diagnostics): per
launch entry / PDL-wait release / first operand stage / epilogue done /
exit, relative to the first launch's entry. Direct launches (no graph)."""
import ctypes as C
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e, runtime  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(1)
if len(sys.argv) > 1 and sys.argv[1] == "resnet18":
    from paper_2210_12415_b200 import workloads
    fac = workloads.tune_resnet18(1, lambda sub: e2e.make_inputs(sub, gen))
    g, _, p = e2e.build_resnet18(1, fac, flags=0)
    ins = e2e.make_inputs(g, gen)
elif len(sys.argv) > 1 and sys.argv[1] == "encoder":  # packed-QKV encoder, 2 layers
    g, gm, p = e2e.build_encoder(2, 64, flags=0, packed_qkv=True)
    ins = e2e.make_encoder_inputs(g, gen)
else:
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    g, gm, p = e2e.build_bert(layers, 64, flags=0)
    ins = e2e.make_bert_inputs(g, gen)
for k, x in ins.items():
    p.set_input_device(k, x)
steps = {}
for i in range(len(g.nodes)):
    steps[i] = p.node_kernel(i)
for _ in range(3):
    p.run()
torch.cuda.synchronize()
n = 64
buf = torch.zeros(n * 8, dtype=torch.int64, device="cuda")
b = buf.view(n, 8)
b[:, 0] = b[:, 1] = b[:, 3] = torch.iinfo(torch.int64).max
runtime.lib().lfgpu_debug_chain_trace(C.c_void_p(buf.data_ptr()))
p.run()
torch.cuda.synchronize()
runtime.lib().lfgpu_debug_chain_trace(None)
t = buf.view(n, 8).cpu().numpy()
rows = [r for r in t if r[4] > 0]
t0 = rows[0][0]
prev_exit = None
print("launch  entry   wait-min wait-max first-data epi-done  exit   (us; gap = entry - previous exit)")
for i, r in enumerate(rows):
    f = lambda v: (v - t0) / 1e3
    gap = "" if prev_exit is None else "gap %.2f" % ((r[0] - prev_exit) / 1e3)
    print(f"{i:3d} {f(r[0]):8.2f} {f(r[1]):8.2f} {f(r[2]):8.2f} {f(r[3]):8.2f} {f(r[5]):8.2f} {f(r[4]):8.2f}  {gap}")
    prev_exit = r[4]
