"""Per-CTA phase timeline of the fused attention kernel (tensor-core path) in
one BERT-base layer's plan (diagnostics): entry, PDL release, operands
landed, scores done, softmax done, context done, exit."""
import ctypes as C
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e, ir, runtime  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(1)
g, gm, p = e2e.build_encoder(1, 64, flags=0, packed_qkv=True)
for k, x in e2e.make_encoder_inputs(g, gen).items():
    p.set_input_device(k, x)
p.run()
torch.cuda.synchronize()
buf = torch.zeros(8 * 4096, dtype=torch.int64, device="cuda")
runtime.lib().lfgpu_debug_umma_trace(C.c_void_p(buf.data_ptr()))
p.run()
torch.cuda.synchronize()
runtime.lib().lfgpu_debug_umma_trace(None)
t = buf[16384:].view(-1, 8).cpu().numpy()
t = t[t[:, 0] > 0][:96]
rel = (t - t[:, 0].min()) / 1e3
names = ["entry", "released", "landed", "scores", "softmax", "context", "exit"]
for i, n in enumerate(names):
    print(f"{n:9s} min {rel[:, i].min():6.2f} med {np.median(rel[:, i]):6.2f} max {rel[:, i].max():6.2f} us")
