"""Per-stage timeline of the CTA-pair GEMM (diagnostics only): stage period
seen by the MMA issuer, producer slot-acquire to data-landed latency, tile
period and epilogue duration. usage: python tools/pair_trace.py n [m_t k_t n_t]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
f = [int(x) for x in sys.argv[2:5]] if len(sys.argv) > 4 else [256, 64, 256]
g = ir.gemm(n, n, n)
seqs = runtime.decode_layout(g, 0, f)
x = (torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.float32) / 64)
y = (torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.float32) / 64)
p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
p.set_input_device("a", x)
p.set_input_device("b", y)
for _ in range(3):
    p.run()
torch.cuda.synchronize()
buf = torch.zeros(512 * 160, dtype=torch.int64, device="cuda")
runtime.lib().lfgpu_debug_umma_trace(C.c_void_p(buf.data_ptr()))
p2 = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
p2.set_input_device("a", x)
p2.set_input_device("b", y)
torch.cuda.synchronize()
if os.environ.get("TRACE_COLD"):
    fl = torch.zeros(64 << 20, device="cuda")
    fl.add_(1.0)
    fl.amax()
    torch.cuda.synchronize()
p2.run()
torch.cuda.synchronize()
runtime.lib().lfgpu_debug_umma_trace(None)
print(p2.node_kernel(0))
t = buf.cpu().numpy().reshape(-1, 512).astype(np.int64)
ncta = int((t[:, 320] != 0).sum())
t = t[:ncta]
t0 = t[t > 0].min()
ent = (t[:, 320] - t0) / 1e3
print("blob copied %.2f, tmem alloc done %.2f" % (np.median(t[:, 324] - t0) / 1e3, np.median(t[:, 325] - t0) / 1e3))
print("producer0: elected %.2f, tile coords %.2f, before first wait %.2f" % tuple(np.median(t[:, k] - t0) / 1e3 for k in (326, 327, 328)))
print("entry spread (us): min %.2f max %.2f; setup done %.2f; pdl wait done %.2f; exit max %.2f" % (
    ent.min(), ent.max(), np.median(t[:, 321] - t0) / 1e3, np.median(t[:, 322] - t0) / 1e3,
    (t[:, 323].max() - t0) / 1e3))
for cta in (0, 1, 2, 3, ncta // 2):
    r = t[cta]
    prod = r[0:64][r[0:64] > 0] - t0
    full = r[64:128][r[64:128] > 0] - t0
    ready = r[128:192][r[128:192] > 0] - t0
    done = r[192:256][r[192:256] > 0] - t0
    print(f"cta {cta}: producer acquire (us) first 12:", np.round(prod[:12] / 1e3, 2))
    if len(full):
        print("   mma full-wait done (us) first 12:", np.round(full[:12] / 1e3, 2))
        d = np.diff(full)
        print("   stage period median %.1f ns, p90 %.1f ns" % (np.median(d), np.percentile(d, 90)))
        k = min(len(prod), len(full))
        print("   acquire->landed latency median %.1f ns" % np.median(full[:k] - prod[:k]))
    ch = r[256:320]
    if (ch > 0).any():
        c = ch[ch > 0] - t0
        print("   tile0 chunks: ld/store stamps (us):", np.round(c[:16] / 1e3, 2))
    print("   tile ready (us):", np.round(ready[:6] / 1e3, 2), " epilogue done:", np.round(done[:6] / 1e3, 2))
