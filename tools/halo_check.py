import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle_lib as O
from paper_2210_12415_b200 import _abi, ir, runtime, tuner
for (nb, ci, co, h, f) in [(1, 64, 64, 56, (7, 14, 32, 32, 32, 32)), (1, 64, 64, 56, (8, 14, 64, 32, 32, 64)),
                          (1, 64, 64, 56, (4, 14, 64, 32, 32, 64)), (2, 128, 128, 28, (4, 14, 64, 64, 64, 64)),
                          (1, 64, 128, 28, (14, 14, 128, 32, 32, 128)), (2, 64, 64, 56, (8, 28, 64, 32, 32, 64)),
                          (1, 32, 64, 14, (14, 14, 64, 16, 16, 32)), (1, 256, 256, 14, (14, 14, 64, 64, 64, 64)),
                          (2, 256, 256, 14, (14, 7, 128, 64, 64, 128)), (1, 512, 512, 7, (7, 7, 64, 64, 64, 64)),
                          (1, 128, 128, 28, (28, 28, 32, 64, 64, 32))]:
    g = ir.pad_conv(nb, ci, co, h, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(f))
    bufs = O.random_inputs(g, 42)
    ins = {"x": bufs[0].copy(), "ker": bufs[1].copy()}
    O.reference_eval(g, bufs)
    try:
        p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
    except Exception as e:
        print(f, "plan error", e); continue
    for k, v in ins.items():
        p.set_input(k, v)
    p.run()
    y = p.get_output("y")
    bad = np.sum(y != bufs[3])
    print(f, "mismatches", int(bad), "of", y.size, "|", p.node_kernel(1)[:110])
