"""Channels-as-rows halo C2D (schedule unroll=2) vs the default
orientation: bit-exactness against the oracle and cold device time."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_lib as O
from paper_2210_12415_b200 import _abi, ir, runtime
cases = [(1, 128, 128, 28, (28, 28, 128, 64, 64, 128)), (1, 256, 256, 14, (14, 14, 128, 64, 64, 128)),
         (1, 128, 128, 14, (14, 14, 128, 64, 64, 128)), (1, 512, 512, 7, (7, 7, 128, 64, 64, 128)),
         (1, 256, 256, 14, (14, 14, 256, 64, 64, 256)), (1, 512, 512, 7, (7, 7, 512, 64, 64, 512)),
         (1, 64, 128, 7, (7, 7, 128, 32, 32, 128))]
for (nb, ci, co, h, f) in cases:
    g = ir.pad_conv(nb, ci, co, h, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(f))
    bufs = O.random_inputs(g, 42)
    ins = {"x": bufs[0].copy(), "ker": bufs[1].copy()}
    O.reference_eval(g, bufs)
    for unroll in (2, 0):
        try:
            p = runtime.Plan(g, seqs, [runtime.sched(1, unroll=unroll, fuse=1)], flags=_abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH)
        except Exception as e:
            print(nb, ci, co, h, f, f"unroll={unroll}: plan error {e}")
            continue
        for k, v in ins.items():
            p.set_input(k, v)
        p.run()
        y = p.get_output("y")
        bad = int(np.sum(y != bufs[3]))
        m = p.measure(warmup=3, reps=20, flush_l2=True)
        k = p.node_kernel(1)
        print(nb, ci, co, h, f, f"unroll={unroll}: mismatches {bad}/{y.size}  {m.cost:.2f} us | {k[:40]} .. {k[k.find('BN='):][:80]}", flush=True)
        p.close()
