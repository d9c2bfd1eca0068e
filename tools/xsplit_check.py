import os, sys
R = __file__.rsplit("/tools/", 1)[0]; sys.path.insert(0, R); sys.path.insert(0, R + "/tests")
import numpy as np
import oracle_lib as O
from paper_2210_12415_b200 import _abi, ir, runtime
for (M, K, N, f, tl) in [(128, 768, 768, (128, 64, 64), 64), (128, 768, 768, (128, 128, 128), 128),
                         (128, 3072, 768, (128, 128, 128), 128), (128, 768, 3072, (128, 128, 128), 128),
                         (128, 3072, 768, (128, 64, 64), 64)]:
    g = ir.gemm(M, K, N)
    seqs = runtime.decode_layout(g, 0, list(f))
    bufs = O.random_inputs(g, 5)
    O.reference_eval(g, bufs)
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=tl)], flags=_abi.PLAN_REQUIRE_TC)
    p.set_input("a", bufs[0]); p.set_input("b", bufs[1]); p.run()
    got = p.get_output("c")
    print(M, K, N, f, p.node_kernel(0)[:150], "exact" if np.array_equal(got, bufs[2]) else "MISMATCH %g" % np.abs(got - bufs[2]).max())
# K-major B (one 128-row box for BN = 128) under the cluster exchange
from paper_2210_12415_b200.layout import reorder, split
for (M, K, N) in [(128, 768, 768), (128, 3072, 768)]:
    g = ir.gemm(M, K, N)
    seqs = runtime.decode_layout(g, 0, [128, 128, 128])
    seqs["b"] = [split(0, [K // 64, 64]), reorder([0, 2, 1])]
    bufs = O.random_inputs(g, 5)
    O.reference_eval(g, bufs)
    p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=128)], flags=_abi.PLAN_REQUIRE_TC)
    p.set_input("a", bufs[0]); p.set_input("b", bufs[1]); p.run()
    got = p.get_output("c")
    print(M, K, N, "bk", p.node_kernel(0)[:150], "exact" if np.array_equal(got, bufs[2]) else "MISMATCH %g" % np.abs(got - bufs[2]).max())
