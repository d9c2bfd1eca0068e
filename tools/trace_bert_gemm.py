"""Per-CTA timeline of one BERT-chain GEMM (M=128, K=768, N=768, 64-bricks),
with and without split-K (diagnostics)."""
import os
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import trace_umma as T  # noqa: E402
from paper_2210_12415_b200 import ir, runtime, tuner  # noqa: E402

for (M, K, N) in [(128, 768, 768), (128, 3072, 768)]:
    g = ir.gemm(M, K, N)
    for order in (0, 1):
        T.timeline(g, tuner.Candidate({0: (128, 64, 64)}, [runtime.sched(0, tile_last=64, order=order)]),
                   {"a": T.k64((M, K)), "b": T.k64((K, N))}, f"bert gemm {M}x{K}x{N} order={order}")
