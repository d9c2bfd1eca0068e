"""Run the hot kernels a few times each for ncu (one GPU). Not a benchmark.

  ncu --set full -k regex:umma_kernel -c 2 python tools/profile_kernels.py gemm
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402
from paper_2210_12415_b200.layout import reorder, split  # noqa: E402


def k64(shape):
    return torch.randint(-64, 65, shape, device="cuda").float() / 64


def gemm(reps=3, factors=(128, 64, 1024), tile=64, order=0):
    g = ir.gemm(1024, 1024, 1024)
    c = tuner.Candidate({0: factors}, [runtime.sched(0, tile_last=tile, order=order)])
    p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC)
    p.set_input_device("a", k64((1024, 1024)))
    p.set_input_device("b", k64((1024, 1024)))
    print(p.node_kernel(0))
    for _ in range(reps):
        p.run()
    torch.cuda.synchronize()


def conv(reps=3, nb=16, factors=(56, 56, 64, 16, 16, 64)):
    g = ir.pad_conv(nb, 64, 64, 56, 3, 1, 1)
    c = tuner.Candidate({1: factors}, [runtime.sched(1)])
    p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC)
    p.set_input_device("x", k64((nb, 64, 56, 56)))
    p.set_input_device("ker", k64((64, 64, 3, 3)))
    print(p.node_kernel(0), "|", p.node_kernel(1))
    for _ in range(reps):
        p.run()
    torch.cuda.synchronize()


def transform(reps=3, n=64):
    x = k64((n, 64, 56, 56))
    y = torch.empty_like(x).view(-1)
    dims = [("N", n), ("C", 64), ("H", 56), ("W", 56)]
    for _ in range(reps):
        runtime.layout_convert(x, dims, [], [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])], y)
    torch.cuda.synchronize()


def gemm_split(reps=3):
    gemm(reps, (128, 64, 256), 128, 0)


def conv_trans(reps=3):
    g = ir.pad_conv(1, 512, 512, 7, 3, 1, 1)
    c = tuner.Candidate({1: (7, 7, 128, 64, 64, 128)}, [runtime.sched(1, unroll=2)])
    p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC)
    p.set_input_device("x", k64((1, 512, 7, 7)))
    p.set_input_device("ker", k64((512, 512, 3, 3)))
    print(p.node_kernel(1))
    for _ in range(reps):
        p.run()
    torch.cuda.synchronize()


def conv_halo(reps=3, nb=16, factors=(7, 14, 32, 32, 32, 32)):
    conv(reps, nb, factors)


def conv_b16best(reps=3):
    conv(reps, 16, (8, 28, 64, 32, 32, 64))


def transform_rotating(reps=12, n=64):
    """K1 back to back over 6 rotating source/destination pairs (617 MB, the
    bench's regime): profile a late launch with --cache-control none so the
    L2 write-backs of earlier destinations land in its DRAM counters."""
    pairs = [(k64((n, 64, 56, 56)), torch.empty(n * 64 * 56 * 56, device="cuda")) for _ in range(6)]
    dims = [("N", n), ("C", 64), ("H", 56), ("W", 56)]
    seq = [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])]
    for i in range(reps):
        x, y = pairs[i % 6]
        runtime.layout_convert(x, dims, [], seq, y)
    torch.cuda.synchronize()


def gemm_pair(reps=3):
    """cfg2 on the CTA-pair kernel (BN=128, 2 K splits over DSMEM)."""
    gemm(reps, (256, 64, 256), 128, 0)


def gemm_bench(reps=3):
    """cfg2 on the layout the r02 bench tuner picked (1-CTA BM=128 BN=64)."""
    gemm(reps, (512, 512, 256), 64, 0)


def gemm_bench_r03(reps=3):
    """cfg2 on the layout the round-2 final bench tuner picked (1-CTA BM=128
    BN=64, multi-slab KC=256)."""
    gemm(reps, (128, 1024, 128), 64, 1)


def gemm_bench_final(reps=3):
    """The round-2 final bench pick (m_t=256 k_t=64 n_t=128 tile=64 order=1)."""
    gemm(reps, (256, 64, 128), 64, 1)


def conv_b16_final(reps=3):
    """cfg1 b16 on the final round-2 bench pick (halo, resident weights, dual issuer)."""
    conv(reps, 16, (56, 28, 64, 32, 32, 64))


def conv_b16r02(reps=3):
    conv(reps, 16, (28, 28, 64, 32, 32, 64))


def conv_b1r02(reps=3):
    conv(reps, 1, (28, 2, 32, 32, 32, 32))


if __name__ == "__main__":
    which = sys.argv[1:] or ["gemm", "conv", "transform"]
    for w in which:
        globals()[w]()

