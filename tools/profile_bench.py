"""The bench's timed kernels, a few launches each, for ncu (one GPU).
Not a benchmark. Layouts default to the last bench's tuned picks.
  ncu --set full -k regex:umma_kernel -c 2 python tools/profile_bench.py gemm
  ncu --metrics gpu__time_duration.sum --csv python tools/profile_bench.py all"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402
from paper_2210_12415_b200.layout import reorder, split  # noqa: E402


def k64(shape):
    return torch.randint(-64, 65, shape, device="cuda").float() / 64


def gemm(reps=3, f=(128, 1024, 64), tile=64, order=0):
    g = ir.gemm(1024, 1024, 1024)
    c = tuner.Candidate({0: f}, [runtime.sched(0, tile_last=tile, order=order)])
    p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC)
    p.set_input_device("a", k64((1024, 1024)))
    p.set_input_device("b", k64((1024, 1024)))
    print(p.node_kernel(0))
    for _ in range(reps):
        p.run()
    torch.cuda.synchronize()


def conv16(reps=3, f=(28, 28, 64, 32, 32, 64)):
    g = ir.bare_conv(16, 64, 64, 58, 3, 1)
    gp = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
    s = runtime.decode_layout(gp, 1, list(f))
    seqs = {"x": s["xp"], "ker": s["ker"], "y": s["y"]}
    p = runtime.Plan(g, seqs, [runtime.sched(0)], _abi.PLAN_REQUIRE_TC)
    p.set_input_device("x", k64((16, 64, 58, 58)))
    p.set_input_device("ker", k64((64, 64, 3, 3)))
    print(p.node_kernel(0))
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


def dep16(reps=3, f=(56, 28, 32, 32, 32)):
    """K6: depthwise 3x3 over 16x256x56x56 on channel-brick layouts."""
    g = ir.dep_chain(16, 256, 56, 3, 1, 1)
    seqs = runtime.decode_layout(g, 1, list(f))
    seqs["y"] = seqs["conv"]
    p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1)])
    p.set_input_device("x", k64((16, 256, 56, 56)))
    p.set_input_device("ker", k64((256, 3, 3)))
    print([p.node_kernel(i) for i in range(len(g.nodes))])
    for _ in range(reps):
        p.run()
    torch.cuda.synchronize()


if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    if which == ["all"]:
        which = ["gemm", "conv16", "transform"]
    for w in which:
        globals()[w]()
