"""Layout-transform bandwidth probe: NCHW -> NCHWc16 (fp32, N=64) and the
identity copy through lfgpu_layout_convert vs torch. Diagnostics only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import runtime  # noqa: E402
from paper_2210_12415_b200.layout import reorder, split, unfold  # noqa: E402


def t(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph (the
    per-call host work - digit-map compilation - is outside the replay)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def cs():
    return torch.cuda.current_stream().cuda_stream


if __name__ == "__main__":
    n = int(os.environ.get("N", "64"))
    reps = int(os.environ.get("REPS", "20"))
    x = torch.randn(n, 64, 56, 56, device="cuda")
    y = torch.empty_like(x)
    xb = x.bfloat16()
    yb = torch.empty_like(xb)
    dims = [("N", n), ("C", 64), ("H", 56), ("W", 56)]
    c16 = [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])]
    c4 = [split(1, [16, 4]), reorder([0, 1, 3, 4, 2])]
    byts = 2 * x.numel() * 4
    cases = [
        ("torch clone", lambda: y.copy_(x), byts),
        ("torch permute NCHW->NCHWc16", lambda: y.view(n, 4, 56, 56, 16).copy_(
            x.view(n, 4, 16, 56, 56).permute(0, 1, 3, 4, 2)), byts),
        ("lfgpu identity", lambda: runtime.layout_convert(x, dims, [], [], y, stream=cs()), byts),
        ("lfgpu NCHW->NCHWc16", lambda: runtime.layout_convert(x, dims, [], c16, y, stream=cs()), byts),
        ("lfgpu NCHWc16->NCHW", lambda: runtime.layout_convert(x, dims, c16, [], y, stream=cs()), byts),
        ("lfgpu NCHW->NCHWc4", lambda: runtime.layout_convert(x, dims, [], c4, y, stream=cs()), byts),
        ("lfgpu bf16 NCHW->NCHWc16", lambda: runtime.layout_convert(xb, dims, [], c16, yb, stream=cs()), byts // 2),
    ]
    # K2: cfg1 b16 x (fp32 NCHW) -> padded, unfolded bf16 bricks of the C2D template
    from paper_2210_12415_b200 import ir
    gc = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
    xs = torch.randn(16, 64, 56, 56, device="cuda")
    for f in [(28, 14, 64, 32, 32, 64), (4, 14, 16, 16, 16, 16), (56, 2, 64, 16, 16, 64)]:
        xp_seq = runtime.decode_layout(gc, 1, list(f))["xp"]
        pd = runtime.derive_layout([("N", 16), ("I", 64), ("H", 58), ("W", 58)], xp_seq)
        nphys = 1
        for _, e in pd:
            nphys *= e
        xpd = torch.empty(nphys, dtype=torch.bfloat16, device="cuda")
        xdims = [("N", 16), ("I", 64), ("H", 56), ("W", 56)]
        nb = xs.numel() * 4 + nphys * 2
        cases.append((f"K2 pad->xp bf16 {f}",
                      lambda s=xp_seq, d=xpd: runtime.pad_convert(xs, xdims, 1, [], s, d, stream=cs()), nb))
    only = os.environ.get("ONLY")
    for name, fn, nb in cases:
        if only and only not in name:
            continue
        us = t(fn, reps)
        print(f"{name:32s} {us:8.2f} us  {nb / us / 1e3:8.1f} GB/s", flush=True)
    # correctness of the vectorised transforms against torch
    runtime.layout_convert(x, dims, [], c16, y)
    assert torch.equal(y.view(n, 4, 56, 56, 16), x.view(n, 4, 16, 56, 56).permute(0, 1, 3, 4, 2))
    runtime.layout_convert(x, dims, c16, [], y)
    assert torch.equal(y, x.view(n, 4, 56, 56, 16).permute(0, 1, 4, 2, 3).reshape(n, 64, 56, 56))
    print("ok")
