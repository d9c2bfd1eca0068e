"""Per-CTA timeline of the tcgen05 kernel (lfgpu_debug_umma_trace) and a
copy-bandwidth calibration against torch. Diagnostics only."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402
from paper_2210_12415_b200.layout import reorder, split  # noqa: E402


def k64(shape):
    return torch.randint(-64, 65, shape, device="cuda").float() / 64


def timeline(g, cand, inputs, name):
    p = runtime.Plan(g, tuner.seqs_for(g, cand), cand.scheds, _abi.PLAN_REQUIRE_TC)
    for k, v in inputs.items():
        p.set_input_device(k, v)
    p.run()
    torch.cuda.synchronize()
    buf = torch.zeros(32 * 4096, dtype=torch.int64, device="cuda")
    runtime.lib().lfgpu_debug_umma_trace(C.c_void_p(buf.data_ptr()))
    p2 = runtime.Plan(g, tuner.seqs_for(g, cand), cand.scheds, _abi.PLAN_REQUIRE_TC)
    for k, v in inputs.items():
        p2.set_input_device(k, v)
    torch.cuda.synchronize()
    if os.environ.get("TRACE_COLD"):
        fl = torch.zeros(128 << 20, device="cuda")
        fl[: fl.numel() // 2].add_(1.0)
        fl[fl.numel() // 2:].amax()
        torch.cuda.synchronize()
    p2.run()
    torch.cuda.synchronize()
    runtime.lib().lfgpu_debug_umma_trace(None)
    allb = buf.cpu().numpy().astype(np.int64)
    nct = int((allb.reshape(-1, 32)[:, 0] != 0).sum())
    t16 = allb[: 32 * nct].reshape(-1, 32)
    if int(os.environ.get("LFGPU_UMMA_DIAG", "0")) & 256:
        st = [np.median(t16[:, 16 + k] - t16[:, 1]) / 1000.0 for k in range(16) if (t16[:, 16 + k] > 0).all()]
        print("  unit-0 stage landed (us after setup):", " ".join(f"{v:.2f}" for v in st))
    ck = [(np.median(t16[:, 20 + k] - t16[:, 0]) / 1000.0) for k in range(8) if (t16[:, 20 + k] > 0).all()]
    print("  unit-0 chunk ends (us):", " ".join(f"{v:.2f}" for v in ck))
    if (t16[:, 16] > 0).all() and not int(os.environ.get("LFGPU_UMMA_DIAG", "0")) & 256:
        sp = (t16[:, 16:20] - t16[:, :1]) / 1000.0
        print("  split-K: published %.2f fenced %.2f spin-done %.2f slices-landed %.2f us" %
              tuple(np.median(sp, axis=0)))
    if (t16[:, 28] > 0).all():
        print("  unit-0 first tmem_ld: issued %.2f done %.2f us after epi start" %
              (np.median((t16[:, 30] - t16[:, 8]) / 1000.0), np.median((t16[:, 28] - t16[:, 8]) / 1000.0)))
    if int(os.environ.get("LFGPU_UMMA_DIAG", "0")) & 32:
        w = (t16[:, 24:32] - t16[:, 8:9]) / 1000.0
        print("  epilogue warps 4..11 wake after warp 4 (us, median):", " ".join(f"{np.median(w[:, j]):.2f}" for j in range(8)))
        print("  tmem alloc/tfull ready (acc_ready) vs wake of last warp (us, median): %.2f" % np.median(w.max(axis=1)))
    elif (t16[:, 24] > 0).all():
        e0 = 9 if int(os.environ.get("LFGPU_UMMA_DIAG", "0")) & 16 else 8
        r = lambda k: np.median((t16[:, k] - t16[:, e0]) / 1000.0)
        print("  mode-2 chunk0 (us after epi start): waited %.2f ld %.2f staged %.2f barred %.2f | chunk1 waited %.2f"
              % (r(24), r(25), r(26), r(27), r(29)))
    t = t16[:, :8]
    ep = (t16[:, 8:16] - t16[:, :1]) / 1000.0
    for k in range(4):
        if (t16[:, 8 + k] > 0).all():
            print(f"  unit {k}: epi start med {np.median(ep[:, k]):.2f} end {np.median(ep[:, 4 + k]):.2f} us")
    # untraced kernel time (events, back-to-back launches of the same plan)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        p2.run()
    torch.cuda.synchronize()
    ev[0].record(torch.cuda.ExternalStream(p2.stream))
    for _ in range(20):
        p2.run()
    ev[1].record(torch.cuda.ExternalStream(p2.stream))
    torch.cuda.synchronize()
    print(f"  untraced back-to-back: {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.2f} us per launch")
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    labels = ["entry", "setup", "tma_done", "first_full", "mma_done", "acc_ready", "epi_done"]
    print(p2.node_kernel(len(g.nodes) - 1))
    print(f"== {name}: {len(t)} CTAs, kernel span {rel[:, 6].max():.2f} us")
    for i, l in enumerate(labels):
        print(f"  {l:10s} min {rel[:, i].min():7.2f}  med {np.median(rel[:, i]):7.2f}  max {rel[:, i].max():7.2f}")
    d = rel[:, 6] - rel[:, 0]
    print(f"  per-CTA duration med {np.median(d):.2f} max {d.max():.2f}")
    print(f"  setup {np.median(rel[:,1]-rel[:,0]):.2f}  first_full-setup {np.median(rel[:,3]-rel[:,1]):.2f}"
          f"  mma {np.median(rel[:,4]-rel[:,3]):.2f}  epi-after-mma {np.median(rel[:,6]-rel[:,4]):.2f}")


def copy_calib():
    n = 64
    x = k64((n, 64, 56, 56))
    y = torch.empty_like(x)
    dims = [("N", n), ("C", 64), ("H", 56), ("W", 56)]

    def t(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3
    byts = 2 * x.numel() * 4
    for name, fn in [
        ("torch clone", lambda: y.copy_(x)),
        ("torch permute NCHW->NCHWc16", lambda: y.view(n, 4, 56, 56, 16).copy_(x.view(n, 4, 16, 56, 56).permute(0, 1, 3, 4, 2))),
        ("lfgpu identity", lambda: runtime.layout_convert(x, dims, [], [], y)),
        ("lfgpu NCHW->NCHWc16", lambda: runtime.layout_convert(x, dims, [], [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])], y)),
    ]:
        us = t(fn)
        print(f"{name:32s} {us:8.2f} us  {byts / us / 1e3:8.1f} GB/s")


def resnet_b1():
    """The b1 ResNet-18 3x3 convs of stages 2-4 at the tuned bricks."""
    for (c, h, f) in [(128, 28, (28, 28, 16, 64, 64, 16)), (256, 14, (14, 14, 16, 64, 64, 16)),
                      (512, 7, (7, 7, 16, 64, 64, 16))]:
        gc = ir.pad_conv(1, c, c, h, 3, 1, 1)
        timeline(gc, tuner.Candidate({1: f}, [runtime.sched(1)]),
                 {"x": k64((1, c, h, h)), "ker": k64((c, c, 3, 3))}, f"conv b1 {c}@{h} {f}")


def single_cta():
    """One CTA, long K: per-stage TMA issue/landing cost with an idle chip."""
    for (M, K, N, f, tl) in [(128, 4096, 64, (128, 64, 64), 64), (128, 4096, 16, (128, 64, 16), 16),
                             (128, 4096, 256, (128, 64, 256), 256)]:
        g = ir.gemm(M, K, N)
        timeline(g, tuner.Candidate({0: f}, [runtime.sched(0, tile_last=tl)]),
                 {"a": k64((M, K)), "b": k64((K, N))}, f"gemm 1-CTA {M}x{K}x{N} {f}")


if __name__ == "__main__":
    if os.environ.get("TRACE_SINGLE"):
        single_cta()
        sys.exit(0)
    if os.environ.get("TRACE_RESNET"):
        resnet_b1()
        sys.exit(0)
    if os.environ.get("TRACE_CONV_VARIANTS"):
        gc = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
        ins = {"x": k64((16, 64, 56, 56)), "ker": k64((64, 64, 3, 3))}
        for f, sc in [((28, 28, 64, 64, 64, 64), runtime.sched(1, vectorize=1)),
                      ((28, 28, 64, 32, 32, 64), runtime.sched(1, vectorize=1, unroll=1)),
                      ((14, 28, 64, 32, 32, 64), runtime.sched(1, vectorize=1))]:
            try:
                timeline(gc, tuner.Candidate({1: f}, [sc]), ins, f"conv b16 {f} unroll={sc.unroll}")
            except Exception as e:
                print("FAILED", f, e)
        gg = ir.gemm(50176, 576, 64)
        for f, tl in [((128, 64, 64), 64), ((128, 32, 64), 64)]:
            timeline(gg, tuner.Candidate({0: f}, [runtime.sched(0, tile_last=tl, order=1)]),
                     {"a": k64((50176, 576)), "b": k64((576, 64))}, f"gemm 50176x576x64 {f}")
        sys.exit(0)
    if os.environ.get("TRACE_INGEST"):  # main-loop time per tile vs number of CTAs pulling
        for M in (256, 512, 1024):
            g = ir.gemm(M, 1024, 1024)
            timeline(g, tuner.Candidate({0: (128, 1024, 64)}, [runtime.sched(0, tile_last=64, order=1)]),
                     {"a": k64((M, 1024)), "b": k64((1024, 1024))}, f"gemm {M}x1024x1024 BN=64")
        sys.exit(0)
    if os.environ.get("TRACE_CONV_ONLY"):
        gc = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
        f = (28, 28, 64, 32, 32, 64)
        timeline(gc, tuner.Candidate({1: f}, [runtime.sched(1)]),
                 {"x": k64((16, 64, 56, 56)), "ker": k64((64, 64, 3, 3))}, f"conv b16 {f}")
        sys.exit(0)
    g = ir.gemm(1024, 1024, 1024)
    A, B = k64((1024, 1024)), k64((1024, 1024))
    for f, tl, o in [((128, 1024, 64), 64, 0), ((128, 64, 256), 128, 0)]:
        timeline(g, tuner.Candidate({0: f}, [runtime.sched(0, tile_last=tl, order=o)]), {"a": A, "b": B},
                 f"gemm {f} tile {tl} order {o}")
    if os.environ.get("TRACE_GEMM_ONLY"):
        sys.exit(0)
    if os.environ.get("TRACE_TINY"):  # fixed per-kernel cost: one 128x64 tile, one K stage
        gt = ir.gemm(128, 64, 64)
        timeline(gt, tuner.Candidate({0: (128, 64, 64)}, [runtime.sched(0, tile_last=64, order=1)]),
                 {"a": k64((128, 64)), "b": k64((64, 64))}, "gemm 128x64x64 (1 tile, 1 stage)")
        sys.exit(0)
    gc = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
    for f in [(28, 28, 64, 32, 32, 64), (8, 14, 64, 32, 32, 64), (7, 14, 32, 32, 32, 32)]:
        timeline(gc, tuner.Candidate({1: f}, [runtime.sched(1)]),
                 {"x": k64((16, 64, 56, 56)), "ker": k64((64, 64, 3, 3))}, f"conv b16 {f}")
