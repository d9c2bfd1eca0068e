"""Quick probe of the tcgen05 kernel: plan summary (store mode, split-K,
grid) and back-to-back device time for a few GEMM / C2D candidates.
Diagnostics only.  python tools/umma_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402


def k64(shape):
    return torch.randint(-64, 65, shape, device="cuda").float() / 64


def probe(g, cand, inputs, reps=20):
    p = runtime.Plan(g, tuner.seqs_for(g, cand), cand.scheds, _abi.PLAN_REQUIRE_TC)
    for k, v in inputs.items():
        p.set_input_device(k, v)
    for _ in range(3):
        p.run()
    torch.cuda.synchronize()
    s = torch.cuda.ExternalStream(p.stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        p.run()
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    m = p.measure(warmup=3, reps=20, flush_l2=True)
    summ = " | ".join(p.node_kernel(i) for i in range(len(g.nodes)) if p.node_kernel(i))
    p.close()
    return us, m.cost, summ


if __name__ == "__main__":
    g = ir.gemm(1024, 1024, 1024)
    A, B = k64((1024, 1024)), k64((1024, 1024))
    cfgs = [((128, 64, 1024), 64, 0), ((128, 64, 1024), 128, 0), ((128, 64, 1024), 128, 1),
            ((128, 64, 1024), 256, 0), ((128, 64, 1024), 256, 1), ((128, 1024, 1024), 64, 0),
            ((128, 64, 256), 256, 0), ((256, 1024, 256), 64, 0)]
    for f, tl, order in cfgs:
        c = tuner.Candidate({0: f}, [runtime.sched(0, tile_last=tl, order=order)])
        us, cold, summ = probe(g, c, {"a": A, "b": B})
        print(f"gemm {f} tile={tl} order={order}: b2b {us:7.2f} us  cold {cold:7.2f} us  "
              f"{2 * 1024**3 / us / 1e6:7.1f} TFLOP/s  [{summ}]")
    for nb, f in [(1, (7, 14, 16, 32, 32, 16)), (1, (4, 14, 64, 32, 32, 64)), (1, (8, 14, 64, 32, 32, 64)),
                  (16, (7, 14, 32, 32, 32, 32)), (16, (8, 14, 64, 32, 32, 64)), (16, (8, 28, 64, 32, 32, 64)),
                  (16, (4, 28, 64, 32, 32, 64))]:
        gc = ir.pad_conv(nb, 64, 64, 56, 3, 1, 1)
        c = tuner.Candidate({1: f}, [runtime.sched(1)])
        fl = 2.0 * nb * 64 * 64 * 56 * 56 * 9
        us, cold, summ = probe(gc, c, {"x": k64((nb, 64, 56, 56)), "ker": k64((64, 64, 3, 3))})
        print(f"conv b{nb} {f}: graph b2b {us:7.2f} us  cold {cold:7.2f} us  "
              f"{fl / us / 1e6:7.1f} TFLOP/s  [{summ}]")
