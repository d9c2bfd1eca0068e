"""cuDNN (torch.nn.functional.conv2d, bf16, fp32 accumulate) on the cfg1
conv shape at batch 1 / 16 — a yardstick for the tuned tcgen05 C2D numbers
in the bench line, never a path. Per-launch device time over back-to-back
launches: warm (one input) and cold (rotating inputs > 2x L2). NCHW and
channels_last layouts; prints one JSON line per case.

usage: python tools/cudnn_yardstick.py [--batch 1 16]
"""
import argparse
import json

import torch
import torch.nn.functional as F


def per_launch_us(fns, reps=50, warm=5):
    for i in range(warm):
        fns[i % len(fns)]()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000 + 60_000 * reps)  # host enqueues every launch before the GPU reaches them
    s.record()
    for i in range(reps):
        fns[i % len(fns)]()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 16])
    a = ap.parse_args()
    torch.backends.cudnn.benchmark = True
    C, H, K = 64, 56, 3
    for nb in a.batch:
        flops = 2.0 * nb * C * H * H * C * K * K
        for fmt in ("nchw", "channels_last"):
            mf = torch.channels_last if fmt == "channels_last" else torch.contiguous_format
            w = (torch.randint(-64, 65, (C, C, K, K), device="cuda").float() / 64).to(torch.bfloat16)
            w = w.contiguous(memory_format=mf)
            per = nb * C * H * H * 2 * 2  # input + output bytes (bf16)
            nrep = max(2, (256 << 20) // per + 1)
            xs = [(torch.randint(-64, 65, (nb, C, H, H), device="cuda").float() / 64).to(torch.bfloat16)
                  .contiguous(memory_format=mf) for _ in range(nrep)]
            warm = per_launch_us([lambda: F.conv2d(xs[0], w, padding=1)])
            cold = per_launch_us([(lambda x=x: F.conv2d(x, w, padding=1)) for x in xs], reps=max(50, len(xs)))
            print(json.dumps({"op": "cuDNN conv2d bf16 (yardstick)", "shape": f"N={nb} 64->64 3x3 s1 56^2 pad1",
                              "layout": fmt, "us_warm": round(warm, 3), "us_cold": round(cold, 3),
                              "tflops_warm": round(flops / warm / 1e6, 2),
                              "tflops_cold": round(flops / cold / 1e6, 2),
                              "rotating_inputs": len(xs)}), flush=True)


if __name__ == "__main__":
    main()
