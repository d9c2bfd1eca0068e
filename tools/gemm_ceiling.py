"""Large-shape GEMM ceiling of the tcgen05 kernels vs torch.matmul (cuBLAS,
yardstick only). Prints one JSON line per shape: our kernel's per-launch
device time (CUDA events over back-to-back launches on the plan's stream)
and TFLOP/s, the same for torch bf16 matmul, and the fraction of the
MEASURED_PEAKS bf16 figure.

usage: python tools/gemm_ceiling.py [n ...] [--factors m_t k_t n_t] [--reps R]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 1590.0


def time_stream(fn, stream, reps, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)  # host enqueues all reps before the GPU reaches them
        s.record(stream)
        for _ in range(reps):
            fn()
        e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sizes", nargs="*", type=int, default=[1024, 2048, 4096, 8192])
    ap.add_argument("--factors", nargs=3, type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tile", type=int, default=1)
    ap.add_argument("--bk", action="store_true", help="K-major B ([K/64][N][64])")
    ap.add_argument("--nograph", action="store_true", help="plain launches instead of a CUDA graph per step")
    ap.add_argument("--cold", action="store_true", help="rotate over replicas > 2x L2 (cold operands)")
    a = ap.parse_args()
    pk = peak()
    for n in a.sizes:
        g = ir.gemm(n, n, n)
        f = a.factors or [256, 64, 256]
        seqs = runtime.decode_layout(g, 0, f)
        if a.bk:
            from paper_2210_12415_b200.layout import reorder, split
            seqs["b"] = [split(0, [n // 64, 64]), reorder([0, 2, 1])]
        p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=a.tile)], flags=_abi.PLAN_REQUIRE_TC | (0 if a.nograph else _abi.PLAN_CUDA_GRAPH))
        x = (torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.float32) / 64).contiguous()
        y = (torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.float32) / 64).contiguous()
        p.set_input_device("a", x)
        p.set_input_device("b", y)
        st = torch.cuda.ExternalStream(p.stream)
        reps = max(3, min(a.reps, int(2e12 / (2 * n ** 3)) + 3))
        plans = [p]
        if a.cold:  # replicas whose operands + results exceed 2x L2
            nrep = max(2, -(-(256 << 20) // (8 * n * n)))
            for _ in range(nrep - 1):
                q = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=a.tile)],
                                 flags=_abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH)
                q.set_input_device("a", x)
                q.set_input_device("b", y)
                plans.append(q)
            reps = max(reps, 2 * nrep)
        it = [0]
        for q in plans:  # instantiate every replica's CUDA graph before timing
            q.run(st.cuda_stream)
        torch.cuda.synchronize()

        def step():
            plans[it[0] % len(plans)].run(st.cuda_stream)
            it[0] += 1
        us = time_stream(step, st, reps)
        flop = 2.0 * n ** 3
        xb, yb = x.to(torch.bfloat16), y.to(torch.bfloat16)
        ts = torch.cuda.current_stream()
        tus = time_stream(lambda: torch.matmul(xb, yb), ts, reps)
        print(json.dumps({"n": n, "layout": f, "kernel": p.node_kernel(0), "us": round(us, 2),
                          "tflops": round(flop / us / 1e6, 1), "frac": round(flop / us / 1e6 / pk, 3),
                          "torch_us": round(tus, 2), "torch_tflops": round(flop / tus / 1e6, 1),
                          "peak": pk}), flush=True)
        p.close()


if __name__ == "__main__":
    main()
