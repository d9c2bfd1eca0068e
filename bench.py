"""bench.py — B200 benchmark of the ALT hot path (BASELINE.json).

Headline (configs[1]): GEMM 1024x1024x1024 on tuned tiled/reordered operand
layouts, TFLOP/s. A "step" is one execution of the tuned GMM plan on bf16
bricks already resident in HBM; K steps run back to back rotating over
operand replicas larger than 2x L2, one CUDA event pair around them. The
tuning itself (GPU-measured candidate sweep over the GMM layout template x
loop tile) runs before the timed region.

Also on the same line:
  e2e                 the drop-in C-ABI call with host doubles (the
                      reference's BufferMap): set_input(a, b) + run +
                      get_output(c) per step, copies inside the step;
  e2e_pipelined_fp32  the same GEMM behind a pipelined fp32 serving loop;
  roofline            the GEMM kernel against the measured bf16 peak;
  c2d_cfg1            BASELINE's "tuned C2D TFLOP/s" (cfg1 b1 / b16): tuned
                      layout, warm and cold-L2 timings, its own roofline and
                      the reference's C2D reference_eval as cpu_baseline;
  layout_transform_*  NCHW->NCHWc16 GB/s over rotating buffers > 4x L2, with
                      the reference's materialize_tensor as cpu_baseline;
  tuner               GPU candidates/s with the reference's simulate_cache
                      as cpu_baseline;
  secondary           cfg4 ResNet-18 (b1, b64 batch-sharded), cfg5 BERT chain;
  cpu_baseline        the reference's GEMM reference_eval on this host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun each rank runs its own replica (weak scaling, no collective
on the data path; only the timing max-reduce).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback"


# ---------------------------------------------------------------------------
# distributed plumbing (barrier + max over ranks only)

def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm

def kmul64(torch, shape, gen, device):
    """Synthetic k/64 values in [-1, 1] (the reference's input distribution,
    interp.cpp:497-498), generated on the device."""
    return (torch.randint(-64, 65, shape, generator=gen, device=device).float() / 64.0)


def time_plan_steps(torch, plan, steps, warmup, flush_buf, world):
    """Per-step CUDA events on the plan's stream; L2 flushed between steps."""
    s = torch.cuda.ExternalStream(plan.stream)
    for _ in range(warmup):
        plan.run()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    half = flush_buf.numel() // 2
    for a, b in evs:
        with torch.cuda.stream(s):
            flush_buf[:half].add_(1.0)     # > L2 write between timed steps ...
            flush_buf[half:].amax()         # ... then a > L2 read: cold, clean L2
            a.record(s)
        plan.run()
        with torch.cuda.stream(s):
            b.record(s)
    torch.cuda.synchronize()
    barrier(world)
    wall = time.perf_counter() - t_wall
    per = [a.elapsed_time(b) for a, b in evs]  # ms
    return per, wall


def time_plan_rotating(torch, plans, steps, warmup, world, preroll=True):
    """K back-to-back steps, step i on replica plans[i % R]. The replicas'
    operand + result buffers together exceed 2x the 126 MB L2, so every step
    reads operands that are not L2-resident (the 'inputs larger than L2'
    rule) while no flush kernel sits between timed steps. One event pair on
    the plans' shared stream brackets the K steps.

    Steady state: the timed steps follow, with no gap, a pre-roll of
    max(32, R) untimed steps, so the L2 is already full of earlier steps'
    dirty results when timing starts and every timed step pays the
    write-backs it causes. Without the pre-roll the first ~30 steps' 4 MB
    results sit in the L2 and are written back after the end event: the
    cfg2 per-launch time then grew with K (9.4 us at K=20, 10.8 at 64, 11.8
    at 200; tools/steps_regime_probe.py)."""
    s = torch.cuda.Stream()
    for i in range(max(warmup, len(plans))):
        plans[i % len(plans)].run(s.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pre = max(32, len(plans)) if preroll else 0
    barrier(world)
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    with torch.cuda.stream(s):
        # A device-side sleep (~1 ms + ~30 us per step) lets the host enqueue
        # the pre-roll and all K steps before the GPU reaches them, so the
        # timed region holds back-to-back device work, not host launch gaps.
        torch.cuda._sleep(2_000_000 + 60_000 * (pre + steps))
    for i in range(pre):
        plans[i % len(plans)].run(s.cuda_stream)
    with torch.cuda.stream(s):
        a.record(s)
    for i in range(steps):
        plans[(pre + i) % len(plans)].run(s.cuda_stream)
    with torch.cuda.stream(s):
        b.record(s)
    torch.cuda.synchronize()
    barrier(world)
    wall = time.perf_counter() - t_wall
    return a.elapsed_time(b), wall


def time_rotating_fn(torch, fns, steps, warmup):
    """K back-to-back calls fns[i % R]() on the current stream, one event
    pair around all K (inputs rotate over R sets larger than L2)."""
    for i in range(max(warmup, len(fns))):
        fns[i % len(fns)]()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pre = len(fns)  # untimed pre-roll right before the start: steady-state L2 write-backs
    torch.cuda._sleep(2_000_000 + 60_000 * (pre + steps))
    for i in range(pre):
        fns[i % len(fns)]()
    a.record()
    for i in range(steps):
        fns[(pre + i) % len(fns)]()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / steps  # us per call


def transform_bench(torch, gen, dev, ctx, pk, steps):
    """NCHW -> NCHWc16 fp32 at N=64 (K1): back-to-back conversions rotating
    over 6 (source, destination) pairs of 51.4 MB each — 617 MB, > 4x the
    126 MB L2 — so every conversion reads its source from and writes its
    destination back to HBM (the write-backs of one step land in the next
    ones, as in a stream of conversions)."""
    from paper_2210_12415_b200 import runtime
    from paper_2210_12415_b200.layout import reorder, split
    Nn = 64
    dims = [("N", Nn), ("C", 64), ("H", 56), ("W", 56)]
    seq = [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])]
    pairs = [(kmul64(torch, (Nn, 64, 56, 56), gen, dev), torch.empty(Nn * 64 * 56 * 56, device=dev))
             for _ in range(6)]
    fns = [(lambda x=x, y=y: runtime.layout_convert(x, dims, [], seq, y, ctx=ctx)) for x, y in pairs]
    us = time_rotating_fn(torch, fns, max(steps, 12), 6)
    byts = 2 * pairs[0][0].numel() * 4
    gbs = byts / (us * 1e-6) / 1e9
    # parity of the benchmarked conversion against the oracle's K1 restatement
    # is covered by tests/test_gpu_convert.py; here: a size-independent check
    # (the NCHWc16 buffer is a permutation of the source: same sum / sum of squares)
    x, y = pairs[0]
    fns[0]()
    torch.cuda.synchronize()
    ok = bool(torch.equal(y.view(Nn, 4, 56, 56, 16), x.view(Nn, 4, 16, 56, 56).permute(0, 1, 3, 4, 2)))
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_transform_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    return {"bytes": byts, "us": round(us, 2), "GB_per_s": round(gbs, 1),
            "frac_of_hbm": round(gbs / pk["hbm_gbs"], 4), "verified_exact": ok,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(gbs / pk["hbm_gbs"], 4), "traffic": traffic,
                         "kernel": "digit_transpose_vec (K1)",
                         "algorithmic": f"{byts} B per launch (source read + destination write)"},
            "l2": "6 rotating source/destination pairs, 617 MB (> 4x L2), back to back"}


def c2d_bench(torch, gen, dev, ctx, pk, nb):
    """cfg1 C2D (Padding -> C2D 64->64 3x3, 56x56) at batch nb: GPU-tuned
    layout, whole plan (K2 padding conversion + tcgen05 conv) and the conv
    kernel alone, warm (K back-to-back executions per event pair) and cold
    (each execution after a 1.5x-L2 read, that read's time subtracted)."""
    from paper_2210_12415_b200 import _abi, ir, runtime, tuner
    gc = ir.pad_conv(nb, 64, 64, 56, 3, 1, 1)
    x = kmul64(torch, (nb, 64, 56, 56), gen, dev)
    w = kmul64(torch, (64, 64, 3, 3), gen, dev)
    cc = tuner.conv_candidates(gc, 1)
    t0 = time.perf_counter()
    rc, _ = tuner.sweep(gc, cc, {"x": x, "ker": w}, warmup=2, reps=3, ctx=ctx)
    ts = time.perf_counter() - t0
    br = tuner.best(rc)
    pc = runtime.Plan(gc, tuner.seqs_for(gc, br.candidate), br.candidate.scheds,
                      _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
    pc.set_input_device("x", x)
    pc.set_input_device("ker", w)
    mw = pc.measure(warmup=5, reps=15, flush_l2=False)
    mc = pc.measure(warmup=3, reps=9, flush_l2=True)
    fl = 2.0 * nb * 64 * 64 * 56 * 56 * 9
    # the C2D kernel alone, on the tuned (padded, unfolded) input layout
    gk = ir.bare_conv(nb, 64, 64, 58, 3, 1)
    seqs_k = tuner.seqs_for(gc, br.candidate)
    seqk = {"x": seqs_k.get("xp", []), "ker": seqs_k.get("ker", []), "y": seqs_k.get("y", [])}
    pk2 = runtime.Plan(gk, seqk, [runtime.sched(0)], _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
    pk2.set_input_device("x", kmul64(torch, (nb, 64, 58, 58), gen, dev))
    pk2.set_input_device("ker", w)
    kw = pk2.measure(warmup=5, reps=15, flush_l2=False)
    kc = pk2.measure(warmup=3, reps=9, flush_l2=True)
    # parity of the benchmarked plan: k/64 inputs make the tcgen05 result exact
    y = torch.tensor(pc.get_output("y"), device=dev).view(nb, 64, 56, 56)
    ref = torch.nn.functional.conv2d(x.double(), w.double(), padding=1)
    out = {
        "layout": br.candidate.label, "candidates": len(rc),
        "legal": sum(r.cost_us is not None for r in rc), "candidates_per_s": round(len(rc) / ts, 1),
        "graph_us_warm": round(mw.cost, 3), "graph_us_cold": round(mc.cost, 3),
        "graph_tflops_warm": round(fl / (mw.cost * 1e-6) / 1e12, 2),
        "kernel_us_warm": round(kw.cost, 3), "kernel_us_cold": round(kc.cost, 3),
        "kernel_tflops_warm": round(fl / (kw.cost * 1e-6) / 1e12, 2),
        "kernel_tflops_cold": round(fl / (kc.cost * 1e-6) / 1e12, 2),
        "measure_resolution_us": round(mw.resolution_us, 4),
        "verified_exact": bool(torch.equal(y.double(), ref)),
        "kernels": pc.node_kernel(0) + " | " + pc.node_kernel(1)}
    out["roofline"] = {"bound": "tensor", "achieved": out["kernel_tflops_cold"], "peak": pk["bf16_tflops"],
                       "unit": "TFLOP/s", "frac": round(out["kernel_tflops_cold"] / pk["bf16_tflops"], 4),
                       "kernel": "umma_conv (tcgen05 implicit GEMM), cold L2",
                       "algorithmic": f"{fl:.0f} FLOP per launch (2*N*O*H*W*I*KH*KW)"}
    pc.close()
    pk2.close()
    return out


def e2e_capi(plan, A, B, M, K, N, steps):
    """The drop-in call with host buffers: every step passes the logical
    inputs as host doubles (the reference's BufferMap, interp.hpp:19-21) to
    lfgpu_plan_set_input (pinned staging, H2D, K1 into the tuned bricks),
    runs the plan and reads the result back with lfgpu_plan_get_output (K1
    back to the logical layout, D2H, host doubles)."""
    import numpy as np
    a = A.double().cpu().numpy().ravel().copy()
    b = B.double().cpu().numpy().ravel().copy()
    c = np.empty(M * N, dtype=np.float64)
    for _ in range(5):  # warm: staging buffers, the host pool's threads, page mappings
        plan.set_input("a", a)
        plan.set_input("b", b)
        plan.run()
        plan.get_output("c", out=c)
    t0 = time.perf_counter()
    for _ in range(steps):
        plan.set_input("a", a)
        plan.set_input("b", b)
        plan.run()
        plan.get_output("c", out=c)
    dt = (time.perf_counter() - t0) / steps
    ok = bool(np.array_equal(c.reshape(M, N), a.reshape(M, K) @ b.reshape(K, N)))
    return dt, ok


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2210_12415_b200 import _abi, ir, runtime, tuner
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    ctx = runtime.context(local)
    pk, pk_kind = peaks()
    gen = torch.Generator(device=dev)
    gen.manual_seed(42 + rank)
    # 2 x 256 MB (> 126 MB L2): written, then read, between isolated steps
    flush = torch.zeros(128 << 20, dtype=torch.float32, device=dev)
    out = {}

    # ---- 1. tune the cfg2 GEMM layout on the GPU (measure backend, cold L2)
    M = K = N = 1024
    g = ir.gemm(M, K, N)
    A = kmul64(torch, (M, K), gen, dev)
    B = kmul64(torch, (K, N), gen, dev)
    cands = tuner.gemm_candidates(M, K, N)
    # Candidates shard over ranks (no collective on the data path); the
    # (index, cost) history is gathered and committed in index order.
    barrier(world)
    res, best_i, local_s, n_local = tuner.sweep_distributed(
        g, cands, {"a": A, "b": B}, warmup=2, reps=5, ctx=ctx)
    tune_s = max_over_ranks(local_s, world)
    ok = [r for r in res if r.cost_us is not None]
    bestr = res[best_i]
    out["tuner"] = {"graph": "cfg2 GEMM 1024^3", "candidates": len(res), "legal": len(ok),
                    "ranks": world, "seconds": round(tune_s, 3),
                    "candidates_per_s": round(len(res) / tune_s, 1),
                    "measure": "cold L2; K executions per CUDA event pair, the 1.5x-L2 reads' time subtracted",
                    "best": bestr.candidate.label, "best_us": round(bestr.cost_us, 3)}
    # measure_top (tuner.cpp:250-272's re-measurement of the top-k): the 8
    # best cold-launch candidates re-timed back to back over rotating
    # replicas (the timed regime below), every rank timing each, the max over
    # ranks deciding; the winner is the one benchmarked.
    top = sorted(ok, key=lambda r: r.cost_us)[:8]
    top_t = []
    for r in top:
        seqs_t = tuner.seqs_for(g, r.candidate)
        reps_t = []
        for _ in range(16):  # 16 x 8 MB of operands + results: > L2 between reuses
            pt = runtime.Plan(g, seqs_t, r.candidate.scheds, _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
            pt.set_input_device("a", A)
            pt.set_input_device("b", B)
            reps_t.append(pt)
        ms, _ = time_plan_rotating(torch, reps_t, 64, 16, world)
        top_t.append(max_over_ranks(ms, world) / 64 * 1e3)
        for pt in reps_t:
            pt.close()
    if top_t:
        bestr = top[min(range(len(top)), key=lambda k: top_t[k])]
        out["tuner"]["measure_top"] = {"k": len(top), "regime": "back to back, 16 rotating replicas",
                                       "us": [round(x, 3) for x in top_t], "picked": bestr.candidate.label}

    # ---- 2. timed region: K steps of the tuned GEMM, rotating over replicas
    # whose operands + results (2+2+4 MB each) total > 2x L2, so each step
    # streams cold operands from HBM.
    seqs_best = tuner.seqs_for(g, bestr.candidate)
    rep_bytes = 2 * M * K + 2 * K * N + 4 * M * N
    n_rep = max(2, -(-(256 << 20) // rep_bytes))
    reps = []
    for _ in range(n_rep):
        r = runtime.Plan(g, seqs_best, bestr.candidate.scheds,
                         _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH, ctx=ctx)
        r.set_input_device("a", A)
        r.set_input_device("b", B)
        reps.append(r)
    plan = reps[0]
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        tot_ms, wall = time_plan_rotating(torch, reps, args.steps, args.warmup, world)
    launches = ctx.launches - launches0 - (max(args.warmup, len(reps)) + max(32, len(reps))) * plan.info().kernels
    total_ms = max_over_ranks(tot_ms, world)
    flops_step = 2.0 * M * N * K
    value = world * args.steps * flops_step / (total_ms * 1e-3) / 1e12
    kern_us = tot_ms / args.steps * 1e3
    # burst view: the same K steps right after the idle sleep, no pre-roll
    # (faster: ~9.4 vs ~12.3 us on cfg2; reported beside, not as `value`)
    burst_ms, _ = time_plan_rotating(torch, reps, args.steps, args.warmup, world, preroll=False)
    burst_us = max_over_ranks(burst_ms, world) / args.steps * 1e3
    # also the isolated-launch view (flush kernels between steps): one kernel
    # launched after a > L2 write+read, incl. its launch/drain latency
    per, _ = time_plan_steps(torch, plan, min(args.steps, 10), 3, flush, world)
    # parity of the benchmarked kernel (k/64 inputs: fp32 accumulation is exact)
    ref_c = A.double() @ B.double()
    verified = True
    for r in (plan, reps[(args.warmup + args.steps - 1) % n_rep]):
        c = torch.tensor(r.get_output("c"), device=dev).view(M, N)
        verified = verified and bool(torch.equal(c.double(), ref_c))

    # ---- 3. e2e through the C-ABI with host buffers (the reference-facing
    # call: host doubles in, host doubles out, copies inside the timed step)
    e2e_steps = max(10, min(args.steps, 30))
    e2e_s, e2e_ok = e2e_capi(plan, A, B, M, K, N, e2e_steps)
    e2e_s = max_over_ranks(e2e_s, world)
    e2e_val = world * flops_step / e2e_s / 1e12
    for r in reps[1:]:
        r.close()

    # ---- 3b. the same GEMM behind a pipelined serving loop with fp32 host
    # buffers: step i+1's H2D (copy stream) overlaps step i's D2H (read-back
    # stream), two buffer sets alternate, events order the three streams.
    Ah = [A.cpu().pin_memory() for _ in range(2)]
    Bh = [B.cpu().pin_memory() for _ in range(2)]
    Ad = [torch.empty_like(A) for _ in range(2)]
    Bd = [torch.empty_like(B) for _ in range(2)]
    Ch = [torch.empty(M * N, dtype=torch.float64).pin_memory() for _ in range(2)]
    Cd = [torch.empty(M * N, dtype=torch.float64, device=dev) for _ in range(2)]
    s = torch.cuda.ExternalStream(plan.stream)
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    c_seq = tuner.seqs_for(g, bestr.candidate).get("c", [])
    c_phys = _view(plan, torch, dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    ev_read = [torch.cuda.Event() for _ in range(2)]
    for j in range(2):
        ev_used[j].record(s)
        ev_read[j].record(s_out)
    e2e_i = [0]

    def e2e_step():
        j = e2e_i[0] % 2
        e2e_i[0] += 1
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_used[j])
            Ad[j].copy_(Ah[j], non_blocking=True)
            Bd[j].copy_(Bh[j], non_blocking=True)
            ev_in[j].record(s_in)
        s.wait_event(ev_in[j])
        plan.set_input_device("a", Ad[j], wait=False)
        plan.set_input_device("b", Bd[j], wait=False)
        ev_used[j].record(s)
        plan.run()
        s.wait_event(ev_read[j])
        runtime.layout_convert(c_phys, [("M", M), ("N", N)], c_seq, [], Cd[j],
                               stream=plan.stream, ctx=ctx)
        ev_out[j].record(s)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_out[j])
            Ch[j].copy_(Cd[j], non_blocking=True)
            ev_read[j].record(s_out)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    pipe_s = max_over_ranks(time.perf_counter() - t0, world)
    pipe_val = world * args.steps * flops_step / pipe_s / 1e12
    assert torch.equal(Ch[(e2e_i[0] - 1) % 2].view(M, N).to(dev), A.double() @ B.double())

    # ---- 4. BASELINE's other headline metrics: tuned C2D (cfg1, b1 / b16)
    # and layout-transform bandwidth, each with its own roofline
    c2d = {f"b{nb}": c2d_bench(torch, gen, dev, ctx, pk, nb) for nb in (1, 16)}
    transform = transform_bench(torch, gen, dev, ctx, pk, args.steps)

    # ---- 4a. the same tcgen05 GEMM at large shapes (the kernel's ceiling,
    # separated from 1024^3's fixed costs); torch.matmul as a yardstick only
    ceiling = {}
    for n in (4096, 8192):
        try:
            gn = ir.gemm(n, n, n)
            sq = runtime.decode_layout(gn, 0, [256, 64, 256])
            pn = runtime.Plan(gn, sq, [runtime.sched(0, tile_last=256)], _abi.PLAN_REQUIRE_TC, ctx=ctx)
            an, bn = kmul64(torch, (n, n), gen, dev), kmul64(torch, (n, n), gen, dev)
            pn.set_input_device("a", an)
            pn.set_input_device("b", bn)
            mn = pn.measure(warmup=2, reps=5, flush_l2=False)
            ab, bb = an.to(torch.bfloat16), bn.to(torch.bfloat16)
            tus = time_rotating_fn(torch, [lambda: torch.matmul(ab, bb)], 10, 3)
            fl = 2.0 * n ** 3
            ok = bool(torch.equal(torch.tensor(pn.get_output("c"), device=dev).view(n, n)[:256].double(),
                                  an[:256].double() @ bn.double())) if n == 4096 else None
            ceiling[f"{n}^3"] = {"us": round(mn.cost, 2), "tflops": round(fl / mn.cost / 1e6, 1),
                                 "frac_of_measured_peak": round(fl / mn.cost / 1e6 / pk["bf16_tflops"], 4),
                                 "kernel": pn.node_kernel(0)[:120], "rows_0_255_exact": ok,
                                 "torch_matmul_us_yardstick": round(tus, 2)}
            pn.close()
            del an, bn, ab, bb
        except Exception as e:
            ceiling[f"{n}^3"] = {"error": str(e)[:200]}

    # ---- 4b. end-to-end graphs: cfg4 ResNet-18 b1 (tuned per-conv layouts,
    # fused epilogues, whole-graph CUDA graph) and cfg5 BERT-base GEMM chain
    # (seq 128, 12 layers); device time per inference step, cold L2.
    sec = {}
    if not args.no_e2e_graphs:
        from paper_2210_12415_b200 import e2e, workloads
        try:
            t0 = time.perf_counter()
            fac = workloads.tune_resnet18(1, lambda sub: e2e.make_inputs(sub, gen), ctx=ctx)
            tune_s = time.perf_counter() - t0
            g18, _, p18 = e2e.build_resnet18(1, fac, ctx=ctx)
            for k, x in e2e.make_inputs(g18, gen).items():
                p18.set_input_device(k, x)
            m18 = p18.measure(warmup=5, reps=9, flush_l2=True)
            m18w = p18.measure(warmup=3, reps=9, flush_l2=False)
            kinds = [p18.node_kernel(i) for i in range(len(g18.nodes))]
            sec["resnet18_b1_inference"] = {
                "latency_us": round(m18.cost, 2), "latency_us_warm": round(m18w.cost, 2),
                "launches": int(m18.kernels),
                "tflops": round(3.628e9 / (m18.cost * 1e-6) / 1e12, 3),
                "tc_convs": sum(k.startswith("umma") for k in kinds), "tuning_s": round(tune_s, 1)}
            p18.close()
        except Exception as e:  # reported, not hidden
            sec["resnet18_b1_inference"] = {"error": str(e)[:200]}
        # cfg4 b64 batch-sharded over the ranks (shard.py): each rank runs
        # its contiguous shard through its own plan; throughput from the
        # max-over-ranks step time (the logits gather is outside the step).
        try:
            from paper_2210_12415_b200 import shard
            gb = 64
            _, nloc = shard.batch_shard(gb, rank, world)
            t0 = time.perf_counter()
            facb = workloads.tune_resnet18(nloc, lambda sub: e2e.make_inputs(sub, gen), ctx=ctx)
            tune_b = time.perf_counter() - t0
            gbb, _, pbb = e2e.build_resnet18(nloc, facb, ctx=ctx)
            for k, x in e2e.make_inputs(gbb, gen).items():
                pbb.set_input_device(k, x)
            mbb = pbb.measure(warmup=3, reps=5, flush_l2=True)
            step_us = max_over_ranks(mbb.cost, world)
            sec["resnet18_b64_batch_sharded"] = {
                "global_batch": gb, "ranks": world, "per_rank_batch": nloc,
                "step_us_max_over_ranks": round(step_us, 2),
                "images_per_s": round(gb / (step_us * 1e-6), 1),
                "tflops": round(3.628e9 * gb / (step_us * 1e-6) / 1e12, 2),
                "launches": int(mbb.kernels), "tuning_s": round(tune_b, 1)}
            pbb.close()
        except Exception as e:
            sec["resnet18_b64_batch_sharded"] = {"error": str(e)[:200]}
        try:
            best = None
            for t in (64, 128):
                gbert, _, pb = e2e.build_bert(12, t, 0, ctx=ctx)
                for k, x in e2e.make_bert_inputs(gbert, gen).items():
                    pb.set_input_device(k, x)
                mb = pb.measure(warmup=5, reps=9, flush_l2=True)
                if best is None or mb.cost < best[0]:
                    best = (mb.cost, t, int(mb.kernels))
                pb.close()
            fl = workloads.BERT_FLOPS_PER_LAYER * 12
            sec["bert_base_gemm_chain_seq128_12l"] = {
                "latency_us": round(best[0], 2), "brick_t": best[1], "launches": best[2],
                "tflops": round(fl / (best[0] * 1e-6) / 1e12, 2)}
        except Exception as e:
            sec["bert_base_gemm_chain_seq128_12l"] = {"error": str(e)[:200]}
        # cfg5 as the full encoder: attention (BmmQK, Softmax, BmmPV),
        # LayerNorm and GELU on the op-set extension, GMMs on tcgen05
        try:
            best = None
            for packed in (False, True):  # three q/k/v GMMs, or one packed QKV GMM
                for t in (64, 128):
                    genc, _, pe = e2e.build_encoder(12, t, 0, ctx=ctx, packed_qkv=packed)
                    for k, x in e2e.make_encoder_inputs(genc, gen).items():
                        pe.set_input_device(k, x)
                    me = pe.measure(warmup=3, reps=7, flush_l2=True)
                    if best is None or me.cost < best[0]:
                        best = (me.cost, t, int(me.kernels), packed)
                    pe.close()
            fl = workloads.bert_encoder_flops(12)
            sec["bert_base_encoder_seq128_12l"] = {
                "latency_us": round(best[0], 2), "brick_t": best[1], "launches": best[2], "packed_qkv": best[3],
                "tflops": round(fl / (best[0] * 1e-6) / 1e12, 2), "gflop": round(fl / 1e9, 3)}
        except Exception as e:
            sec["bert_base_encoder_seq128_12l"] = {"error": str(e)[:200]}

    # ---- 5. cpu baselines (rank 0, N=1): the reference's own code on bounded
    # samples of each workload, single core
    cpu = cpu_extra = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_gemm(rows=args.cpu_rows)
        cpu_extra = cpu_baselines_other(out["tuner"], c2d, transform)

    ach = flops_step / (kern_us * 1e-6) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    if cpu_extra:
        c2d["b1"]["cpu_baseline"] = cpu_extra["c2d"]
        transform["cpu_baseline"] = cpu_extra["transform"]
        out["tuner"]["cpu_baseline"] = cpu_extra["tuner"]
    line = {
        "metric": "tuned GEMM TFLOP/s (BASELINE: tuned C2D/GEMM TFLOP/s, layout-transform GB/s)",
        "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 6),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic k/64 inputs (the reference's random_inputs distribution)",
        "config": {"workload": "cfg2: GEMM 1024x1024x1024 on the tuned GMM template layout",
                   "layout": bestr.candidate.label, "kernel": plan.node_kernel(0),
                   "l2": f"inputs larger than L2: {len(reps)} rotating operand replicas "
                         f"({n_rep * rep_bytes >> 20} MB)",
                   "regime": "sustained: the K timed steps follow max(32, R) untimed steps with no gap "
                             "(steady-state L2 write-backs inside the timed region)",
                   "burst_us_per_step_no_preroll": round(burst_us, 3),
                   "isolated_step_us_after_l2_flush": round(statistics.median(per) * 1e3, 3),
                   "parallelism": f"replicas x{world}", "verified_exact": verified},
        "e2e": {"value": round(e2e_val, 4), "unit": "TFLOP/s",
                "h2d_bytes_per_step": 2 * M * K * 8, "d2h_bytes_per_step": M * N * 8,
                "path": "lfgpu_plan_set_input(a, b: host doubles) + lfgpu_plan_run + "
                        "lfgpu_plan_get_output(c: host doubles), one step at a time; the user's "
                        "doubles narrowed on the host to the operands' bf16 storage (bit-identical "
                        "to the device conversion) and c widened back there",
                "link_bytes_per_step": {"h2d": 2 * M * K * 2, "d2h": M * N * 4},
                "ms_per_step": round(e2e_s * 1e3, 3), "verified_exact": e2e_ok},
        "e2e_pipelined_fp32": {"value": round(pipe_val, 4), "unit": "TFLOP/s",
                               "h2d_bytes_per_step": 2 * M * K * 4, "d2h_bytes_per_step": M * N * 8,
                               "pipelining": "step i+1 H2D overlaps step i D2H (2 buffer sets, 3 streams)"},
        "roofline": {"bound": "tensor", "achieved": round(ach, 2),
                     "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": round(ach / pk["bf16_tflops"], 4), "traffic": traffic,
                     "kernel": plan.node_kernel(0), "peak_source": pk_kind,
                     "algorithmic": "2*1024^3 FLOP per launch"},
        "c2d_cfg1": c2d,
        "gemm_large_shape_ceiling": ceiling,
        "layout_transform_nchw_to_nchwc16_n64": transform,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "wall_s_timed_region": round(wall, 4),
        "tuner": out["tuner"],
        "secondary": sec,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line))


def _view(plan, torch, dev):
    """A torch view of the plan's physical fp32 buffer of `c` (no copy)."""
    ptr, elem, n = plan.buffer("c")

    class _T:  # minimal object exposing data_ptr/dtype/device for layout_convert
        def __init__(self):
            self.dtype = torch.float32
            self.device = dev

        def data_ptr(self):
            return ptr
    return _T()


# ---------------------------------------------------------------------------
# reference CPU path

def cpu_baseline_gemm(rows=256, K=1024, N=1024):
    """reference_eval of GMM on a bounded sample (the first `rows` rows of the
    1024^3 product) — the reference's own code (oracle/_ref) when present,
    else the oracle's C port; single thread."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    from paper_2210_12415_b200 import ir
    g = ir.gemm(rows, K, N)
    kind = "reference" if O.ref_available() else "port"
    bufs = O.random_inputs(g, 42)
    t0 = time.perf_counter()
    O.reference_eval(g, bufs, lib="ref" if kind == "reference" else None)
    dt = time.perf_counter() - t0
    fl = 2.0 * rows * K * N
    return {"value": round(fl / dt / 1e12, 9), "unit": "TFLOP/s", "cores": 1, "kind": kind,
            "sample": f"reference_eval GMM {rows}x{K}x{N} (rows 0..{rows} of cfg2), {dt:.2f} s",
            "gflops": round(fl / dt / 1e9, 4)}


def cpu_baselines_other(tuner_out, c2d, transform):
    """Same-run CPU baselines of the other metrics, the reference's own code
    (oracle/_ref) when present, single core, bounded samples:
    C2D reference_eval at cfg1 b1 (interp.cpp:70-89), materialize_tensor of
    NCHW -> NCHWc16 at N=8 (interp.cpp:280-337), and one simulate_cache
    measurement of a cfg1 candidate (cachesim.cpp:152-174, the tuner's
    measure function)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_lib as O
    from paper_2210_12415_b200 import ir, runtime, tuner
    from paper_2210_12415_b200.layout import reorder, split
    ref = O.ref_available()
    kind = "reference" if ref else "port"
    lib = "ref" if ref else None
    gc = ir.pad_conv(1, 64, 64, 56, 3, 1, 1)
    bufs = O.random_inputs(gc, 42)
    t0 = time.perf_counter()
    O.reference_eval(gc, bufs, lib=lib)
    dt = time.perf_counter() - t0
    fl = 2.0 * 64 * 64 * 56 * 56 * 9
    out = {"c2d": {"value": round(fl / dt / 1e12, 9), "unit": "TFLOP/s", "cores": 1, "kind": kind,
                   "sample": f"reference_eval Padding->C2D cfg1 b1, {dt:.2f} s"}}
    ext = [8, 64, 56, 56]
    src = np.random.default_rng(42).integers(-64, 65, int(np.prod(ext))).astype(np.float64) / 64
    seq = [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])]
    t0 = time.perf_counter()
    O.materialize(ext, seq, src, lib=lib)
    dt = time.perf_counter() - t0
    byts = 2 * src.size * 4
    out["transform"] = {"value": round(byts / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": kind,
                        "sample": f"materialize_tensor NCHW->NCHWc16 N=8 ({src.size} elements, fp32-equivalent bytes), {dt:.2f} s"}
    if ref:
        cand = tuner.conv_candidates(gc, 1)[0]
        t0 = time.perf_counter()
        O.ref_simulate_cache(gc, tuner.seqs_for(gc, cand), cand.scheds)
        dt = time.perf_counter() - t0
        out["tuner"] = {"value": round(1.0 / dt, 4), "unit": "candidates/s", "cores": 1, "kind": kind,
                        "sample": f"one simulate_cache measurement of cfg1 candidate '{cand.label}', {dt:.1f} s"}
    else:
        out["tuner"] = None
    return out


def _ref_worker(rows):
    return cpu_baseline_gemm(rows=rows)


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation of the path on this
    host's cores (one process per core, bounded sample per step)."""
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    rows = args.ref_rows
    per_step_flops = 2.0 * rows * 1024 * 1024 * cores
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_worker, [rows] * cores)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = pool.map(_ref_worker, [rows] * cores)
        dt = time.perf_counter() - t0
    kind = r[0]["kind"]
    val = args.steps * per_step_flops / dt / 1e12
    line = {"impl": "reference", "metric": "tuned GEMM TFLOP/s (BASELINE: tuned C2D/GEMM TFLOP/s, "
            "layout-transform GB/s)", "value": round(val, 9), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic k/64 inputs (random_inputs, seed 42)",
            "config": {"workload": "cfg2: GEMM 1024x1024x1024 (reference_eval, interp.cpp:109-122)",
                       "sample_per_step": f"{cores} processes x {rows} rows of the 1024^3 product"},
            "cpu_baseline": {"value": round(val, 9), "unit": "TFLOP/s", "cores": cores, "kind": kind,
                             "sample": f"{rows}x1024x1024 GMM rows per process per step"},
            "e2e": {"value": round(val, 9), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e-graphs", action="store_true", help="skip ResNet-18 / BERT secondaries")
    ap.add_argument("--cpu-rows", type=int, default=192)
    ap.add_argument("--ref-rows", type=int, default=16)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup(args.gpus)
    run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
