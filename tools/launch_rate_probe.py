"""Back-to-back launch regime of one cfg2 plan (diagnostics): per-launch
device time over K launches after a long device sleep, with the host's
enqueue time per run() beside it; LFGPU_PDL=0 in the environment disables
programmatic dependent launch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402

g = ir.gemm(1024, 1024, 1024)
c = tuner.Candidate({0: (256, 64, 128)}, [runtime.sched(0, tile_last=64, order=1)])
A = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
B = torch.randint(-64, 65, (1024, 1024), device="cuda").float() / 64
p = runtime.Plan(g, tuner.seqs_for(g, c), c.scheds, _abi.PLAN_REQUIRE_TC | _abi.PLAN_CUDA_GRAPH)
p.set_input_device("a", A)
p.set_input_device("b", B)
s = torch.cuda.ExternalStream(p.stream)
for _ in range(10):
    p.run()
torch.cuda.synchronize()
for K in (4, 16, 64, 256):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    with torch.cuda.stream(s):
        torch.cuda._sleep(2_000_000 + 100_000 * K)
    t0 = time.perf_counter()
    for i in range(K):
        ev[i].record(s)
        p.run()
    ev[K].record(s)
    host = (time.perf_counter() - t0) / K * 1e6
    torch.cuda.synchronize()
    d = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(K)]
    q = [round(x, 2) for x in (d[:4] + d[-4:])]
    print(f"PDL={os.environ.get('LFGPU_PDL', '1')} K={K}: mean {sum(d) / K:.3f} us/launch, host {host:.2f} us/run, first/last {q}", flush=True)
