"""Per-CTA timeline of the cfg2 GEMM (1024^3, tuned brick layout m_t=128
k_t=64 n_t=64) on the 1-CTA kernel at each K per stage (diagnostics)."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for kcs in ("64", "128", "256"):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, LFGPU_GEMM_KCS=kcs), check=False)
    sys.exit(0)
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import trace_umma as T  # noqa: E402
from paper_2210_12415_b200 import ir, runtime, tuner  # noqa: E402

g = ir.gemm(1024, 1024, 1024)
T.timeline(g, tuner.Candidate({0: (128, 64, 64)}, [runtime.sched(0, tile_last=64, tile_second=128)]),
           {"a": T.k64((1024, 1024)), "b": T.k64((1024, 1024))}, f"cfg2 KCS={os.environ['LFGPU_GEMM_KCS']}")
