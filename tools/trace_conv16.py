"""Per-CTA timeline of the cfg1 b16 conv on the final bench layout (diagnostics)."""
import os
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import trace_umma as T  # noqa: E402
from paper_2210_12415_b200 import ir, runtime, tuner  # noqa: E402

fac = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (56, 28, 64, 32, 32, 64)
g = ir.pad_conv(16, 64, 64, 56, 3, 1, 1)
T.timeline(g, tuner.Candidate({1: fac}, [runtime.sched(1)]),
           {"x": T.k64((16, 64, 56, 56)), "ker": T.k64((64, 64, 3, 3))}, f"cfg1 b16 {fac}")
