"""List C2D template candidates of the ResNet-18 3x3 stride-1 shapes whose
halo plan falls back (and why). Diagnostics only."""
import os
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_12415_b200 import _abi, ir, runtime, tuner  # noqa: E402

for (c, h) in [(64, 56), (128, 28), (256, 14), (512, 7)]:
    g = ir.pad_conv(1, c, c, h, 3, 1, 1)
    why = Counter()
    n = 0
    for cand in tuner.conv_candidates(g, 1):
        try:
            p = runtime.Plan(g, tuner.seqs_for(g, cand), cand.scheds, _abi.PLAN_REQUIRE_TC)
        except runtime.LfError as e:
            why["plan error: " + str(e)[:90]] += 1
            continue
        k = p.node_kernel(1)
        n += 1
        if "halo:" in k:
            why[k[k.index("halo:"):][:90]] += 1
        else:
            why["halo ok"] += 1
        p.close()
    print(f"== {c}@{h}: {n} plans")
    for w, k in why.most_common(8):
        print(f"  {k:4d}  {w}")
