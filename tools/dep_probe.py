"""DEP (depthwise C2D) on the GPU plan: per-node kernels and device time on
template layouts, checked against the oracle. Diagnostics only.
  python tools/dep_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_lib as O  # noqa: E402
from paper_2210_12415_b200 import ir, runtime  # noqa: E402


def main():
    for (n, c, h, k, s) in [(1, 256, 56, 3, 1), (16, 256, 56, 3, 1), (1, 512, 28, 3, 2)]:
        g = ir.dep_chain(n, c, h, k, s, k // 2)
        tmpl = None
        f = [h // s if h // s <= 56 else 28, (h // s) // 2, 32, 32, 32]
        tl = runtime.decode_layout(g, 1, f)
        tl["y"] = tl["conv"]
        for name, seqs in [("logical", {}), (f"template {f}", tl)]:
            bufs = O.random_inputs(g, 3)
            inputs = {t.id: bufs[i].copy() for i, t in enumerate(g.tensors) if t.role in (ir.INPUT, ir.CONSTANT)}
            O.reference_eval(g, bufs)
            p = runtime.Plan(g, seqs, [runtime.sched(1, fuse=1)])
            for tid, v in inputs.items():
                p.set_input(tid, v)
            p.run()
            d = O.max_rel_diff(p.get_output("y"), bufs[g.tensor_index("y")])
            us = p.measure().cost
            byts = (n * c * (h + 2 * (k // 2)) ** 2 + n * c * (h // s) ** 2) * 4
            print(f"DEP n={n} c={c} h={h} k={k} s={s} {name}: {[p.node_kernel(i) for i in range(len(g.nodes))]} "
                  f"diff={d:.1e} plan {us:.1f} us  (~{byts / us / 1e3:.0f} GB/s on the conv's bytes), tmpl={tmpl}")


if __name__ == "__main__":
    main()
