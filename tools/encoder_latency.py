import sys; sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2210_12415_b200 import e2e, workloads
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
for t in (64, 128):
    g, gm, p = e2e.build_encoder(12, t)
    for k, x in e2e.make_encoder_inputs(g, gen).items(): p.set_input_device(k, x)
    m = p.measure(warmup=3, reps=7, flush_l2=True); mw = p.measure(warmup=3, reps=7, flush_l2=False)
    kinds = {}
    for i in range(len(g.nodes)):
        k = p.node_kernel(i).split(" ")[0]; kinds[k] = kinds.get(k, 0) + 1
    print(t, "cold us", round(m.cost, 1), "warm", round(mw.cost, 1), "launches", m.kernels, kinds)
