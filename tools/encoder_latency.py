"""cfg5 full encoder latency per brick width and q/k/v packing (L2 flushed
and warm), with the kernel mix."""
import sys; sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2210_12415_b200 import e2e
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
for packed in (False, True):
    for t in (64, 128):
        g, gm, p = e2e.build_encoder(12, t, packed_qkv=packed)
        for k, x in e2e.make_encoder_inputs(g, gen).items(): p.set_input_device(k, x)
        m = p.measure(warmup=3, reps=7, flush_l2=True); mw = p.measure(warmup=3, reps=7, flush_l2=False)
        kinds = {}
        for i in range(len(g.nodes)):
            k = p.node_kernel(i).split(" ")[0]; kinds[k] = kinds.get(k, 0) + 1
        print("packed" if packed else "qkv3", t, "cold us", round(m.cost, 1), "warm", round(mw.cost, 1),
              "launches", m.kernels, kinds, flush=True)
        p.close()
