"""cfg5 full encoder / GEMM chain latency per brick width, q/k/v packing and
activation layout (row bricks from decode_layout, or column bricks
"kouter"), L2 flushed and warm, with the kernel mix (diagnostics)."""
import sys; sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2210_12415_b200 import e2e
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
for kouter in (False, True):
    for packed in (False, True):
        for t in (64, 128):
            g, gm, p = e2e.build_encoder(12, t, packed_qkv=packed, kouter=kouter)
            for k, x in e2e.make_encoder_inputs(g, gen).items(): p.set_input_device(k, x)
            m = p.measure(warmup=3, reps=7, flush_l2=True); mw = p.measure(warmup=3, reps=7, flush_l2=False)
            kinds = {}
            for i in range(len(g.nodes)):
                k = p.node_kernel(i).split(" ")[0]; kinds[k] = kinds.get(k, 0) + 1
            kc = sorted({p.node_kernel(i).split("KC=")[1].split(" ")[0] for i in gm})
            print("kouter" if kouter else "rows  ", "packed" if packed else "qkv3", t, "cold us", round(m.cost, 1),
                  "warm", round(mw.cost, 1), "launches", m.kernels, "KC", kc, flush=True)
            p.close()
    for t in (64, 128):
        g, gm, p = e2e.build_bert(12, t, kouter=kouter)
        for k, x in e2e.make_bert_inputs(g, gen).items(): p.set_input_device(k, x)
        m = p.measure(warmup=3, reps=7, flush_l2=True)
        kc = sorted({p.node_kernel(i).split("KC=")[1].split(" ")[0] for i in gm})
        print("kouter" if kouter else "rows  ", "bert-chain", t, "cold us", round(m.cost, 1), "KC", kc, flush=True)
        p.close()
