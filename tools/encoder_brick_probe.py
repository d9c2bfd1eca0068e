import sys; sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2210_12415_b200 import e2e
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
for t in (32, 64):
    g, gm, p = e2e.build_encoder(12, t, packed_qkv=True)
    for k, x in e2e.make_encoder_inputs(g, gen).items(): p.set_input_device(k, x)
    m = p.measure(warmup=3, reps=7, flush_l2=True)
    ks = sorted({p.node_kernel(i).split("splits=")[1].split(" ")[0] + "/" + p.node_kernel(i).split("BN=")[1].split(" ")[0] for i in gm})
    print("encoder t", t, round(m.cost, 1), ks, flush=True)
    p.close()
    g, gm, p = e2e.build_bert(12, t)
    for k, x in e2e.make_bert_inputs(g, gen).items(): p.set_input_device(k, x)
    m = p.measure(warmup=3, reps=7, flush_l2=True)
    print("chain t", t, round(m.cost, 1), flush=True)
    p.close()
