"""BERT GEMM-chain / encoder latency with and without PDL (diagnostics)."""
import os
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import e2e  # noqa: E402
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
for name, build, mk in (("chain", lambda: e2e.build_bert(12, 64), e2e.make_bert_inputs),
                        ("encoder", lambda: e2e.build_encoder(12, 64), e2e.make_encoder_inputs)):
    g, gm, p = build()
    for k, x in mk(g, gen).items():
        p.set_input_device(k, x)
    m = p.measure(warmup=3, reps=5, flush_l2=False)
    print(name, "PDL" if os.environ.get("LFGPU_PDL", "1") != "0" else "noPDL", round(m.cost, 1), "us", m.kernels, "launches")
