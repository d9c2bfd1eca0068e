"""Per-node error of the encoder layer (diagnostics): EXACT plan vs the
oracle at reduced width, and the fused tcgen05 plan vs the bf16-emulating
float64 model at full size."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle_lib as O  # noqa: E402
from paper_2210_12415_b200 import _abi, e2e, ir, runtime, workloads  # noqa: E402

g, _ = workloads.bert_encoder(1, 128, 128, 2, 256)
bufs = O.random_inputs(g, 21)
bufs[g.tensor_index("l0_q_w")] *= 1.0 / 8
ins = {t.id: bufs[i].copy() for i, t in enumerate(g.tensors) if t.role in (ir.INPUT, ir.CONSTANT)}
O.reference_eval(g, bufs)
got = runtime.interpret(g, {}, [], ins, flags=_abi.PLAN_EXACT)
for nd in g.nodes:
    r = bufs[g.tensor_index(nd.output)]
    print("exact", ir.OP_NAMES[nd.kind], nd.output, "%.3g" % O.max_rel_diff(got[nd.output], r),
          "max|ref| %.3g" % abs(r).max())

g, gmms, plan = e2e.build_encoder(1, 128, flags=_abi.PLAN_CUDA_GRAPH | _abi.PLAN_KEEP_ALL)
gen = torch.Generator(device="cuda")
gen.manual_seed(7)
ins = e2e.make_encoder_inputs(g, gen)
for k, x in ins.items():
    plan.set_input_device(k, x)
plan.run()
emu = e2e.reference(g, ins, frozenset(gmms), emulate=True)
ex = e2e.reference(g, ins)
for i, nd in enumerate(g.nodes):
    o = torch.tensor(plan.get_output(nd.output), device="cuda").view(emu[nd.output].shape)
    print("tc", ir.OP_NAMES[nd.kind], nd.output, plan.node_kernel(i)[:20], "vs emu %.3g" % e2e.max_rel(o, emu[nd.output]),
          "vs exact %.3g" % e2e.max_rel(o, ex[nd.output]), "max %.3g" % float(emu[nd.output].abs().max()))
