"""cfg5 BERT-base GEMM chain through one fused whole-graph plan
(workloads.bert_chain): every GMM on tcgen05 with its BiasAdd / residual
EwAdd / ReLU fused into the epilogue, activations chained in one brick
layout (each GMM's output feeds the next GMM's A operand through its bf16
shadow). Checked against float64 torch: exactly emulating the plan's
numerics (bf16 operands, fp32 storage) and within the stated chained-bf16
tolerance of the exact result."""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layers,hid,ffn,qkv,t,order", [
    (2, 128, 256, 384, 64, 0),    # split-K chain
    (2, 128, 256, 384, 64, 1),    # no split
    (1, 768, 3072, 2304, 128, 0),  # one full-size BERT-base layer
])
def test_bert_chain_fused(layers, hid, ffn, qkv, t, order):
    from paper_2210_12415_b200 import e2e as R
    from paper_2210_12415_b200 import _abi, runtime, workloads
    g, gmms = workloads.bert_chain(layers, 128, hid, ffn, qkv)
    seqs, scheds = {}, []
    for ni in gmms:
        nd = g.nodes[ni]
        K = g.tensor(nd.inputs[0]).extents[1]
        N = g.tensor(nd.output).extents[1]
        seqs.update(runtime.decode_layout(g, ni, [128, min(t, K), min(t, N)]))
        scheds.append(runtime.sched(ni, tile_last=min(t, N), order=order, fuse=1))
    seqs = workloads.propagate_elementwise(g, seqs)
    plan = runtime.Plan(g, seqs, scheds, _abi.PLAN_CUDA_GRAPH)
    kinds = [plan.node_kernel(i) for i in range(len(g.nodes))]
    assert all(kinds[i].startswith("umma_gemm") for i in gmms), kinds
    assert all(k in ("fused", "bf16_shadow") or k.startswith("umma") for k in kinds), kinds
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    ins = R.make_bert_inputs(g, gen)
    for k, x in ins.items():
        plan.set_input_device(k, x)
    plan.run()
    out = torch.tensor(plan.get_output("out"), device="cuda").view(128, hid)
    tc = frozenset(gmms)
    emu = R.reference(g, ins, tc, emulate=True)["out"]
    ex = R.reference(g, ins)["out"]
    assert R.max_rel(out, emu) <= 1e-4
    assert R.max_rel(out, ex) <= 2e-2 * layers
