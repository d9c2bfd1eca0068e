"""Per-tensor check of a small BERT chain against float64 torch (diagnostics)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
from paper_2210_12415_b200 import _abi, ir, runtime, workloads
from resnet18_run import max_rel, reference
from bert_run import make_inputs

for (layers, hid, ffn, qkv, t, order, keep) in [(1, 128, 256, 384, 64, 1, 8), (1, 128, 256, 384, 64, 0, 8),
                                               (2, 128, 256, 384, 64, 0, 0), (1, 768, 3072, 2304, 64, 0, 8)]:
    g, gmms = workloads.bert_chain(layers, 128, hid, ffn, qkv)
    seqs, scheds = {}, []
    for ni in gmms:
        nd = g.nodes[ni]
        K = g.tensor(nd.inputs[0]).extents[1]; N = g.tensor(nd.output).extents[1]
        seqs.update(runtime.decode_layout(g, ni, [128, min(t, K), min(t, N)]))
        scheds.append(runtime.sched(ni, tile_last=min(t, N), order=order, fuse=1))
    seqs = workloads.propagate_elementwise(g, seqs)
    plan = runtime.Plan(g, seqs, scheds, keep)
    gen = torch.Generator(device="cuda"); gen.manual_seed(1)
    ins = make_inputs(g, gen)
    for k, x in ins.items():
        plan.set_input_device(k, x)
    plan.run()
    kinds = [plan.node_kernel(i) for i in range(len(g.nodes))]
    tc = frozenset(i for i, k in enumerate(kinds) if k.startswith("umma"))
    emu = reference(g, ins, tc, emulate=True)
    print(f"== layers={layers} hid={hid} t={t} order={order} keep={keep}")
    for i, nd in enumerate(g.nodes):
        tid = nd.output
        try:
            got = torch.tensor(plan.get_output(tid), device="cuda").view_as(emu[tid])
            print(f"  node {i} {ir.OP_NAMES[nd.kind]:8s} {tid:12s} rel {max_rel(got, emu[tid]):.3g}  {kinds[i][:70]}")
        except Exception as e:
            print(f"  node {i} {ir.OP_NAMES[nd.kind]:8s} {tid:12s} n/a ({str(e)[:60]})  {kinds[i][:60]}")
