"""End-to-end graphs of BASELINE.json cfg4 / cfg5 on the GPU backend.

cfg4: ResNet-18 inference through one whole-graph plan (tuned per-conv
template layouts from workloads.tune_resnet18, fused epilogues, CUDA graph).
cfg5: the BERT-base encoder GEMM chain (seq 128, 12 layers) on GMM brick
layouts shared by every activation, so each GMM's output is the next GMM's
A operand with no conversion and the residual EwAdd fuses into the epilogue.

Also the float64 torch model of a graph (`reference`): exact, or emulating
the plan's numerics (bf16 operands on tensor-core contractions, fp32
storage) — test and report infrastructure for chained graphs, where bf16
operand rounding makes bit-exactness against reference_eval impossible.
"""
import math

import torch
import torch.nn.functional as F

from . import _abi, ir, runtime, workloads


def k64(shape, gen, scale=1.0):
    return torch.randint(-64, 65, shape, generator=gen, device="cuda").float() / 64 * scale


def make_inputs(g, gen):  # ResNet-18 (also used by BERT's weight scaling rule)
    """k/64 values; conv / FC weights scaled by a power of two ~ 1/sqrt(fan_in)
    so activations stay O(1) and every weight stays exact in bf16."""
    out = {}
    for t in g.tensors:
        if t.role not in (ir.INPUT, ir.CONSTANT):
            continue
        shape = t.extents
        if t.id.endswith("_w"):
            fan_in = math.prod(shape[1:]) if len(shape) == 4 else shape[0]
            out[t.id] = k64(shape, gen, 2.0 ** -round(math.log2(math.sqrt(fan_in))))
        elif t.id.endswith("_b"):
            out[t.id] = k64(shape, gen, 1.0 / 8)
        else:
            out[t.id] = k64(shape, gen)
    return out


def reference(g, ins, tc_nodes=frozenset(), emulate=False):
    """Float64 forward of the graph; with emulate, tensor-core contraction
    operands are rounded to bf16 and node outputs to fp32."""
    v = {k: x.double() for k, x in ins.items()}

    def rb(x):
        return x.bfloat16().double() if emulate else x

    def rf(x):
        return x.float().double() if emulate else x

    for i, nd in enumerate(g.nodes):
        a = [v[t] for t in nd.inputs]
        if nd.kind == ir.PADDING:
            p = nd.attr("pad", 0)
            r = F.pad(a[0], (p, p, p, p))
        elif nd.kind == ir.LAYOUT_CONVERT:
            r = a[0]
        elif nd.kind == ir.C2D:
            tc = i in tc_nodes
            r = rf(F.conv2d(rb(a[0]) if tc else a[0], rb(a[1]) if tc else a[1],
                            stride=nd.attr("stride", 1)))
        elif nd.kind == ir.GMM:
            tc = i in tc_nodes
            r = rf((rb(a[0]) if tc else a[0]) @ (rb(a[1]) if tc else a[1]))
        elif nd.kind == ir.BIASADD:
            r = rf(a[0] + (a[1].view(1, -1, 1, 1) if a[0].dim() == 4 else a[1].view(1, -1)))
        elif nd.kind == ir.EWADD:
            r = rf(a[0] + a[1])
        elif nd.kind == ir.RELU:
            r = a[0].clamp_min(0)
        elif nd.kind == ir.MAXPOOL:
            r = F.max_pool2d(a[0], nd.attr("window", 1), nd.attr("stride", 1))
        elif nd.kind == ir.GLOBAL_AVGPOOL:
            r = rf(a[0].mean(dim=(2, 3)))
        elif nd.kind == ir.GELU:
            r = rf(0.5 * a[0] * (1.0 + torch.special.erf(a[0] / math.sqrt(2.0))))
        elif nd.kind == ir.SOFTMAX:
            r = rf(torch.softmax(a[0], dim=-1))
        elif nd.kind == ir.LAYERNORM:
            x = a[0]
            mu = x.mean(dim=-1, keepdim=True)
            var = ((x - mu) ** 2).mean(dim=-1, keepdim=True)
            eps = 10.0 ** -nd.attr("eps_exp", 12)
            r = rf((x - mu) / torch.sqrt(var + eps) * a[1][0] + a[1][1])
        elif nd.kind == ir.BMM_QK:
            H, dh = nd.attr("heads", 1), nd.attr("head_dim", 0)
            q, k = a[0], a[1]
            if dh:  # column slices of packed operands
                a0, b0 = nd.attr("a_col0", 0), nd.attr("b_col0", 0)
                q, k = q[:, a0:a0 + H * dh], k[:, b0:b0 + H * dh]
            r = rf(torch.einsum("ihd,jhd->hij", q.reshape(q.shape[0], H, -1), k.reshape(k.shape[0], H, -1)))
        elif nd.kind == ir.BMM_PV:
            H, dh = nd.attr("heads", 1), nd.attr("head_dim", 0)
            pr, vv = a[0], a[1]
            if dh:
                b0 = nd.attr("b_col0", 0)
                vv = vv[:, b0:b0 + H * dh]
            o = torch.einsum("hij,jhd->ihd", pr, vv.reshape(vv.shape[0], H, -1))
            r = rf(o.reshape(o.shape[0], -1))
        else:
            raise ValueError(nd.kind)
        v[nd.output] = r
    return v


def max_rel(a, b):
    s = torch.maximum(torch.ones_like(a), torch.maximum(a.abs(), b.abs()))
    return float(((a - b).abs() / s).max())


def build_resnet18(n, factors, ctx=None, flags=_abi.PLAN_CUDA_GRAPH):
    g, convs = workloads.resnet18(n)
    seqs = workloads.resnet18_seqs(g, convs, factors)
    scheds = [runtime.sched(c["node"], fuse=1) for c in convs]
    gi = len(g.nodes) - 2  # the FC GMM
    scheds.append(runtime.sched(gi, fuse=1))
    plan = runtime.Plan(g, seqs, scheds, flags, ctx=ctx)
    return g, convs, plan




def make_bert_inputs(g, gen):
    out = {}
    for t in g.tensors:
        if t.role not in (ir.INPUT, ir.CONSTANT):
            continue
        if t.id.endswith("_w"):
            out[t.id] = k64(t.extents, gen, 2.0 ** -round(math.log2(math.sqrt(t.extents[0]))))
        elif t.id.endswith("_b"):
            out[t.id] = k64(t.extents, gen, 1.0 / 8)
        else:
            out[t.id] = k64(t.extents, gen)
    return out


def make_encoder_inputs(g, gen, head_dim=64):
    """BERT encoder inputs: k/64 activations, weights scaled by a power of
    two ~ 1/sqrt(fan_in), the query projection also by 1/sqrt(head_dim) (a
    power of two for Dh = 64, so bf16-exact), LayerNorm gamma = 1 + k/512,
    beta = k/512."""
    out = {}
    qs = 2.0 ** -round(math.log2(math.sqrt(head_dim)))
    for t in g.tensors:
        if t.role not in (ir.INPUT, ir.CONSTANT):
            continue
        q = qs if "_q_" in t.id else 1.0
        packed = "_qkv_" in t.id  # packed [., 3*hidden]: the query third carries the scale
        if t.id.endswith("_w"):
            w = k64(t.extents, gen, q * 2.0 ** -round(math.log2(math.sqrt(t.extents[0]))))
            if packed:
                w[:, :t.extents[1] // 3] *= qs
            out[t.id] = w
        elif t.id.endswith("_b"):
            bb = k64(t.extents, gen, q / 8)
            if packed:
                bb[:t.extents[0] // 3] *= qs
            out[t.id] = bb
        elif t.id.endswith("_gb"):
            gb = k64(t.extents, gen, 1.0 / 8)
            gb[0] += 1.0
            out[t.id] = gb
        else:
            out[t.id] = k64(t.extents, gen)
    return out


def kouter_activations(g, seqs, t):
    """Activations [M, N] as column bricks [N/t][M][t] (split + reorder, a
    layout of the reference's language): a GEMM reading one as its A operand
    gets several 64-wide K slabs per TMA box (K bricks outside the rows),
    which the row-major bricks [M][N/t][t] that decode_layout gives at
    m_t = M cannot. Weights, biases and LayerNorm parameters keep theirs."""
    from .layout import reorder, split
    for tdecl in g.tensors:
        if len(tdecl.extents) != 2 or tdecl.id.endswith(("_w", "_b", "_gb")):
            continue
        n = tdecl.extents[1]
        tt = min(t, n)
        if n % tt:
            continue
        seqs[tdecl.id] = [split(1, [n // tt, tt]), reorder([1, 0, 2])]
    return seqs


def build_encoder(layers, t, order=0, ctx=None, flags=_abi.PLAN_CUDA_GRAPH, seq=128, hidden=768, heads=12,
                  ffn=3072, packed_qkv=False, kouter=True):
    """cfg5 as a full BERT-base encoder (workloads.bert_encoder): every GMM
    on tcgen05 in GMM brick layouts (m_t = seq, k_t = n_t = t) with its
    BiasAdd / residual EwAdd / GELU fused into the epilogue; attention
    (BmmQK, Softmax, BmmPV) and LayerNorm read and write those bricks
    through separable offset tables."""
    g, gmms = workloads.bert_encoder(layers, seq, hidden, heads, ffn, packed_qkv)
    seqs, scheds = {}, []
    for ni in gmms:
        nd = g.nodes[ni]
        K = g.tensor(nd.inputs[0]).extents[1]
        N = g.tensor(nd.output).extents[1]
        seqs.update(runtime.decode_layout(g, ni, [seq, min(t, K), min(t, N)]))
        scheds.append(runtime.sched(ni, tile_last=min(t, N), order=order, fuse=1))
    seqs = workloads.propagate_elementwise(g, seqs)
    if kouter:
        seqs = kouter_activations(g, seqs, t)
    return g, gmms, runtime.Plan(g, seqs, scheds, flags, ctx=ctx)


def build_bert(layers, t, order=0, ctx=None, flags=_abi.PLAN_CUDA_GRAPH, kouter=True):
    g, gmms = workloads.bert_chain(layers)
    seqs, scheds = {}, []
    for ni in gmms:
        nd = g.nodes[ni]
        K = g.tensor(nd.inputs[0]).extents[1]
        N = g.tensor(nd.output).extents[1]
        seqs.update(runtime.decode_layout(g, ni, [128, min(t, K), min(t, N)]))
        scheds.append(runtime.sched(ni, tile_last=min(t, N), order=order, fuse=1))
    seqs = workloads.propagate_elementwise(g, seqs)
    if kouter:
        seqs = kouter_activations(g, seqs, t)
    return g, gmms, runtime.Plan(g, seqs, scheds, flags, ctx=ctx)
