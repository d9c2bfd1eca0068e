"""Benchmark workloads named by BASELINE.json configs.

cfg3 is the ResNet-50 convolution sweep: the 24 distinct conv layers of
ResNet-50 v1.5 (stride on the 3x3), explicit Padding for p > 0 and the
C2D `stride` attribute (the reference C2D has no implicit padding,
SPEC.md:80). cfg5 is the BERT-base per-layer GMM chain at seq 128
(GELU replaced by ReLU, the reference op set has no GELU).
"""
from . import ir

# (name, in_channels, out_channels, input H=W, kernel, stride, pad)
RESNET50_CONVS = [
    ("conv1_7x7s2", 3, 64, 224, 7, 2, 3),
    ("l1_1x1_64_64", 64, 64, 56, 1, 1, 0),
    ("l1_3x3_64", 64, 64, 56, 3, 1, 1),
    ("l1_1x1_64_256", 64, 256, 56, 1, 1, 0),
    ("l1_1x1_256_64", 256, 64, 56, 1, 1, 0),
    ("l1_ds_64_256", 64, 256, 56, 1, 1, 0),
    ("l2_1x1_256_128", 256, 128, 56, 1, 1, 0),
    ("l2_3x3s2_128", 128, 128, 56, 3, 2, 1),
    ("l2_1x1_128_512", 128, 512, 28, 1, 1, 0),
    ("l2_1x1_512_128", 512, 128, 28, 1, 1, 0),
    ("l2_3x3_128", 128, 128, 28, 3, 1, 1),
    ("l2_ds_256_512s2", 256, 512, 56, 1, 2, 0),
    ("l3_1x1_512_256", 512, 256, 28, 1, 1, 0),
    ("l3_3x3s2_256", 256, 256, 28, 3, 2, 1),
    ("l3_1x1_256_1024", 256, 1024, 14, 1, 1, 0),
    ("l3_1x1_1024_256", 1024, 256, 14, 1, 1, 0),
    ("l3_3x3_256", 256, 256, 14, 3, 1, 1),
    ("l3_ds_512_1024s2", 512, 1024, 28, 1, 2, 0),
    ("l4_1x1_1024_512", 1024, 512, 14, 1, 1, 0),
    ("l4_3x3s2_512", 512, 512, 14, 3, 2, 1),
    ("l4_1x1_512_2048", 512, 2048, 7, 1, 1, 0),
    ("l4_1x1_2048_512", 2048, 512, 7, 1, 1, 0),
    ("l4_3x3_512", 512, 512, 7, 3, 1, 1),
    ("l4_ds_1024_2048s2", 1024, 2048, 14, 1, 2, 0),
]


def conv_graph(n, ci, co, h, k, stride, pad):
    """(graph, C2D node index) for one conv layer at batch n."""
    if pad:
        return ir.pad_conv(n, ci, co, h, k, stride, pad), 1
    return ir.bare_conv(n, ci, co, h, k, stride), 0


def conv_flops(n, ci, co, h, k, stride, pad):
    ho = (h + 2 * pad - k) // stride + 1
    return 2.0 * n * co * ho * ho * ci * k * k


# BERT-base layer at seq 128: (name, K, N, epilogue)
BERT_GEMMS = [
    ("qkv", 768, 2304, "bias"),
    ("attn_out", 768, 768, "bias+residual"),
    ("ffn1", 768, 3072, "bias+relu"),
    ("ffn2", 3072, 768, "bias+residual"),
]


def bert_chain(layers=12, seq=128, hidden=768, ffn=3072, qkv=2304):
    """cfg5: the BERT-base encoder GEMM chain at seq 128 as one graph.

    Per layer, on h[seq, hidden]:
      qkv   = GMM(h, Wqkv) + b          (graph output: the attention core -
                                          softmax / batched matmul - is not in
                                          the reference op set, ir.hpp:42)
      a     = GMM(h, Wo) + bo + h        (attention-output projection with its
                                          residual; h stands in for the
                                          attention context)
      f     = ReLU(GMM(a, W1) + b1)      (GELU -> ReLU: no GELU in the op set)
      h'    = GMM(f, W2) + b2 + a
    1.812 GFLOP per layer. Returns (graph, gmm node
    indices)."""
    b = Builder()
    I, C, O = ir.INPUT, ir.CONSTANT, ir.OUTPUT
    gmms = []

    def mat(tid, m, n, role=ir.INTERMEDIATE):
        return b.t(tid, [("M", m), ("N", n)], role)

    def linear(name, x, k, n, role_out=ir.INTERMEDIATE):
        w = b.t(f"{name}_w", [("K", k), ("N", n)], C)
        bias = b.t(f"{name}_b", [("N", n)], C)
        y = mat(f"{name}_y", seq, n)
        b.op(ir.GMM, [x, w], y)
        gmms.append(len(b.g.nodes) - 1)
        yb = mat(f"{name}_yb", seq, n, role_out)
        b.op(ir.BIASADD, [y, bias], yb)
        return yb

    h = mat("h0", seq, hidden, I)
    for l in range(layers):
        last = l == layers - 1
        linear(f"l{l}_qkv", h, hidden, qkv, O)
        ao = linear(f"l{l}_ao", h, hidden, hidden)
        a = b.op(ir.EWADD, [ao, h], mat(f"l{l}_a", seq, hidden))
        f1 = linear(f"l{l}_f1", a, hidden, ffn)
        f = b.op(ir.RELU, [f1], mat(f"l{l}_f", seq, ffn))
        f2 = linear(f"l{l}_f2", f, ffn, hidden)
        h = b.op(ir.EWADD, [f2, a], mat(f"l{l + 1}_h" if not last else "out", seq, hidden,
                                       O if last else ir.INTERMEDIATE))
    return b.g, gmms


BERT_FLOPS_PER_LAYER = 2.0 * 128 * (768 * 2304 + 768 * 768 + 768 * 3072 + 3072 * 768)


def bert_encoder(layers=12, seq=128, hidden=768, heads=12, ffn=3072, packed_qkv=False):
    """cfg5 as a real BERT-base encoder (post-LN, as in BERT) on the op-set
    extension (lfgpu.h: GELU, Softmax, LayerNorm, BmmQK, BmmPV). Per layer,
    on h[seq, hidden]:
      q, k, v = GMM(h, W{q,k,v}) + b{q,k,v}  (Wq, bq carry the 1/sqrt(Dh)
                                               attention scale)
      p       = Softmax(BmmQK(q, k))          [heads, seq, seq]
      c       = BmmPV(p, v)                   [seq, hidden]
      h1      = LayerNorm(GMM(c, Wo) + bo + h)
      h'      = LayerNorm(GELU(GMM(h1, W1) + b1) @ W2 + b2 + h1)
    packed_qkv: one GMM(h, Wqkv[hidden, 3*hidden]) + bqkv instead of three;
    BmmQK reads q and k, BmmPV reads v as column slices of it (a_col0 /
    b_col0 / head_dim) — the same arithmetic per element, 2 fewer launches
    per layer.
    Returns (graph, gmm node indices)."""
    b = Builder()
    I, C, O = ir.INPUT, ir.CONSTANT, ir.OUTPUT
    gmms = []

    def mat(tid, m, n, role=ir.INTERMEDIATE):
        return b.t(tid, [("M", m), ("N", n)], role)

    def linear(name, x, k, n, out_id=None):
        w = b.t(f"{name}_w", [("K", k), ("N", n)], C)
        bias = b.t(f"{name}_b", [("N", n)], C)
        y = mat(f"{name}_y", seq, n)
        b.op(ir.GMM, [x, w], y)
        gmms.append(len(b.g.nodes) - 1)
        return b.op(ir.BIASADD, [y, bias], mat(out_id or f"{name}_yb", seq, n))

    def layernorm(name, x, out_id, role=ir.INTERMEDIATE):
        gb = b.t(f"{name}_gb", [("P", 2), ("N", hidden)], C)
        return b.op(ir.LAYERNORM, [x, gb], mat(out_id, seq, hidden, role), eps_exp=12)

    h = mat("h0", seq, hidden, I)
    for l in range(layers):
        last = l == layers - 1
        dh = hidden // heads
        if packed_qkv:
            qkv = linear(f"l{l}_qkv", h, hidden, 3 * hidden)
            s_ = b.op(ir.BMM_QK, [qkv, qkv], b.t(f"l{l}_s", [("H", heads), ("M", seq), ("T", seq)]), heads=heads,
                      a_col0=0, b_col0=hidden, head_dim=dh)
            p_ = b.op(ir.SOFTMAX, [s_], b.t(f"l{l}_p", [("H", heads), ("M", seq), ("T", seq)]))
            c = b.op(ir.BMM_PV, [p_, qkv], mat(f"l{l}_c", seq, hidden), heads=heads, b_col0=2 * hidden, head_dim=dh)
        else:
            q = linear(f"l{l}_q", h, hidden, hidden)
            k = linear(f"l{l}_k", h, hidden, hidden)
            v = linear(f"l{l}_v", h, hidden, hidden)
            s_ = b.op(ir.BMM_QK, [q, k], b.t(f"l{l}_s", [("H", heads), ("M", seq), ("T", seq)]), heads=heads)
            p_ = b.op(ir.SOFTMAX, [s_], b.t(f"l{l}_p", [("H", heads), ("M", seq), ("T", seq)]))
            c = b.op(ir.BMM_PV, [p_, v], mat(f"l{l}_c", seq, hidden), heads=heads)
        ao = linear(f"l{l}_ao", c, hidden, hidden)
        a = b.op(ir.EWADD, [ao, h], mat(f"l{l}_a", seq, hidden))
        h1 = layernorm(f"l{l}_ln1", a, f"l{l}_h1")
        f1 = linear(f"l{l}_f1", h1, hidden, ffn)
        f = b.op(ir.GELU, [f1], mat(f"l{l}_f", seq, ffn))
        f2 = linear(f"l{l}_f2", f, ffn, hidden)
        o = b.op(ir.EWADD, [f2, h1], mat(f"l{l}_o", seq, hidden))
        h = layernorm(f"l{l}_ln2", o, "out" if last else f"l{l + 1}_h", O if last else ir.INTERMEDIATE)
    return b.g, gmms


def bert_encoder_flops(layers=12, seq=128, hidden=768, heads=12, ffn=3072):
    gemm = 2.0 * seq * (4 * hidden * hidden + 2 * hidden * ffn)
    attn = 2.0 * 2 * seq * seq * hidden  # BmmQK + BmmPV over all heads
    return layers * (gemm + attn)


# ---------------------------------------------------------------------------
# cfg4: ResNet-18 inference graph (BatchNorm folded into the conv bias).

class Builder:
    """Small helper to declare tensors and nodes in order."""

    def __init__(self):
        self.g = ir.Graph()

    def t(self, tid, dims, role=ir.INTERMEDIATE):
        self.g.tensors.append(ir.TensorDecl(tid, list(dims), role))
        return tid

    def op(self, kind, inputs, out, **attrs):
        self.g.nodes.append(ir.OperatorNode(kind, list(inputs), out, dict(attrs)))
        return out


RESNET18_STAGES = [(64, 1), (128, 2), (256, 2), (512, 2)]


def resnet18(n, classes=1000, h=224):
    """ResNet-18 v1 inference as one graph. Returns (graph, info) where info
    lists the C2D nodes with their role:
      stem   7x7 s2 3->64 (+ bias + ReLU), then Padding(1) + MaxPool 3 s2
      per basic block: Padding -> C2D 3x3 (stride s) -> BiasAdd -> ReLU ->
        Padding -> C2D 3x3 -> BiasAdd -> EwAdd(residual) -> ReLU; the first
        block of stages 2-4 has a LayoutConvert -> C2D 1x1 s2 -> BiasAdd
        downsample branch as the residual
      GlobalAvgPool -> GMM 512x1000 -> BiasAdd -> logits
    The downsample nodes are declared before the block's main path so the
    residual exists when the fused epilogue of the second conv reads it."""
    b = Builder()
    I, C, O = ir.INPUT, ir.CONSTANT, ir.OUTPUT

    def nchw(tid, c, hh, role=ir.INTERMEDIATE):
        return b.t(tid, [("N", n), ("C", c), ("H", hh), ("W", hh)], role)

    convs = []

    def conv(name, x, cin, cout, hin, k, stride, pad, role):
        """Padding (if pad) -> C2D -> BiasAdd; returns (biased tensor, hout)."""
        xin = x
        hp = hin + 2 * pad
        if pad:
            xin = nchw(f"{name}_xp", cin, hp)
            b.op(ir.PADDING, [x], xin, pad=pad)
        else:
            xin = nchw(f"{name}_xcv", cin, hin)
            b.op(ir.LAYOUT_CONVERT, [x], xin)
        ho = (hp - k) // stride + 1
        w = b.t(f"{name}_w", [("O", cout), ("I", cin), ("KH", k), ("KW", k)], C)
        bias = b.t(f"{name}_b", [("O", cout)], C)
        y = nchw(f"{name}_y", cout, ho)
        b.op(ir.C2D, [xin, w], y, stride=stride)
        convs.append({"name": name, "node": len(b.g.nodes) - 1, "cin": cin, "cout": cout,
                      "h": hin, "k": k, "stride": stride, "pad": pad, "role": role})
        yb = nchw(f"{name}_yb", cout, ho)
        b.op(ir.BIASADD, [y, bias], yb)
        return yb, ho

    x = nchw("x", 3, h, I)
    s, hh = conv("stem", x, 3, 64, h, 7, 2, 3, "stem")
    r = nchw("stem_r", 64, hh)
    b.op(ir.RELU, [s], r)
    mp_in = nchw("pool_xp", 64, hh + 2)
    b.op(ir.PADDING, [r], mp_in, pad=1)
    hh = (hh + 2 - 3) // 2 + 1
    cur = nchw("pool_y", 64, hh)
    b.op(ir.MAXPOOL, [mp_in], cur, window=3, stride=2)
    cin = 64
    for si, (cout, stride) in enumerate(RESNET18_STAGES):
        for bi in range(2):
            st = stride if bi == 0 else 1
            name = f"s{si + 1}b{bi + 1}"
            res = cur
            if st != 1 or cin != cout:
                res, _ = conv(f"{name}_ds", cur, cin, cout, hh, 1, st, 0, f"s{si + 1}_ds")
            a, ho = conv(f"{name}_a", cur, cin, cout, hh, 3, st, 1, f"s{si + 1}_a")
            ar = nchw(f"{name}_ar", cout, ho)
            b.op(ir.RELU, [a], ar)
            bb, _ = conv(f"{name}_b", ar, cout, cout, ho, 3, 1, 1, f"s{si + 1}_b")
            sm = nchw(f"{name}_sum", cout, ho)
            b.op(ir.EWADD, [bb, res], sm)
            cur = nchw(f"{name}_out", cout, ho)
            b.op(ir.RELU, [sm], cur)
            cin, hh = cout, ho
    gp = b.t("gap", [("N", n), ("C", cin)])
    b.op(ir.GLOBAL_AVGPOOL, [cur], gp)
    fw = b.t("fc_w", [("K", cin), ("M", classes)], C)
    fb = b.t("fc_b", [("M", classes)], C)
    lg = b.t("fc_y", [("N", n), ("M", classes)])
    b.op(ir.GMM, [gp, fw], lg)
    b.op(ir.BIASADD, [lg, fb], b.t("logits", [("N", n), ("M", classes)], O))
    return b.g, convs


def propagate_elementwise(g, seqs):
    """Element-wise outputs inherit their first input's layout (the
    reference's forward propagation through element-wise chains,
    propagation.cpp); returns a new SeqMap."""
    out = dict(seqs)
    for nd in g.nodes:
        if ir.is_elementwise_op(nd.kind) and nd.output not in out and nd.inputs[0] in out:
            out[nd.output] = out[nd.inputs[0]]
    return out


def resnet18_seqs(g, convs, factors_of):
    """SeqMap for the ResNet-18 graph from per-conv C2D template factors
    (name -> (h_t, w_t, o_t, i_t, i'_t, o'_t); missing -> logical layouts).
    The MaxPool writes stage 1's residual layout; element-wise outputs
    inherit their producer's layout."""
    from . import runtime
    seqs = {}
    for c in convs:
        f = factors_of.get(c["name"])
        if f:
            seqs.update(runtime.decode_layout(g, c["node"], list(f)))
    if "s1b1_b_y" in seqs:
        seqs["pool_y"] = seqs["s1b1_b_y"]
    return propagate_elementwise(g, seqs)


def tune_resnet18(n, inputs_for, ctx=None, log=None):
    """Per-conv GPU-measured layout choice under the residual constraint:
    within a stage, the two second convs of the blocks (3x3, stride 1) and
    the downsample conv must share one output brick (h_t, w_t, o_t) so the
    residual EwAdd fuses into the tcgen05 epilogue. The brick minimises
    2*t(second conv) + t(downsample) over bricks legal for both; the other
    convs are tuned freely. `inputs_for(graph)` returns device inputs for a
    sub-graph. Returns name -> factors (absent: logical layouts)."""
    from . import tuner
    g, convs = resnet18(n)
    chosen, memo = {}, {}

    def shape_key(c):
        return (c["cin"], c["cout"], c["h"], c["k"], c["stride"], c["pad"])

    def sweep(c):
        """{factors: cost_us} over the template candidates of conv c's shape."""
        key = shape_key(c)
        if key not in memo:
            sub, node = conv_graph(n, *key)
            res, _ = tuner.sweep(sub, tuner.conv_candidates(sub, node), inputs_for(sub),
                                 warmup=1, reps=3, ctx=ctx)
            memo[key] = {tuple(r.candidate.factors[node]): r.cost_us
                         for r in res if r.cost_us is not None}
        return memo[key]

    def best_of(costs, brick=None):
        ok = {f: t for f, t in costs.items() if brick is None or f[:3] == brick}
        return min(ok, key=ok.get) if ok else None

    for si in range(len(RESNET18_STAGES)):
        tag = f"s{si + 1}"
        seconds = [c for c in convs if c["role"] == tag + "_b"]
        ds = [c for c in convs if c["role"] == tag + "_ds"]
        cb = sweep(seconds[0])
        brick = None
        if ds:
            cd = sweep(ds[0])
            tb = {}
            for f, t in cb.items():
                tb[f[:3]] = min(t, tb.get(f[:3], float("inf")))
            td = {}
            for f, t in cd.items():
                td[f[:3]] = min(t, td.get(f[:3], float("inf")))
            both = [k for k in tb if k in td]
            if both:
                brick = min(both, key=lambda k: 2 * tb[k] + td[k])
            fd = best_of(cd, brick)
            if fd:
                chosen[ds[0]["name"]] = fd
        fb = best_of(cb, brick)
        for c in seconds:
            if fb:
                chosen[c["name"]] = fb
    for c in convs:
        if c["name"] in chosen or c["role"] == "stem" or c["role"].endswith(("_b", "_ds")):
            continue
        f = best_of(sweep(c))
        if f:
            chosen[c["name"]] = f
    if log:
        for c in convs:
            log(f"{c['name']}: {chosen.get(c['name'])}")
    return chosen
