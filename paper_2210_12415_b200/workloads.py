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
