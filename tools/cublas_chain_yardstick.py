"""Yardstick only (never a path): cuBLAS (torch.matmul, bf16 in / bf16 out)
on the BERT-base layer's GEMM shapes at M = 128, each timed back to back in
a CUDA graph of 100 launches, and the 4-GEMM layer chain with bias / GELU /
residual as separate torch ops."""
import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
shapes = [(128, 768, 2304), (128, 768, 768), (128, 768, 3072), (128, 3072, 768), (1024, 1024, 1024)]


def graph_time(fn, reps=100):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for m, k, n in shapes:
    a = torch.randn(m, k, device=dev, dtype=torch.bfloat16)
    b = torch.randn(k, n, device=dev, dtype=torch.bfloat16)
    c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    us = graph_time(lambda: torch.matmul(a, b, out=c))
    print(f"cuBLAS {m}x{k}x{n}: {us:.2f} us  {2*m*k*n/us/1e6:.1f} TFLOP/s", flush=True)
    cf = torch.empty(m, n, device=dev, dtype=torch.float32)
    af, bf_ = a.float(), b.float()
    us = graph_time(lambda: torch.matmul(af, bf_, out=cf))
    print(f"cuBLAS fp32 {m}x{k}x{n}: {us:.2f} us", flush=True)

h = torch.randn(128, 768, device=dev, dtype=torch.bfloat16)
W = [torch.randn(768, 2304, device=dev, dtype=torch.bfloat16), torch.randn(768, 768, device=dev, dtype=torch.bfloat16),
     torch.randn(768, 3072, device=dev, dtype=torch.bfloat16), torch.randn(3072, 768, device=dev, dtype=torch.bfloat16)]
bias = [torch.randn(w.shape[1], device=dev, dtype=torch.bfloat16) for w in W]
ln = torch.nn.LayerNorm(768, device=dev, dtype=torch.bfloat16)


def layer():
    qkv = torch.addmm(bias[0], h, W[0])
    q, k, v = qkv.view(128, 3, 12, 64).unbind(1)
    att = torch.nn.functional.scaled_dot_product_attention(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1))
    c = att.transpose(0, 1).reshape(128, 768)
    a = ln(torch.addmm(bias[1], c, W[1]) + h)
    f = torch.nn.functional.gelu(torch.addmm(bias[2], a, W[2]))
    return ln(torch.addmm(bias[3], f, W[3]) + a)


us = graph_time(layer, reps=12)
print(f"torch BERT-base layer (bf16, cuBLAS + SDPA, graph): {us:.1f} us per layer, {12*us:.0f} us per 12 layers")
