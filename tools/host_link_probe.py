"""Host-link probe (diagnostics): pageable vs pinned H2D/D2H of 16 MB, host
memcpy rates, and cudaHostRegister cost on this box."""
import ctypes, time
import numpy as np
import torch
n = 2 << 20  # doubles = 16 MB
a = np.random.rand(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64).pin_memory()
def t(f, r=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(r): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / r
ta = torch.from_numpy(a)
print("pageable H2D GB/s", 16e-3 * 1 / t(lambda: d.copy_(ta)))
print("pinned H2D GB/s", 16e-3 / t(lambda: d.copy_(pin, non_blocking=True)))
print("pinned D2H GB/s", 16e-3 / t(lambda: pin.copy_(d, non_blocking=True)))
print("pageable D2H GB/s", 16e-3 / t(lambda: ta.copy_(d)))
b = np.empty_like(a)
print("np memcpy GB/s", 16e-3 / t(lambda: np.copyto(b, a)))
pn = pin.numpy()
print("memcpy to pinned GB/s", 16e-3 / t(lambda: np.copyto(pn, a)))
cudart = ctypes.CDLL("libcudart.so") if False else None
import os
print("cpus", os.cpu_count())
