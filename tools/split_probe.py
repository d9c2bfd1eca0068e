"""GEMM precision probe (diagnostics): bf16 tensor cores vs split mode on
general fp32 inputs against float64 numpy."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

for (M, K, N, f, tl) in [(512, 1024, 512, (256, 64, 128), 128), (128, 768, 768, (128, 64, 64), 64)]:
    g = ir.gemm(M, K, N)
    seqs = runtime.decode_layout(g, 0, list(f))
    rng = np.random.default_rng(11)
    for dist in ("normal", "uniform", "k64"):
        if dist == "normal":
            a, b = rng.standard_normal((M, K)), rng.standard_normal((K, N))
        elif dist == "uniform":
            a, b = rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N))
        else:
            a, b = rng.integers(-64, 65, (M, K)) / 64.0, rng.integers(-64, 65, (K, N)) / 64.0
        a, b = a.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
        ref = a @ b
        for name, flags in (("bf16", _abi.PLAN_REQUIRE_TC), ("split", _abi.PLAN_REQUIRE_TC | _abi.PLAN_TC_SPLIT),
                            ("exact", _abi.PLAN_EXACT)):
            p = runtime.Plan(g, seqs, [runtime.sched(0, tile_last=tl)], flags=flags)
            p.set_input("a", a.ravel())
            p.set_input("b", b.ravel())
            p.run()
            c = p.get_output("c").reshape(M, N)
            d = np.abs(c - ref) / np.maximum(1, np.maximum(np.abs(c), np.abs(ref)))
            i = np.unravel_index(np.argmax(d), d.shape)
            print(M, K, N, dist, name, "maxrel %.3g at %s got %.6g want %.6g" % (d.max(), i, c[i], ref[i]), p.node_kernel(0)[:60])
