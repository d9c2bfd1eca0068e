"""Mismatch map of the CTA-pair GEMM against the oracle for one shape / knob
setting (debugging aid: prints, per 64x64 block of C, the count of wrong
elements). usage: LFGPU_PAIR_S=2 python tools/pair_debug.py M K N [m_t k_t n_t]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as O  # noqa: E402
from paper_2210_12415_b200 import _abi, ir, runtime  # noqa: E402

M, K, N = (int(x) for x in sys.argv[1:4])
f = [int(x) for x in sys.argv[4:7]] if len(sys.argv) > 6 else None
g = ir.gemm(M, K, N)
seqs = runtime.decode_layout(g, 0, f) if f else {}
if os.environ.get("BK"):  # K-major B: [K/64][N][64]
    from paper_2210_12415_b200.layout import reorder, split
    seqs["b"] = [split(0, [K // 64, 64]), reorder([0, 2, 1])]
bufs = O.random_inputs(g, 42)
a, b = bufs[0].copy(), bufs[1].copy()
ref = (a.reshape(M, K) @ b.reshape(K, N))
ds = os.environ.get("LFGPU_PAIR_DBG_SPLIT")
if ds is not None:  # only split `ds` of S: its K range
    S = int(os.environ.get("LFGPU_PAIR_S", "1"))
    k0, k1 = int(ds) * K // S, (int(ds) + 1) * K // S
    ref = a.reshape(M, K)[:, k0:k1] @ b.reshape(K, N)[k0:k1, :]
p = runtime.Plan(g, seqs, [], flags=_abi.PLAN_REQUIRE_TC)
p.set_input("a", a)
p.set_input("b", b)
p.run()
got = p.get_output("c").reshape(M, N)
print(p.node_kernel(0))
bad = got != ref
print("wrong:", int(bad.sum()), "of", bad.size)
for i in range(0, M, 64):
    print(" ".join("%4d" % bad[i:i + 64, j:j + 64].sum() for j in range(0, N, 64)))
if ds is not None and bad.any():
    S = int(os.environ.get("LFGPU_PAIR_S", "1"))
    A2, B2 = a.reshape(M, K), b.reshape(K, N)
    rr, cc = np.argwhere(bad)[0]
    print("first wrong at", rr, cc, "got", got[rr, cc], "want", ref[rr, cc])
    cands = {}
    for sa in range(S):
        for sb in range(S):
            ka = slice(sa * K // S, (sa + 1) * K // S)
            kb = slice(sb * K // S, (sb + 1) * K // S)
            for sh in (-128, -64, 0, 64, 128):
                c = (cc + sh) % N
                cands[f"A_s{sa} B_s{sb} col{sh:+d}"] = A2[rr, ka] @ B2[kb, c]
    for k, v in cands.items():
        if v == got[rr, cc]:
            print("  matches", k)
    print("  zero?", got[rr, cc] == 0)
