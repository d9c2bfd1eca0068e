"""K1 / K2 on the GPU against the oracle: bit-exact, as layout conversion is a
copy. Calls go through the C-ABI (liblfgpu.so)."""
import numpy as np
import pytest

import oracle_lib as O
from paper_2210_12415_b200 import runtime
from paper_2210_12415_b200.layout import fuse, padding, reorder, split, unfold
from test_oracle import seq_from, src_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(x, dtype=torch.float32):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def gpu_convert(ext, src_seq, dst_seq, src_np, dtype=torch.float32, out_dtype=None):
    out_dtype = out_dtype or dtype
    n_out = int(np.prod(O.derive(ext, dst_seq)))
    src = dev(src_np, dtype)
    dst = torch.full((n_out,), float("nan"), dtype=out_dtype, device="cuda")
    runtime.layout_convert(src, [(f"D{i}", e) for i, e in enumerate(ext)], src_seq, dst_seq, dst)
    torch.cuda.synchronize()
    return dst.double().cpu().numpy()


def test_materialize_golden_bitexact(golden):
    for case in golden["materialize"]:
        seq = seq_from(case["seq"])
        src = src_for(case)
        got = gpu_convert(case["extents"], [], seq, src)
        assert O.fnv1a(got) == case["out"]["fnv"], case["name"]
        want = O.materialize(case["extents"], seq, src)
        assert np.array_equal(got, want), case["name"]


def test_materialize_to_bf16_exact(golden):
    # k/64 values are exact in bf16: the tensor-core operand packing is lossless.
    for case in golden["materialize"]:
        seq = seq_from(case["seq"])
        src = src_for(case)
        got = gpu_convert(case["extents"], [], seq, src, out_dtype=torch.bfloat16)
        assert np.array_equal(got, O.materialize(case["extents"], seq, src)), case["name"]


def random_seq(rng, ext):
    seq, cur = [], list(ext)
    for _ in range(int(rng.integers(1, 5))):
        k = int(rng.integers(0, 5))
        d = int(rng.integers(0, len(cur)))
        if k == 0 and cur[d] > 1:
            divs = [f for f in range(1, cur[d] + 1) if cur[d] % f == 0]
            f = int(rng.choice(divs))
            p = split(d, [cur[d] // f, f])
        elif k == 1:
            p = reorder([int(v) for v in rng.permutation(len(cur))])
        elif k == 2 and d + 1 < len(cur):
            p = fuse(d, 2)
        elif k == 3:
            b = int(rng.integers(1, cur[d] + 1))
            p = unfold(d, b, int(rng.integers(1, b + 1)))
        else:
            p = padding(d, int(rng.integers(0, 3)))
        try:
            cur = O.derive(cur, [p])
        except ValueError:
            continue
        if len(cur) > 10:
            break
        seq.append(p)
    return seq


def test_materialize_fuzz_bitexact():
    rng = np.random.default_rng(2024)
    kinds = {0: 0, 1: 0}
    for it in range(300):
        rank = int(rng.integers(1, 5))
        ext = [int(rng.integers(1, 9)) for _ in range(rank)]
        seq = random_seq(rng, ext)
        x = rng.integers(-64, 65, int(np.prod(ext))) / 64.0
        got = gpu_convert(ext, [], seq, x)
        want = O.materialize(ext, seq, x)
        assert np.array_equal(got, want), (ext, seq)
        kinds[runtime.convert_kind([(f"D{i}", e) for i, e in enumerate(ext)], [], seq)] += 1
    assert kinds[1] > 50 and kinds[0] > 5  # both the digit map and the general program ran


def test_back_conversion_and_relayout():
    rng = np.random.default_rng(5)
    for it in range(120):
        rank = int(rng.integers(1, 5))
        ext = [int(rng.integers(1, 8)) for _ in range(rank)]
        s1, s2 = random_seq(rng, ext), random_seq(rng, ext)
        x = rng.integers(-64, 65, int(np.prod(ext))) / 64.0
        p1 = O.materialize(ext, s1, x)
        # physical (s1) -> logical: interpret's forward-map read-back
        back = gpu_convert(ext, s1, [], p1)
        assert np.array_equal(back, O.to_logical(ext, s1, p1)), (ext, s1)
        # physical (s1) -> physical (s2) through the logical index
        got = gpu_convert(ext, s1, s2, p1)
        assert np.array_equal(got, O.materialize(ext, s2, O.to_logical(ext, s1, p1))), (s1, s2)


def test_large_nchw_to_nchwc16():
    # Many CTAs / tiles: N=64 NCHW -> NCHWc16 against a torch permute.
    N, Cc, H, W = 64, 64, 56, 56
    x = torch.randint(-64, 65, (N, Cc, H, W), device="cuda").float() / 64
    dst = torch.empty(N * Cc * H * W, device="cuda")
    runtime.layout_convert(x, [("N", N), ("C", Cc), ("H", H), ("W", W)], [],
                           [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])], dst)
    want = x.view(N, 4, 16, H, W).permute(0, 1, 3, 4, 2).contiguous().view(-1)
    assert torch.equal(dst, want)


PAD_CASES = [
    # (input NCHW, pad, src seq, dst seq)
    ([1, 64, 56, 56], 1, [],
     [unfold(3, 16, 14), unfold(2, 6, 4), split(1, [4, 16]), reorder([0, 3, 5, 1, 4, 6, 2])]),
    ([1, 64, 56, 56], 1, [split(1, [4, 16]), reorder([0, 1, 3, 4, 2])],
     [unfold(3, 16, 14), unfold(2, 6, 4), split(1, [4, 16]), reorder([0, 3, 5, 1, 4, 6, 2])]),
    ([2, 3, 9, 7], 2, [], [unfold(2, 5, 4), reorder([0, 2, 1, 3, 4])]),  # overhang -> 0
    ([1, 4, 6, 6], 1, [], []),
    ([1, 8, 6, 6], 3, [], [split(1, [2, 4]), reorder([0, 1, 3, 4, 2])]),
]


def test_pad_convert_bitexact():
    rng = np.random.default_rng(8)
    for in_ext, pad, sseq, dseq in PAD_CASES:
        x = rng.integers(-64, 65, int(np.prod(in_ext))) / 64.0
        xs = O.materialize(in_ext, sseq, x)
        rc, want = O.padding_nest(in_ext, pad, sseq, dseq, xs)
        assert rc == 0
        for dt in (torch.float32, torch.bfloat16):
            src = dev(xs)
            dst = torch.full((want.size,), float("nan"), dtype=dt, device="cuda")
            runtime.pad_convert(src, [(f"D{i}", e) for i, e in enumerate(in_ext)], pad, sseq,
                                dseq, dst)
            torch.cuda.synchronize()
            assert np.array_equal(dst.double().cpu().numpy(), want), (in_ext, pad, dseq, dt)
