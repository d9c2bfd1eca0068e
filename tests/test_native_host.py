"""Host-side checks of the native library (no GPU needed): it loads, exports
every symbol include/lfgpu.h declares, the ctypes structs match the C
layout, and the host layout algebra / template decoding agree with the
reference's golden outputs."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib as O
from paper_2210_12415_b200 import _abi, ir, runtime
from paper_2210_12415_b200.layout import fuse, padding, reorder, split, unfold
from test_oracle import GRAPHS, seq_from

HEADER = os.path.join(O.ROOT, "include", "lfgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lfgpu_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = runtime.lib()
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), f"{name} declared in lfgpu.h but not exported"
    assert sorted(runtime.EXPORTS) == decl


def test_struct_sizes_match_header(tmp_path):
    # The C compiler's view of include/lfgpu.h against the ctypes mirror.
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "lfgpu.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(lfgpu_prim), sizeof(lfgpu_dim), sizeof(lfgpu_tensor),'
                   'sizeof(lfgpu_node), sizeof(lfgpu_seq), sizeof(lfgpu_graph),'
                   'sizeof(lfgpu_sched), sizeof(lfgpu_counters),'
                   'offsetof(lfgpu_prim, tile), offsetof(lfgpu_tensor, dims));return 0;}\n')
    exe = tmp_path / "sizes"
    import subprocess
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(_abi.Prim), C.sizeof(_abi.Dim), C.sizeof(_abi.Tensor), C.sizeof(_abi.Node),
            C.sizeof(_abi.Seq), C.sizeof(_abi.GraphDesc), C.sizeof(_abi.Sched),
            C.sizeof(_abi.Counters), _abi.Prim.tile.offset, _abi.Tensor.dims.offset]
    assert got == want
    assert runtime.lib().lfgpu_version() == 1


def test_derive_layout_matches_oracle(golden):
    for case in golden["materialize"]:
        seq = seq_from(case["seq"])
        got = runtime.derive_layout(case["extents"], seq)
        assert [e for _, e in got] == case["phys"], case["name"]


def test_derive_layout_names_and_errors():
    dims = [("N", 1), ("O", 32), ("H", 6), ("W", 6)]
    got = runtime.derive_layout(dims, [split(1, [2, 16]), reorder([0, 1, 3, 4, 2])])
    assert got == [("N", 1), ("O0", 2), ("H", 6), ("W", 6), ("O1", 16)]
    with pytest.raises(runtime.LfError) as e:
        runtime.derive_layout(dims, [split(1, [3, 16])])
    assert e.value.code == _abi.EINVAL and "factors multiply to 48" in str(e.value)
    with pytest.raises(runtime.LfError):
        runtime.derive_layout(dims, [unfold(2, 7, 2)])  # tile > extent
    with pytest.raises(runtime.LfError):
        runtime.derive_layout(dims, [reorder([0, 0, 1, 2])])


def test_decode_layout_matches_reference(golden):
    for case in golden["decode_layout"]:
        g = GRAPHS[case["graph"]]()
        got = runtime.decode_layout(g, case["node"], case["factors"], case["levels"])
        want = {k: seq_from(v) for k, v in case["seqs"].items()}
        assert set(got) == set(want), case
        for k in want:
            assert got[k] == want[k], (case["graph"], case["factors"], k)


def test_layout_template_matches_reference(golden):
    for case in golden["layout_template"]:
        g = GRAPHS[case["graph"]]()
        t = runtime.layout_template(g, case["node"], case["levels"])
        assert [e for _, e in t] == case["extents"]
        nd = [len([d for d in range(1, e + 1) if e % d == 0]) for _, e in t]
        assert nd == case["ndivisors"]


def test_tuner_layouts_compile_to_digit_maps():
    # Every template layout (split / reorder / unfold) takes the affine fast path.
    g = GRAPHS["cfg1_pad_conv"]()
    seqs = runtime.decode_layout(g, 1, [4, 14, 16, 16, 16, 16])
    for tid, seq in seqs.items():
        dims = g.tensor(tid).dims
        assert runtime.convert_kind(dims, [], seq) == 1, tid
        # Reading an overlapped tile back needs min(l/S, T-1) when S does not
        # divide the extent (58 % 14 != 0): the general program handles it.
        assert runtime.convert_kind(dims, seq, []) == (0 if tid == "xp" else 1), tid
    # fuse across a misaligned split needs the general program
    assert runtime.convert_kind([("A", 6), ("B", 4)], [], [fuse(0, 2), split(0, [8, 3])]) == 0
    assert runtime.convert_kind([("A", 6)], [], [padding(0, 2), split(0, [2, 4])]) == 1
