"""Test-side bindings of the oracle (oracle/liblforacle.so) and of the
reference build (oracle/_ref/libref.so). TEST INFRASTRUCTURE ONLY."""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2210_12415_b200 import _abi
from paper_2210_12415_b200.ir import Graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liblforacle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref.so")

_DP = C.POINTER(C.c_double)
_I64P = C.POINTER(C.c_int64)


def build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        lib = C.CDLL(ORACLE_SO)
        lib.lfo_fnv1a_f32.restype = C.c_uint64
        lib.lfo_max_rel_diff.restype = C.c_double
        _oracle = lib
    return _oracle


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_SO)
        _ref.ref_last_error.restype = C.c_char_p
    return _ref


def dptr(a):
    return a.ctypes.data_as(_DP)


def i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(_I64P)


def alloc_buffers(g: Graph):
    return [np.zeros(t.num_elements(), dtype=np.float64) for t in g.tensors]


def buf_ptrs(bufs):
    arr = (_DP * len(bufs))()
    for i, b in enumerate(bufs):
        arr[i] = dptr(b)
    return arr


def random_inputs(g: Graph, seed, lib=None):
    """lf::random_inputs via the oracle (or the reference when lib='ref')."""
    bufs = alloc_buffers(g)
    cg = g.to_c()
    if lib == "ref":
        rc = ref().ref_random_inputs(cg.ptr(), C.c_uint64(seed), buf_ptrs(bufs))
        assert rc == 0, ref().ref_last_error()
    else:
        oracle().lfo_random_inputs(cg.ptr(), C.c_uint64(seed), buf_ptrs(bufs))
    return bufs


def reference_eval(g: Graph, bufs, lib=None):
    cg = g.to_c()
    if lib == "ref":
        rc = ref().ref_reference_eval(cg.ptr(), buf_ptrs(bufs))
        assert rc == 0, ref().ref_last_error()
    else:
        rc = oracle().lfo_reference_eval(cg.ptr(), buf_ptrs(bufs))
        assert rc == 0
    return bufs


def derive(extents, seq):
    ext, p = i64(extents)
    prims = _abi.prim_array(seq)
    out = np.zeros(_abi.MAX_RANK, dtype=np.int64)
    r = C.c_int(0)
    rc = oracle().lfo_derive(len(extents), p, len(seq), prims, C.byref(r),
                             out.ctypes.data_as(_I64P))
    if rc:
        raise ValueError("invalid layout sequence")
    return [int(x) for x in out[: r.value]]


def materialize(extents, seq, src, lib=None):
    """lf::materialize_seq: logical -> physical (doubles)."""
    phys = derive(extents, seq)
    dst = np.zeros(int(np.prod(phys)), dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.float64)
    prims = _abi.prim_array(seq)
    if lib == "ref":
        dims = _abi.dim_array([(f"D{i}", e) for i, e in enumerate(extents)])
        rc = ref().ref_materialize(len(extents), dims, len(seq), prims, dptr(src), dptr(dst))
        assert rc == 0, ref().ref_last_error()
    else:
        ext, p = i64(extents)
        rc = oracle().lfo_materialize(len(extents), p, len(seq), prims, dptr(src), dptr(dst))
        assert rc == 0
    return dst


def to_logical(extents, seq, phys):
    ext, p = i64(extents)
    out = np.zeros(int(np.prod(extents)), dtype=np.float64)
    phys = np.ascontiguousarray(phys, dtype=np.float64)
    prims = _abi.prim_array(seq)
    rc = oracle().lfo_to_logical(len(extents), p, len(seq), prims, dptr(phys), dptr(out))
    assert rc == 0
    return out


def padding_nest(in_extents, pad, src_seq, dst_seq, src_phys):
    ext, p = i64(in_extents)
    out_ext = [in_extents[0], in_extents[1], in_extents[2] + 2 * pad, in_extents[3] + 2 * pad]
    dst = np.zeros(int(np.prod(derive(out_ext, dst_seq))), dtype=np.float64)
    sp, dp = _abi.prim_array(src_seq), _abi.prim_array(dst_seq)
    src_phys = np.ascontiguousarray(src_phys, dtype=np.float64)
    rc = oracle().lfo_padding_nest(p, C.c_int64(pad), len(src_seq), sp, len(dst_seq), dp,
                                   dptr(src_phys), dptr(dst))
    return rc, dst


def convert_nest(extents, src_seq, dst_seq, src_phys):
    ext, p = i64(extents)
    dst = np.zeros(int(np.prod(derive(extents, dst_seq))), dtype=np.float64)
    sp, dp = _abi.prim_array(src_seq), _abi.prim_array(dst_seq)
    src_phys = np.ascontiguousarray(src_phys, dtype=np.float64)
    rc = oracle().lfo_convert_nest(len(extents), p, len(src_seq), sp, len(dst_seq), dp,
                                   dptr(src_phys), dptr(dst))
    return rc, dst


def fnv1a(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    return "%016x" % oracle().lfo_fnv1a_f32(dptr(v), C.c_int64(v.size))


def max_rel_diff(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.size == b.size
    return oracle().lfo_max_rel_diff(dptr(a), dptr(b), C.c_int64(a.size))


def ref_interpret(g: Graph, seqs, scheds, bufs):
    cg = g.to_c(seqs)
    ns = len(scheds)
    sarr = (_abi.Sched * max(1, ns))(*scheds)
    rc = ref().ref_interpret(cg.ptr(), ns, sarr, buf_ptrs(bufs))
    return rc


def ref_simulate_cache(g: Graph, seqs, scheds):
    """lf::simulate_cache(lower(g, seqs, scheds), CacheConfig{}) (cachesim.cpp:152-174):
    the reference's measurement backend. Returns (cost, l1_misses)."""
    cg = g.to_c(seqs)
    ns = len(scheds)
    sarr = (_abi.Sched * max(1, ns))(*scheds)
    cost, miss = C.c_double(), C.c_int64()
    rc = ref().ref_simulate_cache(cg.ptr(), ns, sarr, C.byref(cost), C.byref(miss))
    assert rc == 0, ref().ref_last_error()
    return cost.value, miss.value


def ref_decode_layout(g: Graph, node, factors, tiling_levels=1):
    cg = g.to_c()
    f, fp = i64(factors)
    out = (_abi.Seq * 16)()
    storage = (_abi.Prim * 128)()
    n = C.c_int(0)
    rc = ref().ref_decode_layout(cg.ptr(), node, tiling_levels, fp, len(factors), out, 16,
                                 C.byref(n), storage, 128)
    assert rc == 0, ref().ref_last_error()
    from paper_2210_12415_b200.layout import LayoutPrimitive
    res = {}
    for i in range(n.value):
        res[g.tensors[out[i].tensor].id] = [
            LayoutPrimitive.from_c(out[i].prims[k], lambda t: g.tensors[t].id)
            for k in range(out[i].nprims)]
    return res


def ref_layout_template(g: Graph, node, tiling_levels=1):
    cg = g.to_c()
    ext = np.zeros(16, dtype=np.int64)
    nd = np.zeros(16, dtype=np.int64)
    n = C.c_int(0)
    rc = ref().ref_layout_template(cg.ptr(), node, tiling_levels, C.byref(n),
                                   ext.ctypes.data_as(_I64P), nd.ctypes.data_as(_I64P))
    assert rc == 0, ref().ref_last_error()
    return [int(x) for x in ext[: n.value]], [int(x) for x in nd[: n.value]]


def ref_plan_context(g: Graph, factors, tiling_levels=1):
    """Reference planner + insert_conversions; returns (graph, seqs)."""
    cg = g.to_c()
    f, fp = i64(factors)
    tensors = (_abi.Tensor * 64)()
    nodes = (_abi.Node * 64)()
    seqs = (_abi.Seq * 64)()
    storage = (_abi.Prim * 512)()
    nt, nn, ns = C.c_int(0), C.c_int(0), C.c_int(0)
    rc = ref().ref_plan_context(cg.ptr(), tiling_levels, fp, tensors, 64, nodes, 64, seqs, 64,
                                storage, 512, C.byref(nt), C.byref(nn), C.byref(ns))
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    desc = _abi.GraphDesc()
    desc.ntensors, desc.nnodes, desc.nseqs = nt.value, nn.value, ns.value
    desc.tensors = C.cast(tensors, C.POINTER(_abi.Tensor))
    desc.nodes = C.cast(nodes, C.POINTER(_abi.Node))
    desc.seqs = C.cast(seqs, C.POINTER(_abi.Seq))
    return Graph.from_c(desc)
