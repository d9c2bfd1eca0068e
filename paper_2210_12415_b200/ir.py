"""Graph IR — the Python face of lf::Graph / TensorDecl / OperatorNode.

Mirrors proj/include/layoutforge/ir.hpp:17-83 and the micrograph builders of
proj/tests/graphs.hpp:10-106 (conv_chain, dep_chain, gmm_chain, bare_conv).
Graphs are handed to the native library as POD descriptors (lfgpu_graph);
`Graph.to_c(seqs)` builds one and keeps the ctypes storage alive.
"""
import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import _abi
from .layout import LayoutPrimitive

F32, I32 = _abi.F32, _abi.I32
INPUT, CONSTANT, INTERMEDIATE, OUTPUT = _abi.INPUT, _abi.CONSTANT, _abi.INTERMEDIATE, _abi.OUTPUT
C2D, DEP, GMM, PADDING, RELU, BIASADD, EWADD, LAYOUT_CONVERT = (
    _abi.C2D, _abi.DEP, _abi.GMM, _abi.PADDING, _abi.RELU, _abi.BIASADD, _abi.EWADD,
    _abi.LAYOUT_CONVERT)
# Op-set extension: the pools ResNet-18 needs.
MAXPOOL, GLOBAL_AVGPOOL = _abi.MAXPOOL, _abi.GLOBAL_AVGPOOL
# ... and the rest of a BERT encoder (lfgpu.h documents each op's semantics).
GELU, SOFTMAX, LAYERNORM, BMM_QK, BMM_PV = (_abi.GELU, _abi.SOFTMAX, _abi.LAYERNORM,
                                            _abi.BMM_QK, _abi.BMM_PV)

OP_NAMES = {C2D: "C2D", DEP: "DEP", GMM: "GMM", PADDING: "Padding", RELU: "ReLU",
            BIASADD: "BiasAdd", EWADD: "EwAdd", LAYOUT_CONVERT: "LayoutConvert",
            MAXPOOL: "MaxPool", GLOBAL_AVGPOOL: "GlobalAvgPool", GELU: "GELU",
            SOFTMAX: "Softmax", LAYERNORM: "LayerNorm", BMM_QK: "BmmQK", BMM_PV: "BmmPV"}


def is_complex_op(k):  # ir.cpp:26-28
    return k in (C2D, DEP, GMM)


def is_elementwise_op(k):  # ir.cpp:30-32 (+ GELU, fused into epilogues like ReLU)
    return k in (RELU, BIASADD, EWADD, GELU)


@dataclass
class TensorDecl:
    id: str
    dims: List[Tuple[str, int]]
    role: int = INTERMEDIATE
    dtype: int = F32

    @property
    def extents(self):
        return [e for _, e in self.dims]

    def num_elements(self):
        n = 1
        for _, e in self.dims:
            n *= e
        return n


@dataclass
class OperatorNode:
    kind: int
    inputs: List[str]
    output: str
    attrs: Dict[str, int] = field(default_factory=dict)

    def attr(self, key, fallback):
        return self.attrs.get(key, fallback)


@dataclass
class Graph:
    tensors: List[TensorDecl] = field(default_factory=list)
    nodes: List[OperatorNode] = field(default_factory=list)

    def tensor_index(self, tid):
        for i, t in enumerate(self.tensors):
            if t.id == tid:
                return i
        raise KeyError(f"unknown tensor '{tid}'")

    def _target_index(self, tid):
        """store_at target index, -1 when unknown (the plan reports it, lower.cpp:54)."""
        for i, t in enumerate(self.tensors):
            if t.id == tid:
                return i
        return -1

    def tensor(self, tid):
        return self.tensors[self.tensor_index(tid)]

    def producer_of(self, tid):
        for i, n in enumerate(self.nodes):
            if n.output == tid:
                return i
        return -1

    def consumers_of(self, tid):
        return [i for i, n in enumerate(self.nodes) if tid in n.inputs]

    def to_c(self, seqs: Optional[Dict[str, List[LayoutPrimitive]]] = None):
        """lfgpu_graph descriptor; the returned object owns all storage."""
        return CGraph(self, seqs or {})

    @staticmethod
    def from_c(desc):
        g = Graph()
        for t in range(desc.ntensors):
            td = desc.tensors[t]
            dims = [(td.dims[d].name.decode(), td.dims[d].extent) for d in range(td.rank)]
            g.tensors.append(TensorDecl(td.id.decode(), dims, td.role, td.dtype))
        for i in range(desc.nnodes):
            nd = desc.nodes[i]
            attrs = {}
            if nd.kind in (C2D, DEP, MAXPOOL):
                attrs["stride"] = nd.stride
            if nd.kind == MAXPOOL:
                attrs["window"] = nd.window
            if nd.kind in (BMM_QK, BMM_PV):
                attrs["heads"] = nd.heads
                if nd.a_col0:
                    attrs["a_col0"] = nd.a_col0
                if nd.b_col0:
                    attrs["b_col0"] = nd.b_col0
                if nd.head_dim:
                    attrs["head_dim"] = nd.head_dim
            if nd.kind == LAYERNORM:
                attrs["eps_exp"] = nd.eps_exp
            if nd.kind == PADDING:
                attrs["pad"] = nd.pad
            g.nodes.append(OperatorNode(nd.kind,
                                        [g.tensors[nd.inputs[j]].id for j in range(nd.ninputs)],
                                        g.tensors[nd.output].id, attrs))
        seqs = {}
        for s in range(desc.nseqs):
            sq = desc.seqs[s]
            seqs[g.tensors[sq.tensor].id] = [
                LayoutPrimitive.from_c(sq.prims[k], lambda i: g.tensors[i].id)
                for k in range(sq.nprims)]
        return g, seqs


class CGraph:
    """Owns the ctypes arrays behind one lfgpu_graph."""

    def __init__(self, g: Graph, seqs):
        self.graph = g
        nt, nn = len(g.tensors), len(g.nodes)
        self.tensors = (_abi.Tensor * max(1, nt))()
        for i, t in enumerate(g.tensors):
            d = self.tensors[i]
            d.id = t.id.encode()[: _abi.ID_LEN - 1]
            d.rank = len(t.dims)
            d.dtype = t.dtype
            d.role = t.role
            for k, (name, ext) in enumerate(t.dims):
                d.dims[k].name = name.encode()[: _abi.NAME_LEN - 1]
                d.dims[k].extent = int(ext)
        self.nodes = (_abi.Node * max(1, nn))()
        for i, n in enumerate(g.nodes):
            d = self.nodes[i]
            d.kind = n.kind
            d.ninputs = len(n.inputs)
            for j, tid in enumerate(n.inputs):
                d.inputs[j] = g.tensor_index(tid)
            d.output = g.tensor_index(n.output)
            d.stride = int(n.attr("stride", 1))
            d.pad = int(n.attr("pad", 0))
            d.window = int(n.attr("window", 0))
            d.heads = int(n.attr("heads", 0))
            d.eps_exp = int(n.attr("eps_exp", 12 if n.kind == LAYERNORM else 0))
            d.a_col0 = int(n.attr("a_col0", 0))
            d.b_col0 = int(n.attr("b_col0", 0))
            d.head_dim = int(n.attr("head_dim", 0))
        items = [(k, v) for k, v in seqs.items() if v]
        self.prim_arrays = []
        self.seqs = (_abi.Seq * max(1, len(items)))()
        for i, (tid, seq) in enumerate(items):
            arr = (_abi.Prim * len(seq))()
            for k, p in enumerate(seq):
                p.fill(arr[k], g._target_index)
            self.prim_arrays.append(arr)
            self.seqs[i].tensor = g.tensor_index(tid)
            self.seqs[i].nprims = len(seq)
            self.seqs[i].prims = C.cast(arr, C.POINTER(_abi.Prim))
        self.desc = _abi.GraphDesc()
        self.desc.ntensors = nt
        self.desc.nnodes = nn
        self.desc.nseqs = len(items)
        self.desc.tensors = C.cast(self.tensors, C.POINTER(_abi.Tensor))
        self.desc.nodes = C.cast(self.nodes, C.POINTER(_abi.Node))
        self.desc.seqs = C.cast(self.seqs, C.POINTER(_abi.Seq))

    def ptr(self):
        return C.byref(self.desc)


# ---------------------------------------------------------------------------
# Micrograph builders (proj/tests/graphs.hpp) and benchmark graphs.

def conv_chain(n, ci, co, h, k, stride, pad, dtype=F32):
    """Padding -> C2D(kxk) -> BiasAdd -> ReLU (graphs.hpp:32-53)."""
    hp = h + 2 * pad
    ho = (hp - k) // stride + 1
    g = Graph()
    g.tensors = [
        TensorDecl("x", [("N", n), ("I", ci), ("H", h), ("W", h)], INPUT, dtype),
        TensorDecl("ker", [("O", co), ("I", ci), ("KH", k), ("KW", k)], CONSTANT, dtype),
        TensorDecl("bias", [("O", co)], CONSTANT, dtype),
        TensorDecl("xp", [("N", n), ("I", ci), ("H", hp), ("W", hp)], INTERMEDIATE, dtype),
        TensorDecl("conv", [("N", n), ("O", co), ("H", ho), ("W", ho)], INTERMEDIATE, dtype),
        TensorDecl("biased", [("N", n), ("O", co), ("H", ho), ("W", ho)], INTERMEDIATE, dtype),
        TensorDecl("y", [("N", n), ("O", co), ("H", ho), ("W", ho)], OUTPUT, dtype),
    ]
    g.nodes = [
        OperatorNode(PADDING, ["x"], "xp", {"pad": pad}),
        OperatorNode(C2D, ["xp", "ker"], "conv", {"stride": stride}),
        OperatorNode(BIASADD, ["conv", "bias"], "biased"),
        OperatorNode(RELU, ["biased"], "y"),
    ]
    return g


def dep_chain(n, c, h, k, stride, pad):
    """Padding -> DEP(kxk) -> ReLU (graphs.hpp:56-73)."""
    hp = h + 2 * pad
    ho = (hp - k) // stride + 1
    g = Graph()
    g.tensors = [
        TensorDecl("x", [("N", n), ("C", c), ("H", h), ("W", h)], INPUT),
        TensorDecl("ker", [("C", c), ("KH", k), ("KW", k)], CONSTANT),
        TensorDecl("xp", [("N", n), ("C", c), ("H", hp), ("W", hp)], INTERMEDIATE),
        TensorDecl("conv", [("N", n), ("C", c), ("H", ho), ("W", ho)], INTERMEDIATE),
        TensorDecl("y", [("N", n), ("C", c), ("H", ho), ("W", ho)], OUTPUT),
    ]
    g.nodes = [
        OperatorNode(PADDING, ["x"], "xp", {"pad": pad}),
        OperatorNode(DEP, ["xp", "ker"], "conv", {"stride": stride}),
        OperatorNode(RELU, ["conv"], "y"),
    ]
    return g


def gmm_chain(m, k, n):
    """GMM -> BiasAdd -> ReLU (graphs.hpp:76-92)."""
    g = Graph()
    g.tensors = [
        TensorDecl("a", [("M", m), ("K", k)], INPUT),
        TensorDecl("b", [("K", k), ("N", n)], CONSTANT),
        TensorDecl("bias", [("N", n)], CONSTANT),
        TensorDecl("c", [("M", m), ("N", n)], INTERMEDIATE),
        TensorDecl("biased", [("M", m), ("N", n)], INTERMEDIATE),
        TensorDecl("y", [("M", m), ("N", n)], OUTPUT),
    ]
    g.nodes = [
        OperatorNode(GMM, ["a", "b"], "c"),
        OperatorNode(BIASADD, ["c", "bias"], "biased"),
        OperatorNode(RELU, ["biased"], "y"),
    ]
    return g


def bare_conv(n, ci, co, hin, k, stride):
    """Single C2D without padding (graphs.hpp:95-106)."""
    ho = (hin - k) // stride + 1
    g = Graph()
    g.tensors = [
        TensorDecl("x", [("N", n), ("I", ci), ("H", hin), ("W", hin)], INPUT),
        TensorDecl("ker", [("O", co), ("I", ci), ("KH", k), ("KW", k)], CONSTANT),
        TensorDecl("y", [("N", n), ("O", co), ("H", ho), ("W", ho)], OUTPUT),
    ]
    g.nodes = [OperatorNode(C2D, ["x", "ker"], "y", {"stride": stride})]
    return g


def pad_conv(n, ci, co, h, k, stride, pad, dtype=F32):
    """Padding -> C2D: the cfg1 graph (BASELINE.json configs[0])."""
    hp = h + 2 * pad
    ho = (hp - k) // stride + 1
    g = Graph()
    g.tensors = [
        TensorDecl("x", [("N", n), ("I", ci), ("H", h), ("W", h)], INPUT, dtype),
        TensorDecl("ker", [("O", co), ("I", ci), ("KH", k), ("KW", k)], CONSTANT, dtype),
        TensorDecl("xp", [("N", n), ("I", ci), ("H", hp), ("W", hp)], INTERMEDIATE, dtype),
        TensorDecl("y", [("N", n), ("O", co), ("H", ho), ("W", ho)], OUTPUT, dtype),
    ]
    g.nodes = [
        OperatorNode(PADDING, ["x"], "xp", {"pad": pad}),
        OperatorNode(C2D, ["xp", "ker"], "y", {"stride": stride}),
    ]
    return g


def gemm(m, k, n):
    """Single GMM: the cfg2 graph (a, b, c)."""
    g = Graph()
    g.tensors = [
        TensorDecl("a", [("M", m), ("K", k)], INPUT),
        TensorDecl("b", [("K", k), ("N", n)], INPUT),
        TensorDecl("c", [("M", m), ("N", n)], OUTPUT),
    ]
    g.nodes = [OperatorNode(GMM, ["a", "b"], "c")]
    return g
