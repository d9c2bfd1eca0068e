"""ctypes binding of liblfgpu.so — the Python face of the C-ABI.

Mirrors the reference's execution/measure functions:
  materialize_tensor (interp.cpp:280-337)   -> layout_convert / Plan.set_input
  interpret          (interp.cpp:424-470)   -> interpret / Plan
  simulate_cache     (cachesim.cpp:152-174) -> Plan.measure
and the errors of lf::Error: LfError carries the status code; code
EUNSUPPORTED is how a candidate the GPU cannot legalise is rejected.
There is no fallback: if liblfgpu.so is missing this module raises.
"""
import ctypes as C
import os

import numpy as np

from . import _abi
from .ir import Graph

_PKG = os.path.dirname(os.path.abspath(__file__))
# LFGPU_LIB_PATH: diagnostics only (an alternate build of the same sources)
LIB_PATH = os.environ.get("LFGPU_LIB_PATH") or os.path.join(_PKG, "liblfgpu.so")

# Every entry point include/lfgpu.h declares (tests check the exports).
EXPORTS = [
    "lfgpu_version", "lfgpu_last_error", "lfgpu_device_count", "lfgpu_derive_layout",
    "lfgpu_convert_kind", "lfgpu_layout_template", "lfgpu_decode_layout", "lfgpu_ctx_create",
    "lfgpu_ctx_destroy",
    "lfgpu_ctx_launch_count", "lfgpu_layout_convert", "lfgpu_pad_convert", "lfgpu_plan_build",
    "lfgpu_plan_destroy", "lfgpu_plan_set_input", "lfgpu_plan_set_input_device",
    "lfgpu_plan_set_input_device_async",
    "lfgpu_plan_run", "lfgpu_plan_run_on", "lfgpu_plan_get_output", "lfgpu_plan_tensor_buffer", "lfgpu_plan_stream",
    "lfgpu_plan_info", "lfgpu_plan_node_kernel", "lfgpu_plan_measure", "lfgpu_interpret",
    "lfgpu_debug_umma_trace", "lfgpu_materialize_host", "lfgpu_random_inputs",
]


class LfError(RuntimeError):
    """lf::Error with the C-ABI status code attached."""

    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2210_12415_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.lfgpu_last_error.restype = C.c_char_p
        P = C.POINTER
        L.lfgpu_derive_layout.argtypes = [C.c_int32, P(_abi.Dim), C.c_int32, P(_abi.Prim),
                                          P(C.c_int32), P(_abi.Dim)]
        L.lfgpu_layout_convert.argtypes = [C.c_void_p, C.c_int32, P(_abi.Dim), C.c_int32,
                                           P(_abi.Prim), C.c_int32, P(_abi.Prim), C.c_int32,
                                           C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lfgpu_pad_convert.argtypes = [C.c_void_p, P(_abi.Dim), C.c_int64, C.c_int32,
                                        P(_abi.Prim), C.c_int32, P(_abi.Prim), C.c_int32,
                                        C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lfgpu_plan_build.argtypes = [C.c_void_p, P(_abi.GraphDesc), C.c_int32, P(_abi.Sched),
                                       C.c_int32, P(C.c_void_p)]
        L.lfgpu_plan_set_input.argtypes = [C.c_void_p, C.c_int32, P(C.c_double), C.c_int64]
        L.lfgpu_plan_set_input_device.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]
        L.lfgpu_plan_set_input_device_async.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]
        L.lfgpu_plan_get_output.argtypes = [C.c_void_p, C.c_int32, P(C.c_double), C.c_int64]
        L.lfgpu_plan_tensor_buffer.argtypes = [C.c_void_p, C.c_int32, P(C.c_void_p),
                                               P(C.c_int32), P(C.c_int64)]
        L.lfgpu_plan_stream.argtypes = [C.c_void_p, P(C.c_void_p)]
        L.lfgpu_plan_info.argtypes = [C.c_void_p, P(_abi.Counters)]
        L.lfgpu_plan_node_kernel.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32]
        L.lfgpu_plan_measure.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                         P(_abi.Counters)]
        L.lfgpu_plan_run.argtypes = [C.c_void_p]
        L.lfgpu_plan_run_on.argtypes = [C.c_void_p, C.c_void_p]
        L.lfgpu_plan_destroy.argtypes = [C.c_void_p]
        L.lfgpu_ctx_create.argtypes = [C.c_int, P(C.c_void_p)]
        L.lfgpu_ctx_destroy.argtypes = [C.c_void_p]
        L.lfgpu_ctx_launch_count.argtypes = [C.c_void_p, P(C.c_int64)]
        L.lfgpu_random_inputs.argtypes = [P(_abi.GraphDesc), C.c_uint64, P(P(C.c_double))]
        L.lfgpu_interpret.argtypes = [C.c_void_p, P(_abi.GraphDesc), C.c_int32, P(_abi.Sched),
                                      C.c_int32, P(P(C.c_double))]
        L.lfgpu_convert_kind.argtypes = [C.c_int32, P(_abi.Dim), C.c_int32, P(_abi.Prim),
                                         C.c_int32, P(_abi.Prim), P(C.c_int32)]
        L.lfgpu_decode_layout.argtypes = [P(_abi.GraphDesc), C.c_int32, C.c_int32,
                                          P(C.c_int64), C.c_int32, P(_abi.Seq), C.c_int32,
                                          P(C.c_int32), P(_abi.Prim), C.c_int32]
        _lib = L
    return _lib


def check(rc):
    if rc != _abi.OK:
        raise LfError(rc, lib().lfgpu_last_error().decode(errors="replace"))


def _dims(dims):
    return _abi.dim_array([(d if isinstance(d, tuple) else (f"D{i}", d))
                           for i, d in enumerate(dims)])


def derive_layout(dims, seq):
    """lf::derive_layout (layout.cpp:311-322): [(name, extent)] -> physical dims."""
    d = _dims(dims)
    out = (_abi.Dim * _abi.MAX_RANK)()
    r = C.c_int32(0)
    check(lib().lfgpu_derive_layout(len(dims), d, len(seq), _abi.prim_array(seq), C.byref(r), out))
    return [(out[i].name.decode(), out[i].extent) for i in range(r.value)]


def convert_kind(dims, src_seq, dst_seq):
    """1 when the conversion compiles to the affine digit map, 0 for the general program."""
    k = C.c_int32(0)
    check(lib().lfgpu_convert_kind(len(dims), _dims(dims), len(src_seq), _abi.prim_array(src_seq),
                                   len(dst_seq), _abi.prim_array(dst_seq), C.byref(k)))
    return k.value


def layout_template(graph: Graph, node, tiling_levels=1):
    """lf::build_layout_space for one node: [(label, extent)] in template order."""
    cg = graph.to_c()
    n = C.c_int32(0)
    ext = (C.c_int64 * 16)()
    labels = (C.c_char * 8 * 16)()
    check(lib().lfgpu_layout_template(cg.ptr(), node, tiling_levels, C.byref(n), ext, labels, 16))
    return [(labels[i].value.decode(), ext[i]) for i in range(n.value)]


def decode_layout(graph: Graph, node, factors, tiling_levels=1):
    """lf::decode_layout: factors (template order) -> {tensor id: [LayoutPrimitive]}."""
    from .layout import LayoutPrimitive
    cg = graph.to_c()
    f = (C.c_int64 * len(factors))(*[int(x) for x in factors])
    out = (_abi.Seq * 8)()
    storage = (_abi.Prim * 64)()
    n = C.c_int32(0)
    check(lib().lfgpu_decode_layout(cg.ptr(), node, tiling_levels, f, len(factors), out, 8,
                                    C.byref(n), storage, 64))
    res = {}
    for i in range(n.value):
        res[graph.tensors[out[i].tensor].id] = [
            LayoutPrimitive.from_c(out[i].prims[k], lambda t: graph.tensors[t].id)
            for k in range(out[i].nprims)]
    return res


def device_count():
    n = C.c_int(0)
    check(lib().lfgpu_device_count(C.byref(n)))
    return n.value


class Context:
    """One device context (lfgpu_ctx)."""

    def __init__(self, device=0):
        self.ptr = C.c_void_p()
        check(lib().lfgpu_ctx_create(device, C.byref(self.ptr)))
        self.device = device

    def close(self):
        if self.ptr:
            lib().lfgpu_ctx_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self):
        n = C.c_int64(0)
        lib().lfgpu_ctx_launch_count(self.ptr, C.byref(n))
        return n.value


_ctx = {}


def context(device=0):
    if device not in _ctx:
        _ctx[device] = Context(device)
    return _ctx[device]


_ELEM_OF_DTYPE = {"float32": _abi.ELEM_F32, "int32": _abi.ELEM_I32, "bfloat16": _abi.ELEM_BF16,
                  "float64": _abi.ELEM_F64}


def elem_of(t):
    return _ELEM_OF_DTYPE[str(t.dtype).replace("torch.", "")]


def layout_convert(src, dims, src_seq, dst_seq, dst, stream=None, ctx=None):
    """K1 on torch CUDA tensors: dst (physical per dst_seq) <- src (physical per src_seq).

    With src_seq == [] this is lf::materialize_tensor; with dst_seq == [] the
    back-conversion of interpret (interp.cpp:441-468)."""
    ctx = ctx or context(src.device.index or 0)
    s = stream if stream is not None else 0
    check(lib().lfgpu_layout_convert(ctx.ptr, len(dims), _dims(dims), len(src_seq),
                                     _abi.prim_array(src_seq), len(dst_seq),
                                     _abi.prim_array(dst_seq), elem_of(src), elem_of(dst),
                                     C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                     C.c_void_p(s)))
    return dst


def pad_convert(src, in_dims, pad, src_seq, dst_seq, dst, stream=None, ctx=None):
    """K2: the Padding nest writing straight into dst_seq's layout."""
    ctx = ctx or context(src.device.index or 0)
    s = stream if stream is not None else 0
    check(lib().lfgpu_pad_convert(ctx.ptr, _dims(in_dims), pad, len(src_seq),
                                  _abi.prim_array(src_seq), len(dst_seq),
                                  _abi.prim_array(dst_seq), elem_of(src), elem_of(dst),
                                  C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                  C.c_void_p(s)))
    return dst


def sched(node, tile_last=1, tile_second=1, order=0, vectorize=0, parallel=0, unroll=0, fuse=0):
    s = _abi.Sched()
    s.node, s.tile_last, s.tile_second, s.order = node, tile_last, tile_second, order
    s.vectorize, s.parallel, s.unroll, s.fuse = vectorize, parallel, unroll, fuse
    return s


class Plan:
    """A built lfgpu_plan: one graph with its layouts and schedules on one device."""

    def __init__(self, graph: Graph, seqs=None, scheds=(), flags=_abi.PLAN_DEFAULT, ctx=None):
        self.graph = graph
        self.ctx = ctx or context(0)
        self._cg = graph.to_c(seqs or {})
        self._sched = (_abi.Sched * max(1, len(scheds)))(*scheds)
        self.ptr = C.c_void_p()
        check(lib().lfgpu_plan_build(self.ctx.ptr, self._cg.ptr(), len(scheds), self._sched,
                                     flags, C.byref(self.ptr)))

    def close(self):
        if self.ptr:
            lib().lfgpu_plan_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def index(self, tid):
        return self.graph.tensor_index(tid)

    def set_input(self, tid, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        check(lib().lfgpu_plan_set_input(self.ptr, self.index(tid),
                                         v.ctypes.data_as(C.POINTER(C.c_double)), v.size))

    def set_input_device(self, tid, tensor, wait=True):
        """From a torch CUDA tensor in the logical layout (float32/bfloat16/...).
        wait=False enqueues the conversion on the plan's stream and returns at
        once; the caller keeps `tensor` alive and unchanged until then."""
        # The library orders the read after the legacy default stream; a
        # tensor produced on another torch stream is waited for here.
        import torch
        cur = torch.cuda.current_stream(tensor.device)
        if cur != torch.cuda.default_stream(tensor.device):
            cur.synchronize()
        fn = lib().lfgpu_plan_set_input_device if wait else lib().lfgpu_plan_set_input_device_async
        check(fn(self.ptr, self.index(tid), C.c_void_p(tensor.data_ptr()), elem_of(tensor)))

    def run(self, stream=None):
        if stream is None:
            check(lib().lfgpu_plan_run(self.ptr))
        else:
            check(lib().lfgpu_plan_run_on(self.ptr, C.c_void_p(stream)))

    def get_output(self, tid, out=None):
        """Logical doubles of `tid` (the reference's BufferMap entry); `out`
        (a C-contiguous float64 array of the right size) is filled in place."""
        n = self.graph.tensor(tid).num_elements()
        if out is None:
            out = np.empty(n, dtype=np.float64)
        assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == n
        check(lib().lfgpu_plan_get_output(self.ptr, self.index(tid),
                                          out.ctypes.data_as(C.POINTER(C.c_double)), n))
        return out

    def buffer(self, tid):
        p, e, n = C.c_void_p(), C.c_int32(), C.c_int64()
        check(lib().lfgpu_plan_tensor_buffer(self.ptr, self.index(tid), C.byref(p), C.byref(e),
                                             C.byref(n)))
        return p.value, e.value, n.value

    @property
    def stream(self):
        s = C.c_void_p()
        check(lib().lfgpu_plan_stream(self.ptr, C.byref(s)))
        return s.value

    def info(self):
        c = _abi.Counters()
        check(lib().lfgpu_plan_info(self.ptr, C.byref(c)))
        return c

    def node_kernel(self, i):
        buf = C.create_string_buffer(512)
        check(lib().lfgpu_plan_node_kernel(self.ptr, i, buf, 512))
        return buf.value.decode()

    def measure(self, warmup=3, reps=10, flush_l2=True):
        """The GPU measure backend: median device microseconds (ProfileCounters.cost)."""
        c = _abi.Counters()
        check(lib().lfgpu_plan_measure(self.ptr, warmup, reps, 1 if flush_l2 else 0, C.byref(c)))
        return c


def random_inputs(graph: Graph, seed):
    """lf::random_inputs (interp.cpp:487-503), bit-identical to the
    reference: {tensor id: logical float64 array} for Input/Constant tensors."""
    cg = graph.to_c({})
    out, ptrs = {}, (C.POINTER(C.c_double) * max(1, len(graph.tensors)))()
    for i, t in enumerate(graph.tensors):
        if t.role in (_abi.INPUT, _abi.CONSTANT):
            out[t.id] = np.empty(t.num_elements(), dtype=np.float64)
            ptrs[i] = out[t.id].ctypes.data_as(C.POINTER(C.c_double))
    check(lib().lfgpu_random_inputs(cg.ptr(), C.c_uint64(seed), ptrs))
    return out


def interpret(graph: Graph, seqs, scheds, inputs, flags=_abi.PLAN_DEFAULT, ctx=None):
    """lf::interpret(lower(g, seqs, scheds), inputs) on the GPU.

    `inputs` maps Input/Constant tensor ids to logical buffers; returns a dict
    of every node output in its logical layout (doubles), like
    InterpResult.outputs."""
    ctx = ctx or context(0)
    cg = graph.to_c(seqs or {})
    bufs = []
    ptrs = (C.POINTER(C.c_double) * len(graph.tensors))()
    produced = {n.output for n in graph.nodes}
    for i, t in enumerate(graph.tensors):
        if t.id in inputs:
            b = np.ascontiguousarray(inputs[t.id], dtype=np.float64).ravel().copy()
        elif t.id in produced:
            b = np.zeros(t.num_elements(), dtype=np.float64)
        else:
            bufs.append(None)
            continue
        bufs.append(b)
        ptrs[i] = b.ctypes.data_as(C.POINTER(C.c_double))
    sarr = (_abi.Sched * max(1, len(scheds)))(*scheds)
    check(lib().lfgpu_interpret(ctx.ptr, cg.ptr(), len(scheds), sarr, flags, ptrs))
    return {t.id: bufs[i] for i, t in enumerate(graph.tensors) if t.id in produced}
