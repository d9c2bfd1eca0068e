"""ctypes mirror of include/lfgpu.h (the C-ABI boundary).

Struct layouts must match the header byte for byte; tests/test_abi.py checks
the sizes against the compiled library.
"""
import ctypes as C

MAX_RANK = 12
NAME_LEN = 16
ID_LEN = 32

# status codes
OK, EINVAL, EUNSUPPORTED, ECUDA, ERANGE = 0, 1, 2, 3, 4

# lf::PrimKind (layout.hpp:19-29)
SPLIT, REORDER, FUSE, UNFOLD, PAD, STORE_AT, FOLD, UNPAD, DECOUPLE_AT = range(9)
# lf::OpKind (ir.hpp:42)
C2D, DEP, GMM, PADDING, RELU, BIASADD, EWADD, LAYOUT_CONVERT = range(8)
MAXPOOL, GLOBAL_AVGPOOL = 8, 9  # extensions beyond lf::OpKind (lfgpu.h)
GELU, SOFTMAX, LAYERNORM, BMM_QK, BMM_PV = 10, 11, 12, 13, 14  # BERT encoder set
# lf::DType / lf::Role
F32, I32 = 0, 1
INPUT, CONSTANT, INTERMEDIATE, OUTPUT = range(4)
# element storage
ELEM_F32, ELEM_I32, ELEM_BF16, ELEM_F64 = range(4)

PLAN_DEFAULT = 0
PLAN_EXACT = 1
PLAN_REQUIRE_TC = 2
PLAN_CUDA_GRAPH = 4
PLAN_KEEP_ALL = 8
PLAN_TENSOR_CORES = 16  # lfgpu_interpret: opt into tcgen05 (else reference semantics, EXACT)
PLAN_TC_SPLIT = 32  # GMM on tcgen05 with 3-way bf16 operand splits (fp32-level precision)


class Prim(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dim", C.c_int32),
        ("span", C.c_int32),
        ("nfactors", C.c_int32),
        ("factors", C.c_int64 * MAX_RANK),
        ("nperm", C.c_int32),
        ("perm", C.c_int32 * MAX_RANK),
        ("tile", C.c_int64),
        ("stride", C.c_int64),
        ("pad", C.c_int64),
        ("orig_extent", C.c_int64),
        ("target", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Dim(C.Structure):
    _fields_ = [("name", C.c_char * NAME_LEN), ("extent", C.c_int64)]


class Tensor(C.Structure):
    _fields_ = [
        ("id", C.c_char * ID_LEN),
        ("rank", C.c_int32),
        ("dtype", C.c_int32),
        ("role", C.c_int32),
        ("reserved", C.c_int32),
        ("dims", Dim * MAX_RANK),
    ]


class Node(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("ninputs", C.c_int32),
        ("inputs", C.c_int32 * 2),
        ("output", C.c_int32),
        ("window", C.c_int32),
        ("heads", C.c_int32),
        ("eps_exp", C.c_int32),
        ("a_col0", C.c_int32),
        ("b_col0", C.c_int32),
        ("head_dim", C.c_int32),
        ("stride", C.c_int64),
        ("pad", C.c_int64),
    ]


class Seq(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("nprims", C.c_int32), ("prims", C.POINTER(Prim))]


class GraphDesc(C.Structure):
    _fields_ = [
        ("ntensors", C.c_int32),
        ("nnodes", C.c_int32),
        ("nseqs", C.c_int32),
        ("reserved", C.c_int32),
        ("tensors", C.POINTER(Tensor)),
        ("nodes", C.POINTER(Node)),
        ("seqs", C.POINTER(Seq)),
    ]


class Sched(C.Structure):
    _fields_ = [
        ("node", C.c_int32),
        ("tile_last", C.c_int32),
        ("tile_second", C.c_int32),
        ("order", C.c_int32),
        ("vectorize", C.c_int32),
        ("parallel", C.c_int32),
        ("unroll", C.c_int32),
        ("fuse", C.c_int32),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("kernels", C.c_int64),
        ("bytes_moved", C.c_int64),
        ("flops", C.c_int64),
        ("tc_nodes", C.c_int64),
        ("cost", C.c_double),
        ("min_us", C.c_double),
        ("resolution_us", C.c_double),
        ("runs_per_sample", C.c_int64),
    ]


def prim_array(prims):
    """Python LayoutPrimitive list -> ctypes array (kept alive by caller)."""
    arr = (Prim * max(1, len(prims)))()
    for i, p in enumerate(prims):
        p.fill(arr[i])
    return arr


def dim_array(dims):
    arr = (Dim * max(1, len(dims)))()
    for i, d in enumerate(dims):
        name, ext = (d if isinstance(d, tuple) else (d.name, d.extent))
        arr[i].name = name.encode()[: NAME_LEN - 1]
        arr[i].extent = int(ext)
    return arr
