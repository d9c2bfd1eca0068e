/*
 * lfgpu.h — C-ABI of the B200 (sm_100a) backend for layoutforge's execution
 * and measurement path.
 *
 * The reference (/root/reference/proj, "layoutforge") has no FFI: its hot path
 * is a set of free C++ functions in namespace lf. Every entry point below
 * names the reference function it replaces (file:line, relative to
 * /root/reference). Plain C types only: POD descriptors, raw device/host
 * pointers, sizes, an opaque context, and `void*` CUDA streams.
 *
 * Ownership: the caller owns every buffer it passes. Handles (ctx, plan) are
 * opaque and destroyed explicitly. One context per device, used by one host
 * thread at a time; no other global mutable state except the thread-local
 * error string.
 *
 * Errors: every function returns an int status. LFGPU_EUNSUPPORTED means the
 * candidate cannot be legalised for the GPU kernels; the C++ adapter
 * (include/lf_gpu.hpp) rethrows it as lf::Error so the tuner rejects the
 * candidate exactly like a lowering failure (proj/src/tuner.cpp:169-174).
 * LFGPU_ERANGE mirrors the interpreter's out-of-range access error
 * (proj/src/interp.cpp:348-363).
 */
#ifndef LFGPU_H_
#define LFGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFGPU_MAX_RANK 12
#define LFGPU_NAME_LEN 16
#define LFGPU_ID_LEN 32

/* ---- status codes ---------------------------------------------------- */
enum {
  LFGPU_OK = 0,
  LFGPU_EINVAL = 1,       /* malformed descriptor: lf::Error from shape rules */
  LFGPU_EUNSUPPORTED = 2, /* legal for the reference, not legalisable here   */
  LFGPU_ECUDA = 3,        /* CUDA runtime / driver failure                   */
  LFGPU_ERANGE = 4        /* out-of-range access (interp.cpp:352-359)        */
};

/* ---- enums mirroring the reference ------------------------------------ */
/* lf::PrimKind, same order (proj/include/layoutforge/layout.hpp:19-29) */
enum {
  LFGPU_PRIM_SPLIT = 0,
  LFGPU_PRIM_REORDER = 1,
  LFGPU_PRIM_FUSE = 2,
  LFGPU_PRIM_UNFOLD = 3,
  LFGPU_PRIM_PAD = 4,
  LFGPU_PRIM_STORE_AT = 5,
  LFGPU_PRIM_FOLD = 6,
  LFGPU_PRIM_UNPAD = 7,
  LFGPU_PRIM_DECOUPLE_AT = 8
};

/* lf::OpKind, same order (proj/include/layoutforge/ir.hpp:42) */
enum {
  LFGPU_OP_C2D = 0,
  LFGPU_OP_DEP = 1,
  LFGPU_OP_GMM = 2,
  LFGPU_OP_PADDING = 3,
  LFGPU_OP_RELU = 4,
  LFGPU_OP_BIASADD = 5,
  LFGPU_OP_EWADD = 6,
  LFGPU_OP_LAYOUT_CONVERT = 7,
  /* Extensions beyond lf::OpKind (the pools ResNet-18 needs).
   * Like Padding they are not element-wise and block propagation.
   * MaxPool: out[b,c,h,w] = max_{rh,rw < window} in[b,c,V*h+rh,V*w+rw] on an
   *   explicitly padded input (no implicit padding, like C2D).
   * GlobalAvgPool: out[b,c] = (sum_{h,w} in[b,c,h,w]) / (H*W), rank 4 -> 2. */
  LFGPU_OP_MAXPOOL = 8,
  LFGPU_OP_GLOBAL_AVGPOOL = 9,
  /* Extensions for a full BERT encoder; all over the
   * last logical dim or per attention head, f32, not element-wise except
   * GELU (which fuses into a contraction's epilogue like ReLU):
   * GELU:      y = 0.5 x (1 + erf(x / sqrt(2)))
   * Softmax:   y[.., j] = exp(x[.., j] - max) / sum_j' exp(x[.., j'] - max)
   * LayerNorm: inputs x[.., D], gb[2, D] (row 0 gamma, row 1 beta);
   *            y = (x - mean) / sqrt(var + 10^-eps_exp) * gamma + beta,
   *            mean / biased var over the last dim (eps_exp default 12)
   * BmmQK:     per-head scores; q[T, Cq], k[T', Ck] -> s[H, T, T'],
   *            s[h,i,j] = sum_d q[i, a0+h*Dh+d] * k[j, b0+h*Dh+d]
   *            (attrs heads = H, a_col0 = a0, b_col0 = b0, head_dim = Dh;
   *            head_dim 0 means Dh = Cq / H with Cq == Ck and a0 = b0 = 0).
   *            With column offsets q and k are slices of one packed QKV
   *            tensor; a0 + H*Dh <= Cq and b0 + H*Dh <= Ck.
   * BmmPV:     per-head context; p[H, T, T'], v[T', Cv] -> o[T, H*Dh],
   *            o[i, h*Dh+d] = sum_j p[h,i,j] * v[j, b0+h*Dh+d]
   *            (Dh = head_dim, 0 = Cv / H; o has H*Dh columns; b0 + H*Dh <= Cv)
   * Reductions run in index order (d, j ascending), like interp.cpp. */
  LFGPU_OP_GELU = 10,
  LFGPU_OP_SOFTMAX = 11,
  LFGPU_OP_LAYERNORM = 12,
  LFGPU_OP_BMM_QK = 13,
  LFGPU_OP_BMM_PV = 14
};

/* lf::DType (ir.hpp:26) and lf::Role (ir.hpp:27) */
enum { LFGPU_DTYPE_F32 = 0, LFGPU_DTYPE_I32 = 1 };
enum {
  LFGPU_ROLE_INPUT = 0,
  LFGPU_ROLE_CONSTANT = 1,
  LFGPU_ROLE_INTERMEDIATE = 2,
  LFGPU_ROLE_OUTPUT = 3
};

/* Element storage of raw device buffers handed to the conversion kernels. */
enum {
  LFGPU_ELEM_F32 = 0,
  LFGPU_ELEM_I32 = 1,
  LFGPU_ELEM_BF16 = 2,
  LFGPU_ELEM_F64 = 3
};

/* ---- POD descriptors ---------------------------------------------------- */

/* lf::LayoutPrimitive (layout.hpp:33-52). Dims are 0-based (the reference's
 * in-memory convention; its JSON wire format is 1-based, json_io.cpp:112). */
typedef struct lfgpu_prim {
  int32_t kind;      /* LFGPU_PRIM_*                                     */
  int32_t dim;       /* split/unfold/pad/store_at/fold/unpad anchor, fuse first dim */
  int32_t span;      /* fuse/fold/decouple_at: number of dims merged      */
  int32_t nfactors;  /* split                                             */
  int64_t factors[LFGPU_MAX_RANK];
  int32_t nperm;     /* reorder: new dim j reads old dim perm[j]          */
  int32_t perm[LFGPU_MAX_RANK];
  int64_t tile, stride;   /* unfold B, S (fold reuses both)              */
  int64_t pad;            /* pad/unpad size                              */
  int64_t orig_extent;    /* fold: extent of the refolded dimension      */
  int32_t target;         /* store_at: target tensor index, else -1      */
  int32_t reserved;
} lfgpu_prim;

/* lf::Dim (ir.hpp:21-24) */
typedef struct lfgpu_dim {
  char name[LFGPU_NAME_LEN];
  int64_t extent;
} lfgpu_dim;

/* lf::TensorDecl (ir.hpp:29-41) */
typedef struct lfgpu_tensor {
  char id[LFGPU_ID_LEN];
  int32_t rank;
  int32_t dtype; /* LFGPU_DTYPE_* */
  int32_t role;  /* LFGPU_ROLE_*  */
  int32_t reserved;
  lfgpu_dim dims[LFGPU_MAX_RANK];
} lfgpu_tensor;

/* lf::OperatorNode (ir.hpp:48-58); tensors referenced by declaration index. */
typedef struct lfgpu_node {
  int32_t kind; /* LFGPU_OP_* */
  int32_t ninputs;
  int32_t inputs[2];
  int32_t output;
  int32_t window; /* MaxPool window (KH = KW); 0 elsewhere */
  int32_t heads;  /* attrs["heads"], BmmQK / BmmPV; 0 elsewhere */
  int32_t eps_exp; /* attrs["eps_exp"], LayerNorm: eps = 10^-eps_exp (default 12) */
  int32_t a_col0;  /* attrs["a_col0"], BmmQK: first column of q in its operand (packed QKV); 0 elsewhere */
  int32_t b_col0;  /* attrs["b_col0"], BmmQK / BmmPV: first column of k / v in their operand */
  int32_t head_dim; /* attrs["head_dim"], BmmQK / BmmPV: Dh (0 = operand width / heads) */
  int64_t stride; /* attrs["stride"], C2D/DEP/MaxPool (default 1) */
  int64_t pad;    /* attrs["pad"], Padding (default 0)    */
} lfgpu_node;

/* One entry of lf::SeqMap (lower.hpp:16): the tensor's primitive sequence. */
typedef struct lfgpu_seq {
  int32_t tensor;
  int32_t nprims;
  const lfgpu_prim* prims;
} lfgpu_seq;

/* lf::Graph (ir.hpp:60-73) plus the SeqMap the tuner assigns to it. */
typedef struct lfgpu_graph {
  int32_t ntensors;
  int32_t nnodes;
  int32_t nseqs;
  int32_t reserved;
  const lfgpu_tensor* tensors;
  const lfgpu_node* nodes;
  const lfgpu_seq* seqs; /* tensors without an entry keep their logical layout */
} lfgpu_graph;

/* A decoded loop point for one complex node: the parameter values of
 * lf::LoopSpace (space.hpp:70-90; space.cpp:483-507) before
 * decode_loop_point turns them into loop primitives. SURVEY.md §8(a+) /
 * DESIGN.md §4 give how each maps to the GPU kernel configuration. */
typedef struct lfgpu_sched {
  int32_t node;
  int32_t tile_last;   /* factor chosen for the innermost spatial loop (1 = none) */
  int32_t tile_second; /* factor for the second-innermost spatial loop            */
  int32_t order;       /* 0..2 spatial loops sunk below the reductions            */
  int32_t vectorize;
  int32_t parallel;
  int32_t unroll;
  int32_t fuse; /* absorb the single element-wise consumer chain (lower.cpp:566-608) */
} lfgpu_sched;

/* lf::ProfileCounters (cachesim.hpp:25-31) as the GPU measure backend fills
 * it: cost = median device microseconds of the whole lowered graph; the
 * counter fields are repurposed (documented in DESIGN.md §5). */
typedef struct lfgpu_counters {
  int64_t kernels;     /* kernel launches per graph execution        */
  int64_t bytes_moved; /* algorithmic HBM bytes of the graph          */
  int64_t flops;       /* algorithmic FLOPs (2*MACs)                   */
  int64_t tc_nodes;    /* nodes executed on tcgen05 tensor cores       */
  double cost;         /* median device time, microseconds            */
  double min_us;
  double resolution_us;    /* timer granularity of one sample (event tick / runs) */
  int64_t runs_per_sample; /* graph executions between one CUDA event pair   */
} lfgpu_counters;

/* ---- plan flags ----------------------------------------------------------- */
enum {
  LFGPU_PLAN_DEFAULT = 0,
  /* Contractions on CUDA cores with fp32 storage and fp64 accumulation: the
   * reference's double arithmetic up to fp32 storage of intermediates. */
  LFGPU_PLAN_EXACT = 1 << 0,
  /* Fail with LFGPU_EUNSUPPORTED instead of using the CUDA-core contraction
   * when a C2D/GMM layout cannot run on tcgen05 (tuner measurement mode). */
  LFGPU_PLAN_REQUIRE_TC = 1 << 1,
  /* Capture the kernel sequence in a CUDA graph. */
  LFGPU_PLAN_CUDA_GRAPH = 1 << 2,
  /* Materialize every node output (no epilogue fusion); lfgpu_interpret
   * sets it so all node outputs can be compared with reference_eval. */
  LFGPU_PLAN_KEEP_ALL = 1 << 3,
  /* lfgpu_interpret only: opt into the tcgen05 contractions (bf16 operands,
   * fp32 accumulation; bit-exact on the reference's k/64 inputs, ~2^-9
   * relative per chained contraction otherwise). Without it (or
   * LFGPU_PLAN_REQUIRE_TC) lfgpu_interpret runs LFGPU_PLAN_EXACT: the
   * reference's double arithmetic up to fp32 storage (1e-5 rule,
   * proj/src/cli.cpp:30-49). Plans (lfgpu_plan_build) use tensor cores by
   * default. */
  LFGPU_PLAN_TENSOR_CORES = 1 << 4,
  /* GMM on tensor cores at fp32-level precision: each fp32 operand is split
   * into three bf16 pieces (x = x0 + x1 + x2, 24 significand bits) and the six
   * leading piece products are one bf16 GEMM with K' = 6K (the operands
   * concatenated along K, fp32 accumulation in TMEM), at 6x the tensor-core
   * work. Operand rounding disappears; the fp32 accumulation remains (max
   * rel diff ~1e-5..1e-4 on general inputs at K ~ 1e3, stated tolerance
   * 1e-4; LFGPU_PLAN_EXACT is the 1e-5 path). */
  LFGPU_PLAN_TC_SPLIT = 1 << 5
};

typedef struct lfgpu_ctx lfgpu_ctx;
typedef struct lfgpu_plan lfgpu_plan;

/* ---- library ---------------------------------------------------------------- */
int lfgpu_version(void);
/* Thread-local message of the last failing call on this thread. */
const char* lfgpu_last_error(void);
int lfgpu_device_count(int* count);

/* ---- host-only layout algebra (no GPU needed) --------------------------------- */
/* lf::derive_layout (layout.cpp:311-322) over lf::apply_primitive_shape
 * (layout.cpp:94-184): physical dims (names + extents) of a sequence. */
int lfgpu_derive_layout(int32_t rank, const lfgpu_dim* dims, int32_t nprims,
                        const lfgpu_prim* prims, int32_t* out_rank, lfgpu_dim* out_dims);

/* Classify how the GPU will execute a conversion: 1 = affine digit map
 * (tiled/vectorised kernel), 0 = general index program. For tests/diagnostics. */
int lfgpu_convert_kind(int32_t rank, const lfgpu_dim* logical, int32_t nsrc,
                       const lfgpu_prim* src_seq, int32_t ndst, const lfgpu_prim* dst_seq,
                       int32_t* kind);

/* lf::build_layout_space (space.cpp:49-104) for one complex node: the
 * tunable labels ("h_t", "o_t2", ...) in template order and the extents
 * whose divisors they range over. */
int lfgpu_layout_template(const lfgpu_graph* g, int32_t node, int32_t tiling_levels,
                          int32_t* ntunables, int64_t* extents, char (*labels)[8], int32_t cap);

/* lf::decode_layout (space.cpp:174-417) for the template of complex node
 * `node`: factors in template order (space.cpp:49-104). Writes at most
 * `cap` sequences (prims stored in `prim_storage`, `prim_cap` entries). */
int lfgpu_decode_layout(const lfgpu_graph* g, int32_t node, int32_t tiling_levels,
                        const int64_t* factors, int32_t nfactors, lfgpu_seq* out_seqs,
                        int32_t cap, int32_t* nout, lfgpu_prim* prim_storage,
                        int32_t prim_cap);

/* ---- device context ------------------------------------------------------------ */
int lfgpu_ctx_create(int device, lfgpu_ctx** out);
int lfgpu_ctx_destroy(lfgpu_ctx* ctx);
/* Number of kernels this context launched since creation (evidence counter). */
int lfgpu_ctx_launch_count(lfgpu_ctx* ctx, int64_t* count);

/* ---- K1: layout conversion ----------------------------------------------------------
 * Replaces lf::materialize_tensor / materialize_seq (interp.cpp:181-337)
 * when src_seq is empty, the back-conversion of interpret
 * (interp.cpp:441-468) when dst_seq is empty, and the LayoutConvert nest
 * (lower.cpp:239-243) otherwise. Unfold overhang reads clamp to D-1
 * (interp.cpp:210-213); pad cells are zero (interp.cpp:225-233). Element
 * types may differ (e.g. F32 -> BF16 for tensor-core operands). Async on
 * `stream` (cudaStream_t, NULL = legacy default stream). */
int lfgpu_layout_convert(lfgpu_ctx* ctx, int32_t rank, const lfgpu_dim* logical,
                         int32_t nsrc, const lfgpu_prim* src_seq, int32_t ndst,
                         const lfgpu_prim* dst_seq, int32_t src_elem, int32_t dst_elem,
                         const void* d_src, void* d_dst, void* stream);

/* K1 with host buffers: lf::materialize_tensor for one Input/Constant tensor
 * (interp.cpp:280-337) — logical doubles in, physical doubles out (stored
 * on the device as `elem`, LFGPU_ELEM_F32 reproduces float32 tensors
 * bit-exactly). Synchronous. */
int lfgpu_materialize_host(lfgpu_ctx* ctx, int32_t rank, const lfgpu_dim* logical,
                           int32_t nprims, const lfgpu_prim* seq, int32_t elem,
                           const double* host_logical, double* host_physical);

/* ---- K2: Padding written straight into the consumer's layout ----------------------
 * The Padding nest of lower.cpp:228-238 / 391-403 on a propagated output
 * layout: out-of-interior and unfold-overhang cells get 0. `in_logical` is
 * the rank-4 NCHW input shape; output logical shape is NC(H+2p)(W+2p)
 * (ir.cpp:230-235). */
int lfgpu_pad_convert(lfgpu_ctx* ctx, const lfgpu_dim* in_logical, int64_t pad,
                      int32_t nsrc, const lfgpu_prim* src_seq, int32_t ndst,
                      const lfgpu_prim* dst_seq, int32_t src_elem, int32_t dst_elem,
                      const void* d_src, void* d_dst, void* stream);

/* ---- whole-graph plans (interpret / measure) ------------------------------------------
 * Build: the GPU lowering of lf::lower (lower.cpp:545-610) for a graph that
 * already carries its LayoutConvert nodes (propagation.cpp:265-313). One
 * kernel (or fused kernel) per node, buffers in physical layouts. */
int lfgpu_plan_build(lfgpu_ctx* ctx, const lfgpu_graph* g, int32_t nsched,
                     const lfgpu_sched* sched, int32_t flags, lfgpu_plan** out);
int lfgpu_plan_destroy(lfgpu_plan* plan);

/* Upload an Input/Constant tensor from a host buffer in its logical layout
 * (doubles, as lf::BufferMap holds them; interp.hpp:19-21) and materialize
 * it into the plan's physical layout on the device (K1). The host buffer has
 * been read in full when the call returns (by-value, like BufferMap); float
 * tensors are narrowed to their f32 / bf16 storage on the host, bit-identical
 * to the device conversion, and the copy to the device is stream-ordered
 * before the plan's next run / get_output (LFGPU_STAGE_F64=1: stage the
 * doubles and convert on the device, synchronously). */
int lfgpu_plan_set_input(lfgpu_plan* plan, int32_t tensor, const double* host_logical,
                         int64_t n);
/* Same, from a device buffer of `elem` type already in the logical layout.
 * The conversion reads `d_logical` after all work enqueued before the call
 * on the legacy default stream (the plan's own stream is non-blocking);
 * producers on other streams must be synchronised by the caller. Returns
 * once the conversion has consumed `d_logical`. */
int lfgpu_plan_set_input_device(lfgpu_plan* plan, int32_t tensor, const void* d_logical,
                                int32_t elem);
/* Same, stream-ordered: the conversion is enqueued on the plan's stream and
 * the call returns at once; `d_logical` must stay valid and unchanged until
 * the plan's stream passes this point (the serving / pipelined path). */
int lfgpu_plan_set_input_device_async(lfgpu_plan* plan, int32_t tensor, const void* d_logical,
                                      int32_t elem);
/* Execute every node once on the plan's stream (asynchronous). */
int lfgpu_plan_run(lfgpu_plan* plan);
/* Same, enqueued on the caller's stream instead of the plan's own (NULL:
 * the plan's stream). Stream-ordered like a kernel launch; several plans
 * may share one stream. The run is joined to the plan's own stream both
 * ways (events): it starts after work already enqueued there (e.g.
 * lfgpu_plan_set_input_device_async) and later plan-stream work
 * (lfgpu_plan_get_output, set-input) starts after it.
 * Co-residency: 1-CTA split-K contractions meet at per-tile counters and
 * assume all CTAs of their grid are resident at once; do not run two such
 * plans concurrently on different streams of one device (the CTA-pair
 * kernel's splits meet inside a thread-block cluster and have no such
 * requirement). */
int lfgpu_plan_run_on(lfgpu_plan* plan, void* stream);
/* Convert a node output back to its logical layout and copy it to host
 * doubles (interp.cpp:441-468). Synchronises the plan's stream. */
int lfgpu_plan_get_output(lfgpu_plan* plan, int32_t tensor, double* host_logical, int64_t n);
/* Device pointer of a tensor's physical buffer and its element type. */
int lfgpu_plan_tensor_buffer(lfgpu_plan* plan, int32_t tensor, void** d_ptr, int32_t* elem,
                             int64_t* numel);
/* Raw CUDA stream the plan runs on. */
int lfgpu_plan_stream(lfgpu_plan* plan, void** stream);
/* Per-plan facts: launches per run, tensor-core nodes, algorithmic bytes/flops. */
int lfgpu_plan_info(lfgpu_plan* plan, lfgpu_counters* info);
/* Name of the kernel used for node i ("umma_c2d", "digit_copy", ...). */
int lfgpu_plan_node_kernel(lfgpu_plan* plan, int32_t node, char* buf, int32_t cap);

/* The measure backend: replaces lf::simulate_cache (cachesim.cpp:152-174)
 * at the tuner's seam (tuner.cpp:178). Runs `warmup` untimed executions,
 * then `reps` samples; each sample brackets K back-to-back executions with
 * one CUDA event pair (K sized so a sample spans ~100 us: a single event
 * pair around a microsecond-scale graph sits on the event timer's ~1 us
 * ladder). flush_l2 == 0: warm steady state, sample = span / K.
 * flush_l2 != 0: cold and clean L2 — every execution is preceded by a
 * read of a buffer 1.5x the L2 (evicting, and writing back, whatever the
 * previous execution left), and the same K reads are timed alone right
 * after: sample = (span(read+run) - span(read)) / K.
 * cost = median sample (us), min_us = min sample, resolution_us = 1.024 / K
 * (the event tick observed on this B200 spread over K executions). */
int lfgpu_plan_measure(lfgpu_plan* plan, int32_t warmup, int32_t reps, int32_t flush_l2,
                       lfgpu_counters* out);

/* lf::random_inputs (interp.cpp:487-503), bit-identical (same libstdc++
 * mt19937_64 and distributions): fills bufs[t] (numel doubles, logical
 * row-major) for every Input/Constant tensor t in declaration order;
 * other entries may be NULL. Host-only (no device work). */
int lfgpu_random_inputs(const lfgpu_graph* g, uint64_t seed, double* const* bufs);

/* One-call interpret: lf::interpret(lower(g, seqs, sched), inputs)
 * (interp.cpp:424-470). host_bufs has one pointer per tensor (declaration
 * order): Input/Constant entries are read (logical doubles), node-output
 * entries are written (logical doubles), other entries may be NULL.
 * Reference semantics by default (LFGPU_PLAN_EXACT is implied unless
 * LFGPU_PLAN_TENSOR_CORES or LFGPU_PLAN_REQUIRE_TC is passed). */
int lfgpu_interpret(lfgpu_ctx* ctx, const lfgpu_graph* g, int32_t nsched,
                    const lfgpu_sched* sched, int32_t flags, double* const* host_bufs);

/* ---- diagnostics ------------------------------------------------------------------------
 * When d_buf is non-NULL, every subsequent tcgen05 contraction launch writes
 * eight %globaltimer stamps (ns) per CTA into d_buf[8*cta + i]: entry, setup
 * done, last TMA issued, first stage landed, last MMA committed, accumulator
 * ready, epilogue done. NULL disables. Not thread-safe; profiling only. */
int lfgpu_debug_umma_trace(void* d_buf);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* LFGPU_H_ */
