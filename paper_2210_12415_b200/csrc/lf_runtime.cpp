// lf_runtime.cpp — device context, whole-graph plans and the C-ABI.
//
// A plan is the GPU lowering of one (Graph, SeqMap, schedules) triple: the
// reference's lower() (proj/src/lower.cpp:545-610) emits one loop nest per
// node in topological order and interpret() runs it after materializing
// inputs (interp.cpp:424-470). Here every node becomes one kernel launch on
// physical-layout device buffers:
//   Padding / LayoutConvert -> digit_copy (K2/K1) or ix_copy
//   C2D / GMM               -> tcgen05 kernels (K4/K3) when the layouts are
//                              tensor-core legal, else gen_contract
//   DEP                     -> gen_contract
//   ReLU / BiasAdd / EwAdd  -> fused into the tcgen05 epilogue when the
//                              schedule asks for it, else gen_eltwise
// and measure() replaces simulate_cache (cachesim.cpp:152-174) at the
// tuner's seam (tuner.cpp:178).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <random>
#include <string>
#include <thread>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "lf_alloc.hpp"
#include "lf_rows.hpp"
#include "lf_core.hpp"
#include "lf_direct.hpp"
#include "lf_generic.hpp"
#include "lf_kernels.hpp"
#include "lf_small.hpp"
#include "lf_umma.hpp"

using namespace lfg;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_OK(expr)                                                               \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      fail(LFGPU_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));        \
  } while (0)

std::vector<Dim> dims_of(int rank, const lfgpu_dim* d) {
  std::vector<Dim> out;
  for (int i = 0; i < rank; ++i) out.push_back({std::string(d[i].name), d[i].extent});
  return out;
}

Seq seq_of(int n, const lfgpu_prim* p) { return Seq(p, p + n); }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return LFGPU_OK;
  } catch (const Error& e) {
    return set_error(e.code, e.what());
  } catch (const std::exception& e) {
    return set_error(LFGPU_EINVAL, e.what());
  }
}

}  // namespace

namespace lfg {
int set_error_external(int code, const std::string& msg) { return set_error(code, msg); }
}  // namespace lfg

// ---------------------------------------------------------------------------
// context

struct lfgpu_ctx {
  int device = 0;
  int* d_err = nullptr;
  int64_t launches = 0;
  void* flush = nullptr;  // > L2 buffer for cache flushing between timings
  size_t flush_bytes = 0;
};

namespace {

struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t bytes) {
    if (bytes && !(p = dev_alloc(bytes))) fail(LFGPU_ECUDA, "device allocation of " + std::to_string(bytes) + " bytes");
  }
  ~DevBuf() {
    if (p) dev_free(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Upload a POD value / vector into a device buffer kept alive by `keep`.
template <typename T>
T* upload(std::vector<std::unique_ptr<DevBuf>>& keep, const T* host, size_t count) {
  keep.push_back(std::make_unique<DevBuf>(sizeof(T) * std::max<size_t>(count, 1)));
  CUDA_OK(cudaMemcpy(keep.back()->p, host, sizeof(T) * count, cudaMemcpyHostToDevice));
  return static_cast<T*>(keep.back()->p);
}

// One conversion (K1/K2) compiled for launch.
struct CopyKernel {
  bool digit = false;
  DigitMap map;
  const int32_t* d_tab = nullptr;  // DigitMap source offset tables (ntab > 0)
  IxProgram* d_progs = nullptr;
  int64_t n = 0;
  int src_elem = 0, dst_elem = 0;
  const char* name = "";
};

CopyKernel compile_copy(const CopySpec& spec, int se, int de,
                        std::vector<std::unique_ptr<DevBuf>>& keep, bool* oob) {
  CopyKernel k;
  k.src_elem = se;
  k.dst_elem = de;
  k.n = numel(derive(spec.lmap.dst_logical, spec.dst_seq));
  *oob = false;
  // fp32 sources may use offset tables for a non-affine source side.
  std::vector<int32_t> tabs;
  if (compile_digit_map(spec, &k.map, oob, se == LFGPU_ELEM_F32 ? &tabs : nullptr)) {
    k.digit = true;
    if (k.map.ntab > 0) k.d_tab = upload(keep, tabs.data(), tabs.size());
    return k;
  }
  IxProgram progs[2];
  compile_ix_programs(spec, &progs[0], &progs[1]);
  k.d_progs = upload(keep, progs, 2);
  k.name = "ix_copy";
  return k;
}

cudaError_t run_copy(const CopyKernel& k, const void* src, void* dst, int* d_err,
                     cudaStream_t s) {
  KernelInfo info;
  if (k.digit) return launch_digit_copy(k.map, k.src_elem, k.dst_elem, src, dst, s, &info, k.d_tab);
  return launch_ix_copy(k.d_progs, k.n, k.src_elem, k.dst_elem, src, dst, d_err, s, &info);
}

const char* copy_name(const CopyKernel& k) {
  if (!k.digit) return "ix_copy";
  // Mirrors make_params()'s choice in k_copy.cu.
  int a = k.map.ndig - 1;
  bool transpose = false;
  if (k.map.ndig >= 2 && k.map.src_stride[a] != 1)
    for (int d = 0; d < k.map.ndig - 1; ++d)
      if (k.map.src_stride[d] == 1) transpose = true;
  if (k.map.ntab > 0) return transpose ? "digit_copy_transpose_tab" : "digit_copy_direct_tab";
  return transpose ? "digit_copy_transpose" : "digit_copy_direct";
}

LogicalMap identity_map(const std::vector<Dim>& logical) {
  LogicalMap m;
  m.dst_logical = logical;
  m.src_logical = logical;
  return m;
}

LogicalMap padding_map(const std::vector<Dim>& in, int64_t pad) {
  LogicalMap m;
  m.src_logical = in;
  m.dst_logical = in;
  m.dst_logical[2].extent += 2 * pad;
  m.dst_logical[3].extent += 2 * pad;
  m.shift = {0, 0, -pad, -pad};
  m.lo = {0, 0, pad, pad};
  m.hi = {in[0].extent, in[1].extent, pad + in[2].extent, pad + in[3].extent};
  m.has_guard = true;
  return m;
}

}  // namespace

// ---------------------------------------------------------------------------
// plans

struct PTensor {
  std::string id;
  // Input conversions (logical -> storage) compiled once per source element
  // type; key = src elem * 8 + dst elem (tables live in the plan's `keep`).
  std::map<int, CopyKernel> in_copy;
  // Host-buffer entry points (lfgpu_plan_set_input / get_output, the
  // reference's BufferMap of doubles): a device f64 staging buffer, a pinned
  // host staging buffer and the output conversion, all kept with the plan so
  // a repeated call is copies + K1 launches only.
  void* d_f64 = nullptr;
  double* h_pin = nullptr;
  cudaEvent_t staged = nullptr;  // the last staging DMA / K1 out of h_pin / d_f64
  bool out_copy_ready = false;
  CopyKernel out_copy;
  int dtype = LFGPU_DTYPE_F32;
  int role = LFGPU_ROLE_INTERMEDIATE;
  std::vector<Dim> logical, phys;
  Seq seq;
  int elem = LFGPU_ELEM_F32;  // primary storage
  void* d = nullptr;
  void* d_bf16 = nullptr;     // tensor-core operand shadow (same layout)
  int64_t numel = 0;
  int producer = -1;
  std::vector<int> consumers;
  bool need_f32 = false, need_bf16 = false;
  bool valid = true;  // false: fused away, never materialized
  bool shadow_by_producer = false;  // the producer's epilogue writes d_bf16 too
};

// LFGPU_OUT_STREAM=1: a graph output no node reads back is written with
// streaming (evict-first) stores by the 1-CTA tcgen05 epilogue. Measured
// neutral on the cfg2 back-to-back steady state (12.30 vs 12.30 us per
// launch, tools/steps_regime_probe.py), so off by default.
static int out_stream_for(const PTensor& t) {
  static const bool on = [] {
    const char* e = getenv("LFGPU_OUT_STREAM");
    return e && atoi(e) != 0;
  }();
  return on && t.role == LFGPU_ROLE_OUTPUT && t.consumers.empty() ? 1 : 0;
}

struct PStep {
  int node = -1;
  int launches = 1;  // kernels this step launches
  std::string kernel;
  std::function<cudaError_t(cudaStream_t)> run;
};

struct lfgpu_plan {
  lfgpu_ctx* ctx = nullptr;
  int flags = 0;
  std::vector<PTensor> t;
  std::vector<lfgpu_node> nodes;
  std::vector<PStep> steps;
  std::vector<std::string> node_kernel;
  std::map<int, std::string> summary;
  std::vector<std::unique_ptr<DevBuf>> keep;
  cudaStream_t stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // run_on(user stream) joins the plan stream both ways: the run waits for
  // work already enqueued on the plan stream (async set-input conversions),
  // later plan-stream work (get_output, set-input) waits for the run.
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaEvent_t ev_dev_in = nullptr;  // legacy-stream join of device-buffer inputs
  std::vector<cudaEvent_t> stage_ev;  // per-chunk events of the host staging
  int* h_err = nullptr;               // pinned: the device error flag read back with outputs
  int64_t bytes = 0, flops = 0, tc_nodes = 0;
  std::vector<int> order;

  ~lfgpu_plan() {
    // Buffers go back to the allocator cache for the next plan: no launch
    // of this plan may still be reading or writing them.
    if (stream) cudaStreamSynchronize(stream);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_dev_in) cudaEventDestroy(ev_dev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    for (auto e : stage_ev) cudaEventDestroy(e);
    if (h_err) cudaFreeHost(h_err);
    for (auto& x : t) {
      if (x.staged) cudaEventDestroy(x.staged);
      if (x.d_f64) dev_free(x.d_f64);
      if (x.h_pin) cudaFreeHost(x.h_pin);
    }
    keep.clear();
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

std::vector<int> topo(const std::vector<lfgpu_node>& nodes, const std::vector<PTensor>& t) {
  // Kahn with insertion-order ties (ir.cpp:266-295).
  int n = static_cast<int>(nodes.size());
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> succ(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < nodes[i].ninputs; ++j) {
      int p = t[nodes[i].inputs[j]].producer;
      if (p >= 0 && p != i) {
        succ[p].push_back(i);
        ++indeg[i];
      }
    }
  std::set<int> ready;
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) ready.insert(i);
  std::vector<int> order;
  while (!ready.empty()) {
    int i = *ready.begin();
    ready.erase(ready.begin());
    order.push_back(i);
    for (int s : succ[i])
      if (--indeg[s] == 0) ready.insert(s);
  }
  if (static_cast<int>(order.size()) != n) fail(LFGPU_EINVAL, "topo_order: graph has a cycle");
  return order;
}

int64_t* tables_for(lfgpu_plan* P, const PTensor& t, std::vector<int64_t>* off) {
  std::vector<int64_t> tab;
  if (!separable_tables(t.logical, t.seq, &tab, off))
    fail(LFGPU_EUNSUPPORTED, "layout of '" + t.id + "' is not separable per logical dim: " +
                                 seq_str(t.seq));
  return upload(P->keep, tab.data(), tab.size());
}

// Columns [c0, c0 + width) of a rank-2 separable tensor: every row offset a
// multiple of 4 and the columns contiguous in runs of 4 starting 16-byte
// aligned (the fused attention kernel's 16-byte gathers).
bool cols_vec4(const PTensor& t, int64_t c0, int64_t width) {
  std::vector<int64_t> tab, off;
  if (t.logical.size() != 2 || c0 % 4 || width % 4 || !separable_tables(t.logical, t.seq, &tab, &off)) return false;
  for (int64_t i = 0; i < t.logical[0].extent; ++i)
    if (tab[off[0] + i] % 4) return false;
  for (int64_t c = c0; c < c0 + width; c += 4) {
    const int64_t b = tab[off[1] + c];
    if (b % 4) return false;
    for (int k = 1; k < 4; ++k)
      if (tab[off[1] + c + k] != b + k) return false;
  }
  return true;
}

bool same_extents(const std::vector<Dim>& a, const std::vector<Dim>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].extent != b[i].extent) return false;
  return true;
}

// Row / column offsets of a separable layout seen as [rows, last dim]: the
// row base of every multi-index of the leading dims (row-major order) and
// the offset of every last-dim index.
void row_col_offsets(const PTensor& t, std::vector<int64_t>* rows, std::vector<int64_t>* cols) {
  std::vector<int64_t> tab, off;
  if (!separable_tables(t.logical, t.seq, &tab, &off))
    fail(LFGPU_EUNSUPPORTED, "layout of '" + t.id + "' is not separable per logical dim: " + seq_str(t.seq));
  const size_t r = t.logical.size();
  const int64_t d = t.logical.back().extent;
  cols->assign(d, 0);
  for (int64_t j = 0; j < d; ++j) (*cols)[j] = tab[off[r - 1] + j];
  rows->assign(1, 0);
  for (size_t k = 0; k + 1 < r; ++k) {
    std::vector<int64_t> next;
    next.reserve(rows->size() * t.logical[k].extent);
    for (int64_t base : *rows)
      for (int64_t i = 0; i < t.logical[k].extent; ++i) next.push_back(base + tab[off[k] + i]);
    rows->swap(next);
  }
}

IxProgram* out_program(lfgpu_plan* P, const PTensor& t) {
  CopySpec spec;
  spec.lmap = identity_map(t.logical);
  spec.dst_seq = t.seq;
  spec.mode = FoldMode::Nest;
  IxProgram progs[2];
  compile_ix_programs(spec, &progs[0], &progs[1]);
  return upload(P->keep, &progs[0], 1);
}

int storage_elem(const PTensor& t) {
  return t.dtype == LFGPU_DTYPE_I32 ? LFGPU_ELEM_I32 : LFGPU_ELEM_F32;
}

// store_at is folded offline (lower.cpp:32-82): the attachment only
// co-locates a constant with its target's storage, one extra slot along
// `dim`, so values are unaffected. The plan applies the reference's
// validation (source constant, attachment last, target known and not itself
// attached, shape compatible, the grown target still derivable), then
// keeps the source in its own buffer in the absorb-prefix layout and the
// target in its own layout: every consumer reads the same values the fused
// storage would hold.
void fold_store_at(lfgpu_plan* P, int ntensors) {
  std::vector<int> target(ntensors, -1), dim(ntensors, 0);
  for (int i = 0; i < ntensors; ++i) {
    PTensor& t = P->t[i];
    for (size_t j = 0; j < t.seq.size(); ++j) {
      const lfgpu_prim& p = t.seq[j];
      if (p.kind == LFGPU_PRIM_DECOUPLE_AT)
        fail(LFGPU_EINVAL, "decouple_at cannot appear in a compilation sequence");
      if (p.kind != LFGPU_PRIM_STORE_AT) continue;
      if (t.role != LFGPU_ROLE_CONSTANT)
        fail(LFGPU_EINVAL, "store_at on non-constant tensor '" + t.id +
                               "': layout fusion is offline only");
      if (j + 1 != t.seq.size())
        fail(LFGPU_EINVAL, "store_at must be the final primitive of '" + t.id + "'");
      if (p.target < 0 || p.target >= ntensors)
        fail(LFGPU_EINVAL, "store_at target of '" + t.id + "' unknown");
      target[i] = p.target;
      dim[i] = p.dim;
    }
  }
  std::map<int, std::vector<Dim>> grown;  // target -> dims with its slots
  for (int i = 0; i < ntensors; ++i) {
    if (target[i] < 0) continue;
    PTensor& src = P->t[i];
    PTensor& dst = P->t[target[i]];
    if (target[target[i]] >= 0)
      fail(LFGPU_EINVAL, "store_at target '" + dst.id + "' is itself attached elsewhere");
    src.seq.pop_back();  // the absorb prefix (lower.cpp:59)
    std::vector<Dim> sd;
    try {
      sd = derive(src.logical, src.seq);
    } catch (const Error& e) {
      fail(e.code, "tensor '" + src.id + "': " + e.what());
    }
    // apply_store_at (layout.cpp:450-467)
    // Each attachment sees the target as grown by the earlier ones.
    auto it = grown.emplace(target[i], dst.logical).first;
    std::vector<Dim>& td = it->second;
    const int d = dim[i], rank = static_cast<int>(td.size());
    if (d < 0 || d >= rank) fail(LFGPU_EINVAL, "store_at: dim out of range");
    if (static_cast<int>(sd.size()) + 1 != rank)
      fail(LFGPU_EINVAL, "store_at: source must match target with one dim removed");
    for (int k = 0, j = 0; k < rank; ++k) {
      if (k == d) continue;
      if (sd[j].extent != td[k].extent)
        fail(LFGPU_EINVAL, "store_at: shape incompatibility at target dim " + std::to_string(k));
      ++j;
    }
    td[d].extent += 1;
  }
  // The target's sequence must still derive on the grown dims (lower.cpp:84-95).
  for (const auto& [ti, td] : grown) {
    try {
      (void)derive(td, P->t[ti].seq);
    } catch (const Error& e) {
      fail(e.code, "tensor '" + P->t[ti].id + "': " + e.what());
    }
  }
}

void build_plan(lfgpu_plan* P, const lfgpu_graph* g, int nsched, const lfgpu_sched* sched) {
  if (!g || g->ntensors <= 0) fail(LFGPU_EINVAL, "empty graph");
  P->t.resize(g->ntensors);
  for (int i = 0; i < g->ntensors; ++i) {
    const lfgpu_tensor& td = g->tensors[i];
    PTensor& t = P->t[i];
    t.id = td.id;
    t.dtype = td.dtype;
    t.role = td.role;
    t.logical = dims_of(td.rank, td.dims);
    for (const auto& d : t.logical)
      if (d.extent < 1) fail(LFGPU_EINVAL, "tensor '" + t.id + "' has an extent < 1");
  }
  for (int s = 0; s < g->nseqs; ++s) {
    const lfgpu_seq& sq = g->seqs[s];
    if (sq.tensor < 0 || sq.tensor >= g->ntensors) fail(LFGPU_EINVAL, "seq names no tensor");
    P->t[sq.tensor].seq = seq_of(sq.nprims, sq.prims);
  }
  fold_store_at(P, g->ntensors);
  for (auto& t : P->t) {
    try {
      t.phys = derive(t.logical, t.seq);
    } catch (const Error& e) {
      fail(e.code, "tensor '" + t.id + "': " + e.what());
    }
    t.numel = numel(t.phys);
    t.elem = storage_elem(t);
  }
  P->nodes.assign(g->nodes, g->nodes + g->nnodes);
  for (int i = 0; i < g->nnodes; ++i) {
    const auto& n = P->nodes[i];
    if (n.output < 0 || n.output >= g->ntensors) fail(LFGPU_EINVAL, "node output out of range");
    if (P->t[n.output].producer >= 0) fail(LFGPU_EINVAL, "tensor produced twice");
    P->t[n.output].producer = i;
    for (int j = 0; j < n.ninputs; ++j) {
      if (n.inputs[j] < 0 || n.inputs[j] >= g->ntensors) fail(LFGPU_EINVAL, "input out of range");
      P->t[n.inputs[j]].consumers.push_back(i);
    }
  }
  P->order = topo(P->nodes, P->t);
  P->node_kernel.assign(P->nodes.size(), "");

  std::map<int, lfgpu_sched> sched_of;
  for (int i = 0; i < nsched; ++i) sched_of[sched[i].node] = sched[i];
  const bool exact = P->flags & LFGPU_PLAN_EXACT;

  // 1. Tensor-core eligibility per contraction and fusion chains.
  std::map<int, UmmaPlan> umma;
  std::map<int, std::vector<EpiOp>> direct;  // CUDA-core direct convs (k_direct.cu)
  std::map<int, std::vector<EpiOp>> depd;    // K6 depthwise (k_direct.cu)
  std::map<int, std::vector<EpiOp>> gemv;    // small-M GMM on CUDA cores (k_small.cu)
  std::map<int, UmmaPlan> im2col;            // small-I C2D: im2col + tcgen05 GEMM
  struct SplitGmm {                          // LFGPU_PLAN_TC_SPLIT operands (K' = 6K)
    std::vector<Dim> a_log, b_log;
    Seq a_seq, b_seq;
  };
  std::map<int, SplitGmm> split_gmm;
  std::map<int, int> im2col_pad;             // im2col node -> Padding node it reads through
  std::set<int> fused_away;  // element-wise nodes absorbed into an epilogue
  std::vector<int> pos(P->nodes.size(), 0);
  for (size_t k = 0; k < P->order.size(); ++k) pos[P->order[k]] = static_cast<int>(k);
  // Epilogue fusion of the single-consumer element-wise chain after node ni
  // (lower.cpp:566-608) while every member keeps the output's physical layout.
  // GELU fuses only into the tcgen05 epilogues (tc = true).
  auto fuse_chain = [&](int ni, const PTensor& Cc, bool tc = false) {
    std::vector<EpiOp> epi;
    int cur = P->nodes[ni].output;
    while (true) {
      const auto& cons = P->t[cur].consumers;
      if (cons.size() != 1) break;
      const auto& c = P->nodes[cons[0]];
      if (c.kind != LFGPU_OP_RELU && c.kind != LFGPU_OP_BIASADD && c.kind != LFGPU_OP_EWADD &&
          !(tc && c.kind == LFGPU_OP_GELU))
        break;
      if (c.inputs[0] != cur) break;
      if (!seq_equal(P->t[c.output].seq, Cc.seq)) break;
      if (c.kind == LFGPU_OP_EWADD && !seq_equal(P->t[c.inputs[1]].seq, Cc.seq)) break;
      if (c.kind == LFGPU_OP_BIASADD && !P->t[c.inputs[1]].seq.empty()) break;
      if (static_cast<int>(epi.size()) >= kMaxEpi) break;
      if (c.kind == LFGPU_OP_RELU && !epi.empty() && epi.back().kind == EPI_RELU) break;
      // The epilogue reads a residual / bias when the contraction runs: its
      // producer must already have run (e.g. a ResNet downsample branch).
      const bool unary = c.kind == LFGPU_OP_RELU || c.kind == LFGPU_OP_GELU;
      if (!unary) {
        const int pr = P->t[c.inputs[1]].producer;
        if (pr >= 0 && pos[pr] > pos[ni]) break;
      }
      EpiOp e;
      e.kind = c.kind == LFGPU_OP_RELU ? EPI_RELU
               : c.kind == LFGPU_OP_GELU ? EPI_GELU
               : c.kind == LFGPU_OP_BIASADD ? EPI_BIAS
                                            : EPI_RESIDUAL;
      e.tensor = unary ? -1 : c.inputs[1];
      e.out_tensor = c.output;
      epi.push_back(e);
      fused_away.insert(cons[0]);
      cur = c.output;
    }
    return epi;
  };
  for (int ni : P->order) {
    const auto& n = P->nodes[ni];
    if (n.kind == LFGPU_OP_DEP && !exact && P->t[n.output].dtype == LFGPU_DTYPE_F32) {
      // K6 when every operand's layout is separable per logical dim.
      std::vector<int64_t> tb, of;
      bool ok = true;
      for (int t : {n.inputs[0], n.inputs[1], n.output})
        ok = ok && separable_tables(P->t[t].logical, P->t[t].seq, &tb, &of);
      if (ok) {
        lfgpu_sched s{};
        s.node = ni;
        if (sched_of.count(ni)) s = sched_of[ni];
        depd[ni] = s.fuse && !(P->flags & LFGPU_PLAN_KEEP_ALL) ? fuse_chain(ni, P->t[n.output])
                                                               : std::vector<EpiOp>{};
      }
      continue;
    }
    if (n.kind != LFGPU_OP_C2D && n.kind != LFGPU_OP_GMM) continue;
    if (exact || P->t[n.output].dtype != LFGPU_DTYPE_F32) continue;
    UmmaPlan up;
    std::string why;
    const PTensor& A = P->t[n.inputs[0]];
    const PTensor& B = P->t[n.inputs[1]];
    const PTensor& Cc = P->t[n.output];
    lfgpu_sched s{};
    s.node = ni;
    if (sched_of.count(ni)) s = sched_of[ni];
    if (n.kind == LFGPU_OP_GMM && (P->flags & LFGPU_PLAN_TC_SPLIT)) {
      // fp32-level precision on tensor cores: the node's operands are split
      // into bf16 pieces concatenated along K (lf_rows.hpp), laid out in
      // plain GMM bricks; the output keeps the node's own layout.
      const int64_t M = A.logical[0].extent, K = A.logical[1].extent, N = B.logical[1].extent;
      const int64_t K6 = kSplitTerms * K, bn = N % 128 == 0 ? 128 : N % 64 == 0 ? 64 : 0;
      SplitGmm sg;
      std::string w3;
      bool ok3 = bn && M % 128 == 0 && K6 % 64 == 0;
      if (ok3) {
        sg.a_log = {{"M", M}, {"K", K6}};
        sg.b_log = {{"K", K6}, {"N", N}};
        sg.a_seq = {make_split(0, {M / 128, 128}), make_split(2, {K6 / 64, 64}), make_reorder({0, 2, 1, 3})};
        sg.b_seq = {make_split(0, {K6 / 64, 64}), make_split(2, {N / bn, bn}), make_reorder({0, 2, 1, 3})};
        lfgpu_sched s3 = s;
        s3.tile_last = static_cast<int32_t>(bn);
        ok3 = umma_plan_gemm(sg.a_log, sg.a_seq, sg.b_log, sg.b_seq, Cc.logical, Cc.seq, s3, &up, &w3);
      }
      if (ok3) {
        if (s.fuse && !(P->flags & LFGPU_PLAN_KEEP_ALL)) {
          std::vector<EpiOp> epi = fuse_chain(ni, Cc, true);
          for (const auto& e : epi) up.epi[up.epi_count++] = e;
        }
        up.summary += " split=bf16x3";
        umma[ni] = up;
        split_gmm[ni] = sg;
        continue;
      }
      if (P->flags & LFGPU_PLAN_REQUIRE_TC)
        fail(LFGPU_EUNSUPPORTED, "node " + std::to_string(ni) + " not tensor-core legal (split mode): " +
                                     (w3.empty() ? "needs M % 128, N % 64" : w3));
      continue;
    }
    bool ok = n.kind == LFGPU_OP_GMM
                  ? umma_plan_gemm(A.logical, A.seq, B.logical, B.seq, Cc.logical, Cc.seq, s,
                                   &up, &why)
                  : umma_plan_conv(A.logical, A.seq, B.logical, B.seq, Cc.logical, Cc.seq,
                                   n.stride, s, &up, &why);
    if (!ok) {
      // Small-I convolutions on logical operands: the CUDA-core direct kernel.
      const bool dc = n.kind == LFGPU_OP_C2D && A.seq.empty() && B.seq.empty() &&
                      direct_conv_applies(B.logical[1].extent, B.logical[2].extent,
                                          B.logical[3].extent, B.logical[0].extent);
      if (dc) {
        // Tensor cores through an im2col operand when the pixel count tiles
        // by 128 and O fits one UMMA N; else the CUDA-core direct kernel.
        const int64_t Nb = A.logical[0].extent, Ho = Cc.logical[2].extent, Wo = Cc.logical[3].extent;
        const int64_t O = B.logical[0].extent;
        const int64_t K = B.logical[1].extent * B.logical[2].extent * B.logical[3].extent;
        const int64_t M = Nb * Ho * Wo, Kp = (K + 63) / 64 * 64;
        UmmaPlan ug;
        std::string w2;
        // Rows per tile: whole output rows (the C layout splits Ho and Wo).
        int64_t RT = 0;
        if (Wo <= 128) {
          for (int64_t r = 128 / Wo; r >= 1 && !RT; --r)
            if (Ho % r == 0) RT = r * Wo;
        } else {
          for (int64_t d = 128; d >= 16 && !RT; --d)
            if (Wo % d == 0) RT = d;
        }
        bool ic = !getenv("LFGPU_NO_IM2COL") && RT >= 16 && M % RT == 0 && O % 16 == 0 && O <= 256;
        if (ic) {
          const std::vector<Dim> a_log{{"M", M}, {"K", Kp}}, b_log{{"K", Kp}, {"N", O}},
              c_log{{"M", M}, {"N", O}};
          const Seq a_seq{make_split(0, {M / RT, RT}), make_split(2, {Kp / 64, 64}),
                          make_reorder({0, 2, 1, 3})};
          const Seq b_seq{make_split(0, {Kp / 64, 64}), make_split(2, {1, O}), make_reorder({2, 0, 3, 1})};
          // C rows are pixels (n, ho, wo): reshape to the conv output's
          // logical NCHW, then its own sequence: the GEMM writes it in place.
          Seq c_seq{make_split(0, {Nb, Ho, Wo}), make_reorder({0, 3, 1, 2})};
          c_seq.insert(c_seq.end(), Cc.seq.begin(), Cc.seq.end());
          lfgpu_sched s2 = s;
          s2.tile_last = static_cast<int32_t>(O);
          s2.order = 1;
          ic = umma_plan_gemm(a_log, a_seq, b_log, b_seq, c_log, c_seq, s2, &ug, &w2, static_cast<int>(RT));
          if (!ic && getenv("LFGPU_DEBUG_IM2COL")) fprintf(stderr, "im2col gemm rejected: %s\n", w2.c_str());
        }
        if (ic) {
          if (s.fuse && !(P->flags & LFGPU_PLAN_KEEP_ALL)) {
            std::vector<EpiOp> epi = fuse_chain(ni, Cc, true);
            for (const auto& e : epi) ug.epi[ug.epi_count++] = e;
          }
          im2col[ni] = ug;
          // The Padding feeding only this conv is folded into the im2col
          // reads (zero outside x): its step and its buffer's writes vanish.
          const int pn = A.producer;
          if (pn >= 0 && P->nodes[pn].kind == LFGPU_OP_PADDING && A.consumers.size() == 1 &&
              P->t[P->nodes[pn].inputs[0]].seq.empty() && A.role == LFGPU_ROLE_INTERMEDIATE &&
              !(P->flags & LFGPU_PLAN_KEEP_ALL) && !getenv("LFGPU_NO_PAD_ABSORB")) {
            im2col_pad[ni] = pn;
            fused_away.insert(pn);
          }
          continue;
        }
        direct[ni] = s.fuse && !(P->flags & LFGPU_PLAN_KEEP_ALL) ? fuse_chain(ni, Cc)
                                                                 : std::vector<EpiOp>{};
        continue;
      }
      if (P->flags & LFGPU_PLAN_REQUIRE_TC)
        fail(LFGPU_EUNSUPPORTED, "node " + std::to_string(ni) + " not tensor-core legal: " + why);
      // Small-M GMM (the batch-1 classifier): k_small.cu's GEMV with the
      // element-wise chain fused, when every operand layout is separable.
      if (n.kind == LFGPU_OP_GMM && A.logical[0].extent <= 16) {
        std::vector<int64_t> tb, of;
        bool sep = true;
        for (int t : {n.inputs[0], n.inputs[1], n.output})
          sep = sep && separable_tables(P->t[t].logical, P->t[t].seq, &tb, &of);
        if (sep)
          gemv[ni] = s.fuse && !(P->flags & LFGPU_PLAN_KEEP_ALL) ? fuse_chain(ni, Cc) : std::vector<EpiOp>{};
      }
      continue;
    }
    if (s.fuse && !(P->flags & LFGPU_PLAN_KEEP_ALL)) {
      std::vector<EpiOp> epi = fuse_chain(ni, Cc, true);
      for (const auto& e : epi) up.epi[up.epi_count++] = e;
    }
    umma[ni] = up;
  }

  // 1b. Padding absorbed into the producing C2D's epilogue: when a Padding's
  // input is the final tensor of a tcgen05 C2D (after its fused chain) and
  // the padded tensor feeds only tensor-core contractions, the producer
  // writes the padded (possibly unfolded) bf16 layout itself and the
  // Padding step disappears (the paper's "producer yields the consumer's
  // layout"; lower.cpp:228-238).
  std::map<int, int> absorbed_pad;  // umma node -> Padding node it absorbs
  if (!(P->flags & (LFGPU_PLAN_KEEP_ALL | LFGPU_PLAN_EXACT)) && !getenv("LFGPU_NO_PAD_ABSORB")) {
    for (int pn : P->order) {
      const auto& pnode = P->nodes[pn];
      if (pnode.kind != LFGPU_OP_PADDING) continue;
      const int tin = pnode.inputs[0];
      int u = P->t[tin].producer;
      while (u >= 0 && fused_away.count(u)) u = P->t[P->nodes[u].inputs[0]].producer;
      if (u < 0 || !umma.count(u) || P->nodes[u].kind != LFGPU_OP_C2D || absorbed_pad.count(u))
        continue;
      const UmmaPlan& up = umma[u];
      if (up.trans) continue;  // accumulator columns are pixels there, not channels
      const int final_t = up.epi_count ? up.epi[up.epi_count - 1].out_tensor : P->nodes[u].output;
      if (final_t != tin) continue;
      const PTensor& xp = P->t[pnode.output];
      bool all_tc = !xp.consumers.empty() && xp.role != LFGPU_ROLE_OUTPUT;
      for (int c : xp.consumers)
        if (!umma.count(c)) all_tc = false;
      if (!all_tc) continue;
      ScatterDesc sd;
      std::string why;
      if (!umma_scatter_desc(xp.logical, xp.seq, pnode.pad, &sd, &why) || sd.sC1 != 1 || sd.ic % 4 ||
          up.BN % 8)
        continue;
      umma[u].scatter = sd;
      absorbed_pad[u] = pn;
      fused_away.insert(pn);
    }
  }

  // 1c. LayoutConvert absorbed into its producer (propagation.cpp:265-313
  // inserts the conversion; the paper's producer-yields-the-consumer's-layout,
  // PAPER.md:379-381): when the converted tensor is the final tensor of a
  // tcgen05 contraction (after its fused chain) and feeds only the
  // conversion, the contraction is re-planned to write the conversion's
  // layout directly and the conversion step disappears.
  std::map<int, int> out_redirect;  // umma node -> tensor it writes instead of its chain's final tensor
  if (!(P->flags & (LFGPU_PLAN_KEEP_ALL | LFGPU_PLAN_EXACT)) && !getenv("LFGPU_NO_CONVERT_ABSORB")) {
    for (int cn : P->order) {
      const auto& cnode = P->nodes[cn];
      if (cnode.kind != LFGPU_OP_LAYOUT_CONVERT || fused_away.count(cn)) continue;
      const int tin = cnode.inputs[0];
      const PTensor& T = P->t[tin];
      if (T.consumers.size() != 1 || T.role == LFGPU_ROLE_OUTPUT) continue;
      int u = T.producer;
      while (u >= 0 && fused_away.count(u)) u = P->t[P->nodes[u].inputs[0]].producer;
      if (u < 0 || !umma.count(u) || absorbed_pad.count(u) || split_gmm.count(u) || out_redirect.count(u)) continue;
      const UmmaPlan& old = umma[u];
      const int final_t = old.epi_count ? old.epi[old.epi_count - 1].out_tensor : P->nodes[u].output;
      if (final_t != tin) continue;
      bool residual = false;  // a residual operand is read in the output's own layout
      for (int e = 0; e < old.epi_count; ++e) residual = residual || old.epi[e].kind == EPI_RESIDUAL;
      if (residual) continue;
      const auto& un = P->nodes[u];
      const PTensor& UA = P->t[un.inputs[0]];
      const PTensor& UB = P->t[un.inputs[1]];
      const PTensor& U = P->t[cnode.output];
      lfgpu_sched su{};
      su.node = u;
      if (sched_of.count(u)) su = sched_of[u];
      UmmaPlan np;
      std::string why;
      const bool ok = un.kind == LFGPU_OP_GMM
                          ? umma_plan_gemm(UA.logical, UA.seq, UB.logical, UB.seq, U.logical, U.seq, su, &np, &why)
                          : umma_plan_conv(UA.logical, UA.seq, UB.logical, UB.seq, U.logical, U.seq, un.stride, su,
                                           &np, &why);
      if (!ok) continue;
      for (int e = 0; e < old.epi_count; ++e) np.epi[e] = old.epi[e];
      np.epi_count = old.epi_count;
      np.summary += " (writes " + U.id + ": LayoutConvert absorbed)";
      umma[u] = np;
      out_redirect[u] = cnode.output;
      fused_away.insert(cn);
    }
  }

  // 1c'. A Padding feeding only a MaxPool is absorbed into its reads
  // (k_small.cu: zeros outside the unpadded input take part in the max);
  // the padded tensor is never materialized.
  std::map<int, int> maxpool_pad;  // MaxPool node -> Padding node it reads through
  if (!(P->flags & (LFGPU_PLAN_KEEP_ALL | LFGPU_PLAN_EXACT)) && !getenv("LFGPU_NO_PAD_ABSORB")) {
    for (int mn = 0; mn < static_cast<int>(P->nodes.size()); ++mn) {
      const auto& mp = P->nodes[mn];
      if (mp.kind != LFGPU_OP_MAXPOOL) continue;
      const PTensor& XP = P->t[mp.inputs[0]];
      const int pn = XP.producer;
      if (pn < 0 || P->nodes[pn].kind != LFGPU_OP_PADDING || XP.consumers.size() != 1 ||
          XP.role != LFGPU_ROLE_INTERMEDIATE || fused_away.count(pn))
        continue;
      const PTensor& X = P->t[P->nodes[pn].inputs[0]];
      const PTensor& Y = P->t[mp.output];
      std::vector<int64_t> tb, of;
      if (X.logical.size() != 4 || X.dtype != LFGPU_DTYPE_F32 || Y.dtype != LFGPU_DTYPE_F32 ||
          !separable_tables(X.logical, X.seq, &tb, &of) || !separable_tables(Y.logical, Y.seq, &tb, &of))
        continue;
      maxpool_pad[mn] = pn;
      fused_away.insert(pn);
      P->t[mp.inputs[0]].valid = false;
      P->t[P->nodes[pn].inputs[0]].need_f32 = true;
    }
  }

  // 1d. Attention fusion: BmmQK -> Softmax -> BmmPV whose scores and
  // probabilities are single-consumer intermediates runs as one kernel
  // (k_rows.cu attn_kernel) at the BmmPV's position; s and p are never
  // materialized. The shapes are checked when the BmmPV step is built.
  std::map<int, int> attn_of;  // BmmPV node -> its BmmQK node
  if (!(P->flags & LFGPU_PLAN_KEEP_ALL) && !getenv("LFGPU_NO_ATTN_FUSE")) {
    for (int qn = 0; qn < static_cast<int>(P->nodes.size()); ++qn) {
      const auto& qk = P->nodes[qn];
      if (qk.kind != LFGPU_OP_BMM_QK) continue;
      const PTensor& S = P->t[qk.output];
      if (S.role != LFGPU_ROLE_INTERMEDIATE || S.consumers.size() != 1) continue;
      const auto& sm = P->nodes[S.consumers[0]];
      if (sm.kind != LFGPU_OP_SOFTMAX || sm.inputs[0] != qk.output) continue;
      const PTensor& Pr = P->t[sm.output];
      if (Pr.role != LFGPU_ROLE_INTERMEDIATE || Pr.consumers.size() != 1) continue;
      const int pn = Pr.consumers[0];
      const auto& pv = P->nodes[pn];
      if (pv.kind != LFGPU_OP_BMM_PV || pv.inputs[0] != sm.output || pv.heads != qk.heads) continue;
      if (S.logical.size() != 3 || S.logical[2].extent > 512) continue;
      attn_of[pn] = qn;
      fused_away.insert(qn);
      fused_away.insert(S.consumers[0]);
      P->t[qk.output].valid = false;  // never allocated or written
      P->t[sm.output].valid = false;
    }
  }

  // 2. Storage decisions: bf16 for tensor-core operands, f32/i32 otherwise.
  for (auto& t : P->t) {
    for (int c : t.consumers) {
      bool tc_operand = umma.count(c) && !split_gmm.count(c) && (P->nodes[c].inputs[0] == &t - &P->t[0] ||
                                          P->nodes[c].inputs[1] == &t - &P->t[0]);
      // A tensor read only as an epilogue residual/bias stays fp32.
      if (tc_operand) t.need_bf16 = true;
      else t.need_f32 = true;
    }
    if (t.producer >= 0 || t.role == LFGPU_ROLE_OUTPUT) t.need_f32 = true;
    if (t.consumers.empty()) t.need_f32 = true;
    // A Padding / LayoutConvert output feeding only tensor cores is written in
    // bf16 directly: the conversion absorbed into the producer.
    if (t.producer >= 0 && t.need_bf16) {
      const auto& pn = P->nodes[t.producer];
      bool all_tc = true;
      for (int c : t.consumers)
        if (!umma.count(c)) all_tc = false;
      if ((pn.kind == LFGPU_OP_PADDING || pn.kind == LFGPU_OP_LAYOUT_CONVERT) && all_tc)
        t.need_f32 = false;
    }
  }
  // An absorbed LayoutConvert's output is written by the contraction's
  // epilogue, which stores fp32 (and the bf16 copy alongside).
  for (const auto& kv : out_redirect) P->t[kv.second].need_f32 = true;
  for (auto& t : P->t) {
    if (!t.valid) continue;  // fused away before storage (attention scores)
    size_t es = elem_size(t.elem);
    if (t.need_f32 || !t.need_bf16) {
      P->keep.push_back(std::make_unique<DevBuf>(es * t.numel));
      t.d = P->keep.back()->p;
    }
    if (t.need_bf16) {
      P->keep.push_back(std::make_unique<DevBuf>(2 * t.numel));
      t.d_bf16 = P->keep.back()->p;
    }
    if (!t.d) t.elem = LFGPU_ELEM_BF16;  // bf16-only storage
  }
  for (auto& kv : absorbed_pad) {
    PTensor& xp = P->t[P->nodes[kv.second].output];
    if (!xp.d_bf16 || xp.d) fail(LFGPU_EINVAL, "absorbed Padding output must be bf16-only");
    CUDA_OK(cudaMemset(xp.d_bf16, 0, 2 * xp.numel));  // the pad ring, never written
    umma[kv.first].scatter.dst = xp.d_bf16;
  }
  int* d_err = P->ctx->d_err;

  // Mixed consumers: refresh a tensor's bf16 shadow right after it is
  // written (by its own node, or by the fused epilogue of the chain it ends).
  auto refresh_shadow = [&](int ni, PTensor& out) {
    if (!(out.d && out.d_bf16) || out.shadow_by_producer) return;
    CopySpec spec;
    spec.lmap = identity_map(out.logical);
    spec.dst_seq = out.seq;
    spec.src_seq = out.seq;
    bool oob;
    CopyKernel k = compile_copy(spec, out.elem, LFGPU_ELEM_BF16, P->keep, &oob);
    const void* src = out.d;
    void* dst = out.d_bf16;
    PStep sh;
    sh.node = ni;
    sh.kernel = "bf16_shadow";
    sh.run = [k, src, dst, d_err](cudaStream_t s) { return run_copy(k, src, dst, d_err, s); };
    P->steps.push_back(std::move(sh));
  };

  // Batched-matmul parameters of node bn (BmmQK / BmmPV): shape checks,
  // separable tables, column slices.
  auto bmm_params = [&](int bn) {
    const auto& n = P->nodes[bn];
    const PTensor& out = P->t[n.output];
    const PTensor& A = P->t[n.inputs[0]];
    const PTensor& B = P->t[n.inputs[1]];
    const int64_t H = n.heads;
    if (H < 1) fail(LFGPU_EINVAL, "batched matmul needs heads >= 1");
    if ((!A.d && A.valid) || !B.d) fail(LFGPU_EUNSUPPORTED, "batched matmul reads f32 operands");
    if (out.dtype != LFGPU_DTYPE_F32) fail(LFGPU_EUNSUPPORTED, "batched matmul is defined for f32 only");
    BmmParams M;
    M.mode = n.kind == LFGPU_OP_BMM_QK ? 0 : 1;
    M.H = static_cast<int32_t>(H);
    if (n.kind == LFGPU_OP_BMM_QK) {  // q [T, Cq], k [T2, Ck] -> s [H, T, T2]
      if (A.logical.size() != 2 || B.logical.size() != 2 || out.logical.size() != 3 ||
          out.logical[0].extent != H || out.logical[1].extent != A.logical[0].extent ||
          out.logical[2].extent != B.logical[0].extent)
        fail(LFGPU_EINVAL, "BmmQK shapes: q [T, Cq], k [T2, Ck] -> s [H, T, T2]");
      int64_t dh = n.head_dim;
      if (dh == 0) {
        if (A.logical[1].extent != B.logical[1].extent || A.logical[1].extent % H || n.a_col0 || n.b_col0)
          fail(LFGPU_EINVAL, "BmmQK without head_dim: q [T, H*Dh], k [T2, H*Dh], no column offsets");
        dh = A.logical[1].extent / H;
      }
      if (n.a_col0 < 0 || n.b_col0 < 0 || n.a_col0 + H * dh > A.logical[1].extent ||
          n.b_col0 + H * dh > B.logical[1].extent)
        fail(LFGPU_EINVAL, "BmmQK column slice out of range");
      M.T = static_cast<int32_t>(A.logical[0].extent);
      M.T2 = static_cast<int32_t>(B.logical[0].extent);
      M.Dh = static_cast<int32_t>(dh);
    } else {  // p [H, T, T2], v [T2, Cv] -> o [T, H*Dh]
      if (A.logical.size() != 3 || B.logical.size() != 2 || out.logical.size() != 2 ||
          A.logical[0].extent != H || A.logical[2].extent != B.logical[0].extent ||
          out.logical[1].extent % H || out.logical[0].extent != A.logical[1].extent || n.a_col0 ||
          n.b_col0 < 0 || n.b_col0 + out.logical[1].extent > B.logical[1].extent)
        fail(LFGPU_EINVAL, "BmmPV shapes: p [H, T, T2], v [T2, Cv] -> o [T, H*Dh], b_col0 + H*Dh <= Cv");
      M.T = static_cast<int32_t>(A.logical[1].extent);
      M.T2 = static_cast<int32_t>(A.logical[2].extent);
      M.Dh = static_cast<int32_t>(out.logical[1].extent / H);
      if ((n.head_dim && n.head_dim != M.Dh) || (!n.head_dim && out.logical[1].extent != B.logical[1].extent))
        fail(LFGPU_EINVAL, "BmmPV: o columns must be heads * head_dim (head_dim 0: o and v equally wide)");
    }
    if (M.Dh > 128 || M.Dh % 2) fail(LFGPU_EUNSUPPORTED, "batched matmul head dim must be even and <= 128");
    if (M.mode == 1 && M.T2 > 512) fail(LFGPU_EUNSUPPORTED, "BmmPV reduction length > 512");
    std::vector<int64_t> oa, ob, oo;
    M.ta = tables_for(P, A, &oa);
    M.tb = tables_for(P, B, &ob);
    M.to = tables_for(P, out, &oo);
    for (size_t j = 0; j < oa.size() && j < 3; ++j) M.a_off[j] = oa[j];
    for (size_t j = 0; j < ob.size() && j < 3; ++j) M.b_off[j] = ob[j];
    // packed operands: a column slice is the same column table entered
    // a_col0 / b_col0 entries later
    if (n.kind == LFGPU_OP_BMM_QK) M.a_off[1] += n.a_col0;
    M.b_off[1] += n.b_col0;
    for (size_t j = 0; j < oo.size() && j < 3; ++j) M.o_off[j] = oo[j];
    M.a = static_cast<const float*>(A.d);
    M.b = static_cast<const float*>(B.d);
    M.out = static_cast<float*>(out.d);
    return M;
  };

  // 3. One step per node.
  for (int ni : P->order) {
    if (fused_away.count(ni)) {
      P->node_kernel[ni] = "fused";
      // The chain's final tensor was written by the producer's epilogue.
      PTensor& fo = P->t[P->nodes[ni].output];
      if (fo.valid) refresh_shadow(ni, fo);
      continue;
    }
    const auto& n = P->nodes[ni];
    PTensor& out = P->t[n.output];
    PStep step;
    step.node = ni;
    switch (n.kind) {
      case LFGPU_OP_PADDING:
      case LFGPU_OP_LAYOUT_CONVERT: {
        const PTensor& in = P->t[n.inputs[0]];
        CopySpec spec;
        if (n.kind == LFGPU_OP_PADDING) {
          if (in.logical.size() != 4) fail(LFGPU_EINVAL, "Padding input must be rank 4");
          spec.lmap = padding_map(in.logical, n.pad);
        } else {
          spec.lmap = identity_map(in.logical);
        }
        spec.dst_seq = out.seq;
        spec.src_seq = in.seq;
        spec.mode = FoldMode::Nest;
        bool oob = false;
        int se = in.d ? in.elem : LFGPU_ELEM_BF16;
        const void* src = in.d ? in.d : in.d_bf16;
        // Write the primary buffer, and the bf16 shadow in the same pass when
        // this is the only consumer-facing copy.
        int de = out.d ? out.elem : LFGPU_ELEM_BF16;
        void* dst = out.d ? out.d : out.d_bf16;
        CopyKernel k = compile_copy(spec, se, de, P->keep, &oob);
        if (oob)
          fail(LFGPU_ERANGE, std::string("out-of-range access: ") +
                                 (n.kind == LFGPU_OP_PADDING ? "Padding" : "LayoutConvert") +
                                 " into '" + out.id + "' reads outside '" + in.id + "'");
        step.kernel = copy_name(k);
        step.run = [k, src, dst, d_err](cudaStream_t s) { return run_copy(k, src, dst, d_err, s); };
        P->bytes += in.numel * elem_size(se) + out.numel * elem_size(de);
        break;
      }
      case LFGPU_OP_RELU:
      case LFGPU_OP_BIASADD:
      case LFGPU_OP_EWADD: {
        GenEltwise G;
        G.op = n.kind == LFGPU_OP_RELU ? GEN_RELU : n.kind == LFGPU_OP_BIASADD ? GEN_BIASADD : GEN_EWADD;
        G.rank = static_cast<int32_t>(out.logical.size());
        G.n = out.numel;
        const PTensor& x = P->t[n.inputs[0]];
        if (!x.d) fail(LFGPU_EUNSUPPORTED, "element-wise read of a bf16-only tensor");
        std::vector<int64_t> off;
        G.tab0 = tables_for(P, x, &off);
        for (size_t j = 0; j < off.size(); ++j) G.tab_off[j] = off[j];
        G.in0 = x.d;
        if (n.kind != LFGPU_OP_RELU) {
          const PTensor& y = P->t[n.inputs[1]];
          std::vector<int64_t> off1;
          G.tab1 = tables_for(P, y, &off1);
          G.in1 = y.d;
          if (n.kind == LFGPU_OP_EWADD)
            for (size_t j = 0; j < off1.size(); ++j)
              if (off1[j] != off[j]) fail(LFGPU_EINVAL, "EwAdd operands differ in shape");
          G.bias_dim = out.logical.size() == 4 ? 1 : static_cast<int32_t>(out.logical.size()) - 1;
          P->bytes += y.numel * elem_size(y.elem);
        }
        IxProgram* prog = out_program(P, out);
        int elem = out.elem;
        void* dst = out.d;
        step.kernel = "gen_eltwise";
        step.run = [prog, G, elem, dst, d_err](cudaStream_t s) {
          return launch_gen_eltwise(prog, G, elem, dst, d_err, s);
        };
        P->bytes += x.numel * elem_size(x.elem) + out.numel * elem_size(out.elem);
        break;
      }
      case LFGPU_OP_C2D:
      case LFGPU_OP_GMM:
      case LFGPU_OP_DEP: {
        const PTensor& A = P->t[n.inputs[0]];
        const PTensor& B = P->t[n.inputs[1]];
        int64_t macs = 0;
        if (n.kind == LFGPU_OP_GMM) macs = out.logical[0].extent * out.logical[1].extent * A.logical[1].extent;
        else if (n.kind == LFGPU_OP_C2D)
          macs = numel(out.logical) * B.logical[1].extent * B.logical[2].extent * B.logical[3].extent;
        else
          macs = numel(out.logical) * B.logical[1].extent * B.logical[2].extent;
        P->flops += 2 * macs;
        auto it = umma.find(ni);
        auto dt = direct.find(ni);
        auto dp = depd.find(ni);
        auto ic = im2col.find(ni);
        if (ic != im2col.end()) {
          UmmaPlan up = ic->second;
          Im2col Q;
          Q.N = static_cast<int32_t>(A.logical[0].extent);
          Q.I = static_cast<int32_t>(A.logical[1].extent);
          Q.H = static_cast<int32_t>(A.logical[2].extent);
          Q.W = static_cast<int32_t>(A.logical[3].extent);
          Q.O = static_cast<int32_t>(B.logical[0].extent);
          Q.KH = static_cast<int32_t>(B.logical[2].extent);
          Q.KW = static_cast<int32_t>(B.logical[3].extent);
          Q.V = static_cast<int32_t>(n.stride);
          Q.Ho = static_cast<int32_t>(out.logical[2].extent);
          Q.Wo = static_cast<int32_t>(out.logical[3].extent);
          Q.K = Q.I * Q.KH * Q.KW;
          Q.Kp = (Q.K + 63) / 64 * 64;
          Q.RT = up.tiles.empty() ? 128 : up.tiles[0].rows;  // rows per A brick = rows per tile
          if (!A.d || !B.d) fail(LFGPU_EUNSUPPORTED, "im2col conv on a bf16-only operand");
          Q.x = static_cast<const float*>(A.d);
          auto ipd = im2col_pad.find(ni);
          if (ipd != im2col_pad.end()) {  // read the unpadded input
            const auto& pnode = P->nodes[ipd->second];
            PTensor& xin = P->t[pnode.inputs[0]];
            if (!xin.d) fail(LFGPU_EUNSUPPORTED, "im2col: padded input has no fp32 buffer");
            Q.x = static_cast<const float*>(xin.d);
            Q.H = static_cast<int32_t>(xin.logical[2].extent);
            Q.W = static_cast<int32_t>(xin.logical[3].extent);
            Q.pad = static_cast<int32_t>(pnode.pad);
            const_cast<PTensor&>(A).valid = false;  // the padded tensor is never materialized
          }
          Q.w = static_cast<const float*>(B.d);
          const int64_t M = static_cast<int64_t>(Q.N) * Q.Ho * Q.Wo;
          P->keep.push_back(std::make_unique<DevBuf>(2 * static_cast<size_t>(M) * Q.Kp));
          Q.a = P->keep.back()->p;
          P->keep.push_back(std::make_unique<DevBuf>(2 * static_cast<size_t>(Q.O) * Q.Kp));
          Q.b = P->keep.back()->p;
          up.a = Q.a;
          up.b = Q.b;
          int final_t = up.epi_count ? up.epi[up.epi_count - 1].out_tensor : n.output;
          if (out_redirect.count(ni)) {  // the absorbed LayoutConvert's output, in its layout
            P->t[final_t].valid = false;
            final_t = out_redirect.at(ni);
          }
          up.out = static_cast<float*>(P->t[final_t].d);
          up.out_stream = out_stream_for(P->t[final_t]);
          if (P->t[final_t].d && P->t[final_t].d_bf16 && P->t[final_t].elem == LFGPU_ELEM_F32) {
            up.out_bf16 = P->t[final_t].d_bf16;
            P->t[final_t].shadow_by_producer = true;
          }
          for (int e = 0; e < up.epi_count; ++e) {
            if (up.epi[e].tensor >= 0) {
              const PTensor& et = P->t[up.epi[e].tensor];
              if (!et.d) fail(LFGPU_EUNSUPPORTED, "epilogue operand has no fp32 buffer");
              up.epi[e].ptr = static_cast<const float*>(et.d);
            }
          }
          for (int e = 0; e + 1 < up.epi_count; ++e) P->t[up.epi[e].out_tensor].valid = false;
          if (up.epi_count) out.valid = false;
          UmmaLaunch L = umma_prepare(up);
          L.chain_slot = static_cast<int>(P->steps.size());
          step.kernel = "im2col_umma";
          step.launches = 2;
          step.run = [Q, L](cudaStream_t st) {
            cudaError_t e = launch_im2col(Q, st);
            return e != cudaSuccess ? e : umma_launch(L, st);
          };
          P->tc_nodes += 1;
          P->bytes += A.numel * 4 + B.numel * 4 + 4 * M * Q.Kp + P->t[final_t].numel * 4;
          P->summary[ni] = "im2col(Kp=" + std::to_string(Q.Kp) + ") + " + up.summary +
                           " store=" + std::to_string(L.store_mode) + " grid=" + std::to_string(L.grid);
        } else if (dp != depd.end()) {
          DirectDep D;
          D.N = static_cast<int32_t>(out.logical[0].extent);
          D.C = static_cast<int32_t>(out.logical[1].extent);
          D.Ho = static_cast<int32_t>(out.logical[2].extent);
          D.Wo = static_cast<int32_t>(out.logical[3].extent);
          D.KH = static_cast<int32_t>(B.logical[1].extent);
          D.KW = static_cast<int32_t>(B.logical[2].extent);
          D.V = static_cast<int32_t>(n.stride);
          if (!A.d || !B.d) fail(LFGPU_EUNSUPPORTED, "depthwise conv on a bf16-only operand");
          std::vector<int64_t> xo, wo, oo;
          D.x = static_cast<const float*>(A.d);
          D.xt = tables_for(P, A, &xo);
          for (size_t j = 0; j < xo.size(); ++j) D.x_off[j] = xo[j];
          D.w = static_cast<const float*>(B.d);
          D.wt = tables_for(P, B, &wo);
          for (size_t j = 0; j < wo.size(); ++j) D.w_off[j] = wo[j];
          const auto& epi = dp->second;
          const int final_t = epi.empty() ? n.output : epi.back().out_tensor;
          PTensor& fo = P->t[final_t];
          D.ot = tables_for(P, fo, &oo);
          for (size_t j = 0; j < oo.size(); ++j) D.o_off[j] = oo[j];
          D.out = static_cast<float*>(fo.d);
          // Thread order follows the output's unit-stride logical dim.
          {
            std::vector<int64_t> tb, of;
            separable_tables(fo.logical, fo.seq, &tb, &of);
            auto stride_of = [&](int d) {
              return fo.logical[d].extent > 1 ? tb[of[d] + 1] - tb[of[d]] : INT64_MAX;
            };
            D.fast = stride_of(1) <= stride_of(3) ? 1 : 3;
          }
          // float4 over channels when C is unit-stride in aligned groups of
          // 4 in input, weights and output and all other offsets are
          // multiples of 4 (16-byte aligned float4 accesses).
          {
            auto quad_ok = [&](const PTensor& t, int cdim) {
              std::vector<int64_t> tb, of;
              if (!separable_tables(t.logical, t.seq, &tb, &of)) return false;
              if (t.logical[cdim].extent % 4) return false;
              for (size_t d = 0; d < t.logical.size(); ++d)
                for (int64_t i = 0; i < t.logical[d].extent; ++i) {
                  const int64_t v = tb[of[d] + i];
                  if (static_cast<int>(d) == cdim) {
                    if (i % 4 == 0 ? v % 4 != 0 : v != tb[of[d] + i - 1] + 1) return false;
                  } else if (v % 4) {
                    return false;
                  }
                }
              return true;
            };
            bool q = D.fast == 1 && quad_ok(A, 1) && quad_ok(B, 0) && quad_ok(fo, 1);
            for (size_t e = 0; q && e < epi.size(); ++e)
              if (epi[e].kind == EPI_RESIDUAL && !quad_ok(P->t[epi[e].tensor], 1)) q = false;
            D.vec4 = q ? 1 : 0;
          }
          D.nepi = static_cast<int32_t>(epi.size());
          for (size_t e = 0; e < epi.size(); ++e) {
            D.epi_kind[e] = epi[e].kind == EPI_BIAS ? DIRECT_EPI_BIAS
                            : epi[e].kind == EPI_RELU ? DIRECT_EPI_RELU
                                                      : DIRECT_EPI_RESIDUAL;
            if (epi[e].tensor >= 0) {
              const PTensor& et = P->t[epi[e].tensor];
              if (!et.d) fail(LFGPU_EUNSUPPORTED, "epilogue operand has no fp32 buffer");
              D.epi_ptr[e] = static_cast<const float*>(et.d);
            }
          }
          for (size_t e = 0; e + 1 < epi.size(); ++e) P->t[epi[e].out_tensor].valid = false;
          if (!epi.empty()) out.valid = false;
          step.kernel = D.vec4 ? "dep_direct4" : "dep_direct";
          step.run = [D](cudaStream_t st) { return launch_dep_direct(D, st); };
          P->bytes += A.numel * 4 + B.numel * 4 + fo.numel * 4;
        } else if (dt != direct.end()) {
          DirectConv D;
          D.N = static_cast<int32_t>(A.logical[0].extent);
          D.I = static_cast<int32_t>(A.logical[1].extent);
          D.H = static_cast<int32_t>(A.logical[2].extent);
          D.W = static_cast<int32_t>(A.logical[3].extent);
          D.O = static_cast<int32_t>(B.logical[0].extent);
          D.KH = static_cast<int32_t>(B.logical[2].extent);
          D.KW = static_cast<int32_t>(B.logical[3].extent);
          D.V = static_cast<int32_t>(n.stride);
          D.Ho = static_cast<int32_t>(out.logical[2].extent);
          D.Wo = static_cast<int32_t>(out.logical[3].extent);
          if (!A.d || !B.d) fail(LFGPU_EUNSUPPORTED, "direct conv on a bf16-only operand");
          D.x = static_cast<const float*>(A.d);
          D.w = static_cast<const float*>(B.d);
          const auto& epi = dt->second;
          int final_t = epi.empty() ? n.output : epi.back().out_tensor;
          PTensor& fo = P->t[final_t];
          std::vector<int64_t> oo;
          D.tab = tables_for(P, fo, &oo);
          for (size_t j = 0; j < oo.size(); ++j) D.tab_off[j] = oo[j];
          D.out = static_cast<float*>(fo.d);
          D.nepi = static_cast<int32_t>(epi.size());
          for (size_t e = 0; e < epi.size(); ++e) {
            D.epi_kind[e] = epi[e].kind == EPI_BIAS ? DIRECT_EPI_BIAS
                            : epi[e].kind == EPI_RELU ? DIRECT_EPI_RELU
                                                      : DIRECT_EPI_RESIDUAL;
            if (epi[e].tensor >= 0) {
              const PTensor& et = P->t[epi[e].tensor];
              if (!et.d) fail(LFGPU_EUNSUPPORTED, "epilogue operand has no fp32 buffer");
              D.epi_ptr[e] = static_cast<const float*>(et.d);
            }
          }
          for (size_t e = 0; e + 1 < epi.size(); ++e) P->t[epi[e].out_tensor].valid = false;
          if (!epi.empty()) out.valid = false;
          step.kernel = "c2d_direct";
          step.run = [D](cudaStream_t st) { return launch_c2d_direct(D, st); };
          P->bytes += A.numel * 4 + B.numel * 4 + fo.numel * 4;
        } else if (it != umma.end()) {
          UmmaPlan up = it->second;
          up.a = up.swap_ab ? B.d_bf16 : A.d_bf16;
          up.b = up.swap_ab ? A.d_bf16 : B.d_bf16;
          SplitParams sa, sb;
          const bool split3 = split_gmm.count(ni) > 0;
          if (split3) {
            const SplitGmm& sg = split_gmm.at(ni);
            if (!A.d || !B.d) fail(LFGPU_EUNSUPPORTED, "split-precision GMM needs fp32 operands");
            const int64_t M = A.logical[0].extent, K = A.logical[1].extent, N = B.logical[1].extent;
            auto dst_tables = [&](const std::vector<Dim>& lg, const Seq& sq, std::vector<int64_t>* r,
                                  std::vector<int64_t>* c) {
              std::vector<int64_t> tab, off;
              if (!separable_tables(lg, sq, &tab, &off)) fail(LFGPU_EINVAL, "split operand layout");
              r->assign(tab.begin() + off[0], tab.begin() + off[0] + lg[0].extent);
              c->assign(tab.begin() + off[1], tab.begin() + off[1] + lg[1].extent);
            };
            std::vector<int64_t> ar, ac, br, bc, dar, dac, dbr, dbc;
            row_col_offsets(A, &ar, &ac);
            row_col_offsets(B, &br, &bc);
            dst_tables(sg.a_log, sg.a_seq, &dar, &dac);
            dst_tables(sg.b_log, sg.b_seq, &dbr, &dbc);
            P->keep.push_back(std::make_unique<DevBuf>(2 * M * kSplitTerms * K));
            void* a3 = P->keep.back()->p;
            P->keep.push_back(std::make_unique<DevBuf>(2 * kSplitTerms * K * N));
            void* b3 = P->keep.back()->p;
            sa.side = 0;
            sa.R = M;
            sa.C = K;
            sa.K = K;
            sa.src = static_cast<const float*>(A.d);
            sa.src_row = upload(P->keep, ar.data(), ar.size());
            sa.src_col = upload(P->keep, ac.data(), ac.size());
            sa.dst = a3;
            sa.dst_row = upload(P->keep, dar.data(), dar.size());
            sa.dst_col = upload(P->keep, dac.data(), dac.size());
            sb.side = 1;
            sb.R = K;
            sb.C = N;
            sb.K = K;
            sb.src = static_cast<const float*>(B.d);
            sb.src_row = upload(P->keep, br.data(), br.size());
            sb.src_col = upload(P->keep, bc.data(), bc.size());
            sb.dst = b3;
            sb.dst_row = upload(P->keep, dbr.data(), dbr.size());
            sb.dst_col = upload(P->keep, dbc.data(), dbc.size());
            up.a = a3;
            up.b = b3;
          }
          // The chain's final output is the one written; intermediates of a
          // fused chain are also written when the caller keeps them.
          int final_t = up.epi_count ? up.epi[up.epi_count - 1].out_tensor : n.output;
          if (out_redirect.count(ni)) {  // the absorbed LayoutConvert's output, in its layout
            P->t[final_t].valid = false;
            final_t = out_redirect.at(ni);
          }
          up.out = static_cast<float*>(P->t[final_t].d);
          up.out_stream = out_stream_for(P->t[final_t]);
          if (P->t[final_t].d && P->t[final_t].d_bf16 &&
              P->t[final_t].elem == LFGPU_ELEM_F32) {  // dual store: no shadow pass
            up.out_bf16 = P->t[final_t].d_bf16;
            P->t[final_t].shadow_by_producer = true;
          }
          for (int e = 0; e < up.epi_count; ++e) {
            if (up.epi[e].tensor >= 0) {
              const PTensor& et = P->t[up.epi[e].tensor];
              if (!et.d) fail(LFGPU_EUNSUPPORTED, "epilogue operand has no fp32 buffer");
              up.epi[e].ptr = static_cast<const float*>(et.d);
            }
          }
          // Intermediate tensors of a fused chain are never written.
          for (int e = 0; e + 1 < up.epi_count; ++e) P->t[up.epi[e].out_tensor].valid = false;
          if (up.epi_count) out.valid = false;
          UmmaLaunch L = umma_prepare(up);
          L.chain_slot = static_cast<int>(P->steps.size());
          {
            // Resident weights may load before the PDL wait when they are a
            // plan constant (no producer) and this is not the run's first
            // kernel (which may follow a set_input conversion of them).
            const PTensor& W = P->t[n.inputs[1]];
            L.w_prewait = L.wres && !P->steps.empty() && W.producer < 0 && !getenv("LFGPU_NO_W_PREWAIT") ? 1 : 0;
          }
          step.kernel = up.kind == UMMA_CONV ? "umma_conv" : "umma_gemm";
          if (split3) {
            step.launches = 3;
            step.run = [L, sa, sb](cudaStream_t s) {
              cudaError_t e = launch_split_bf16(sa, s);
              if (e == cudaSuccess) e = launch_split_bf16(sb, s);
              return e != cudaSuccess ? e : umma_launch(L, s);
            };
          } else {
            step.run = [L](cudaStream_t s) { return umma_launch(L, s); };
          }
          P->tc_nodes += 1;
          P->bytes += A.numel * 2 + B.numel * 2 + P->t[final_t].numel * 4;
          P->summary[ni] = up.summary + " store=" + std::to_string(L.store_mode) +
                           " splits=" + std::to_string(L.splits) + " grid=" + std::to_string(L.grid) +
                           " ring=" + std::to_string(L.pipe) + (L.epi_alias ? " epi-in-ring" : "") +
                           (L.dual == 1 ? " dual" : L.dual == 2 ? " split-issue" : "");
        } else if (gemv.count(ni)) {
          GemvParams Gv;
          Gv.M = static_cast<int32_t>(A.logical[0].extent);
          Gv.K = static_cast<int32_t>(A.logical[1].extent);
          Gv.N = static_cast<int32_t>(B.logical[1].extent);
          if (!A.d || !B.d) fail(LFGPU_EUNSUPPORTED, "CUDA-core GEMV on a bf16-only operand");
          std::vector<int64_t> ao, bo, oo;
          Gv.a = static_cast<const float*>(A.d);
          Gv.at = tables_for(P, A, &ao);
          Gv.b = static_cast<const float*>(B.d);
          Gv.bt = tables_for(P, B, &bo);
          for (int j = 0; j < 2; ++j) {
            Gv.a_off[j] = ao[j];
            Gv.b_off[j] = bo[j];
          }
          const auto& epi = gemv.at(ni);
          const int final_t = epi.empty() ? n.output : epi.back().out_tensor;
          PTensor& fo = P->t[final_t];
          Gv.ot = tables_for(P, fo, &oo);
          for (int j = 0; j < 2; ++j) Gv.o_off[j] = oo[j];
          Gv.out = static_cast<float*>(fo.d);
          if (fo.d_bf16) {
            Gv.out_bf16 = fo.d_bf16;
            fo.shadow_by_producer = true;
          }
          Gv.nepi = static_cast<int32_t>(epi.size());
          for (size_t e = 0; e < epi.size() && e < 4; ++e) {
            Gv.epi_kind[e] = epi[e].kind;
            if (epi[e].tensor >= 0) {
              const PTensor& et = P->t[epi[e].tensor];
              if (!et.d) fail(LFGPU_EUNSUPPORTED, "epilogue operand has no fp32 buffer");
              Gv.epi_ptr[e] = static_cast<const float*>(et.d);
            }
          }
          if (epi.size() > 4) fail(LFGPU_EUNSUPPORTED, "GEMV epilogue chain longer than 4");
          for (size_t e = 0; e + 1 < epi.size(); ++e) P->t[epi[e].out_tensor].valid = false;
          if (!epi.empty()) out.valid = false;
          step.kernel = "gemv";
          step.run = [Gv](cudaStream_t st) { return launch_gemv(Gv, st); };
          P->bytes += A.numel * 4 + B.numel * 4 + fo.numel * 4;
        } else {
          GenContract G;
          G.op = n.kind == LFGPU_OP_GMM ? GEN_GMM : n.kind == LFGPU_OP_C2D ? GEN_C2D : GEN_DEP;
          G.n = out.numel;
          G.V = n.stride;
          if (n.kind == LFGPU_OP_GMM) {
            G.K = A.logical[1].extent;
          } else if (n.kind == LFGPU_OP_C2D) {
            G.I = B.logical[1].extent;
            G.KH = B.logical[2].extent;
            G.KW = B.logical[3].extent;
          } else {
            G.KH = B.logical[1].extent;
            G.KW = B.logical[2].extent;
          }
          if (!A.d || !B.d) fail(LFGPU_EUNSUPPORTED, "CUDA-core contraction on bf16-only operand");
          std::vector<int64_t> oa, ob;
          G.ta = tables_for(P, A, &oa);
          G.tb = tables_for(P, B, &ob);
          for (size_t j = 0; j < oa.size(); ++j) G.a_off[j] = oa[j];
          for (size_t j = 0; j < ob.size(); ++j) G.b_off[j] = ob[j];
          G.a = A.d;
          G.b = B.d;
          IxProgram* prog = out_program(P, out);
          int elem = out.elem;
          void* dst = out.d;
          step.kernel = "gen_contract";
          step.run = [prog, G, elem, exact, dst](cudaStream_t s) {
            return launch_gen_contract(prog, G, elem, exact, dst, s);
          };
          P->bytes += A.numel * elem_size(A.elem) + B.numel * elem_size(B.elem) +
                      out.numel * elem_size(out.elem);
        }
        break;
      }
      case LFGPU_OP_GELU: {
        // Element-wise (fused into the producing contraction's epilogue when
        // the schedule asks for it; here the stand-alone node).
        GenEltwise G;
        G.op = GEN_GELU;
        G.rank = static_cast<int32_t>(out.logical.size());
        G.n = out.numel;
        const PTensor& x = P->t[n.inputs[0]];
        if (!x.d) fail(LFGPU_EUNSUPPORTED, "element-wise read of a bf16-only tensor");
        if (out.dtype != LFGPU_DTYPE_F32) fail(LFGPU_EUNSUPPORTED, "GELU is defined for f32 tensors only");
        std::vector<int64_t> off;
        G.tab0 = tables_for(P, x, &off);
        for (size_t j = 0; j < off.size(); ++j) G.tab_off[j] = off[j];
        G.in0 = x.d;
        IxProgram* prog = out_program(P, out);
        int elem = out.elem;
        void* dst = out.d;
        step.kernel = "gen_eltwise";
        step.run = [prog, G, elem, dst, d_err](cudaStream_t s) {
          return launch_gen_eltwise(prog, G, elem, dst, d_err, s);
        };
        P->bytes += x.numel * elem_size(x.elem) + out.numel * elem_size(out.elem);
        break;
      }
      case LFGPU_OP_SOFTMAX:
      case LFGPU_OP_LAYERNORM: {
        // Row reductions over the last logical dim (k_rows.cu), every operand
        // through its separable offset tables.
        const PTensor& X = P->t[n.inputs[0]];
        const char* nm = n.kind == LFGPU_OP_SOFTMAX ? "Softmax" : "LayerNorm";
        if (out.dtype != LFGPU_DTYPE_F32 || X.dtype != LFGPU_DTYPE_F32)
          fail(LFGPU_EUNSUPPORTED, std::string(nm) + " is defined for f32 tensors only");
        if (!same_extents(X.logical, out.logical))
          fail(LFGPU_EINVAL, std::string(nm) + " output shape mismatch for '" + out.id + "'");
        const int64_t d = out.logical.back().extent;
        if (d > 2048) fail(LFGPU_EUNSUPPORTED, std::string(nm) + " rows longer than 2048");
        if (!X.d) fail(LFGPU_EUNSUPPORTED, "row read of a bf16-only tensor");
        RowsParams R;
        R.op = n.kind == LFGPU_OP_SOFTMAX ? ROWS_SOFTMAX : ROWS_LAYERNORM;
        R.d = static_cast<int32_t>(d);
        R.rows = out.numel / std::max<int64_t>(d, 1);
        std::vector<int64_t> rx, cx, ry, cy;
        row_col_offsets(X, &rx, &cx);
        row_col_offsets(out, &ry, &cy);
        R.row_x = upload(P->keep, rx.data(), rx.size());
        R.col_x = upload(P->keep, cx.data(), cx.size());
        R.row_y = upload(P->keep, ry.data(), ry.size());
        R.col_y = upload(P->keep, cy.data(), cy.size());
        R.x = static_cast<const float*>(X.d);
        R.y = static_cast<float*>(out.d);
        if (out.d_bf16) {  // a tensor-core consumer's operand, written in the same pass
          R.y_bf16 = out.d_bf16;
          out.shadow_by_producer = true;
        }
        if (n.kind == LFGPU_OP_LAYERNORM) {
          const PTensor& GB = P->t[n.inputs[1]];
          if (GB.logical.size() != 2 || GB.logical[0].extent != 2 || GB.logical[1].extent != d)
            fail(LFGPU_EINVAL, "LayerNorm parameters must be [2, " + std::to_string(d) + "] (gamma; beta)");
          if (!GB.d) fail(LFGPU_EUNSUPPORTED, "LayerNorm parameters must be f32");
          std::vector<int64_t> rg, cg;
          row_col_offsets(GB, &rg, &cg);
          std::vector<int64_t> cgb(2 * d);
          for (int64_t j = 0; j < d; ++j) {
            cgb[j] = rg[0] + cg[j];
            cgb[d + j] = rg[1] + cg[j];
          }
          R.col_gb = upload(P->keep, cgb.data(), cgb.size());
          R.gb = static_cast<const float*>(GB.d);
          R.eps = static_cast<float>(std::pow(10.0, -static_cast<double>(n.eps_exp)));
          P->bytes += GB.numel * 4;
        }
        step.kernel = n.kind == LFGPU_OP_SOFTMAX ? "rows_softmax" : "rows_layernorm";
        step.run = [R](cudaStream_t s) { return launch_rows(R, s); };
        P->bytes += X.numel * 4 + out.numel * 4;
        break;
      }
      case LFGPU_OP_BMM_QK:
      case LFGPU_OP_BMM_PV: {
        BmmParams M = bmm_params(ni);
        if (out.d_bf16) {
          M.out_bf16 = out.d_bf16;
          out.shadow_by_producer = true;
        }
        const PTensor& A = P->t[n.inputs[0]];
        P->bytes += (n.kind == LFGPU_OP_BMM_QK ? (int64_t(M.T) + M.T2) * M.H * M.Dh
                                               : A.numel + int64_t(M.T2) * M.H * M.Dh) * 4 +
                    out.numel * 4;
        P->flops += 2 * static_cast<int64_t>(M.H) * M.T * M.T2 * M.Dh;
        if (n.kind == LFGPU_OP_BMM_PV && attn_of.count(ni)) {
          // the fused attention core: QK's operands, PV's v and output
          const int qn = attn_of.at(ni);
          BmmParams Q = bmm_params(qn);
          if (Q.T2 != M.T2 || Q.T != M.T || Q.Dh != M.Dh)
            fail(LFGPU_EINVAL, "attention: BmmQK / BmmPV shapes disagree");
          P->bytes -= A.numel * 4;  // p is never read from memory
          P->flops += 2 * static_cast<int64_t>(Q.H) * Q.T * Q.T2 * Q.Dh;
          P->bytes += (int64_t(Q.T) + Q.T2) * Q.H * Q.Dh * 4;
          const auto& qkn = P->nodes[qn];
          const int64_t w = int64_t(Q.H) * Q.Dh;
          Q.vec = Q.Dh % 4 == 0 && cols_vec4(P->t[qkn.inputs[0]], qkn.a_col0, w) &&
                  cols_vec4(P->t[qkn.inputs[1]], qkn.b_col0, w) && cols_vec4(P->t[n.inputs[1]], n.b_col0, w);
          if (getenv("LFGPU_ATTN_SCALAR")) Q.vec = 0;
          step.kernel = "attention";
          step.run = [Q, M, exact](cudaStream_t s) {
            BmmParams q = Q;
            q.dbg = static_cast<unsigned long long*>(umma_debug_buffer());  // diagnostics only
            return launch_attention(q, M, exact, s);
          };
          break;
        }
        step.kernel = n.kind == LFGPU_OP_BMM_QK ? "bmm_qk" : "bmm_pv";
        step.run = [M, exact](cudaStream_t s) { return launch_bmm(M, exact, s); };
        break;
      }
      case LFGPU_OP_MAXPOOL:
      case LFGPU_OP_GLOBAL_AVGPOOL: {
        // Op-set extension (lfgpu.h): CUDA-core window reductions through the
        // operand's separable offset tables, output walked in physical order.
        const PTensor& A = P->t[n.inputs[0]];
        if (A.logical.size() != 4) fail(LFGPU_EINVAL, "pool input must be rank 4");
        GenContract G;
        G.n = out.numel;
        if (n.kind == LFGPU_OP_MAXPOOL) {
          const int64_t k = n.window, v = n.stride;
          if (k < 1 || v < 1) fail(LFGPU_EINVAL, "MaxPool needs window >= 1 and stride >= 1");
          if (out.logical.size() != 4 || out.logical[0].extent != A.logical[0].extent ||
              out.logical[1].extent != A.logical[1].extent ||
              out.logical[2].extent != (A.logical[2].extent - k) / v + 1 ||
              out.logical[3].extent != (A.logical[3].extent - k) / v + 1 ||
              A.logical[2].extent < k || A.logical[3].extent < k)
            fail(LFGPU_EINVAL, "MaxPool output shape mismatch for '" + out.id + "'");
          G.op = GEN_MAXPOOL;
          G.KH = G.KW = k;
          G.V = v;
        } else {
          if (out.logical.size() != 2 || out.logical[0].extent != A.logical[0].extent ||
              out.logical[1].extent != A.logical[1].extent)
            fail(LFGPU_EINVAL, "GlobalAvgPool output must be [N, C] for '" + out.id + "'");
          if (out.dtype != LFGPU_DTYPE_F32)
            fail(LFGPU_EUNSUPPORTED, "GlobalAvgPool is defined for f32 tensors only");
          G.op = GEN_GLOBAL_AVGPOOL;
          G.H = A.logical[2].extent;
          G.W = A.logical[3].extent;
        }
        {
          // k_small.cu's table-driven pool kernels when both layouts are
          // separable (fp32; the exact mode keeps the generic kernel), reading
          // through an absorbed Padding when 1c' found one
          const auto mpp = maxpool_pad.find(ni);
          const PTensor& X = mpp != maxpool_pad.end() ? P->t[P->nodes[mpp->second].inputs[0]] : A;
          std::vector<int64_t> tb, of;
          if (!exact && out.dtype == LFGPU_DTYPE_F32 && out.d && X.d && separable_tables(X.logical, X.seq, &tb, &of) &&
              separable_tables(out.logical, out.seq, &tb, &of)) {
            PoolParams Pp;
            Pp.op = n.kind == LFGPU_OP_MAXPOOL ? 0 : 1;
            Pp.N = static_cast<int32_t>(X.logical[0].extent);
            Pp.C = static_cast<int32_t>(X.logical[1].extent);
            Pp.H = static_cast<int32_t>(X.logical[2].extent);
            Pp.W = static_cast<int32_t>(X.logical[3].extent);
            if (mpp != maxpool_pad.end()) Pp.pad = static_cast<int32_t>(P->nodes[mpp->second].pad);
            if (Pp.op == 0) {
              Pp.Ho = static_cast<int32_t>(out.logical[2].extent);
              Pp.Wo = static_cast<int32_t>(out.logical[3].extent);
              Pp.K = static_cast<int32_t>(n.window);
              Pp.V = static_cast<int32_t>(n.stride);
            }
            std::vector<int64_t> xo, oo;
            Pp.x = static_cast<const float*>(X.d);
            Pp.xt = tables_for(P, X, &xo);
            for (size_t j = 0; j < xo.size() && j < 4; ++j) Pp.x_off[j] = xo[j];
            Pp.out = static_cast<float*>(out.d);
            Pp.ot = tables_for(P, out, &oo);
            for (size_t j = 0; j < oo.size() && j < 4; ++j) Pp.o_off[j] = oo[j];
            if (out.d_bf16) {
              Pp.out_bf16 = out.d_bf16;
              out.shadow_by_producer = true;
            }
            step.kernel = n.kind == LFGPU_OP_MAXPOOL ? "maxpool" : "global_avgpool";
            step.run = [Pp](cudaStream_t st) { return launch_pool(Pp, st); };
            P->bytes += X.numel * 4 + out.numel * 4;
            break;
          }
          if (mpp != maxpool_pad.end()) fail(LFGPU_EUNSUPPORTED, "absorbed Padding without the pool kernel");
        }
        if (!A.d) fail(LFGPU_EUNSUPPORTED, "pool read of a bf16-only tensor");
        std::vector<int64_t> oa;
        G.ta = tables_for(P, A, &oa);
        for (size_t j = 0; j < oa.size(); ++j) G.a_off[j] = oa[j];
        G.a = A.d;
        IxProgram* prog = out_program(P, out);
        int elem = out.elem;
        void* dst = out.d;
        step.kernel = n.kind == LFGPU_OP_MAXPOOL ? "gen_maxpool" : "gen_global_avgpool";
        step.run = [prog, G, elem, exact, dst](cudaStream_t s) {
          return launch_gen_contract(prog, G, elem, exact, dst, s);
        };
        P->bytes += A.numel * elem_size(A.elem) + out.numel * elem_size(out.elem);
        break;
      }
      default:
        fail(LFGPU_EINVAL, "unknown operator kind " + std::to_string(n.kind));
    }
    P->node_kernel[ni] = step.kernel;
    P->steps.push_back(std::move(step));
    if (out.valid) refresh_shadow(ni, out);
  }
}

void plan_run_steps(lfgpu_plan* P, cudaStream_t on = nullptr) {
  cudaStream_t st = on ? on : P->stream;
  // A plan of one kernel launches it directly: a graph launch costs ~3 us
  // more per step on this B200 (tools/gemm_ceiling.py --nograph) and, unlike
  // a direct PDL launch, cannot overlap the previous kernel's tail.
  int64_t nl = 0;
  for (const auto& s : P->steps) nl += s.launches;
  if ((P->flags & LFGPU_PLAN_CUDA_GRAPH) && nl > 1) {
    if (!P->gexec) {
      CUDA_OK(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal));
      for (auto& s : P->steps) {
        cudaError_t e = s.run(P->stream);
        if (e != cudaSuccess) {
          cudaGraph_t g;
          cudaStreamEndCapture(P->stream, &g);
          if (g) cudaGraphDestroy(g);
          fail(LFGPU_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
        }
      }
      CUDA_OK(cudaStreamEndCapture(P->stream, &P->graph));
      CUDA_OK(cudaGraphInstantiate(&P->gexec, P->graph, 0));
    }
    CUDA_OK(cudaGraphLaunch(P->gexec, st));
  } else {
    for (auto& s : P->steps) {
      cudaError_t e = s.run(st);
      if (e != cudaSuccess)
        fail(LFGPU_ECUDA, "kernel " + s.kernel + " (node " + std::to_string(s.node) +
                              "): " + cudaGetErrorString(e));
    }
  }
  P->ctx->launches += static_cast<int64_t>(P->steps.size());
}

void check_device_error(lfgpu_plan* P) {
  int h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, P->ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
  CUDA_OK(cudaStreamSynchronize(P->stream));
  if (h) {
    CUDA_OK(cudaMemsetAsync(P->ctx->d_err, 0, sizeof(int), P->stream));
    fail(LFGPU_ERANGE, "out-of-range access during execution");
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI

extern "C" {

int lfgpu_version(void) { return 1; }

const char* lfgpu_last_error(void) { return g_last_error.c_str(); }

int lfgpu_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) n = 0;
  *count = n;
  return LFGPU_OK;
}

int lfgpu_derive_layout(int32_t rank, const lfgpu_dim* dims, int32_t nprims,
                        const lfgpu_prim* prims, int32_t* out_rank, lfgpu_dim* out_dims) {
  return guarded([&] {
    auto d = derive(dims_of(rank, dims), seq_of(nprims, prims));
    *out_rank = static_cast<int32_t>(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
      std::memset(out_dims[i].name, 0, LFGPU_NAME_LEN);
      std::strncpy(out_dims[i].name, d[i].name.c_str(), LFGPU_NAME_LEN - 1);
      out_dims[i].extent = d[i].extent;
    }
  });
}

int lfgpu_convert_kind(int32_t rank, const lfgpu_dim* logical, int32_t nsrc,
                       const lfgpu_prim* src_seq, int32_t ndst, const lfgpu_prim* dst_seq,
                       int32_t* kind) {
  return guarded([&] {
    CopySpec spec;
    spec.lmap = identity_map(dims_of(rank, logical));
    spec.src_seq = seq_of(nsrc, src_seq);
    spec.dst_seq = seq_of(ndst, dst_seq);
    DigitMap m;
    bool oob;
    *kind = compile_digit_map(spec, &m, &oob) ? 1 : 0;
  });
}

int lfgpu_ctx_create(int device, lfgpu_ctx** out) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      fail(LFGPU_ECUDA, "no CUDA device available");
    CUDA_OK(cudaSetDevice(device));
    auto* c = new lfgpu_ctx;
    c->device = device;
    cudaError_t e = cudaMalloc(&c->d_err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, sizeof(int));
    if (e != cudaSuccess) {
      delete c;
      fail(LFGPU_ECUDA, cudaGetErrorString(e));
    }
    *out = c;
  });
}

int lfgpu_ctx_destroy(lfgpu_ctx* ctx) {
  if (!ctx) return LFGPU_OK;
  cudaSetDevice(ctx->device);
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->flush) cudaFree(ctx->flush);
  delete ctx;
  return LFGPU_OK;
}

int lfgpu_ctx_launch_count(lfgpu_ctx* ctx, int64_t* count) {
  *count = ctx ? ctx->launches : 0;
  return LFGPU_OK;
}

int lfgpu_layout_convert(lfgpu_ctx* ctx, int32_t rank, const lfgpu_dim* logical, int32_t nsrc,
                         const lfgpu_prim* src_seq, int32_t ndst, const lfgpu_prim* dst_seq,
                         int32_t src_elem, int32_t dst_elem, const void* d_src, void* d_dst,
                         void* stream) {
  return guarded([&] {
    if (!ctx) fail(LFGPU_EINVAL, "null context");
    CUDA_OK(cudaSetDevice(ctx->device));
    CopySpec spec;
    spec.lmap = identity_map(dims_of(rank, logical));
    spec.src_seq = seq_of(nsrc, src_seq);
    spec.dst_seq = seq_of(ndst, dst_seq);
    spec.mode = FoldMode::Clamp;
    std::vector<std::unique_ptr<DevBuf>> keep;
    bool oob;
    CopyKernel k = compile_copy(spec, src_elem, dst_elem, keep, &oob);
    auto s = static_cast<cudaStream_t>(stream);
    CUDA_OK(run_copy(k, d_src, d_dst, ctx->d_err, s));
    ctx->launches += 1;
    if (!keep.empty()) CUDA_OK(cudaStreamSynchronize(s));  // program buffers die here
  });
}

int lfgpu_materialize_host(lfgpu_ctx* ctx, int32_t rank, const lfgpu_dim* logical,
                           int32_t nprims, const lfgpu_prim* seq, int32_t elem,
                           const double* host_logical, double* host_physical) {
  return guarded([&] {
    if (!ctx) fail(LFGPU_EINVAL, "null context");
    CUDA_OK(cudaSetDevice(ctx->device));
    auto dims = dims_of(rank, logical);
    Seq s = seq_of(nprims, seq);
    const int64_t nl = numel(dims), np = numel(derive(dims, s));
    DevBuf in(sizeof(double) * std::max<int64_t>(nl, 1)), mid(elem_size(elem) * std::max<int64_t>(nl, 1)),
        phys(elem_size(elem) * std::max<int64_t>(np, 1)), out(sizeof(double) * std::max<int64_t>(np, 1));
    CUDA_OK(cudaMemcpy(in.p, host_logical, sizeof(double) * nl, cudaMemcpyHostToDevice));
    std::vector<std::unique_ptr<DevBuf>> keep;
    bool oob;
    CopySpec id;
    id.lmap = identity_map(dims);
    CopySpec mat = id;
    mat.dst_seq = s;
    mat.mode = FoldMode::Clamp;
    // logical f64 -> logical elem (the tensor's storage type) -> physical elem -> f64
    CUDA_OK(run_copy(compile_copy(id, LFGPU_ELEM_F64, elem, keep, &oob), in.p, mid.p, ctx->d_err, 0));
    CUDA_OK(run_copy(compile_copy(mat, elem, elem, keep, &oob), mid.p, phys.p, ctx->d_err, 0));
    CopySpec back;
    back.lmap = identity_map(derive(dims, s));
    CUDA_OK(run_copy(compile_copy(back, elem, LFGPU_ELEM_F64, keep, &oob), phys.p, out.p, ctx->d_err, 0));
    CUDA_OK(cudaMemcpy(host_physical, out.p, sizeof(double) * np, cudaMemcpyDeviceToHost));
    ctx->launches += 3;
  });
}

int lfgpu_pad_convert(lfgpu_ctx* ctx, const lfgpu_dim* in_logical, int64_t pad, int32_t nsrc,
                      const lfgpu_prim* src_seq, int32_t ndst, const lfgpu_prim* dst_seq,
                      int32_t src_elem, int32_t dst_elem, const void* d_src, void* d_dst,
                      void* stream) {
  return guarded([&] {
    if (!ctx) fail(LFGPU_EINVAL, "null context");
    CUDA_OK(cudaSetDevice(ctx->device));
    CopySpec spec;
    spec.lmap = padding_map(dims_of(4, in_logical), pad);
    spec.src_seq = seq_of(nsrc, src_seq);
    spec.dst_seq = seq_of(ndst, dst_seq);
    spec.mode = FoldMode::Nest;
    std::vector<std::unique_ptr<DevBuf>> keep;
    bool oob;
    CopyKernel k = compile_copy(spec, src_elem, dst_elem, keep, &oob);
    if (oob) fail(LFGPU_ERANGE, "out-of-range access: padding reads outside its input");
    auto s = static_cast<cudaStream_t>(stream);
    CUDA_OK(run_copy(k, d_src, d_dst, ctx->d_err, s));
    ctx->launches += 1;
    if (!keep.empty()) CUDA_OK(cudaStreamSynchronize(s));
  });
}

int lfgpu_plan_build(lfgpu_ctx* ctx, const lfgpu_graph* g, int32_t nsched,
                     const lfgpu_sched* sched, int32_t flags, lfgpu_plan** out) {
  *out = nullptr;
  auto* P = new lfgpu_plan;
  int rc = guarded([&] {
    if (!ctx) fail(LFGPU_EINVAL, "null context");
    CUDA_OK(cudaSetDevice(ctx->device));
    P->ctx = ctx;
    P->flags = flags;
    CUDA_OK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
    build_plan(P, g, nsched, sched);
  });
  if (rc != LFGPU_OK) {
    delete P;
    return rc;
  }
  *out = P;
  return LFGPU_OK;
}

int lfgpu_plan_destroy(lfgpu_plan* plan) {
  if (plan) {
    cudaSetDevice(plan->ctx->device);
    cudaStreamSynchronize(plan->stream);
    delete plan;
  }
  return LFGPU_OK;
}

// Staging bytes per tensor: n doubles, or (narrowed staging) n floats plus
// n bf16 at a 256-byte aligned offset — never more than 8n + 256.
static size_t stage_bytes(int64_t n) { return sizeof(double) * std::max<int64_t>(n, 1) + 256; }
static size_t stage_bf16_offset(int64_t n) { return (sizeof(float) * std::max<int64_t>(n, 1) + 255) & ~size_t(255); }

static void host_stage_alloc(PTensor& t, int64_t n) {
  if (t.d_f64) {
    // the previous call's DMA / conversion out of the staging buffers
    if (t.staged) CUDA_OK(cudaEventSynchronize(t.staged));
    return;
  }
  CUDA_OK(cudaEventCreateWithFlags(&t.staged, cudaEventDisableTiming));
  t.d_f64 = dev_alloc(stage_bytes(n));
  if (!t.d_f64) fail(LFGPU_ECUDA, "device allocation of the f64 staging buffer");
  CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&t.h_pin), stage_bytes(n), cudaHostAllocDefault));
}

// Host restatements of the device conversions the K1 copy applies to f64
// sources (k_copy.cu Elem<float>::from_d = cvt.rn.f32.f64, Elem<bf16>::from_d
// = cvt.rn.bf16.f32 of that float): round to nearest even, subnormals kept,
// any NaN -> the canonical bf16 NaN 0x7fff. Narrowing on the host moves 4 or
// 2 bytes per element over the link instead of 8 with bit-identical values.
static inline uint16_t host_bf16_rn(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  if ((x & 0x7fffffffu) > 0x7f800000u) return 0x7fffu;
  x += 0x7fffu + ((x >> 16) & 1u);
  return static_cast<uint16_t>(x >> 16);
}

// A small pool of host worker threads for the host-buffer entry points:
// one core copies ~15 GB/s on the GPU box (tools/host_link_probe.py), the
// pinned H2D link ~25 GB/s and D2H ~54 GB/s, so staging copies are split
// over workers and overlapped with the DMA chunk by chunk.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p(std::max(2u, std::min(16u, std::thread::hardware_concurrency())));
    return p;
  }
  int size() const { return static_cast<int>(w_.size()); }
  // Run fn(i) for i in [0, n) on the workers; returns when all are done.
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> one_caller(call_);  // plans on several host threads share the pool
    std::unique_lock<std::mutex> lk(m_);
    fn_ = &fn;
    next_ = 0;
    total_ = n;
    left_ = n;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [&] { return left_ == 0; });
    fn_ = nullptr;
  }

 private:
  explicit HostPool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) w_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : w_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < total_); });
      if (stop_) return;
      while (next_ < total_) {
        const int i = next_++;
        const auto* fn = fn_;
        lk.unlock();
        (*fn)(i);
        lk.lock();
        if (--left_ == 0) done_.notify_all();
      }
      seen = gen_;
    }
  }
  std::vector<std::thread> w_;
  std::mutex call_, m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int next_ = 0, total_ = 0, left_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// memcpy of `bytes` split over the pool's workers
static void host_copy_bytes(void* dst, const void* src, size_t bytes) {
  HostPool& pool = HostPool::get();
  const int nt = bytes >= (size_t(1) << 20) ? pool.size() : 1;
  if (nt == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes / nt + 63) & ~size_t(63);
  pool.run(nt, [&](int i) {
    const size_t a = std::min(bytes, per * i), b = std::min(bytes, per * (i + 1));
    if (a < b) std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  });
}

constexpr size_t kStageChunk = size_t(2) << 20;  // bytes per overlapped staging chunk

// user host -> pinned staging -> device, chunk by chunk: chunk i+1's host
// copy overlaps chunk i's DMA (stream-ordered on `st`, not synchronised).
static void stage_h2d(void* d_dst, void* h_pin, const void* src, size_t bytes, cudaStream_t st) {
  for (size_t off = 0; off < bytes; off += kStageChunk) {
    const size_t len = std::min(kStageChunk, bytes - off);
    host_copy_bytes(static_cast<char*>(h_pin) + off, static_cast<const char*>(src) + off, len);
    CUDA_OK(cudaMemcpyAsync(static_cast<char*>(d_dst) + off, static_cast<char*>(h_pin) + off, len,
                            cudaMemcpyHostToDevice, st));
  }
}

// device -> pinned staging -> user host, chunk by chunk: chunk i's host copy
// overlaps chunk i+1's DMA. Returns after the last chunk has been copied.
static void stage_d2h(void* dst, void* h_pin, const void* d_src, size_t bytes, cudaStream_t st,
                      std::vector<cudaEvent_t>& ev) {
  const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
  while (ev.size() < nch) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
  }
  for (size_t c = 0; c < nch; ++c) {
    const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
    CUDA_OK(cudaMemcpyAsync(static_cast<char*>(h_pin) + off, static_cast<const char*>(d_src) + off, len,
                            cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaEventRecord(ev[c], st));
  }
  for (size_t c = 0; c < nch; ++c) {
    const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
    CUDA_OK(cudaEventSynchronize(ev[c]));
    host_copy_bytes(static_cast<char*>(dst) + off, static_cast<char*>(h_pin) + off, len);
  }
}

// user doubles -> (host threads: narrow to f32 and / or bf16) -> pinned ->
// device staging, chunk by chunk: chunk i+1's conversion overlaps chunk i's DMA.
static void stage_h2d_narrow(PTensor& t, const double* src, int64_t n, bool want_f32, bool want_bf16,
                             cudaStream_t st) {
  float* hf = reinterpret_cast<float*>(t.h_pin);
  uint16_t* hb = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(t.h_pin) + stage_bf16_offset(n));
  char* df = static_cast<char*>(t.d_f64);
  char* db = df + stage_bf16_offset(n);
  HostPool& pool = HostPool::get();
  // each worker narrows one contiguous slice and enqueues its slice's DMA at
  // once, so early slices travel while later ones are still converted
  const int nt = n >= 65536 ? pool.size() : 1;
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  auto work = [&](int i) {
    CUDA_OK(cudaSetDevice(dev));  // pool threads: the plan's device
    const int64_t per = ((n + nt - 1) / nt + 127) & ~int64_t(127);
    const int64_t a = std::min(n, per * i), b = std::min(n, per * (i + 1));
    if (a >= b) return;
    for (int64_t e = a; e < b; ++e) {
      const float f = static_cast<float>(src[e]);
      if (want_f32) hf[e] = f;
      if (want_bf16) hb[e] = host_bf16_rn(f);
    }
    if (want_f32) CUDA_OK(cudaMemcpyAsync(df + 4 * a, hf + a, 4 * (b - a), cudaMemcpyHostToDevice, st));
    if (want_bf16) CUDA_OK(cudaMemcpyAsync(db + 2 * a, hb + a, 2 * (b - a), cudaMemcpyHostToDevice, st));
  };
  if (nt == 1) work(0);
  else pool.run(nt, work);
}

// device f32 staging -> pinned -> user doubles (float -> double is exact),
// chunk i's widening overlapping chunk i+1's DMA.
static void stage_d2h_widen(double* dst, const PTensor& t, int64_t n, cudaStream_t st, std::vector<cudaEvent_t>& ev) {
  HostPool& pool = HostPool::get();
  const int nt = n >= 65536 ? pool.size() : 1;
  const int64_t per = ((n + nt - 1) / nt + 127) & ~int64_t(127);
  while (static_cast<int>(ev.size()) < nt) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
  }
  float* hf = reinterpret_cast<float*>(t.h_pin);
  const float* df = static_cast<const float*>(t.d_f64);
  for (int i = 0; i < nt; ++i) {  // one DMA + event per worker slice
    const int64_t a = std::min(n, per * i), b = std::min(n, per * (i + 1));
    if (a < b) CUDA_OK(cudaMemcpyAsync(hf + a, df + a, 4 * (b - a), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaEventRecord(ev[i], st));
  }
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  auto work = [&](int i) {  // slice i widens as soon as its DMA landed
    CUDA_OK(cudaSetDevice(dev));
    const int64_t a = std::min(n, per * i), b = std::min(n, per * (i + 1));
    CUDA_OK(cudaEventSynchronize(ev[i]));
    for (int64_t e = a; e < b; ++e) dst[e] = hf[e];
  };
  if (nt == 1) work(0);
  else pool.run(nt, work);
}

// The K1 conversion from a logical source of element type `se` into tensor
// t's physical storage of element type `de`, compiled once per pair.
static const CopyKernel& in_copy_kernel(lfgpu_plan* P, PTensor& t, int se, int de) {
  const int key = se * 8 + de;
  auto it = t.in_copy.find(key);
  if (it == t.in_copy.end()) {
    CopySpec spec;
    spec.lmap = identity_map(t.logical);
    spec.dst_seq = t.seq;  // materialize_tensor (interp.cpp:280-337)
    spec.mode = FoldMode::Clamp;
    bool oob;
    it = t.in_copy.emplace(key, compile_copy(spec, se, de, P->keep, &oob)).first;
  }
  return it->second;
}

static void set_input_impl(lfgpu_plan* P, int32_t tensor, const void* d_logical, int32_t elem) {
  if (tensor < 0 || tensor >= static_cast<int32_t>(P->t.size()))
    fail(LFGPU_EINVAL, "tensor index out of range");
  PTensor& t = P->t[tensor];
  // The plan's stream is non-blocking: order the read of `d_logical` after
  // the work already enqueued on the legacy default stream (where a caller
  // such as torch's default stream produced it).
  if (!P->ev_dev_in) CUDA_OK(cudaEventCreateWithFlags(&P->ev_dev_in, cudaEventDisableTiming));
  CUDA_OK(cudaEventRecord(P->ev_dev_in, cudaStreamLegacy));
  CUDA_OK(cudaStreamWaitEvent(P->stream, P->ev_dev_in, 0));
  // Compiled once per (source, destination) element pair and kept with the
  // plan, so a repeated call is only the K1 launch(es), stream-ordered on the
  // plan's stream with no host synchronisation (the serving / e2e path).
  if (t.d) CUDA_OK(run_copy(in_copy_kernel(P, t, elem, t.elem), d_logical, t.d, P->ctx->d_err, P->stream));
  if (t.d_bf16)
    CUDA_OK(run_copy(in_copy_kernel(P, t, elem, LFGPU_ELEM_BF16), d_logical, t.d_bf16, P->ctx->d_err, P->stream));
}

int lfgpu_plan_set_input(lfgpu_plan* plan, int32_t tensor, const double* host_logical, int64_t n) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(plan->ctx->device));
    const PTensor& t = plan->t.at(tensor);
    if (n != numel(t.logical))
      fail(LFGPU_EINVAL, "input '" + t.id + "' has " + std::to_string(n) + " values, expected " +
                             std::to_string(numel(t.logical)));
    PTensor& tt = plan->t[tensor];
    host_stage_alloc(tt, n);
    // user doubles -> pinned staging (host threads) -> device staging (DMA)
    // -> K1 into the plan's physical layout(s); synchronous like the
    // reference's by-value BufferMap.
    const bool f32 = tt.d && tt.elem == LFGPU_ELEM_F32, bf = tt.d_bf16 != nullptr;
    if ((f32 || !tt.d) && !getenv("LFGPU_STAGE_F64")) {
      // float storage: narrowed on the host exactly as the device would
      stage_h2d_narrow(tt, host_logical, n, f32, bf, plan->stream);
      int* d_err = plan->ctx->d_err;
      if (f32)
        CUDA_OK(run_copy(in_copy_kernel(plan, tt, LFGPU_ELEM_F32, LFGPU_ELEM_F32), tt.d_f64, tt.d, d_err,
                         plan->stream));
      if (bf)
        CUDA_OK(run_copy(in_copy_kernel(plan, tt, LFGPU_ELEM_BF16, LFGPU_ELEM_BF16),
                         static_cast<char*>(tt.d_f64) + stage_bf16_offset(n), tt.d_bf16, d_err, plan->stream));
      // The user's buffer has been read in full; the DMA and K1 stay
      // stream-ordered before the next run / get_output (staging reuse
      // waits on `staged`).
      CUDA_OK(cudaEventRecord(tt.staged, plan->stream));
    } else {
      stage_h2d(tt.d_f64, tt.h_pin, host_logical, sizeof(double) * n, plan->stream);
      set_input_impl(plan, tensor, tt.d_f64, LFGPU_ELEM_F64);
      CUDA_OK(cudaStreamSynchronize(plan->stream));
    }
  });
}

int lfgpu_plan_set_input_device(lfgpu_plan* plan, int32_t tensor, const void* d_logical,
                                int32_t elem) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(plan->ctx->device));
    set_input_impl(plan, tensor, d_logical, elem);
    CUDA_OK(cudaStreamSynchronize(plan->stream));
  });
}

int lfgpu_plan_set_input_device_async(lfgpu_plan* plan, int32_t tensor, const void* d_logical,
                                      int32_t elem) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(plan->ctx->device));
    set_input_impl(plan, tensor, d_logical, elem);
  });
}

int lfgpu_plan_run(lfgpu_plan* plan) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(plan->ctx->device));
    plan_run_steps(plan);
  });
}

int lfgpu_plan_run_on(lfgpu_plan* plan, void* stream) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(plan->ctx->device));
    cudaStream_t us = static_cast<cudaStream_t>(stream);
    if (!us || us == plan->stream) {
      plan_run_steps(plan, plan->stream);
      return;
    }
    if (!plan->ev_in) {
      CUDA_OK(cudaEventCreateWithFlags(&plan->ev_in, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&plan->ev_out, cudaEventDisableTiming));
    }
    CUDA_OK(cudaEventRecord(plan->ev_in, plan->stream));
    CUDA_OK(cudaStreamWaitEvent(us, plan->ev_in, 0));
    plan_run_steps(plan, us);
    CUDA_OK(cudaEventRecord(plan->ev_out, us));
    CUDA_OK(cudaStreamWaitEvent(plan->stream, plan->ev_out, 0));
  });
}

int lfgpu_plan_get_output(lfgpu_plan* plan, int32_t tensor, double* host_logical, int64_t n) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(plan->ctx->device));
    PTensor& t = plan->t.at(tensor);
    if (n != numel(t.logical)) fail(LFGPU_EINVAL, "output size mismatch for '" + t.id + "'");
    if (!t.valid)
      fail(LFGPU_EUNSUPPORTED, "'" + t.id + "' was fused away (epilogue or attention core) and not materialized");
    // float storage comes back as f32 (exact for f32 and bf16) and is
    // widened on the host; int32 as f64
    const int se = t.d ? t.elem : LFGPU_ELEM_BF16;
    const bool narrow = se != LFGPU_ELEM_I32 && !getenv("LFGPU_STAGE_F64");
    if (!t.out_copy_ready) {
      CopySpec spec;
      spec.lmap = identity_map(t.logical);
      spec.src_seq = t.seq;  // forward map back to logical (interp.cpp:441-468)
      spec.mode = FoldMode::Clamp;
      bool oob;
      t.out_copy = compile_copy(spec, se, narrow ? LFGPU_ELEM_F32 : LFGPU_ELEM_F64, plan->keep, &oob);
      t.out_copy_ready = true;
    }
    host_stage_alloc(t, n);
    if (!plan->h_err) {
      CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&plan->h_err), sizeof(int), cudaHostAllocDefault));
      *plan->h_err = 0;
    }
    const void* src = t.d ? t.d : t.d_bf16;
    CUDA_OK(run_copy(t.out_copy, src, t.d_f64, plan->ctx->d_err, plan->stream));
    int* h = plan->h_err;  // the out-of-range flag of this execution, read with the data
    CUDA_OK(cudaMemcpyAsync(h, plan->ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, plan->stream));
    if (narrow) stage_d2h_widen(host_logical, t, n, plan->stream, plan->stage_ev);
    else stage_d2h(host_logical, t.h_pin, t.d_f64, sizeof(double) * n, plan->stream, plan->stage_ev);
    if (*h) {
      CUDA_OK(cudaMemsetAsync(plan->ctx->d_err, 0, sizeof(int), plan->stream));
      CUDA_OK(cudaStreamSynchronize(plan->stream));
      fail(LFGPU_ERANGE, "out-of-range access during execution");
    }
  });
}

int lfgpu_plan_tensor_buffer(lfgpu_plan* plan, int32_t tensor, void** d_ptr, int32_t* elem,
                             int64_t* n) {
  return guarded([&] {
    const PTensor& t = plan->t.at(tensor);
    *d_ptr = t.d ? t.d : t.d_bf16;
    *elem = t.d ? t.elem : LFGPU_ELEM_BF16;
    *n = t.numel;
  });
}

int lfgpu_plan_stream(lfgpu_plan* plan, void** stream) {
  *stream = plan->stream;
  return LFGPU_OK;
}

int lfgpu_plan_info(lfgpu_plan* plan, lfgpu_counters* info) {
  std::memset(info, 0, sizeof(*info));
  info->kernels = 0;
  for (const auto& st : plan->steps) info->kernels += st.launches;
  info->bytes_moved = plan->bytes;
  info->flops = plan->flops;
  info->tc_nodes = plan->tc_nodes;
  return LFGPU_OK;
}

int lfgpu_plan_node_kernel(lfgpu_plan* plan, int32_t node, char* buf, int32_t cap) {
  return guarded([&] {
    std::string s = plan->node_kernel.at(node);
    auto it = plan->summary.find(node);
    if (it != plan->summary.end()) s += " [" + it->second + "]";
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  });
}

int lfgpu_plan_measure(lfgpu_plan* plan, int32_t warmup, int32_t reps, int32_t flush_l2,
                       lfgpu_counters* out) {
  return guarded([&] {
    lfgpu_ctx* ctx = plan->ctx;
    CUDA_OK(cudaSetDevice(ctx->device));
    if (flush_l2 && !ctx->flush) {
      ctx->flush_bytes = size_t(192) << 20;  // 1.5x the 126 MB L2, read once per execution
      CUDA_OK(cudaMalloc(&ctx->flush, ctx->flush_bytes));
      CUDA_OK(cudaMemsetAsync(ctx->flush, 0, ctx->flush_bytes, plan->stream));
    }
    auto touch = [&] {
      CUDA_OK(launch_l2_touch(ctx->flush, ctx->flush_bytes, static_cast<int*>(ctx->flush), plan->stream));
    };
    for (int i = 0; i < warmup; ++i) plan_run_steps(plan);
    reps = std::max(reps, 1);
    cudaEvent_t e[4];
    for (auto& x : e) CUDA_OK(cudaEventCreate(&x));
    auto span = [&](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, a, b));
      return ms * 1000.0;
    };
    // K: executions per event pair, from a 4-execution estimate (warm)
    CUDA_OK(cudaEventRecord(e[0], plan->stream));
    for (int i = 0; i < 4; ++i) plan_run_steps(plan);
    CUDA_OK(cudaEventRecord(e[1], plan->stream));
    CUDA_OK(cudaStreamSynchronize(plan->stream));
    const double est = std::max(0.5, span(e[0], e[1]) / 4.0);
    int K = static_cast<int>(std::lround(100.0 / est));
    K = std::max(flush_l2 ? 2 : 4, std::min(flush_l2 ? 4 : 64, K));
    std::vector<double> us;
    for (int r = 0; r < reps; ++r) {
      CUDA_OK(cudaEventRecord(e[0], plan->stream));
      for (int k = 0; k < K; ++k) {
        if (flush_l2) touch();
        plan_run_steps(plan);
      }
      CUDA_OK(cudaEventRecord(e[1], plan->stream));
      if (flush_l2) {
        CUDA_OK(cudaEventRecord(e[2], plan->stream));
        for (int k = 0; k < K; ++k) touch();
        CUDA_OK(cudaEventRecord(e[3], plan->stream));
      }
      CUDA_OK(cudaStreamSynchronize(plan->stream));
      double t = span(e[0], e[1]);
      if (flush_l2) t -= span(e[2], e[3]);
      us.push_back(t / K);
    }
    for (auto& x : e) cudaEventDestroy(x);
    check_device_error(plan);
    std::sort(us.begin(), us.end());
    lfgpu_plan_info(plan, out);
    out->cost = us[us.size() / 2];
    out->min_us = us.front();
    out->runs_per_sample = K;
    out->resolution_us = 1.024 / K;
  });
}

int lfgpu_random_inputs(const lfgpu_graph* g, uint64_t seed, double* const* bufs) {
  // lf::random_inputs (interp.cpp:487-503) with the same standard-library
  // engine and distributions, so the values are the reference's bit for bit:
  // one mt19937_64 stream over the Input/Constant tensors in declaration
  // order; floats U(-1, 1) rounded to k/64, int32 U{-4..4}.
  return guarded([&] {
    std::mt19937_64 rng(seed);
    for (int t = 0; t < g->ntensors; ++t) {
      const lfgpu_tensor& td = g->tensors[t];
      if (td.role != LFGPU_ROLE_INPUT && td.role != LFGPU_ROLE_CONSTANT) continue;
      if (!bufs[t]) fail(LFGPU_EINVAL, std::string("missing buffer for tensor '") + td.id + "'");
      int64_t n = 1;
      for (int d = 0; d < td.rank; ++d) n *= td.dims[d].extent;
      double* b = bufs[t];
      if (td.dtype == LFGPU_DTYPE_I32) {
        std::uniform_int_distribution<int> dist(-4, 4);
        for (int64_t i = 0; i < n; ++i) b[i] = dist(rng);
      } else {
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        for (int64_t i = 0; i < n; ++i) b[i] = std::round(dist(rng) * 64.0) / 64.0;
      }
    }
  });
}

int lfgpu_interpret(lfgpu_ctx* ctx, const lfgpu_graph* g, int32_t nsched,
                    const lfgpu_sched* sched, int32_t flags, double* const* host_bufs) {
  lfgpu_plan* P = nullptr;
  // Reference semantics unless the caller opts into tensor cores.
  if (!(flags & (LFGPU_PLAN_TENSOR_CORES | LFGPU_PLAN_REQUIRE_TC | LFGPU_PLAN_TC_SPLIT))) flags |= LFGPU_PLAN_EXACT;
  int rc = lfgpu_plan_build(ctx, g, nsched, sched, (flags & ~LFGPU_PLAN_TENSOR_CORES) | LFGPU_PLAN_KEEP_ALL, &P);
  if (rc != LFGPU_OK) return rc;
  rc = guarded([&] {
    for (int i = 0; i < g->ntensors; ++i) {
      int role = g->tensors[i].role;
      if (role != LFGPU_ROLE_INPUT && role != LFGPU_ROLE_CONSTANT) continue;
      if (!host_bufs[i]) fail(LFGPU_EINVAL, std::string("missing input buffer for tensor '") +
                                                g->tensors[i].id + "'");
      int r = lfgpu_plan_set_input(P, i, host_bufs[i], numel(P->t[i].logical));
      if (r) fail(r, g_last_error);
    }
    int r = lfgpu_plan_run(P);
    if (r) fail(r, g_last_error);
    for (const auto& n : P->nodes) {
      if (!host_bufs[n.output]) continue;
      r = lfgpu_plan_get_output(P, n.output, host_bufs[n.output], numel(P->t[n.output].logical));
      if (r) fail(r, g_last_error);
    }
  });
  lfgpu_plan_destroy(P);
  return rc;
}

}  // extern "C"

namespace lfg {
void umma_set_chain_buffer(void* p);
}
// Diagnostics: per-launch [entry, wait, first data, exit] timestamps of the
// tcgen05 kernels of a plan (8 uint64 per plan step; the caller
// initialises the min slots to ~0 and the max slots to 0).
extern "C" int lfgpu_debug_chain_trace(void* d_buf) {
  lfg::umma_set_chain_buffer(d_buf);
  return LFGPU_OK;
}

extern "C" int lfgpu_debug_umma_trace(void* d_buf) {
  lfg::umma_set_debug_buffer(d_buf);
  return LFGPU_OK;
}
