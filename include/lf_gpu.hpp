// lf_gpu.hpp — header-only drop-in adapter from the reference's C++ API
// (layoutforge, proj/include/layoutforge) to the B200 backend's C-ABI
// (include/lfgpu.h).
//
// A layoutforge maintainer compiles this header inside the reference build
// and links liblfgpu.so. It converts the reference's own types (lf::Graph,
// lf::SeqMap, lf::LoopSchedule, lf::BufferMap) to the POD descriptors and
// rethrows every non-OK status as lf::Error, so callers keep the
// reference's error contract (proj/include/layoutforge/ir.hpp:17-19;
// tuner.cpp:169-174 rejects candidates that throw). See INTEGRATION.md.
//
//   lf::gpu::interpret(...)   replaces lf::interpret(lower(...), inputs)  interp.cpp:424-470
//   lf::gpu::materialize(...) replaces lf::materialize_tensor           interp.cpp:280-337
//   lf::gpu::measure(...)     replaces lf::simulate_cache at tuner.cpp:178 cachesim.cpp:152-174
//   lf::gpu::measure_batch(...) the top-k of Tuner::measure_top (tuner.cpp:243-274)
//                             over several devices, results in candidate order
#pragma once

#include <algorithm>
#include <atomic>
#include <cctype>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "layoutforge/cachesim.hpp"
#include "layoutforge/interp.hpp"
#include "layoutforge/lower.hpp"
#include "lfgpu.h"

namespace lf::gpu {

inline void check(int rc) {
  if (rc != LFGPU_OK) throw lf::Error(std::string("lfgpu: ") + lfgpu_last_error());
}

/// One device context (one host thread at a time).
class Context {
 public:
  explicit Context(int device = 0) : device_(device) { check(lfgpu_ctx_create(device, &ctx_)); }
  ~Context() { lfgpu_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lfgpu_ctx* get() const { return ctx_; }
  int device() const { return device_; }

 private:
  int device_ = 0;
  lfgpu_ctx* ctx_ = nullptr;
};

inline lfgpu_prim to_c(const LayoutPrimitive& p, const Graph* g) {
  lfgpu_prim c;
  std::memset(&c, 0, sizeof(c));
  c.kind = static_cast<int32_t>(p.kind);  // same enumerator order (layout.hpp:19-29)
  c.dim = p.dim;
  c.span = p.span;
  c.nfactors = static_cast<int32_t>(p.factors.size());
  for (size_t i = 0; i < p.factors.size() && i < LFGPU_MAX_RANK; ++i) c.factors[i] = p.factors[i];
  c.nperm = static_cast<int32_t>(p.perm.size());
  for (size_t i = 0; i < p.perm.size() && i < LFGPU_MAX_RANK; ++i) c.perm[i] = p.perm[i];
  c.tile = p.tile;
  c.stride = p.stride;
  c.pad = p.pad;
  c.orig_extent = p.orig_extent;
  c.target = (g && !p.target.empty()) ? g->tensor_index(p.target) : -1;
  return c;
}

inline std::vector<lfgpu_dim> to_c(const std::vector<Dim>& dims) {
  std::vector<lfgpu_dim> out(dims.size());
  for (size_t i = 0; i < dims.size(); ++i) {
    std::memset(out[i].name, 0, LFGPU_NAME_LEN);
    std::strncpy(out[i].name, dims[i].name.c_str(), LFGPU_NAME_LEN - 1);
    out[i].extent = dims[i].extent;
  }
  return out;
}

/// Owns the POD description of one (Graph, SeqMap).
struct Desc {
  std::vector<lfgpu_tensor> tensors;
  std::vector<lfgpu_node> nodes;
  std::vector<std::vector<lfgpu_prim>> prims;
  std::vector<lfgpu_seq> seqs;
  lfgpu_graph g{};
};

inline Desc describe(const Graph& g, const SeqMap& seqs) {
  Desc d;
  for (const auto& t : g.tensors) {
    lfgpu_tensor c;
    std::memset(&c, 0, sizeof(c));
    std::strncpy(c.id, t.id.c_str(), LFGPU_ID_LEN - 1);
    c.rank = static_cast<int32_t>(t.dims.size());
    c.dtype = static_cast<int32_t>(t.dtype);
    c.role = static_cast<int32_t>(t.role);
    auto dims = to_c(t.dims);
    for (size_t i = 0; i < dims.size() && i < LFGPU_MAX_RANK; ++i) c.dims[i] = dims[i];
    d.tensors.push_back(c);
  }
  for (const auto& n : g.nodes) {
    lfgpu_node c;
    std::memset(&c, 0, sizeof(c));
    c.kind = static_cast<int32_t>(n.kind);  // same order as lf::OpKind (ir.hpp:42)
    c.ninputs = static_cast<int32_t>(n.inputs.size());
    for (size_t j = 0; j < n.inputs.size() && j < 2; ++j) c.inputs[j] = g.tensor_index(n.inputs[j]);
    c.output = g.tensor_index(n.output);
    c.stride = n.attr("stride", 1);
    c.pad = n.attr("pad", 0);
    d.nodes.push_back(c);
  }
  for (const auto& [id, seq] : seqs) {
    if (seq.empty()) continue;
    std::vector<lfgpu_prim> v;
    for (const auto& p : seq) v.push_back(to_c(p, &g));
    d.prims.push_back(std::move(v));
  }
  size_t k = 0;
  for (const auto& [id, seq] : seqs) {
    if (seq.empty()) continue;
    lfgpu_seq s;
    s.tensor = g.tensor_index(id);
    s.nprims = static_cast<int32_t>(d.prims[k].size());
    s.prims = d.prims[k].data();
    d.seqs.push_back(s);
    ++k;
  }
  d.g.ntensors = static_cast<int32_t>(d.tensors.size());
  d.g.nnodes = static_cast<int32_t>(d.nodes.size());
  d.g.nseqs = static_cast<int32_t>(d.seqs.size());
  d.g.tensors = d.tensors.data();
  d.g.nodes = d.nodes.data();
  d.g.seqs = d.seqs.data();
  return d;
}

/// LoopSchedule primitives (as decode_loop_point emits them, space.cpp:509-589)
/// back to the loop-point parameters the GPU kernels are configured by.
inline lfgpu_sched to_sched(const Graph& g, const SeqMap& seqs, const LoopSchedule& s) {
  lfgpu_sched r;
  std::memset(&r, 0, sizeof(r));
  r.node = s.node;
  r.tile_last = r.tile_second = 1;
  // Loop names mirror the transformed output dims (lower.cpp:169-172).
  const auto& out = g.tensor(g.nodes[s.node].output);
  auto it = seqs.find(out.id);
  auto dims = derive_layout(out.dims, it == seqs.end() ? std::vector<LayoutPrimitive>{} : it->second);
  auto lower = [](std::string x) {
    for (auto& ch : x) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return x;
  };
  const std::string last = dims.empty() ? "" : lower(dims.back().name);
  for (const auto& p : s.prims) {
    switch (p.kind) {
      case LoopSchedPrim::Kind::Split:
        (p.var == last ? r.tile_last : r.tile_second) = static_cast<int32_t>(p.factor);
        break;
      case LoopSchedPrim::Kind::Reorder: {
        // order = spatial[:-sink] + reductions + spatial[-sink:]
        static const char* red[] = {"ri", "rh", "rw", "rk"};
        int last_red = -1;
        for (size_t i = 0; i < p.order.size(); ++i)
          for (const char* rn : red)
            if (p.order[i] == rn) last_red = static_cast<int>(i);
        r.order = last_red < 0 ? 0 : static_cast<int32_t>(p.order.size()) - 1 - last_red;
        break;
      }
      case LoopSchedPrim::Kind::Annotate:
        if (p.ann == Annotation::Vectorize) r.vectorize = 1;
        if (p.ann == Annotation::Parallel) r.parallel = 1;
        if (p.ann == Annotation::Unroll) r.unroll = 1;
        break;
      case LoopSchedPrim::Kind::FuseConsumer:
        r.fuse = 1;
        break;
    }
  }
  return r;
}

inline std::vector<lfgpu_sched> to_scheds(const Graph& g, const SeqMap& seqs,
                                          const std::vector<LoopSchedule>& scheds) {
  std::vector<lfgpu_sched> v;
  for (const auto& s : scheds) v.push_back(to_sched(g, seqs, s));
  return v;
}

/// interpret(lower(g, seqs, scheds), inputs) on the GPU; every node output in
/// its logical layout, like InterpResult::outputs (interp.hpp:33-42).
/// Default: reference semantics (LFGPU_PLAN_EXACT, the 1e-5 rule of
/// cli.cpp:30-49 holds on chained graphs). Pass LFGPU_PLAN_TENSOR_CORES to
/// run the tcgen05 kernels (bf16 operands: exact on k/64 inputs, ~2^-9
/// relative per chained contraction otherwise).
inline BufferMap interpret(Context& ctx, const Graph& g, const SeqMap& seqs,
                           const std::vector<LoopSchedule>& scheds, const BufferMap& inputs,
                           int flags = LFGPU_PLAN_EXACT) {
  Desc d = describe(g, seqs);
  auto sc = to_scheds(g, seqs, scheds);
  BufferMap out;
  std::vector<std::vector<double>> bufs(g.tensors.size());
  std::vector<double*> ptrs(g.tensors.size(), nullptr);
  for (size_t i = 0; i < g.tensors.size(); ++i) {
    const auto& t = g.tensors[i];
    if (t.role == Role::Input || t.role == Role::Constant) {
      auto it = inputs.find(t.id);
      if (it == inputs.end()) throw lf::Error("missing input buffer for tensor '" + t.id + "'");
      bufs[i] = it->second;
    } else if (g.producer_of(t.id) >= 0) {
      bufs[i].assign(t.num_elements(), 0.0);
    } else {
      continue;
    }
    ptrs[i] = bufs[i].data();
  }
  check(lfgpu_interpret(ctx.get(), &d.g, static_cast<int32_t>(sc.size()), sc.data(), flags,
                        ptrs.data()));
  for (const auto& n : g.nodes) out[n.output] = bufs[g.tensor_index(n.output)];
  return out;
}

/// materialize_tensor for an Input/Constant tensor with its own sequence.
inline std::vector<double> materialize(Context& ctx, const std::vector<Dim>& logical,
                                       const std::vector<LayoutPrimitive>& seq,
                                       const std::vector<double>& raw,
                                       DType dtype = DType::Float32) {
  auto dims = to_c(logical);
  std::vector<lfgpu_prim> prims;
  for (const auto& p : seq) prims.push_back(to_c(p, nullptr));
  auto phys = derive_layout(logical, seq);
  int64_t n = 1;
  for (const auto& d : phys) n *= d.extent;
  std::vector<double> out(n);
  check(lfgpu_materialize_host(ctx.get(), static_cast<int32_t>(dims.size()), dims.data(),
                               static_cast<int32_t>(prims.size()), prims.data(),
                               dtype == DType::Int32 ? LFGPU_ELEM_I32 : LFGPU_ELEM_F32, raw.data(),
                               out.data()));
  return out;
}

/// The tuner's measurement on the GPU: cost = median device microseconds of
/// the whole lowered graph. Counter fields: insts = kernel launches,
/// l1_loads = algorithmic bytes, l1_misses = 0, l1_stores = tensor-core nodes.
/// Default flags never reject a point the reference's lowering accepted:
/// tcgen05 where the layout allows it, the CUDA-core contraction otherwise
/// (its cost then ranks the point). The seam at tuner.cpp:178 sits outside
/// Tuner::evaluate's try/catch (tuner.cpp:169-174), so a throwing measure
/// would abort lf::tune; pass LFGPU_PLAN_REQUIRE_TC only from callers that
/// catch lf::Error themselves.
inline ProfileCounters measure(Context& ctx, const Graph& g, const SeqMap& seqs,
                               const std::vector<LoopSchedule>& scheds, int warmup = 3,
                               int reps = 10, bool flush_l2 = true,
                               int flags = LFGPU_PLAN_CUDA_GRAPH) {
  Desc d = describe(g, seqs);
  auto sc = to_scheds(g, seqs, scheds);
  lfgpu_plan* plan = nullptr;
  check(lfgpu_plan_build(ctx.get(), &d.g, static_cast<int32_t>(sc.size()), sc.data(), flags,
                         &plan));
  lfgpu_counters c;
  int rc = lfgpu_plan_measure(plan, warmup, reps, flush_l2 ? 1 : 0, &c);
  lfgpu_plan_destroy(plan);
  check(rc);
  ProfileCounters p;
  p.insts = c.kernels;
  p.l1_loads = c.bytes_moved;
  p.l1_misses = 0;
  p.l1_stores = c.tc_nodes;
  p.cost = c.cost;
  return p;
}


/// One measured candidate of a batch: the counters, or the lf::Error text of
/// a candidate the backend rejected; `device` is the context index that
/// measured it.
struct BatchOutcome {
  bool ok = false;
  ProfileCounters counters;
  std::string error;
  int device = -1;
};

/// Tuner::measure_top's top-k (tuner.cpp:243-274) measured across devices:
/// one host thread per context takes the next unmeasured candidate (dynamic
/// dealing, so a slow candidate does not stall a device), and the outcomes
/// come back indexed like `scheds`, so the caller commits them in candidate
/// order exactly as the serial loop would (tuner.cpp:259-272). A candidate
/// the backend rejects (lf::Error other than a device fault) is recorded as
/// not ok. A device fault (LFGPU_ECUDA) retires that context and puts its
/// candidate back on the queue for the others; when every context has
/// faulted, measure_batch throws. Contexts on distinct devices measure
/// concurrently; contexts sharing a device take turns for the timed part
/// (one device mutex), so one context's plan build overlaps the other's
/// measurement without disturbing it.
inline std::vector<BatchOutcome> measure_batch(const std::vector<Context*>& ctxs, const Graph& g,
                                               const SeqMap& seqs,
                                               const std::vector<std::vector<LoopSchedule>>& scheds,
                                               int warmup = 3, int reps = 10, bool flush_l2 = true,
                                               int flags = LFGPU_PLAN_CUDA_GRAPH) {
  if (ctxs.empty()) throw lf::Error("lfgpu: measure_batch needs at least one context");
  std::vector<BatchOutcome> out(scheds.size());
  std::mutex m;
  std::deque<size_t> queue;
  for (size_t i = 0; i < scheds.size(); ++i) queue.push_back(i);
  int alive = static_cast<int>(ctxs.size()), inflight = 0;
  std::condition_variable cv;  // a faulted device may re-queue work for the others
  std::string fault;
  std::vector<int> devs;  // one timing mutex per distinct device
  for (auto* c : ctxs)
    if (std::find(devs.begin(), devs.end(), c->device()) == devs.end()) devs.push_back(c->device());
  std::vector<std::mutex> dev_m(devs.size());
  auto worker = [&](int dev) {
    std::mutex& timing =
        dev_m[std::find(devs.begin(), devs.end(), ctxs[dev]->device()) - devs.begin()];
    for (;;) {
      size_t i;
      {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return !queue.empty() || inflight == 0; });
        if (queue.empty()) return;
        i = queue.front();
        queue.pop_front();
        ++inflight;
      }
      Desc d = describe(g, seqs);
      auto sc = to_scheds(g, seqs, scheds[i]);
      lfgpu_plan* plan = nullptr;
      lfgpu_counters c;
      int rc = lfgpu_plan_build(ctxs[dev]->get(), &d.g, static_cast<int32_t>(sc.size()), sc.data(),
                                flags, &plan);
      if (rc == LFGPU_OK) {
        {
          std::lock_guard<std::mutex> t(timing);
          rc = lfgpu_plan_measure(plan, warmup, reps, flush_l2 ? 1 : 0, &c);
        }
        lfgpu_plan_destroy(plan);
      }
      std::lock_guard<std::mutex> lk(m);
      --inflight;
      cv.notify_all();
      if (rc == LFGPU_ECUDA) {  // device fault: retire this context, re-queue
        fault = lfgpu_last_error();
        queue.push_front(i);
        --alive;
        return;
      }
      BatchOutcome& o = out[i];
      o.device = dev;
      if (rc != LFGPU_OK) {
        o.error = std::string("lfgpu: ") + lfgpu_last_error();
        continue;
      }
      o.ok = true;
      o.counters.insts = c.kernels;
      o.counters.l1_loads = c.bytes_moved;
      o.counters.l1_misses = 0;
      o.counters.l1_stores = c.tc_nodes;
      o.counters.cost = c.cost;
    }
  };
  if (ctxs.size() == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (size_t k = 0; k < ctxs.size(); ++k) th.emplace_back(worker, static_cast<int>(k));
    for (auto& t : th) t.join();
  }
  if (alive == 0 && !queue.empty())
    throw lf::Error("lfgpu: every device faulted during measure_batch: " + fault);
  return out;
}

}  // namespace lf::gpu
