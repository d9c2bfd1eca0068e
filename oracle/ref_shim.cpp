// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library (layoutforge,
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/). Used to pin oracle/lf_oracle.c, to generate the golden
// vectors under tests/golden/, and as the "reference" CPU baseline in
// bench.py. The product never links this.
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../include/lfgpu.h"
#include "layoutforge/cachesim.hpp"
#include "layoutforge/interp.hpp"
#include "layoutforge/lower.hpp"
#include "layoutforge/propagation.hpp"
#include "layoutforge/space.hpp"

namespace {

thread_local std::string g_err;

lf::LayoutPrimitive to_prim(const lfgpu_prim& p, const lf::Graph* g) {
  lf::LayoutPrimitive q;
  q.kind = static_cast<lf::PrimKind>(p.kind);
  q.dim = p.dim;
  q.span = p.span;
  for (int i = 0; i < p.nfactors; ++i) q.factors.push_back(p.factors[i]);
  for (int i = 0; i < p.nperm; ++i) q.perm.push_back(p.perm[i]);
  q.tile = p.tile;
  q.stride = p.stride;
  q.pad = p.pad;
  q.orig_extent = p.orig_extent;
  if (p.target >= 0 && g) q.target = g->tensors[p.target].id;
  return q;
}

void from_prim(const lf::LayoutPrimitive& q, const lf::Graph* g, lfgpu_prim* p) {
  std::memset(p, 0, sizeof(*p));
  p->kind = static_cast<int32_t>(q.kind);
  p->dim = q.dim;
  p->span = q.span;
  p->nfactors = static_cast<int32_t>(q.factors.size());
  for (size_t i = 0; i < q.factors.size(); ++i) p->factors[i] = q.factors[i];
  p->nperm = static_cast<int32_t>(q.perm.size());
  for (size_t i = 0; i < q.perm.size(); ++i) p->perm[i] = q.perm[i];
  p->tile = q.tile;
  p->stride = q.stride;
  p->pad = q.pad;
  p->orig_extent = q.orig_extent;
  p->target = (g && !q.target.empty()) ? g->tensor_index(q.target) : -1;
}

std::vector<lf::Dim> to_dims(int rank, const lfgpu_dim* d) {
  std::vector<lf::Dim> out;
  for (int i = 0; i < rank; ++i) out.push_back({d[i].name, d[i].extent});
  return out;
}

lf::Graph to_graph(const lfgpu_graph* gg) {
  lf::Graph g;
  for (int t = 0; t < gg->ntensors; ++t) {
    const lfgpu_tensor& td = gg->tensors[t];
    lf::TensorDecl d;
    d.id = td.id;
    d.dims = to_dims(td.rank, td.dims);
    d.dtype = static_cast<lf::DType>(td.dtype);
    d.role = static_cast<lf::Role>(td.role);
    g.tensors.push_back(d);
  }
  for (int i = 0; i < gg->nnodes; ++i) {
    const lfgpu_node& nd = gg->nodes[i];
    lf::OperatorNode n;
    n.kind = static_cast<lf::OpKind>(nd.kind);
    for (int j = 0; j < nd.ninputs; ++j) n.inputs.push_back(g.tensors[nd.inputs[j]].id);
    n.output = g.tensors[nd.output].id;
    if (nd.kind == LFGPU_OP_C2D || nd.kind == LFGPU_OP_DEP) n.attrs["stride"] = nd.stride;
    if (nd.kind == LFGPU_OP_PADDING) n.attrs["pad"] = nd.pad;
    g.nodes.push_back(n);
  }
  return g;
}

lf::SeqMap to_seqs(const lfgpu_graph* gg, const lf::Graph& g) {
  lf::SeqMap m;
  for (int s = 0; s < gg->nseqs; ++s) {
    const lfgpu_seq& sq = gg->seqs[s];
    std::vector<lf::LayoutPrimitive> v;
    for (int k = 0; k < sq.nprims; ++k) v.push_back(to_prim(sq.prims[k], &g));
    m[g.tensors[sq.tensor].id] = v;
  }
  return m;
}

// lfgpu_sched -> loop-schedule primitives through the reference's own loop
// space (space.cpp:483-589): parameter values are matched to indices.
std::vector<lf::LoopSchedule> to_scheds(const lf::Graph& g, const lf::SeqMap& seqs, int n,
                                        const lfgpu_sched* s) {
  std::vector<lf::LoopSchedule> out;
  if (n == 0) return out;
  lf::PassResult pass = lf::rewrite_accesses_pass(g, seqs);
  int counter = 0;
  for (int i = 0; i < n; ++i) {
    int node = s[i].node;
    lf::LoopNest nest = lf::build_loop_nest(g, pass, node, &counter);
    auto consumers = g.consumers_of(g.nodes[node].output);
    bool has_ew = consumers.size() == 1 && lf::is_elementwise_op(g.nodes[consumers[0]].kind);
    lf::LoopSpace space = lf::build_loop_space(g, nest, has_ew);
    lf::LoopPoint pt(space.params.size(), 0);
    for (size_t k = 0; k < space.params.size(); ++k) {
      const auto& p = space.params[k];
      int64_t want = 0;
      if (k == 0 && p.name.rfind("tile_", 0) == 0) want = s[i].tile_last;
      else if (k == 1 && p.name.rfind("tile_", 0) == 0) want = s[i].tile_second;
      else if (p.name == "order") want = s[i].order;
      else if (p.name == "vectorize") want = s[i].vectorize;
      else if (p.name == "parallel") want = s[i].parallel;
      else if (p.name == "unroll") want = s[i].unroll;
      else if (p.name == "fuse") want = s[i].fuse;
      for (size_t v = 0; v < p.values.size(); ++v)
        if (p.values[v] == want) pt[k] = static_cast<int>(v);
    }
    lf::LoopSchedule ls;
    ls.node = node;
    ls.prims = lf::decode_loop_point(space, pt);
    out.push_back(ls);
  }
  return out;
}

lf::BufferMap to_buffers(const lf::Graph& g, double* const* bufs) {
  lf::BufferMap m;
  for (size_t t = 0; t < g.tensors.size(); ++t) {
    const auto& td = g.tensors[t];
    if (td.role != lf::Role::Input && td.role != lf::Role::Constant) continue;
    m[td.id] = std::vector<double>(bufs[t], bufs[t] + td.num_elements());
  }
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// lf::random_inputs (interp.cpp:487-503).
int ref_random_inputs(const lfgpu_graph* gg, uint64_t seed, double** out) {
  try {
    lf::Graph g = to_graph(gg);
    lf::BufferMap m = lf::random_inputs(g, seed);
    for (size_t t = 0; t < g.tensors.size(); ++t) {
      auto it = m.find(g.tensors[t].id);
      if (it == m.end()) continue;
      std::memcpy(out[t], it->second.data(), it->second.size() * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// lf::reference_eval (interp.cpp:50-176).
int ref_reference_eval(const lfgpu_graph* gg, double** bufs) {
  try {
    lf::Graph g = to_graph(gg);
    lf::BufferMap out = lf::reference_eval(g, to_buffers(g, bufs));
    for (size_t t = 0; t < g.tensors.size(); ++t) {
      auto it = out.find(g.tensors[t].id);
      if (it == out.end()) continue;
      std::memcpy(bufs[t], it->second.data(), it->second.size() * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// lf::derive_layout (layout.cpp:311-322).
int ref_derive_layout(int rank, const lfgpu_dim* dims, int nprims, const lfgpu_prim* prims,
                      int* out_rank, lfgpu_dim* out) {
  try {
    std::vector<lf::LayoutPrimitive> seq;
    for (int i = 0; i < nprims; ++i) seq.push_back(to_prim(prims[i], nullptr));
    auto d = lf::derive_layout(to_dims(rank, dims), seq);
    *out_rank = static_cast<int>(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
      std::memset(out[i].name, 0, sizeof(out[i].name));
      std::strncpy(out[i].name, d[i].name.c_str(), sizeof(out[i].name) - 1);
      out[i].extent = d[i].extent;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// lf::materialize_tensor (interp.cpp:280-337) for one stand-alone input tensor.
int ref_materialize(int rank, const lfgpu_dim* dims, int nprims, const lfgpu_prim* prims,
                    const double* src, double* dst) {
  try {
    lf::Program p;
    lf::ProgTensor t;
    t.id = "t";
    t.orig_dims = to_dims(rank, dims);
    for (int i = 0; i < nprims; ++i) t.seq.push_back(to_prim(prims[i], nullptr));
    t.dims = lf::derive_layout(t.orig_dims, t.seq);
    t.role = lf::Role::Input;
    p.tensors.push_back(t);
    lf::BufferMap raw{{"t", std::vector<double>(src, src + lf::TensorDecl{"t", t.orig_dims}.num_elements())}};
    auto buf = lf::materialize_tensor(p, 0, raw);
    std::memcpy(dst, buf.data(), buf.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// lf::interpret(lf::lower(g, seqs, scheds), inputs) (interp.cpp:424-470).
// Returns 2 on lf::Error (the CLI's "invalid" exit code, cli.cpp:67-92).
int ref_interpret(const lfgpu_graph* gg, int nsched, const lfgpu_sched* sched, double** bufs) {
  try {
    lf::Graph g = to_graph(gg);
    lf::SeqMap seqs = to_seqs(gg, g);
    auto scheds = to_scheds(g, seqs, nsched, sched);
    lf::Program prog = lf::lower(g, seqs, scheds);
    lf::InterpResult r = lf::interpret(prog, to_buffers(g, bufs));
    for (size_t t = 0; t < g.tensors.size(); ++t) {
      auto it = r.outputs.find(g.tensors[t].id);
      if (it == r.outputs.end()) continue;
      std::memcpy(bufs[t], it->second.data(), it->second.size() * sizeof(double));
    }
    return 0;
  } catch (const lf::Error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// lf::simulate_cache (cachesim.cpp:152-174) with the default CacheConfig:
// the reference's measurement backend, timed as the tuner CPU baseline.
int ref_simulate_cache(const lfgpu_graph* gg, int nsched, const lfgpu_sched* sched,
                       double* cost, int64_t* misses) {
  try {
    lf::Graph g = to_graph(gg);
    lf::SeqMap seqs = to_seqs(gg, g);
    auto scheds = to_scheds(g, seqs, nsched, sched);
    lf::Program prog = lf::lower(g, seqs, scheds);
    lf::ProfileCounters c = lf::simulate_cache(prog, lf::CacheConfig{});
    *cost = c.cost;
    *misses = c.l1_misses;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// lf::decode_layout (space.cpp:174-417) on build_layout_space's template.
int ref_decode_layout(const lfgpu_graph* gg, int node, int tiling_levels,
                      const int64_t* factors, int nfactors, lfgpu_seq* out, int cap, int* nout,
                      lfgpu_prim* storage, int prim_cap) {
  try {
    lf::Graph g = to_graph(gg);
    auto templates = lf::build_layout_space(g, tiling_levels);
    auto it = templates.find(node);
    if (it == templates.end()) throw lf::Error("node has no layout template");
    std::vector<int64_t> f(factors, factors + nfactors);
    lf::SeqMap m = lf::decode_layout(g, it->second, f);
    int k = 0, used = 0;
    for (const auto& [id, seq] : m) {
      if (k >= cap || used + static_cast<int>(seq.size()) > prim_cap)
        throw lf::Error("output capacity");
      out[k].tensor = g.tensor_index(id);
      out[k].nprims = static_cast<int32_t>(seq.size());
      out[k].prims = storage + used;
      for (const auto& p : seq) from_prim(p, &g, &storage[used++]);
      ++k;
    }
    *nout = k;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// Template shape of build_layout_space (space.cpp:49-104): tunable count,
// extents and divisor counts for node `node`.
int ref_layout_template(const lfgpu_graph* gg, int node, int tiling_levels, int* ntun,
                        int64_t* extents, int64_t* ndivisors) {
  try {
    lf::Graph g = to_graph(gg);
    auto templates = lf::build_layout_space(g, tiling_levels);
    auto it = templates.find(node);
    if (it == templates.end()) throw lf::Error("node has no layout template");
    *ntun = static_cast<int>(it->second.tunables.size());
    for (size_t i = 0; i < it->second.tunables.size(); ++i) {
      extents[i] = it->second.tunables[i].extent;
      ndivisors[i] = static_cast<int64_t>(it->second.tunables[i].divisors.size());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// The tuner's context build (tuner.cpp:108-121): every complex node claims
// its decoded template layout in topological order (propagation.cpp:232-251),
// then insert_conversions splices LayoutConvert nodes (propagation.cpp:265-313).
// Output graph/seq storage is caller-provided; returns the new graph shape.
int ref_plan_context(const lfgpu_graph* gg, int tiling_levels, const int64_t* factors,
                     lfgpu_tensor* out_tensors, int tensor_cap, lfgpu_node* out_nodes,
                     int node_cap, lfgpu_seq* out_seqs, int seq_cap, lfgpu_prim* storage,
                     int prim_cap, int* ntensors, int* nnodes, int* nseqs) {
  try {
    lf::Graph g = to_graph(gg);
    auto templates = lf::build_layout_space(g, tiling_levels);
    lf::LayoutPlanner planner(g);
    int off = 0;
    for (int op : lf::topo_order(g)) {
      auto it = templates.find(op);
      if (it == templates.end()) continue;
      std::vector<int64_t> f(factors + off, factors + off + it->second.tunables.size());
      off += static_cast<int>(it->second.tunables.size());
      planner.claim_operator(op, lf::decode_layout(g, it->second, f));
    }
    lf::PropagationPlan plan = planner.take_plan();
    lf::ConversionResult conv = lf::insert_conversions(g, &plan);
    lf::Graph g2 = lf::infer_shapes(conv.graph);
    if (static_cast<int>(g2.tensors.size()) > tensor_cap ||
        static_cast<int>(g2.nodes.size()) > node_cap)
      throw lf::Error("output capacity");
    for (size_t t = 0; t < g2.tensors.size(); ++t) {
      lfgpu_tensor& td = out_tensors[t];
      std::memset(&td, 0, sizeof(td));
      std::strncpy(td.id, g2.tensors[t].id.c_str(), sizeof(td.id) - 1);
      td.rank = static_cast<int32_t>(g2.tensors[t].dims.size());
      td.dtype = static_cast<int32_t>(g2.tensors[t].dtype);
      td.role = static_cast<int32_t>(g2.tensors[t].role);
      for (size_t d = 0; d < g2.tensors[t].dims.size(); ++d) {
        std::strncpy(td.dims[d].name, g2.tensors[t].dims[d].name.c_str(),
                     sizeof(td.dims[d].name) - 1);
        td.dims[d].extent = g2.tensors[t].dims[d].extent;
      }
    }
    for (size_t i = 0; i < g2.nodes.size(); ++i) {
      lfgpu_node& nd = out_nodes[i];
      std::memset(&nd, 0, sizeof(nd));
      nd.kind = static_cast<int32_t>(g2.nodes[i].kind);
      nd.ninputs = static_cast<int32_t>(g2.nodes[i].inputs.size());
      for (size_t j = 0; j < g2.nodes[i].inputs.size(); ++j)
        nd.inputs[j] = g2.tensor_index(g2.nodes[i].inputs[j]);
      nd.output = g2.tensor_index(g2.nodes[i].output);
      nd.stride = g2.nodes[i].attr("stride", 1);
      nd.pad = g2.nodes[i].attr("pad", 0);
    }
    int k = 0, used = 0;
    for (const auto& [id, seq] : plan.assignments) {
      if (seq.empty()) continue;
      if (k >= seq_cap || used + static_cast<int>(seq.size()) > prim_cap)
        throw lf::Error("output capacity");
      out_seqs[k].tensor = g2.tensor_index(id);
      out_seqs[k].nprims = static_cast<int32_t>(seq.size());
      out_seqs[k].prims = storage + used;
      for (const auto& p : seq) from_prim(p, &g2, &storage[used++]);
      ++k;
    }
    *ntensors = static_cast<int>(g2.tensors.size());
    *nnodes = static_cast<int>(g2.nodes.size());
    *nseqs = k;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"
