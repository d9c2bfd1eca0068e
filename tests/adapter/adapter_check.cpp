// adapter_check.cpp — TEST INFRASTRUCTURE: the drop-in adapter
// (include/lf_gpu.hpp) exercised from the reference's own C++ API.
//
//   adapter_check host   descriptor / schedule / shape round trips (no GPU)
//   adapter_check gpu    lf::gpu::interpret vs the reference's
//                        lf::interpret(lf::lower(...)) on the same inputs,
//                        plus lf::gpu::materialize vs lf::materialize_tensor
//                        and one lf::gpu::measure call.
// Built by tests/test_adapter.py against /root/reference/proj/include and
// oracle/_ref/libref.so; exits non-zero on any mismatch.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "layoutforge/interp.hpp"
#include "layoutforge/lower.hpp"
#include "layoutforge/propagation.hpp"
#include "layoutforge/space.hpp"
#include "lf_gpu.hpp"

using namespace lf;

static int failures = 0;
#define EXPECT(c, msg)                                  \
  do {                                                  \
    if (!(c)) {                                         \
      std::printf("FAIL: %s (%s:%d)\n", msg, __FILE__, __LINE__); \
      ++failures;                                       \
    }                                                   \
  } while (0)

static TensorDecl T(const std::string& id, std::vector<Dim> d, Role r) {
  TensorDecl t;
  t.id = id;
  t.dims = std::move(d);
  t.role = r;
  return t;
}

static OperatorNode N(OpKind k, std::vector<std::string> in, std::string out,
                      std::map<std::string, int64_t> a = {}) {
  OperatorNode n;
  n.kind = k;
  n.inputs = std::move(in);
  n.output = std::move(out);
  n.attrs = std::move(a);
  return n;
}

// Padding -> C2D -> BiasAdd -> ReLU (proj/tests/graphs.hpp:32-53 shape).
static Graph conv_chain(int64_t n, int64_t ci, int64_t co, int64_t h) {
  Graph g;
  int64_t hp = h + 2, ho = hp - 2;
  g.tensors = {T("x", {{"N", n}, {"I", ci}, {"H", h}, {"W", h}}, Role::Input),
               T("ker", {{"O", co}, {"I", ci}, {"KH", 3}, {"KW", 3}}, Role::Constant),
               T("bias", {{"O", co}}, Role::Constant),
               T("xp", {{"N", n}, {"I", ci}, {"H", hp}, {"W", hp}}, Role::Intermediate),
               T("conv", {{"N", n}, {"O", co}, {"H", ho}, {"W", ho}}, Role::Intermediate),
               T("biased", {{"N", n}, {"O", co}, {"H", ho}, {"W", ho}}, Role::Intermediate),
               T("y", {{"N", n}, {"O", co}, {"H", ho}, {"W", ho}}, Role::Output)};
  g.nodes = {N(OpKind::Padding, {"x"}, "xp", {{"pad", 1}}),
             N(OpKind::C2D, {"xp", "ker"}, "conv", {{"stride", 1}}),
             N(OpKind::BiasAdd, {"conv", "bias"}, "biased"), N(OpKind::ReLU, {"biased"}, "y")};
  return g;
}

// The tuner's context for one layout point (tuner.cpp:108-121).
static void context(const Graph& g, const std::vector<int64_t>& f, Graph* g2, SeqMap* seqs) {
  auto templates = build_layout_space(g, 1);
  LayoutPlanner planner(g);
  planner.claim_operator(1, decode_layout(g, templates.at(1), f));
  PropagationPlan plan = planner.take_plan();
  ConversionResult conv = insert_conversions(g, &plan);
  *g2 = infer_shapes(conv.graph);
  *seqs = plan.assignments;
}

static int host_checks() {
  Graph g = conv_chain(1, 64, 64, 56);
  Graph g2;
  SeqMap seqs;
  context(g, {4, 28, 16, 32, 32, 16}, &g2, &seqs);
  gpu::Desc d = gpu::describe(g2, seqs);
  EXPECT(d.g.ntensors == static_cast<int>(g2.tensors.size()), "tensor count");
  // Physical shapes through the C-ABI equal the reference's derive_layout.
  for (const auto& [id, seq] : seqs) {
    const auto& t = g2.tensor(id);
    auto want = derive_layout(t.dims, seq);
    auto dims = gpu::to_c(t.dims);
    std::vector<lfgpu_prim> prims;
    for (const auto& p : seq) prims.push_back(gpu::to_c(p, &g2));
    int32_t r = 0;
    lfgpu_dim out[LFGPU_MAX_RANK];
    gpu::check(lfgpu_derive_layout(static_cast<int32_t>(dims.size()), dims.data(),
                                   static_cast<int32_t>(prims.size()), prims.data(), &r, out));
    EXPECT(r == static_cast<int>(want.size()), "rank");
    for (int i = 0; i < r; ++i) {
      EXPECT(out[i].extent == want[i].extent, "extent");
      EXPECT(want[i].name == out[i].name, "dim name");
    }
  }
  // Loop points survive decode_loop_point -> to_sched.
  PassResult pass = rewrite_accesses_pass(g2, seqs);
  int counter = 0;
  int conv_node = -1;
  for (size_t i = 0; i < g2.nodes.size(); ++i)
    if (g2.nodes[i].kind == OpKind::C2D) conv_node = static_cast<int>(i);
  LoopNest nest = build_loop_nest(g2, pass, conv_node, &counter);
  LoopSpace space = build_loop_space(g2, nest, true);
  std::mt19937_64 rng(5);
  for (int it = 0; it < 50; ++it) {
    LoopPoint pt = random_loop_point(space, &rng);
    LoopSchedule ls;
    ls.node = conv_node;
    ls.prims = decode_loop_point(space, pt);
    lfgpu_sched s = gpu::to_sched(g2, seqs, ls);
    auto val = [&](const std::string& name) -> int64_t {
      for (size_t i = 0; i < space.params.size(); ++i)
        if (space.params[i].name == name) return space.params[i].values[pt[i]];
      return -1;
    };
    int64_t last = space.params[0].values[pt[0]];
    int64_t second = space.params[1].values[pt[1]];
    int64_t ext_last = space.spatial_extents.back();
    int64_t ext_second = space.spatial_extents[space.spatial_extents.size() - 2];
    EXPECT(s.tile_last == ((last > 1 && last < ext_last) ? last : 1), "tile_last");
    EXPECT(s.tile_second == ((second > 1 && second < ext_second) ? second : 1), "tile_second");
    EXPECT(s.order == val("order"), "order");
    EXPECT(s.parallel == val("parallel"), "parallel");
    EXPECT(s.fuse == val("fuse"), "fuse");
  }
  return failures;
}

static int gpu_checks() {
  gpu::Context ctx(0);
  // 1. interpret parity on small graphs with template layouts (EXACT flags,
  //    test_executor.cpp:413-440 style) and a tensor-core-sized layout.
  struct Case {
    int64_t n, ci, co, h;
    std::vector<int64_t> f;
    int flags;
  };
  std::vector<Case> cases = {{1, 2, 4, 6, {2, 2, 2, 1, 1, 2}, LFGPU_PLAN_EXACT},
                             {1, 3, 6, 8, {4, 2, 3, 1, 3, 2}, LFGPU_PLAN_EXACT},
                             {1, 64, 64, 56, {4, 28, 16, 32, 32, 16}, LFGPU_PLAN_DEFAULT}};
  for (const auto& c : cases) {
    Graph g = conv_chain(c.n, c.ci, c.co, c.h);
    Graph g2;
    SeqMap seqs;
    context(g, c.f, &g2, &seqs);
    BufferMap inputs = random_inputs(g2, 42);
    InterpResult ref = interpret(lower(g2, seqs, {}), inputs);
    BufferMap got = gpu::interpret(ctx, g2, seqs, {}, inputs, c.flags);
    double d = max_rel_diff(ref.outputs, got);
    std::printf("interpret conv_chain(%ld,%ld,%ld,%ld): max_rel_diff %.3g\n", (long)c.n,
                (long)c.ci, (long)c.co, (long)c.h, d);
    EXPECT(d <= 1e-5, "gpu interpret vs reference interpret");
  }
  // 2. materialize parity (interp.cpp:280-337) incl. unfold overhang clamp.
  {
    Program p;
    ProgTensor t;
    t.id = "arr";
    t.orig_dims = {{"N", 1}, {"I", 8}, {"H", 11}, {"W", 9}};
    t.seq = {LayoutPrimitive::unfold(3, 5, 3), LayoutPrimitive::unfold(2, 4, 3),
             LayoutPrimitive::split(1, {2, 4}),
             LayoutPrimitive::reorder({0, 3, 5, 1, 4, 6, 2})};
    t.dims = derive_layout(t.orig_dims, t.seq);
    t.role = Role::Input;
    p.tensors.push_back(t);
    std::vector<double> raw(8 * 11 * 9);
    for (size_t i = 0; i < raw.size(); ++i) raw[i] = static_cast<double>(i % 97) / 64.0;
    auto want = materialize_tensor(p, 0, {{"arr", raw}});
    auto got = gpu::materialize(ctx, t.orig_dims, t.seq, raw);
    EXPECT(want == got, "gpu materialize vs materialize_tensor");
  }
  // 3. the measure hook (tuner.cpp:178 seam) returns a device time.
  {
    Graph g = conv_chain(1, 64, 64, 56);
    Graph g2;
    SeqMap seqs;
    context(g, {4, 28, 16, 32, 32, 16}, &g2, &seqs);
    ProfileCounters c = gpu::measure(ctx, g2, seqs, {});
    std::printf("measure: cost %.3f us, %ld kernels\n", c.cost, (long)c.insts);
    EXPECT(c.cost > 0 && c.insts >= 2, "measure");
  }
  return failures;
}

int main(int argc, char** argv) {
  std::string mode = argc > 1 ? argv[1] : "host";
  try {
    int f = mode == "gpu" ? gpu_checks() : host_checks();
    std::printf("%s: %s\n", mode.c_str(), f ? "FAILED" : "OK");
    return f ? 1 : 0;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 2;
  }
}
