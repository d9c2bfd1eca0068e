// tune_check.cpp — TEST INFRASTRUCTURE: the reference's own two-stage tuner
// (proj/src/tuner.cpp, lf::tune) driven by the GPU measure backend through
// the one-line seam INTEGRATION.md shows (tuner.cpp:178, generated into
// oracle/_ref/tune/tuner_gpu.cpp by `make -C oracle tune`).
//
//   tune_check host                 hook unset: the hooked tuner equals the
//                                   unmodified one (simulate_cache) on a
//                                   small GMM graph (same best cost)
//   tune_check gpu <cfg> <budget> <mode> [parallel]
//                                   cfg: cfg1 (Padding -> C2D 64->64 3x3
//                                   56x56, N=1) | cfg2 (GMM 1024^3);
//                                   mode: tc (LFGPU_PLAN_REQUIRE_TC: points
//                                   the tensor-core kernels cannot take are
//                                   counted as rejected and scored with a
//                                   penalty) | any (the adapter's default:
//                                   tcgen05 where the layout allows it,
//                                   CUDA cores otherwise; never rejects);
//                                   parallel: TuneOptions::parallel_eval.
// Prints one JSON line: measurements, rejected, tensor-core plans, best cost
// (us), wall seconds and candidates/s. Built by tests/test_adapter.py.
#include <chrono>
#include <map>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "layoutforge/cachesim.hpp"
#include "layoutforge/tuner.hpp"
#include "lf_gpu.hpp"

using namespace lf;

lf::ProfileCounters (*lf_gpu_measure_hook)(const lf::Graph&, const lf::SeqMap&,
                                           const std::vector<lf::LoopSchedule>&) = nullptr;
void (*lf_gpu_batch_hook)(const lf::Graph&, const lf::SeqMap&,
                          const std::vector<std::vector<lf::LoopSchedule>>&) = nullptr;

namespace {

gpu::Context* g_ctx = nullptr;
int g_flags = LFGPU_PLAN_CUDA_GRAPH;
int g_calls = 0, g_rejected = 0, g_tc = 0;
constexpr double kPenaltyUs = 1e6;  // a rejected point's score (mode tc)

// measure_top's prefetched top-k (lf::gpu::measure_batch over every
// context), keyed by the candidate's schedules; the per-candidate seam
// consumes them in the tuner's own order, so commits stay index-ordered.
std::vector<gpu::Context*> g_ctxs;
std::map<std::string, gpu::BatchOutcome> g_prefetched;
int g_batched = 0, g_batch_calls = 0, g_prefetch_used = 0;
double g_measure_s = 0.0;  // wall time inside the GPU backend (build + measure)

struct MeasureClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~MeasureClock() { g_measure_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

std::string sched_key(const std::vector<LoopSchedule>& sc) {
  std::string k;
  for (const auto& s : sc) {
    k += "n" + std::to_string(s.node) + ":";
    for (const auto& p : s.prims) {
      k += std::to_string(static_cast<int>(p.kind)) + "," + p.var + "," + std::to_string(p.factor) + "," +
           std::to_string(static_cast<int>(p.ann));
      for (const auto& o : p.order) k += "," + o;
      k += ";";
    }
  }
  return k;
}

void batch_hook(const Graph& g, const SeqMap& seqs, const std::vector<std::vector<LoopSchedule>>& b) {
  // Only points the reference's lowering accepts reach the seam
  // (Tuner::evaluate, tuner.cpp:168-174): filter the same way first.
  std::vector<std::vector<LoopSchedule>> todo;
  for (const auto& sc : b) {
    try {
      (void)lower(g, seqs, sc);
    } catch (const Error&) {
      continue;
    }
    if (!g_prefetched.count(sched_key(sc))) todo.push_back(sc);
  }
  ++g_batch_calls;
  g_batched += static_cast<int>(todo.size());
  MeasureClock clk;
  auto out = gpu::measure_batch(g_ctxs, g, seqs, todo, 1, 3, true, g_flags);
  for (size_t i = 0; i < todo.size(); ++i) g_prefetched[sched_key(todo[i])] = out[i];
}

ProfileCounters gpu_hook(const Graph& g, const SeqMap& seqs, const std::vector<LoopSchedule>& sc) {
  ++g_calls;
  auto it = g_prefetched.find(sched_key(sc));
  if (it != g_prefetched.end()) {
    gpu::BatchOutcome o = it->second;
    g_prefetched.erase(it);
    ++g_prefetch_used;
    if (o.ok) {
      if (o.counters.l1_stores > 0) ++g_tc;
      return o.counters;
    }
    ++g_rejected;
    ProfileCounters p;
    p.cost = kPenaltyUs;
    return p;
  }
  try {
    MeasureClock clk;
    ProfileCounters p = gpu::measure(*g_ctx, g, seqs, sc, 1, 3, true, g_flags);
    if (p.l1_stores > 0) ++g_tc;  // l1_stores = nodes executed on tcgen05
    return p;
  } catch (const Error&) {
    ++g_rejected;
    ProfileCounters p;
    p.cost = kPenaltyUs;
    return p;
  }
}

TensorDecl T(const std::string& id, std::vector<Dim> d, Role r) {
  TensorDecl t;
  t.id = id;
  t.dims = std::move(d);
  t.role = r;
  return t;
}

OperatorNode N(OpKind k, std::vector<std::string> in, std::string out, std::map<std::string, int64_t> a = {}) {
  OperatorNode n;
  n.kind = k;
  n.inputs = std::move(in);
  n.output = std::move(out);
  n.attrs = std::move(a);
  return n;
}

Graph cfg1() {  // BASELINE configs[0]: Padding -> C2D 64->64 3x3 s1, 56x56, N=1
  Graph g;
  g.tensors = {T("x", {{"N", 1}, {"I", 64}, {"H", 56}, {"W", 56}}, Role::Input),
               T("ker", {{"O", 64}, {"I", 64}, {"KH", 3}, {"KW", 3}}, Role::Constant),
               T("xp", {{"N", 1}, {"I", 64}, {"H", 58}, {"W", 58}}, Role::Intermediate),
               T("y", {{"N", 1}, {"O", 64}, {"H", 56}, {"W", 56}}, Role::Output)};
  g.nodes = {N(OpKind::Padding, {"x"}, "xp", {{"pad", 1}}), N(OpKind::C2D, {"xp", "ker"}, "y", {{"stride", 1}})};
  return g;
}

Graph gmm(int64_t m, int64_t k, int64_t n) {  // BASELINE configs[1] at 1024^3
  Graph g;
  g.tensors = {T("a", {{"M", m}, {"K", k}}, Role::Input), T("b", {{"K", k}, {"N", n}}, Role::Constant),
               T("c", {{"M", m}, {"N", n}}, Role::Output)};
  g.nodes = {N(OpKind::GMM, {"a", "b"}, "c")};
  return g;
}

Budget budget(int total) {
  Budget b;
  b.total = total;
  b.joint = total * 3 / 8;
  b.loop_only = total - b.joint;
  b.batch = 32;
  b.top_k = 8;
  b.seed = 42;
  return b;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  if (mode == "host") {
    // With the hook unset the generated tuner is the reference's: same
    // result twice (determinism, test_tuner.cpp:296-300) and a finite cost.
    Graph g = gmm(64, 64, 64);
    CacheConfig cc;
    TuneResult r1 = tune(g, budget(16), cc), r2 = tune(g, budget(16), cc);
    const bool ok = std::isfinite(r1.best_cost) && r1.best_cost == r2.best_cost && r1.sim_calls == r2.sim_calls &&
                    r1.sim_calls > 0;
    std::printf("host: %s best_cost=%.3f sims=%d\n", ok ? "OK" : "FAIL", r1.best_cost, r1.sim_calls);
    return ok ? 0 : 1;
  }
  const std::string cfg = argc > 2 ? argv[2] : "cfg2";
  const int total = argc > 3 ? std::atoi(argv[3]) : 64;
  const std::string m = argc > 4 ? argv[4] : "any";
  // the reference's own parallel lowering + feature extraction (std::async,
  // tuner.cpp:196-221)
  const bool par = argc > 5 && std::string(argv[5]) == "parallel";
  g_flags = LFGPU_PLAN_CUDA_GRAPH | (m == "tc" ? LFGPU_PLAN_REQUIRE_TC : 0);
  // batch N: measure_top's top-k measured by lf::gpu::measure_batch over N
  // contexts (devices 0..N-1 round-robin over the visible GPUs).
  const bool batch = argc > 6 && std::string(argv[6]) == "batch";
  const int nctx = argc > 7 ? std::max(1, std::atoi(argv[7])) : 1;
  int ndev = 1;
  lfgpu_device_count(&ndev);
  std::vector<std::unique_ptr<gpu::Context>> pool;
  for (int i = 0; i < (batch ? nctx : 1); ++i) pool.push_back(std::make_unique<gpu::Context>(i % std::max(1, ndev)));
  for (auto& c : pool) g_ctxs.push_back(c.get());
  g_ctx = pool[0].get();
  lf_gpu_measure_hook = gpu_hook;
  if (batch) lf_gpu_batch_hook = batch_hook;
  Graph g = cfg == "cfg1" ? cfg1() : gmm(1024, 1024, 1024);
  auto t0 = std::chrono::steady_clock::now();
  TuneOptions opts;
  opts.parallel_eval = par;
  TuneResult r = tune(g, budget(total), CacheConfig{}, opts);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf(
      "{\"cfg\": \"%s\", \"mode\": \"%s\", \"parallel_eval\": %d, \"budget\": %d, \"measurements\": %d, \"rejected\": %d, "
      "\"tensor_core_plans\": %d, \"rejected_frac\": %.4f, \"best_cost_us\": %.3f, \"seconds\": %.2f, "
      "\"candidates_per_s\": %.2f, \"contexts\": %d, \"batch_calls\": %d, \"batched\": %d, \"prefetch_used\": %d, \"gpu_backend_s\": %.3f}\n",
      cfg.c_str(), m.c_str(), par ? 1 : 0, total, g_calls, g_rejected, g_tc, g_calls ? double(g_rejected) / g_calls : 0.0,
      r.best_cost, secs, secs > 0 ? g_calls / secs : 0.0, static_cast<int>(g_ctxs.size()), g_batch_calls, g_batched,
      g_prefetch_used, g_measure_s);
  return (g_calls > 0 && std::isfinite(r.best_cost)) ? 0 : 1;
}
