// lf_space.cpp — the layout tuning templates of complex operators and the
// decoding of a factor point into primitive sequences: the candidate
// layouts the GPU kernels consume.
//
// Restates lf::build_layout_space (proj/src/space.cpp:49-104),
// lf::identity_factors (space.cpp:106-111) and lf::decode_layout
// (space.cpp:174-417). Tensor roles: C2D/DEP output NOHW -> N (H/h)(W/w)
// (O/o) [level-2 blocks] h w o; input NIHW -> overlapped tiles
// N (H/h)(W/w)(I/i) B_h B_w i with B = (h-1)V + KH, S = hV; C2D weight
// OIKhKw -> (O/o')(I/i') KH KW i' o'; DEP weight CKhKw -> (C/c') KH KW c';
// GMM operands -> two-level bricks.
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "lf_core.hpp"

namespace lfg {

struct Tunable {
  std::string label;
  int tensor;  // tensor index the factor tiles
  int64_t extent;
};

struct Template {
  int node = -1;
  int kind = 0;
  int levels = 1;
  std::vector<Tunable> t;
};

namespace {

std::vector<int64_t> ext_of(const lfgpu_tensor& t) {
  std::vector<int64_t> e;
  for (int i = 0; i < t.rank; ++i) e.push_back(t.dims[i].extent);
  return e;
}

}  // namespace

Template layout_template(const lfgpu_graph* g, int node, int levels) {
  const lfgpu_node& n = g->nodes[node];
  Template T;
  T.node = node;
  T.kind = n.kind;
  T.levels = levels;
  auto out = ext_of(g->tensors[n.output]);
  auto add = [&](const char* label, int tensor, int64_t extent) {
    T.t.push_back({label, tensor, extent});
  };
  switch (n.kind) {
    case LFGPU_OP_C2D: {
      auto in = ext_of(g->tensors[n.inputs[0]]);
      auto ker = ext_of(g->tensors[n.inputs[1]]);
      add("h_t", n.output, out[2]);
      add("w_t", n.output, out[3]);
      add("o_t", n.output, out[1]);
      add("i_t", n.inputs[0], in[1]);
      add("i_t2", n.inputs[1], ker[1]);
      add("o_t2", n.inputs[1], ker[0]);
      break;
    }
    case LFGPU_OP_DEP: {
      auto in = ext_of(g->tensors[n.inputs[0]]);
      auto ker = ext_of(g->tensors[n.inputs[1]]);
      add("h_t", n.output, out[2]);
      add("w_t", n.output, out[3]);
      add("o_t", n.output, out[1]);
      add("i_t", n.inputs[0], in[1]);
      add("c_t2", n.inputs[1], ker[0]);
      break;
    }
    case LFGPU_OP_GMM: {
      auto a = ext_of(g->tensors[n.inputs[0]]);
      add("m_t", n.output, out[0]);
      add("k_t", n.inputs[0], a[1]);
      add("n_t", n.output, out[1]);
      break;
    }
    default:
      fail(LFGPU_EINVAL, "node has no layout template (not C2D/DEP/GMM)");
  }
  if (levels == 2 && n.kind != LFGPU_OP_GMM) {
    add("h_l2", n.output, out[2]);
    add("w_l2", n.output, out[3]);
    add("o_l2", n.output, out[1]);
  }
  return T;
}

namespace {

int64_t factor(const Template& T, const std::vector<int64_t>& f, const std::string& label,
               int64_t fallback) {
  for (size_t i = 0; i < T.t.size(); ++i)
    if (T.t[i].label == label) return f[i];
  return fallback;
}

// A dim split into parts; `level` -1 marks an untouched dim.
struct Part {
  char which;
  int level;
};

int index_of(const std::vector<Part>& parts, char c, int lvl) {
  for (size_t k = 0; k < parts.size(); ++k)
    if (parts[k].which == c && parts[k].level == lvl) return static_cast<int>(k);
  return -1;
}

void push_parts(std::vector<Part>* parts, char c, bool tiled, bool l2) {
  if (!tiled) {
    parts->push_back({c, -1});
    return;
  }
  parts->push_back({c, 0});
  parts->push_back({c, 1});
  if (l2) parts->push_back({c, 2});
}

void finish_reorder(Seq* seq, const std::vector<int>& perm) {
  for (size_t k = 0; k < perm.size(); ++k)
    if (perm[k] != static_cast<int>(k)) {
      seq->push_back(make_reorder(perm));
      return;
    }
}

Seq two_level(const std::vector<int64_t>& e, int64_t t0, int64_t t1) {
  Seq seq;
  bool s0 = t0 < e[0], s1 = t1 < e[1];
  if (s1) seq.push_back(make_split(1, {e[1] / t1, t1}));
  if (s0) seq.push_back(make_split(0, {e[0] / t0, t0}));
  if (s0 && s1) seq.push_back(make_reorder({0, 2, 1, 3}));
  else if (s0) seq.push_back(make_reorder({0, 2, 1}));
  return seq;
}

}  // namespace

std::map<int, Seq> decode_layout(const lfgpu_graph* g, const Template& T,
                                 const std::vector<int64_t>& f) {
  if (f.size() != T.t.size())
    fail(LFGPU_EINVAL, "decode_layout: expected " + std::to_string(T.t.size()) + " factors");
  for (size_t i = 0; i < f.size(); ++i)
    if (f[i] < 1 || T.t[i].extent % f[i] != 0)
      fail(LFGPU_EINVAL, "decode_layout: factor " + std::to_string(f[i]) + " does not divide " +
                             T.t[i].label + " extent " + std::to_string(T.t[i].extent));
  const lfgpu_node& n = g->nodes[T.node];
  std::map<int, Seq> out;
  if (T.kind == LFGPU_OP_GMM) {
    auto c = ext_of(g->tensors[n.output]);
    auto a = ext_of(g->tensors[n.inputs[0]]);
    auto b = ext_of(g->tensors[n.inputs[1]]);
    int64_t m_t = factor(T, f, "m_t", c[0]), k_t = factor(T, f, "k_t", a[1]),
            n_t = factor(T, f, "n_t", c[1]);
    Seq sc = two_level(c, m_t, n_t), sa = two_level(a, m_t, k_t), sb = two_level(b, k_t, n_t);
    if (!sc.empty()) out[n.output] = sc;
    if (!sa.empty()) out[n.inputs[0]] = sa;
    if (!sb.empty()) out[n.inputs[1]] = sb;
    return out;
  }
  const bool c2d = T.kind == LFGPU_OP_C2D;
  auto yo = ext_of(g->tensors[n.output]);
  auto xi = ext_of(g->tensors[n.inputs[0]]);
  auto kr = ext_of(g->tensors[n.inputs[1]]);
  const int64_t V = n.stride;
  const int64_t kh = c2d ? kr[2] : kr[1], kw = c2d ? kr[3] : kr[2];
  const int64_t h_t = factor(T, f, "h_t", yo[2]), w_t = factor(T, f, "w_t", yo[3]),
                o_t = factor(T, f, "o_t", yo[1]);
  const int64_t h_l2 = factor(T, f, "h_l2", 1), w_l2 = factor(T, f, "w_l2", 1),
                o_l2 = factor(T, f, "o_l2", 1);

  // Output.
  {
    bool th = h_t < yo[2], tw = w_t < yo[3], to = o_t < yo[1];
    bool l2h = T.levels == 2 && th && h_l2 > 1 && h_t % h_l2 == 0 && h_l2 < h_t;
    bool l2w = T.levels == 2 && tw && w_l2 > 1 && w_t % w_l2 == 0 && w_l2 < w_t;
    bool l2o = T.levels == 2 && to && o_l2 > 1 && o_t % o_l2 == 0 && o_l2 < o_t;
    auto fac = [](int64_t D, int64_t t, int64_t l2, bool use) {
      return use ? std::vector<int64_t>{D / t, t / l2, l2} : std::vector<int64_t>{D / t, t};
    };
    Seq seq;
    if (tw) seq.push_back(make_split(3, fac(yo[3], w_t, w_l2, l2w)));
    if (th) seq.push_back(make_split(2, fac(yo[2], h_t, h_l2, l2h)));
    if (to) seq.push_back(make_split(1, fac(yo[1], o_t, o_l2, l2o)));
    if (!seq.empty()) {
      std::vector<Part> parts{{'n', -1}};
      push_parts(&parts, 'o', to, l2o);
      push_parts(&parts, 'h', th, l2h);
      push_parts(&parts, 'w', tw, l2w);
      std::vector<int> perm{index_of(parts, 'n', -1)};
      auto put = [&](char c, int lvl) {
        int k = index_of(parts, c, lvl);
        if (k >= 0) perm.push_back(k);
      };
      put('h', th ? 0 : -1);
      put('w', tw ? 0 : -1);
      put('o', to ? 0 : -1);
      if (l2h) put('h', 1);
      if (l2w) put('w', 1);
      if (l2o) put('o', 1);
      if (th) put('h', l2h ? 2 : 1);
      if (tw) put('w', l2w ? 2 : 1);
      if (to) put('o', l2o ? 2 : 1);
      finish_reorder(&seq, perm);
      out[n.output] = seq;
    }
  }
  // Input: overlapped tiles.
  {
    bool uh = h_t < yo[2], uw = w_t < yo[3];
    int64_t i_t = factor(T, f, "i_t", xi[1]);
    bool ti = i_t < xi[1];
    Seq seq;
    if (uw) seq.push_back(make_unfold(3, (w_t - 1) * V + kw, w_t * V));
    if (uh) seq.push_back(make_unfold(2, (h_t - 1) * V + kh, h_t * V));
    if (ti) seq.push_back(make_split(1, {xi[1] / i_t, i_t}));
    if (!seq.empty()) {
      std::vector<Part> parts{{'n', -1}};
      push_parts(&parts, 'i', ti, false);
      push_parts(&parts, 'h', uh, false);
      push_parts(&parts, 'w', uw, false);
      std::vector<int> perm{index_of(parts, 'n', -1)};
      auto put = [&](char c, int lvl) {
        int k = index_of(parts, c, lvl);
        if (k >= 0) perm.push_back(k);
      };
      put('h', uh ? 0 : -1);
      put('w', uw ? 0 : -1);
      put('i', ti ? 0 : -1);
      if (uh) put('h', 1);
      if (uw) put('w', 1);
      if (ti) put('i', 1);
      finish_reorder(&seq, perm);
      out[n.inputs[0]] = seq;
    }
  }
  // Weight.
  if (c2d) {
    int64_t i2 = factor(T, f, "i_t2", kr[1]), o2 = factor(T, f, "o_t2", kr[0]);
    bool ti = i2 < kr[1], to = o2 < kr[0];
    Seq seq;
    if (ti) seq.push_back(make_split(1, {kr[1] / i2, i2}));
    if (to) seq.push_back(make_split(0, {kr[0] / o2, o2}));
    if (!seq.empty()) {
      std::vector<Part> parts;
      push_parts(&parts, 'o', to, false);
      push_parts(&parts, 'i', ti, false);
      parts.push_back({'h', -1});
      parts.push_back({'w', -1});
      std::vector<int> perm;
      auto put = [&](char c, int lvl) {
        int k = index_of(parts, c, lvl);
        if (k >= 0) perm.push_back(k);
      };
      put('o', to ? 0 : -1);
      put('i', ti ? 0 : -1);
      put('h', -1);
      put('w', -1);
      if (ti) put('i', 1);
      if (to) put('o', 1);
      finish_reorder(&seq, perm);
      out[n.inputs[1]] = seq;
    }
  } else {
    int64_t c2 = factor(T, f, "c_t2", kr[0]);
    if (c2 < kr[0]) out[n.inputs[1]] = {make_split(0, {kr[0] / c2, c2}), make_reorder({0, 2, 3, 1})};
  }
  return out;
}

}  // namespace lfg

using namespace lfg;

extern "C" int lfgpu_decode_layout(const lfgpu_graph* g, int32_t node, int32_t tiling_levels,
                                   const int64_t* factors, int32_t nfactors, lfgpu_seq* out_seqs,
                                   int32_t cap, int32_t* nout, lfgpu_prim* prim_storage,
                                   int32_t prim_cap);
extern "C" int lfgpu_layout_template(const lfgpu_graph* g, int32_t node, int32_t tiling_levels,
                                     int32_t* ntunables, int64_t* extents, char (*labels)[8],
                                     int32_t cap);

namespace lfg {
int set_error_external(int code, const std::string& msg);
}

int lfgpu_decode_layout(const lfgpu_graph* g, int32_t node, int32_t tiling_levels,
                        const int64_t* factors, int32_t nfactors, lfgpu_seq* out_seqs, int32_t cap,
                        int32_t* nout, lfgpu_prim* prim_storage, int32_t prim_cap) {
  try {
    if (!g || node < 0 || node >= g->nnodes) fail(LFGPU_EINVAL, "node out of range");
    Template T = layout_template(g, node, tiling_levels);
    auto m = decode_layout(g, T, std::vector<int64_t>(factors, factors + nfactors));
    int k = 0, used = 0;
    for (const auto& [tensor, seq] : m) {
      if (k >= cap || used + static_cast<int>(seq.size()) > prim_cap)
        fail(LFGPU_EINVAL, "decode_layout: output capacity");
      out_seqs[k].tensor = tensor;
      out_seqs[k].nprims = static_cast<int32_t>(seq.size());
      out_seqs[k].prims = prim_storage + used;
      for (const auto& p : seq) prim_storage[used++] = p;
      ++k;
    }
    *nout = k;
    return LFGPU_OK;
  } catch (const Error& e) {
    return set_error_external(e.code, e.what());
  }
}

int lfgpu_layout_template(const lfgpu_graph* g, int32_t node, int32_t tiling_levels,
                          int32_t* ntunables, int64_t* extents, char (*labels)[8], int32_t cap) {
  try {
    if (!g || node < 0 || node >= g->nnodes) fail(LFGPU_EINVAL, "node out of range");
    Template T = layout_template(g, node, tiling_levels);
    if (static_cast<int>(T.t.size()) > cap) fail(LFGPU_EINVAL, "layout_template: capacity");
    *ntunables = static_cast<int32_t>(T.t.size());
    for (size_t i = 0; i < T.t.size(); ++i) {
      extents[i] = T.t[i].extent;
      std::memset(labels[i], 0, 8);
      std::strncpy(labels[i], T.t[i].label.c_str(), 7);
    }
    return LFGPU_OK;
  } catch (const Error& e) {
    return set_error_external(e.code, e.what());
  }
}
