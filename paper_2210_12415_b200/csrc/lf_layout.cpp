// lf_layout.cpp — layout shape algebra and the compiler from primitive
// sequences to device index maps (DigitMap / IxProgram).
//
// Shape rules follow lf::apply_primitive_shape (proj/src/layout.cpp:94-184)
// and lf::invert_sequence (layout.cpp:337-405); value semantics follow
// lf::materialize_step (interp.cpp:181-264) and the loop-nest accesses
// (layout.cpp:186-309, lower.cpp:152-259).
#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <sstream>

#include "lf_core.hpp"

namespace lfg {

// ---------------------------------------------------------------------------
// Primitive constructors

static Prim blank(int kind) {
  Prim p;
  std::memset(&p, 0, sizeof(p));
  p.kind = kind;
  p.target = -1;
  return p;
}

Prim make_split(int dim, const std::vector<int64_t>& factors) {
  Prim p = blank(LFGPU_PRIM_SPLIT);
  p.dim = dim;
  p.nfactors = static_cast<int32_t>(factors.size());
  for (size_t i = 0; i < factors.size(); ++i) p.factors[i] = factors[i];
  return p;
}

Prim make_reorder(const std::vector<int>& perm) {
  Prim p = blank(LFGPU_PRIM_REORDER);
  p.nperm = static_cast<int32_t>(perm.size());
  for (size_t i = 0; i < perm.size(); ++i) p.perm[i] = perm[i];
  return p;
}

Prim make_fuse(int dim, int span) {
  Prim p = blank(LFGPU_PRIM_FUSE);
  p.dim = dim;
  p.span = span;
  return p;
}

Prim make_unfold(int dim, int64_t tile, int64_t stride) {
  Prim p = blank(LFGPU_PRIM_UNFOLD);
  p.dim = dim;
  p.tile = tile;
  p.stride = stride;
  return p;
}

Prim make_fold(int dim, int64_t tile, int64_t stride, int64_t orig_extent) {
  Prim p = blank(LFGPU_PRIM_FOLD);
  p.dim = dim;
  p.tile = tile;
  p.stride = stride;
  p.orig_extent = orig_extent;
  return p;
}

Prim make_pad(int dim, int64_t pad) {
  Prim p = blank(LFGPU_PRIM_PAD);
  p.dim = dim;
  p.pad = pad;
  return p;
}

Prim make_unpad(int dim, int64_t pad) {
  Prim p = blank(LFGPU_PRIM_UNPAD);
  p.dim = dim;
  p.pad = pad;
  return p;
}

// ---------------------------------------------------------------------------
// Shape algebra

int64_t unfold_tiles(int64_t d, int64_t b, int64_t s) { return (d - b + s - 1) / s + 1; }

static const char* kind_name(int k) {
  static const char* names[] = {"split", "reorder", "fuse",  "unfold",     "pad",
                                "store_at", "fold", "unpad", "decouple_at"};
  return (k >= 0 && k <= 8) ? names[k] : "?";
}

static void check_dim(const std::vector<Dim>& dims, const Prim& p, int dim) {
  if (dim < 0 || dim >= static_cast<int>(dims.size()))
    fail(LFGPU_EINVAL, std::string(kind_name(p.kind)) + ": dim " + std::to_string(dim) +
                           " out of range for rank " + std::to_string(dims.size()));
}

std::vector<Dim> apply_shape(const std::vector<Dim>& dims, const Prim& p) {
  std::vector<Dim> out;
  const std::string k = kind_name(p.kind);
  switch (p.kind) {
    case LFGPU_PRIM_SPLIT: {
      check_dim(dims, p, p.dim);
      if (p.nfactors < 1) fail(LFGPU_EINVAL, k + ": needs at least one factor");
      int64_t prod = 1;
      for (int j = 0; j < p.nfactors; ++j) {
        if (p.factors[j] < 1) fail(LFGPU_EINVAL, k + ": factor < 1");
        prod *= p.factors[j];
      }
      if (prod != dims[p.dim].extent)
        fail(LFGPU_EINVAL, k + ": factors multiply to " + std::to_string(prod) + ", dim " +
                               dims[p.dim].name + " has extent " +
                               std::to_string(dims[p.dim].extent));
      out.assign(dims.begin(), dims.begin() + p.dim);
      for (int j = 0; j < p.nfactors; ++j)
        out.push_back({dims[p.dim].name + std::to_string(j), p.factors[j]});
      out.insert(out.end(), dims.begin() + p.dim + 1, dims.end());
      break;
    }
    case LFGPU_PRIM_REORDER: {
      if (p.nperm != static_cast<int>(dims.size()))
        fail(LFGPU_EINVAL, k + ": permutation length mismatch");
      std::vector<bool> seen(dims.size(), false);
      for (int j = 0; j < p.nperm; ++j) {
        int v = p.perm[j];
        if (v < 0 || v >= static_cast<int>(dims.size()) || seen[v])
          fail(LFGPU_EINVAL, k + ": not a permutation");
        seen[v] = true;
      }
      for (int j = 0; j < p.nperm; ++j) out.push_back(dims[p.perm[j]]);
      break;
    }
    case LFGPU_PRIM_FUSE: {
      check_dim(dims, p, p.dim);
      if (p.span < 1) fail(LFGPU_EINVAL, k + ": span < 1");
      if (p.dim + p.span > static_cast<int>(dims.size()))
        fail(LFGPU_EINVAL, k + ": fused dims must be contiguous and in range");
      out.assign(dims.begin(), dims.begin() + p.dim);
      Dim f{"", 1};
      for (int j = 0; j < p.span; ++j) {
        f.extent *= dims[p.dim + j].extent;
        f.name += dims[p.dim + j].name;
      }
      out.push_back(f);
      out.insert(out.end(), dims.begin() + p.dim + p.span, dims.end());
      break;
    }
    case LFGPU_PRIM_UNFOLD: {
      check_dim(dims, p, p.dim);
      int64_t d = dims[p.dim].extent;
      if (p.stride < 1 || p.stride > p.tile || p.tile > d)
        fail(LFGPU_EINVAL, k + ": requires 1 <= stride <= tile <= extent (tile=" +
                               std::to_string(p.tile) + ", stride=" + std::to_string(p.stride) +
                               ", extent=" + std::to_string(d) + ")");
      out = dims;
      out[p.dim] = {dims[p.dim].name + "0", unfold_tiles(d, p.tile, p.stride)};
      out.insert(out.begin() + p.dim + 1, Dim{dims[p.dim].name + "1", p.tile});
      break;
    }
    case LFGPU_PRIM_PAD:
      check_dim(dims, p, p.dim);
      if (p.pad < 0) fail(LFGPU_EINVAL, k + ": pad size < 0");
      out = dims;
      out[p.dim].extent += p.pad;
      break;
    case LFGPU_PRIM_FOLD: {
      check_dim(dims, p, p.dim);
      if (p.dim + 1 >= static_cast<int>(dims.size()))
        fail(LFGPU_EINVAL, k + ": needs two adjacent dims");
      if (dims[p.dim + 1].extent != p.tile)
        fail(LFGPU_EINVAL, k + ": inner dim does not match tile size");
      out.assign(dims.begin(), dims.begin() + p.dim);
      std::string name = dims[p.dim].name;
      if (!name.empty() && name.back() == '0') name.pop_back();
      out.push_back({name, p.orig_extent});
      out.insert(out.end(), dims.begin() + p.dim + 2, dims.end());
      break;
    }
    case LFGPU_PRIM_UNPAD:
      check_dim(dims, p, p.dim);
      if (p.pad < 0 || p.pad >= dims[p.dim].extent)
        fail(LFGPU_EINVAL, k + ": unpad size out of range");
      out = dims;
      out[p.dim].extent -= p.pad;
      break;
    default:
      fail(LFGPU_EINVAL, k + ": requires graph context; resolved by the plan builder");
  }
  if (out.size() > static_cast<size_t>(kMaxRank))
    fail(LFGPU_EUNSUPPORTED, "rank exceeds " + std::to_string(kMaxRank));
  return out;
}

std::vector<Dim> derive(const std::vector<Dim>& dims, const Seq& seq) {
  std::vector<Dim> cur = dims;
  for (size_t i = 0; i < seq.size(); ++i) {
    try {
      cur = apply_shape(cur, seq[i]);
    } catch (const Error& e) {
      fail(e.code, "primitive #" + std::to_string(i) + ": " + e.what());
    }
  }
  return cur;
}

std::vector<int64_t> extents(const std::vector<Dim>& dims) {
  std::vector<int64_t> e;
  for (const auto& d : dims) e.push_back(d.extent);
  return e;
}

int64_t numel(const std::vector<Dim>& dims) {
  int64_t n = 1;
  for (const auto& d : dims) n *= d.extent;
  return n;
}

std::vector<int64_t> row_strides(const std::vector<int64_t>& ext) {
  std::vector<int64_t> s(ext.size(), 1);
  for (int i = static_cast<int>(ext.size()) - 2; i >= 0; --i) s[i] = s[i + 1] * ext[i + 1];
  return s;
}

Seq invert(const std::vector<Dim>& dims, const Seq& seq) {
  std::vector<std::vector<Dim>> shapes{dims};
  for (const auto& p : seq) shapes.push_back(apply_shape(shapes.back(), p));
  Seq inv;
  for (int i = static_cast<int>(seq.size()) - 1; i >= 0; --i) {
    const Prim& p = seq[i];
    const auto& before = shapes[i];
    switch (p.kind) {
      case LFGPU_PRIM_SPLIT: inv.push_back(make_fuse(p.dim, p.nfactors)); break;
      case LFGPU_PRIM_REORDER: {
        std::vector<int> ip(p.nperm);
        for (int j = 0; j < p.nperm; ++j) ip[p.perm[j]] = j;
        inv.push_back(make_reorder(ip));
        break;
      }
      case LFGPU_PRIM_FUSE: {
        std::vector<int64_t> f;
        for (int j = 0; j < p.span; ++j) f.push_back(before[p.dim + j].extent);
        inv.push_back(make_split(p.dim, f));
        break;
      }
      case LFGPU_PRIM_UNFOLD:
        inv.push_back(make_fold(p.dim, p.tile, p.stride, before[p.dim].extent));
        break;
      case LFGPU_PRIM_PAD: inv.push_back(make_unpad(p.dim, p.pad)); break;
      case LFGPU_PRIM_FOLD: inv.push_back(make_unfold(p.dim, p.tile, p.stride)); break;
      case LFGPU_PRIM_UNPAD: inv.push_back(make_pad(p.dim, p.pad)); break;
      default: fail(LFGPU_EINVAL, "invert: store_at must be folded by the plan builder");
    }
  }
  return inv;
}

bool seq_equal(const Seq& a, const Seq& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    const Prim &x = a[i], &y = b[i];
    if (x.kind != y.kind || x.dim != y.dim || x.span != y.span || x.nfactors != y.nfactors ||
        x.nperm != y.nperm || x.tile != y.tile || x.stride != y.stride || x.pad != y.pad ||
        x.target != y.target)
      return false;
    for (int j = 0; j < x.nfactors; ++j)
      if (x.factors[j] != y.factors[j]) return false;
    for (int j = 0; j < x.nperm; ++j)
      if (x.perm[j] != y.perm[j]) return false;
  }
  return true;
}

std::string seq_str(const Seq& s) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < s.size(); ++i) {
    const Prim& p = s[i];
    if (i) os << ", ";
    os << kind_name(p.kind) << "(";
    switch (p.kind) {
      case LFGPU_PRIM_SPLIT:
        os << p.dim << ", {";
        for (int j = 0; j < p.nfactors; ++j) os << (j ? "," : "") << p.factors[j];
        os << "}";
        break;
      case LFGPU_PRIM_REORDER:
        for (int j = 0; j < p.nperm; ++j) os << (j ? "," : "") << p.perm[j];
        break;
      case LFGPU_PRIM_FUSE: os << p.dim << ", " << p.span; break;
      case LFGPU_PRIM_UNFOLD:
      case LFGPU_PRIM_FOLD: os << p.dim << ", " << p.tile << ", " << p.stride; break;
      default: os << p.dim << ", " << p.pad; break;
    }
    os << ")";
  }
  os << "]";
  return os.str();
}

// ---------------------------------------------------------------------------
// The digit engine: symbolic affine index vectors over a refinable digit set.

namespace {

struct Combo {
  std::map<int, int64_t> t;  // digit -> coefficient
  int64_t c0 = 0;
  bool clamped = false;  // value = min(affine, cmax)
  int64_t cmax = 0;
};

struct Pending {  // Nest mode: a value that may exceed its extent unless guarded
  Combo v;
  int64_t bound;
};

class DigitEngine {
 public:
  std::vector<int64_t> ext, dstr;
  std::vector<Combo> V;              // current index vector
  std::vector<int64_t> E;            // extents of V entries
  std::vector<std::pair<Combo, std::pair<int64_t, int64_t>>> preds;  // lo <= v < hi
  std::vector<Pending> pending;
  bool ok = true;

  explicit DigitEngine(const std::vector<int64_t>& phys) {
    auto st = row_strides(phys);
    for (size_t k = 0; k < phys.size(); ++k) {
      ext.push_back(phys[k]);
      dstr.push_back(st[k]);
      Combo c;
      if (phys[k] > 1) c.t[static_cast<int>(k)] = 1;
      V.push_back(c);
      E.push_back(phys[k]);
    }
  }

  static Combo lin(const std::vector<std::pair<const Combo*, int64_t>>& parts) {
    Combo r;
    for (const auto& [c, k] : parts) {
      r.c0 += c->c0 * k;
      for (const auto& [d, v] : c->t) r.t[d] += v * k;
    }
    for (auto it = r.t.begin(); it != r.t.end();)
      it = it->second == 0 ? r.t.erase(it) : std::next(it);
    return r;
  }

  int64_t max_value(const Combo& c) const {
    int64_t m = c.c0;
    for (const auto& [d, v] : c.t)
      if (v > 0) m += v * (ext[d] - 1);
    return m;
  }
  int64_t min_value(const Combo& c) const {
    int64_t m = c.c0;
    for (const auto& [d, v] : c.t)
      if (v < 0) m += v * (ext[d] - 1);
    return m;
  }

  // x_d = f*x_hi + x_lo; hi keeps index d, lo is appended.
  void refine(int d, int64_t f) {
    int lo = static_cast<int>(ext.size());
    ext.push_back(f);
    dstr.push_back(dstr[d]);
    ext[d] /= f;
    dstr[d] *= f;
    auto fix = [&](Combo& c) {
      auto it = c.t.find(d);
      if (it == c.t.end()) return;
      int64_t v = it->second;
      it->second = v * f;
      c.t[lo] += v;
    };
    for (auto& c : V) fix(c);
    for (auto& p : preds) fix(p.first);
    for (auto& p : pending) fix(p.v);
  }

  // Mixed-radix split of V[idx] (dense over digits, total extent = prod F).
  bool split_entry(int idx, const std::vector<int64_t>& F) {
    int64_t E_total = 1;
    for (auto f : F) E_total *= f;
    for (int guard = 0; guard < 64; ++guard) {
      Combo& v = V[idx];
      if (v.clamped || v.c0 != 0) return false;
      std::vector<std::pair<int64_t, int>> terms;  // (coef, digit)
      for (const auto& [d, c] : v.t)
        if (ext[d] > 1) {
          if (c <= 0) return false;
          terms.push_back({c, d});
        }
      std::sort(terms.begin(), terms.end());
      int64_t expect = 1;
      for (const auto& [c, d] : terms) {
        if (c != expect) return false;
        expect *= ext[d];
      }
      if (expect != E_total) return false;
      // Boundaries at the suffix products s_j (j >= 1).
      bool refined = false;
      for (size_t j = 1; j < F.size() && !refined; ++j) {
        int64_t s = 1;
        for (size_t l = j; l < F.size(); ++l) s *= F[l];
        for (const auto& [c, d] : terms) {
          if (c < s && s < c * ext[d]) {
            if (s % c != 0 || ext[d] % (s / c) != 0) return false;
            refine(d, s / c);
            refined = true;
            break;
          }
        }
      }
      if (refined) continue;
      // Aligned: distribute terms to components.
      std::vector<Combo> parts(F.size());
      std::vector<int64_t> suffix(F.size(), 1);
      for (int j = static_cast<int>(F.size()) - 2; j >= 0; --j) suffix[j] = suffix[j + 1] * F[j + 1];
      for (const auto& [c, d] : terms) {
        for (size_t j = 0; j < F.size(); ++j) {
          if (c >= suffix[j] && c < suffix[j] * F[j]) {
            parts[j].t[d] = c / suffix[j];
            break;
          }
        }
      }
      V.erase(V.begin() + idx);
      E.erase(E.begin() + idx);
      V.insert(V.begin() + idx, parts.begin(), parts.end());
      E.insert(E.begin() + idx, F.begin(), F.end());
      return true;
    }
    return false;
  }

  void fuse_entries(int idx, int span) {
    std::vector<std::pair<const Combo*, int64_t>> parts;
    int64_t total = 1;
    for (int j = span - 1; j >= 0; --j) {
      parts.push_back({&V[idx + j], total});
      total *= E[idx + j];
    }
    for (int j = 0; j < span; ++j)
      if (V[idx + j].clamped) ok = false;
    Combo f = lin(parts);
    V.erase(V.begin() + idx, V.begin() + idx + span);
    E.erase(E.begin() + idx, E.begin() + idx + span);
    V.insert(V.begin() + idx, f);
    E.insert(E.begin() + idx, total);
  }

  void permute(const int32_t* perm, int n, bool inverse) {
    std::vector<Combo> nv(n);
    std::vector<int64_t> ne(n);
    for (int j = 0; j < n; ++j) {
      if (inverse) {
        nv[perm[j]] = V[j];
        ne[perm[j]] = E[j];
      } else {
        nv[j] = V[perm[j]];
        ne[j] = E[perm[j]];
      }
    }
    V = nv;
    E = ne;
  }
};

}  // namespace

bool compile_digit_map(const CopySpec& spec, DigitMap* out, bool* oob,
                       std::vector<int32_t>* tables) {
  *oob = false;
  std::vector<Dim> dst_phys = derive(spec.lmap.dst_logical, spec.dst_seq);
  std::vector<Dim> src_phys = derive(spec.lmap.src_logical, spec.src_seq);
  DigitEngine en(extents(dst_phys));

  // Shapes the destination sequence passes through (for inverse steps).
  std::vector<std::vector<Dim>> shapes{spec.lmap.dst_logical};
  for (const auto& p : spec.dst_seq) shapes.push_back(apply_shape(shapes.back(), p));

  // 1. destination physical -> destination logical (inverse sequence).
  for (int i = static_cast<int>(spec.dst_seq.size()) - 1; i >= 0 && en.ok; --i) {
    const Prim& p = spec.dst_seq[i];
    const auto& before = shapes[i];
    switch (p.kind) {
      case LFGPU_PRIM_SPLIT:  // inverse: fuse
        en.fuse_entries(p.dim, p.nfactors);
        break;
      case LFGPU_PRIM_REORDER:
        en.permute(p.perm, p.nperm, /*inverse=*/true);
        break;
      case LFGPU_PRIM_FUSE: {  // inverse: split into the fused extents
        std::vector<int64_t> f;
        for (int j = 0; j < p.span; ++j) f.push_back(before[p.dim + j].extent);
        if (!en.split_entry(p.dim, f)) return false;
        break;
      }
      case LFGPU_PRIM_UNFOLD: {  // inverse: fold, t*S + o
        if (en.V[p.dim].clamped || en.V[p.dim + 1].clamped) return false;
        Combo f = DigitEngine::lin({{&en.V[p.dim], p.stride}, {&en.V[p.dim + 1], 1}});
        int64_t D = before[p.dim].extent;
        bool overhang = en.max_value(f) > D - 1;
        en.V.erase(en.V.begin() + p.dim, en.V.begin() + p.dim + 2);
        en.E.erase(en.E.begin() + p.dim, en.E.begin() + p.dim + 2);
        if (overhang) {
          if (spec.mode == FoldMode::Clamp) {
            f.clamped = true;
            f.cmax = D - 1;
          } else {
            en.pending.push_back({f, D});
          }
        }
        en.V.insert(en.V.begin() + p.dim, f);
        en.E.insert(en.E.begin() + p.dim, D);
        break;
      }
      case LFGPU_PRIM_PAD: {  // inverse: unpad -> cells beyond the extent
        int64_t D = before[p.dim].extent;
        if (en.V[p.dim].clamped) return false;
        if (spec.mode == FoldMode::Clamp)
          en.preds.push_back({en.V[p.dim], {0, D}});
        else
          en.pending.push_back({en.V[p.dim], D});
        en.E[p.dim] = D;
        break;
      }
      default:
        return false;
    }
  }
  if (!en.ok) return false;

  // 2. logical guard + shift (Padding nest).
  const auto& L = spec.lmap;
  if (L.has_guard) {
    for (size_t j = 0; j < en.V.size(); ++j) {
      bool trivial = L.lo[j] <= en.min_value(en.V[j]) && en.max_value(en.V[j]) < L.hi[j];
      if (!trivial) {
        if (en.V[j].clamped) return false;
        en.preds.push_back({en.V[j], {L.lo[j], L.hi[j]}});
      }
    }
  }
  // Resolve Nest-mode pending bounds: covered iff a guard on an identical
  // logical combo keeps it below the bound.
  for (const auto& pd : en.pending) {
    bool covered = false;
    if (L.has_guard) {
      for (size_t j = 0; j < en.V.size(); ++j)
        if (en.V[j].t == pd.v.t && en.V[j].c0 == pd.v.c0 && L.hi[j] <= pd.bound) covered = true;
    }
    if (!covered) *oob = true;
  }
  if (L.has_guard)
    for (size_t j = 0; j < en.V.size(); ++j) {
      en.V[j].c0 += L.shift[j];
      if (en.V[j].clamped) en.V[j].cmax += L.shift[j];
    }
  for (size_t j = 0; j < en.V.size(); ++j) en.E[j] = L.src_logical[j].extent;

  // 3. source logical -> source physical (forward sequence); on failure
  // (and when allowed) keep the logical forms and use offset tables.
  const DigitEngine logical_state = en;
  auto forward_src = [&]() -> bool {
    std::vector<Dim> cur = L.src_logical;
    for (const auto& p : spec.src_seq) {
      std::vector<Dim> nxt = apply_shape(cur, p);
      switch (p.kind) {
        case LFGPU_PRIM_SPLIT: {
          std::vector<int64_t> f(p.factors, p.factors + p.nfactors);
          if (!en.split_entry(p.dim, f)) return false;
          break;
        }
        case LFGPU_PRIM_REORDER:
          en.permute(p.perm, p.nperm, /*inverse=*/false);
          break;
        case LFGPU_PRIM_FUSE:
          en.fuse_entries(p.dim, p.span);
          if (!en.ok) return false;
          break;
        case LFGPU_PRIM_UNFOLD: {
          int64_t D = cur[p.dim].extent;
          int64_t T = unfold_tiles(D, p.tile, p.stride);
          if (D % p.stride != 0 || D / p.stride > T) return false;
          if (!en.split_entry(p.dim, {D / p.stride, p.stride})) return false;
          en.E[p.dim] = T;
          en.E[p.dim + 1] = p.tile;
          break;
        }
        case LFGPU_PRIM_PAD:
          en.E[p.dim] += p.pad;
          break;
        default:
          return false;
      }
      cur = nxt;
    }
    return true;
  };
  bool use_tables = false;
  std::vector<int64_t> ltab, ltab_off;
  if (!forward_src()) {
    if (!tables || spec.src_seq.empty()) return false;
    en = logical_state;
    if (!separable_tables(L.src_logical, spec.src_seq, &ltab, &ltab_off)) return false;
    use_tables = true;
  }

  // 4. emit.
  auto sstr = row_strides(extents(src_phys));
  DigitMap m;
  std::vector<int64_t> src_coef(en.ext.size(), 0);
  std::vector<Combo> clamps;
  std::vector<int64_t> clamp_stride;
  std::vector<Combo> tabs;
  std::vector<int64_t> tab_max, tab_off;
  int64_t base = 0;
  for (size_t k = 0; k < en.V.size(); ++k) {
    const Combo& c = en.V[k];
    int64_t stride = use_tables ? 0 : sstr[k];
    if (use_tables) {
      // Logical coordinate k: affine table -> a stride, else a table term.
      const int64_t D = L.src_logical[k].extent;
      const int64_t* T = ltab.data() + ltab_off[k];
      stride = D > 1 ? T[1] - T[0] : 0;
      bool affine = true;
      for (int64_t l = 0; l < D && affine; ++l) affine = T[l] == T[0] + l * stride;
      base += T[0];
      if (!affine) {
        if (static_cast<int>(tabs.size()) >= kMaxTab) return false;
        tabs.push_back(c);
        tab_max.push_back(c.clamped ? std::min(c.cmax, D - 1) : D - 1);
        tab_off.push_back(static_cast<int64_t>(tables->size()));
        for (int64_t l = 0; l < D; ++l) {
          const int64_t v = T[l] - T[0];
          if (v > INT32_MAX || v < INT32_MIN) return false;
          tables->push_back(static_cast<int32_t>(v));
        }
        continue;
      }
    }
    if (c.clamped) {
      clamps.push_back(c);
      clamp_stride.push_back(stride);
      continue;
    }
    base += c.c0 * stride;
    for (const auto& [d, v] : c.t) src_coef[d] += v * stride;
  }
  // Digits in destination order (descending dst stride); drop extent-1 digits.
  std::vector<int> order;
  for (size_t d = 0; d < en.ext.size(); ++d)
    if (en.ext[d] > 1) order.push_back(static_cast<int>(d));
  std::sort(order.begin(), order.end(),
            [&](int a, int b) { return en.dstr[a] > en.dstr[b]; });
  // Linear forms over digits: dst, src, preds, clamps — for coalescing.
  auto form_coef = [&](int f, int d) -> int64_t {
    if (f == 0) return en.dstr[d];
    if (f == 1) return src_coef[d];
    int pi = f - 2;
    if (pi < static_cast<int>(en.preds.size())) {
      auto it = en.preds[pi].first.t.find(d);
      return it == en.preds[pi].first.t.end() ? 0 : it->second;
    }
    int ci = pi - static_cast<int>(en.preds.size());
    if (ci < static_cast<int>(clamps.size())) {
      auto it = clamps[ci].t.find(d);
      return it == clamps[ci].t.end() ? 0 : it->second;
    }
    int ti = ci - static_cast<int>(clamps.size());
    auto it = tabs[ti].t.find(d);
    return it == tabs[ti].t.end() ? 0 : it->second;
  };
  int nforms = 2 + static_cast<int>(en.preds.size() + clamps.size() + tabs.size());
  // Groups of consecutive digits merged when every form is contiguous.
  struct G {
    int64_t ext;
    std::vector<int64_t> coef;
  };
  std::vector<G> groups;
  for (int d : order) {
    std::vector<int64_t> co(nforms);
    for (int f = 0; f < nforms; ++f) co[f] = form_coef(f, d);
    if (!groups.empty()) {
      G& g = groups.back();  // g is the outer neighbour of d
      bool merge = true;
      for (int f = 0; f < nforms; ++f)
        if (g.coef[f] != co[f] * en.ext[d]) merge = false;
      if (merge) {
        g.ext *= en.ext[d];
        g.coef = co;
        continue;
      }
    }
    groups.push_back({en.ext[d], co});
  }
  if (groups.size() > static_cast<size_t>(kMaxDig) || en.preds.size() > kMaxPred ||
      clamps.size() > kMaxClamp)
    return false;
  m.ndig = static_cast<int32_t>(groups.size());
  m.npred = static_cast<int32_t>(en.preds.size());
  m.nclamp = static_cast<int32_t>(clamps.size());
  m.ntab = static_cast<int32_t>(tabs.size());
  m.src_base = base;
  for (size_t g = 0; g < groups.size(); ++g) {
    m.ext[g] = groups[g].ext;
    m.dst_stride[g] = groups[g].coef[0];
    m.src_stride[g] = groups[g].coef[1];
    for (int p = 0; p < m.npred; ++p) m.pcoef[p][g] = groups[g].coef[2 + p];
    for (int c = 0; c < m.nclamp; ++c) m.ccoef[c][g] = groups[g].coef[2 + m.npred + c];
    for (int t = 0; t < m.ntab; ++t) m.tcoef[t][g] = groups[g].coef[2 + m.npred + m.nclamp + t];
  }
  for (int t = 0; t < m.ntab; ++t) {
    m.tconst[t] = tabs[t].c0;
    m.tmax[t] = tab_max[t];
    m.toff[t] = tab_off[t];
  }
  for (int p = 0; p < m.npred; ++p) {
    m.pconst[p] = en.preds[p].first.c0;
    m.plo[p] = en.preds[p].second.first;
    m.phi[p] = en.preds[p].second.second;
  }
  for (int c = 0; c < m.nclamp; ++c) {
    m.cconst[c] = clamps[c].c0;
    m.cmax[c] = clamps[c].cmax;
    m.cstride[c] = clamp_stride[c];
  }
  m.dst_numel = numel(dst_phys);
  int64_t check = 1;
  for (int g = 0; g < m.ndig; ++g) check *= m.ext[g];
  if (check != m.dst_numel) return false;
  *out = m;
  return true;
}

// ---------------------------------------------------------------------------
// General index programs

namespace {

void push(IxProgram* p, IxOp op) {
  if (p->nops >= kMaxOps) fail(LFGPU_EUNSUPPORTED, "index program too long");
  p->ops[p->nops++] = op;
}

IxOp op0(int kind, int dim) {
  IxOp o;
  std::memset(&o, 0, sizeof(o));
  o.kind = kind;
  o.dim = dim;
  return o;
}

// Forward access of one primitive (layout.cpp:192-309, numeric form).
void emit_forward(IxProgram* prog, const std::vector<Dim>& before, const Prim& p, bool clamp_fold) {
  switch (p.kind) {
    case LFGPU_PRIM_SPLIT: {
      IxOp o = op0(IX_SPLIT, p.dim);
      o.n = p.nfactors;
      for (int j = 0; j < p.nfactors; ++j) o.a[j] = static_cast<int32_t>(p.factors[j]);
      push(prog, o);
      break;
    }
    case LFGPU_PRIM_REORDER: {
      IxOp o = op0(IX_PERM, 0);
      o.n = p.nperm;
      for (int j = 0; j < p.nperm; ++j) o.a[j] = p.perm[j];
      push(prog, o);
      break;
    }
    case LFGPU_PRIM_FUSE: {
      IxOp o = op0(IX_FUSE, p.dim);
      o.n = p.span;
      for (int j = 0; j < p.span; ++j) o.a[j] = static_cast<int32_t>(before[p.dim + j].extent);
      push(prog, o);
      break;
    }
    case LFGPU_PRIM_UNFOLD: {
      IxOp o = op0(IX_UNFOLD, p.dim);
      o.a[0] = static_cast<int32_t>(p.stride);
      o.a[1] = static_cast<int32_t>(unfold_tiles(before[p.dim].extent, p.tile, p.stride));
      push(prog, o);
      break;
    }
    case LFGPU_PRIM_FOLD: {
      IxOp o = op0(IX_FOLD, p.dim);
      o.a[0] = static_cast<int32_t>(p.stride);
      o.a[1] = clamp_fold ? static_cast<int32_t>(p.orig_extent - 1) : -1;
      push(prog, o);
      if (!clamp_fold) {  // nest semantics: beyond the extent is an error
        IxOp b = op0(IX_BOUND, p.dim);
        b.a[0] = 0;
        b.a[1] = static_cast<int32_t>(p.orig_extent);
        b.flag = 1;
        push(prog, b);
      }
      break;
    }
    case LFGPU_PRIM_UNPAD: {  // identity access; cells past the extent
      IxOp b = op0(IX_BOUND, p.dim);
      b.a[0] = 0;
      b.a[1] = static_cast<int32_t>(before[p.dim].extent - p.pad);
      b.flag = clamp_fold ? 0 : 1;
      push(prog, b);
      break;
    }
    case LFGPU_PRIM_PAD:
      break;  // identity access
    default:
      fail(LFGPU_EINVAL, "index program: unsupported primitive");
  }
}

}  // namespace

void compile_ix_programs(const CopySpec& spec, IxProgram* dst_inv, IxProgram* src_fwd) {
  const auto& L = spec.lmap;
  std::vector<Dim> dst_phys = derive(L.dst_logical, spec.dst_seq);
  std::vector<Dim> src_phys = derive(L.src_logical, spec.src_seq);
  *dst_inv = IxProgram();
  *src_fwd = IxProgram();
  dst_inv->in_rank = static_cast<int32_t>(dst_phys.size());
  for (size_t k = 0; k < dst_phys.size(); ++k)
    dst_inv->in_ext[k] = static_cast<int32_t>(dst_phys[k].extent);
  Seq inv = invert(L.dst_logical, spec.dst_seq);
  std::vector<Dim> cur = dst_phys;
  bool clamp = spec.mode == FoldMode::Clamp;
  for (const auto& p : inv) {
    emit_forward(dst_inv, cur, p, clamp);
    cur = apply_shape(cur, p);
  }
  dst_inv->out_rank = static_cast<int32_t>(L.dst_logical.size());
  for (size_t j = 0; j < L.dst_logical.size(); ++j)
    dst_inv->out_ext[j] = static_cast<int32_t>(L.dst_logical[j].extent);
  // Guard (zero outside) then shift into the source's logical space.
  if (L.has_guard) {
    for (size_t j = 0; j < L.dst_logical.size(); ++j) {
      IxOp b = op0(IX_BOUND, static_cast<int>(j));
      b.a[0] = static_cast<int32_t>(L.lo[j]);
      b.a[1] = static_cast<int32_t>(L.hi[j]);
      b.flag = 0;
      push(dst_inv, b);
    }
    for (size_t j = 0; j < L.dst_logical.size(); ++j)
      if (L.shift[j] != 0) {
        IxOp s = op0(IX_SHIFT, static_cast<int>(j));
        s.a[0] = static_cast<int32_t>(L.shift[j]);
        push(dst_inv, s);
      }
  }
  src_fwd->in_rank = static_cast<int32_t>(L.src_logical.size());
  for (size_t j = 0; j < L.src_logical.size(); ++j)
    src_fwd->in_ext[j] = static_cast<int32_t>(L.src_logical[j].extent);
  // Source logical range check (the interpreter's bounds check).
  for (size_t j = 0; j < L.src_logical.size(); ++j) {
    IxOp b = op0(IX_BOUND, static_cast<int>(j));
    b.a[0] = 0;
    b.a[1] = static_cast<int32_t>(L.src_logical[j].extent);
    b.flag = 1;
    push(src_fwd, b);
  }
  cur = L.src_logical;
  for (const auto& p : spec.src_seq) {
    emit_forward(src_fwd, cur, p, /*clamp_fold=*/true);
    cur = apply_shape(cur, p);
  }
  src_fwd->out_rank = static_cast<int32_t>(src_phys.size());
  for (size_t k = 0; k < src_phys.size(); ++k)
    src_fwd->out_ext[k] = static_cast<int32_t>(src_phys[k].extent);
}

// ---------------------------------------------------------------------------
// Host numeric forward map and separable offset tables

int64_t forward_offset(const std::vector<Dim>& logical, const Seq& seq, const int64_t* idx) {
  std::vector<Dim> cur = logical;
  std::vector<int64_t> v(idx, idx + logical.size());
  for (const auto& p : seq) {
    std::vector<int64_t> nv;
    switch (p.kind) {
      case LFGPU_PRIM_SPLIT: {  // mixed radix (layout.cpp:193-211)
        nv.assign(v.begin(), v.begin() + p.dim);
        int64_t e = v[p.dim];
        int64_t suffix = 1;
        for (int j = 1; j < p.nfactors; ++j) suffix *= p.factors[j];
        for (int j = 0; j < p.nfactors; ++j) {
          int64_t c = e / suffix;
          if (j > 0) c %= p.factors[j];
          nv.push_back(c);
          if (j + 1 < p.nfactors) suffix /= p.factors[j + 1];
        }
        nv.insert(nv.end(), v.begin() + p.dim + 1, v.end());
        break;
      }
      case LFGPU_PRIM_REORDER:
        for (int j = 0; j < p.nperm; ++j) nv.push_back(v[p.perm[j]]);
        break;
      case LFGPU_PRIM_FUSE: {
        nv.assign(v.begin(), v.begin() + p.dim);
        int64_t acc = 0;
        for (int j = 0; j < p.span; ++j) acc = acc * cur[p.dim + j].extent + v[p.dim + j];
        nv.push_back(acc);
        nv.insert(nv.end(), v.begin() + p.dim + p.span, v.end());
        break;
      }
      case LFGPU_PRIM_UNFOLD: {  // plain rewrite (layout.cpp:281-287)
        int64_t T = unfold_tiles(cur[p.dim].extent, p.tile, p.stride);
        for (size_t i = 0; i < v.size(); ++i) {
          if (static_cast<int>(i) == p.dim) {
            int64_t t = std::min(v[i] / p.stride, T - 1);
            nv.push_back(t);
            nv.push_back(v[i] - t * p.stride);
          } else {
            nv.push_back(v[i]);
          }
        }
        break;
      }
      case LFGPU_PRIM_FOLD:
        nv.assign(v.begin(), v.begin() + p.dim);
        nv.push_back(v[p.dim] * p.stride + v[p.dim + 1]);
        nv.insert(nv.end(), v.begin() + p.dim + 2, v.end());
        break;
      case LFGPU_PRIM_PAD:
      case LFGPU_PRIM_UNPAD:
        nv = v;
        break;
      default:
        fail(LFGPU_EINVAL, "forward map: unsupported primitive");
    }
    cur = apply_shape(cur, p);
    v = nv;
  }
  auto st = row_strides(extents(cur));
  int64_t off = 0;
  for (size_t k = 0; k < v.size(); ++k) off += v[k] * st[k];
  return off;
}

bool separable_tables(const std::vector<Dim>& logical, const Seq& seq,
                      std::vector<int64_t>* table, std::vector<int64_t>* off) {
  // Dependency sets (bitmask of logical dims) per current dim.
  std::vector<uint32_t> dep;
  for (size_t j = 0; j < logical.size(); ++j) dep.push_back(1u << j);
  for (const auto& p : seq) {
    std::vector<uint32_t> nd;
    switch (p.kind) {
      case LFGPU_PRIM_SPLIT:
      case LFGPU_PRIM_UNFOLD: {
        if (__builtin_popcount(dep[p.dim]) > 1) return false;
        int parts = p.kind == LFGPU_PRIM_SPLIT ? p.nfactors : 2;
        nd.assign(dep.begin(), dep.begin() + p.dim);
        for (int j = 0; j < parts; ++j) nd.push_back(dep[p.dim]);
        nd.insert(nd.end(), dep.begin() + p.dim + 1, dep.end());
        break;
      }
      case LFGPU_PRIM_REORDER:
        for (int j = 0; j < p.nperm; ++j) nd.push_back(dep[p.perm[j]]);
        break;
      case LFGPU_PRIM_FUSE: {
        nd.assign(dep.begin(), dep.begin() + p.dim);
        uint32_t u = 0;
        for (int j = 0; j < p.span; ++j) u |= dep[p.dim + j];
        nd.push_back(u);
        nd.insert(nd.end(), dep.begin() + p.dim + p.span, dep.end());
        break;
      }
      case LFGPU_PRIM_PAD:
      case LFGPU_PRIM_UNPAD:
        nd = dep;
        break;
      default:
        return false;
    }
    dep = nd;
  }
  table->clear();
  off->clear();
  std::vector<int64_t> idx(logical.size(), 0);
  for (size_t j = 0; j < logical.size(); ++j) {
    off->push_back(static_cast<int64_t>(table->size()));
    for (int64_t l = 0; l < logical[j].extent; ++l) {
      idx[j] = l;
      table->push_back(forward_offset(logical, seq, idx.data()));
    }
    idx[j] = 0;
  }
  return true;
}

}  // namespace lfg
