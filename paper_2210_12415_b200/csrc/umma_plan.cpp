// umma_plan.cpp — legality analysis and table construction for the tcgen05
// contraction kernel (k_umma.cu) on tuned layouts.
//
// The GMM template (space.cpp:388-412) stores A as (M/m_t)(K/k_t) m_t k_t
// bricks, B as (K/k_t)(N/n_t) k_t n_t and C as (M/m_t)(N/n_t) m_t n_t; the
// C2D template (space.cpp:185-375) stores the input as overlapped tiles
// N (H/h_t)(W/w_t)(I/i_t) B_h B_w i_t, the weight as (O/o')(I/i') KH KW i' o'
// and the output as N (H/h_t)(W/w_t)(O/o_t) h_t w_t o_t. Each brick maps to
// TMA boxes (one per CTA tile and K stage); the innermost brick dim decides
// whether the operand is K-major or MN-major for UMMA, and its byte width
// picks the 32/64/128-byte swizzle shared by the tensor map and the SMEM
// descriptor. SURVEY.md §8(a+) derives the mapping; DESIGN.md §4 states the
// legality rules enforced here.
#include <algorithm>
#include <array>
#include <climits>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <sstream>

#include "lf_pair.hpp"
#include "lf_umma.hpp"

namespace lfg {

namespace {

enum { DG_PART = 0, DG_TILE = 1, DG_OFF = 2 };

struct PDigit {
  int lj;        // logical dim
  int kind;      // DG_*
  int64_t div;   // DG_PART: logical = ... + (digit * div)
  int64_t ext;
  int64_t S;     // DG_TILE / DG_OFF: unfold stride
  int64_t stride = 0;  // physical stride (elements)
};

bool analyze(const std::vector<Dim>& logical, const Seq& seq, std::vector<PDigit>* out) {
  std::vector<PDigit> cur;
  for (size_t j = 0; j < logical.size(); ++j)
    cur.push_back({static_cast<int>(j), DG_PART, 1, logical[j].extent, 0});
  for (const auto& p : seq) {
    switch (p.kind) {
      case LFGPU_PRIM_SPLIT: {
        PDigit d = cur.at(p.dim);
        if (d.kind != DG_PART) return false;
        std::vector<PDigit> parts;
        int64_t suffix = 1;
        for (int j = 1; j < p.nfactors; ++j) suffix *= p.factors[j];
        for (int j = 0; j < p.nfactors; ++j) {
          parts.push_back({d.lj, DG_PART, d.div * suffix, p.factors[j], 0});
          if (j + 1 < p.nfactors) suffix /= p.factors[j + 1];
        }
        cur.erase(cur.begin() + p.dim);
        cur.insert(cur.begin() + p.dim, parts.begin(), parts.end());
        break;
      }
      case LFGPU_PRIM_REORDER: {
        std::vector<PDigit> n;
        for (int j = 0; j < p.nperm; ++j) n.push_back(cur.at(p.perm[j]));
        cur = n;
        break;
      }
      case LFGPU_PRIM_UNFOLD: {
        PDigit d = cur.at(p.dim);
        if (d.kind != DG_PART || d.div != 1 || d.ext != logical[d.lj].extent) return false;
        int64_t T = unfold_tiles(d.ext, p.tile, p.stride);
        PDigit t{d.lj, DG_TILE, p.stride, T, p.stride};
        PDigit o{d.lj, DG_OFF, 1, p.tile, p.stride};
        cur.erase(cur.begin() + p.dim);
        cur.insert(cur.begin() + p.dim, {t, o});
        break;
      }
      default:
        return false;
    }
  }
  std::vector<int64_t> ext;
  for (const auto& d : cur) ext.push_back(d.ext);
  auto st = row_strides(ext);
  for (size_t k = 0; k < cur.size(); ++k) cur[k].stride = st[k];
  *out = cur;
  return true;
}

// Value of logical index `v` on digit d (DG_PART only).
inline int64_t digit_of(const PDigit& d, int64_t v) { return (v / d.div) % d.ext; }

// A view dimension before merging: one physical digit plus its box and the
// way its coordinate is formed.
struct VDim {
  int64_t ext = 1;
  int64_t stride = 0;  // elements
  int64_t box = 1;
  int64_t estride = 1;
};

// Merge maximal runs of outer box-1 dims (row-major contiguous) so the view
// fits TMA's 5 dims. `group[k]` receives the merged dim index of phys dim k
// and `mult[k]` its coordinate multiplier inside the merged dim.
bool merge_view(const std::vector<VDim>& phys, OperandView* v, std::vector<int>* group,
                std::vector<int64_t>* mult, std::string* why) {
  // phys is outer->inner. Build merged dims inner->outer for TMA.
  int n = static_cast<int>(phys.size());
  group->assign(n, -1);
  mult->assign(n, 1);
  std::vector<VDim> merged;  // inner -> outer
  int k = n - 1;
  while (k >= 0) {
    if (phys[k].box != 1 || phys[k].estride != 1 || k == n - 1) {
      (*group)[k] = static_cast<int>(merged.size());
      merged.push_back(phys[k]);
      --k;
      continue;
    }
    // run of box-1 dims ending at k (inner end)
    int lo = k;
    while (lo - 1 >= 0 && phys[lo - 1].box == 1 && phys[lo - 1].estride == 1) --lo;
    VDim m;
    m.stride = phys[k].stride;
    m.ext = 1;
    int gi = static_cast<int>(merged.size());
    for (int q = k; q >= lo; --q) {
      (*group)[q] = gi;
      (*mult)[q] = m.ext;
      m.ext *= phys[q].ext;
    }
    merged.push_back(m);
    k = lo - 1;
  }
  if (merged.size() > 5) {
    *why = "operand view needs " + std::to_string(merged.size()) + " TMA dims";
    return false;
  }
  v->rank = static_cast<int32_t>(merged.size());
  for (int d = 0; d < v->rank; ++d) {
    v->dims[d] = static_cast<uint64_t>(merged[d].ext);
    v->strides[d] = static_cast<uint64_t>(merged[d].stride * 2);
    v->box[d] = static_cast<uint32_t>(merged[d].box);
    v->estride[d] = static_cast<uint32_t>(merged[d].estride);
    if (merged[d].box > 256 || merged[d].box < 1) {
      *why = "TMA box dim " + std::to_string(merged[d].box) + " out of range";
      return false;
    }
    if (d > 0 && (v->strides[d] % 16) != 0) {
      *why = "TMA stride not 16-byte aligned";
      return false;
    }
  }
  return true;
}

void finish_descriptor(OperandView* v, int rows_alloc) {
  // Box bytes = product of loaded elements * 2 (bf16).
  int64_t elems = 1;
  for (int d = 0; d < v->rank; ++d) elems *= (v->box[d] + v->estride[d] - 1) / v->estride[d];
  v->box_bytes = static_cast<int32_t>(elems * 2);
  int align = v->swizzle * 8;  // swizzle atom: 8 rows of `swizzle` bytes
  if (v->mn_major) {
    // canonical MN-major: [k rows][swizzle bytes] per box; boxes are the
    // MN atom-columns (LBO), 8-row K groups at SBO.
    v->slot_bytes = (v->box_bytes + align - 1) / align * align;
    v->sbo = static_cast<uint32_t>(8 * v->swizzle);
    v->lbo = static_cast<uint32_t>(v->slot_bytes);
    v->k_adv = static_cast<uint32_t>(16 * v->swizzle);
  } else {
    // canonical K-major: rows of `swizzle` bytes, 8-row groups at SBO;
    // UMMA reads rows_alloc rows even if the box fills fewer.
    int64_t bytes = static_cast<int64_t>(rows_alloc) * v->swizzle;
    v->slot_bytes = static_cast<int32_t>((std::max<int64_t>(bytes, v->box_bytes) + 1023) / 1024 * 1024);
    v->sbo = static_cast<uint32_t>(8 * v->swizzle);
    v->lbo = 16;
    v->k_adv = 32;  // 16 bf16 along the row
  }
}

// Cover `T` consecutive values of a logical dim with its DG_PART digits
// (ascending div); returns per-digit box sizes. Allows an outermost
// overhang (TMA zero-fills beyond the tensor).
bool cover(const std::vector<const PDigit*>& digits_by_div, int64_t T, std::vector<int64_t>* box,
           std::string* why) {
  box->assign(digits_by_div.size(), 1);
  int64_t rem = T;
  int64_t expect_div = 1;
  for (size_t i = 0; i < digits_by_div.size(); ++i) {
    const PDigit& d = *digits_by_div[i];
    if (d.div != expect_div) {
      *why = "non-dense digit order";
      return false;
    }
    expect_div *= d.ext;
    if (rem == 1) continue;
    if (d.ext >= rem) {
      if (d.ext % rem) {
        *why = "tile " + std::to_string(T) + " does not align with brick " + std::to_string(d.ext);
        return false;
      }
      (*box)[i] = rem;
      rem = 1;
    } else {
      if (rem % d.ext) {
        *why = "brick " + std::to_string(d.ext) + " does not divide tile " + std::to_string(T);
        return false;
      }
      (*box)[i] = d.ext;
      rem /= d.ext;
    }
  }
  if (rem != 1) {
    if (digits_by_div.empty()) return false;
    (*box)[digits_by_div.size() - 1] *= rem;  // overhang past the tensor end
  }
  return true;
}

std::vector<const PDigit*> digits_of(const std::vector<PDigit>& ds, int lj) {
  std::vector<const PDigit*> v;
  for (const auto& d : ds)
    if (d.lj == lj) v.push_back(&d);
  std::sort(v.begin(), v.end(), [](const PDigit* a, const PDigit* b) { return a->div < b->div; });
  return v;
}

// Check that the box>1 dims other than dim0 appear outer->inner with
// decreasing div (SMEM rows come out in logical order).
bool rows_ordered(const std::vector<PDigit>& ds, const std::vector<int64_t>& box) {
  int64_t last = INT64_MAX;
  for (size_t k = 0; k + 1 < ds.size(); ++k) {
    if (box[k] <= 1) continue;
    if (ds[k].div >= last) return false;
    last = ds[k].div;
  }
  return true;
}

uint32_t make_idesc(int M, int N, bool a_mn, bool b_mn) {
  uint32_t d = 0;
  d |= 1u << 4;                          // D format: F32
  d |= 1u << 7;                          // A format: BF16
  d |= 1u << 10;                         // B format: BF16
  d |= (a_mn ? 1u : 0u) << 15;           // A major
  d |= (b_mn ? 1u : 0u) << 16;           // B major
  d |= static_cast<uint32_t>(N >> 3) << 17;
  d |= static_cast<uint32_t>(M >> 4) << 24;
  return d;
}

int pick_pipe(const UmmaPlan& p) {
  int per = p.A.slot_bytes * p.A.boxes + p.B.slot_bytes * p.B.boxes;
  // 227 KB per CTA minus alignment slack, the epilogue transpose buffers,
  // barriers, the stage table and the row/column tables (k_umma.cu SMEM layout).
  int fixed = 1024 + 256 + kEpiSmemBytes +
              static_cast<int>(sizeof(StageEntry) * p.stages.size() + 8 * p.col_off.size() + 8 * 128);
  int budget = 227 * 1024 - fixed;
  int cap = 8;
  if (const char* e = getenv("LFGPU_MAX_PIPE")) cap = std::max(2, atoi(e));  // diagnostics
  if (const char* e = getenv("LFGPU_SMEM_BUDGET_KB")) budget = atoi(e) * 1024 - fixed;
  return std::max(2, std::min(cap, budget / std::max(per, 1)));
}

// Split-only operand view for GEMM: `mn_lj`, `k_lj` name the logical dims.
bool gemm_operand(const std::vector<Dim>& log, const Seq& seq, int mn_lj, int k_lj, int T_mn,
                  int KC, OperandView* v, std::vector<PDigit>* ds_out,
                  std::vector<int64_t>* box_out, std::vector<int>* group,
                  std::vector<int64_t>* mult, std::string* why) {
  std::vector<PDigit> ds;
  if (!analyze(log, seq, &ds)) {
    *why = "layout is not a split/reorder brick layout";
    return false;
  }
  for (const auto& d : ds)
    if (d.kind != DG_PART) {
      *why = "unfold in a GEMM operand";
      return false;
    }
  const PDigit& inner = ds.back();
  if (inner.div != 1 || inner.ext % 64 != 0) {
    *why = "innermost brick dim must be a multiple of 64 elements";
    return false;
  }
  v->mn_major = inner.lj == mn_lj ? 1 : 0;
  v->swizzle = 128;
  std::vector<int64_t> box(ds.size(), 1);
  std::vector<int64_t> bmn, bk;
  auto mnd = digits_of(ds, mn_lj), kd = digits_of(ds, k_lj);
  if (v->mn_major) {
    if (T_mn % 64) {
      *why = "MN-major tile not a multiple of 64";
      return false;
    }
    v->boxes = T_mn / 64;
    if (v->boxes > kMaxBoxes) {
      *why = "too many TMA boxes";
      return false;
    }
    if (!cover(kd, KC, &bk, why)) return false;
    for (size_t i = 0; i < kd.size(); ++i) box[kd[i] - ds.data()] = bk[i];
    box[ds.size() - 1] = 64;
  } else {
    v->boxes = 1;
    if (!cover(mnd, T_mn, &bmn, why)) return false;
    for (size_t i = 0; i < mnd.size(); ++i) box[mnd[i] - ds.data()] = bmn[i];
    if (KC > 64) {
      // A stage of KC/64 K slabs in one box: the 64-wide K brick plus the
      // next K digit, landing as KC/64 canonical [rows][64] slabs in SMEM.
      if (inner.ext != 64) {
        *why = "multi-slab K stage needs 64-wide K bricks";
        return false;
      }
      if (!cover(kd, KC, &bk, why)) return false;
      for (size_t i = 0; i < kd.size(); ++i) box[kd[i] - ds.data()] = bk[i];
    } else {
      box[ds.size() - 1] = KC;
      if (inner.ext % KC) {
        *why = "K stage does not divide the K brick";
        return false;
      }
    }
  }
  if (!rows_ordered(ds, box)) {
    *why = "brick digits out of order for the SMEM tile";
    return false;
  }
  std::vector<VDim> phys;
  for (size_t k = 0; k < ds.size(); ++k) phys.push_back({ds[k].ext, ds[k].stride, box[k], 1});
  if (!merge_view(phys, v, group, mult, why)) return false;
  *ds_out = ds;
  *box_out = box;
  return true;
}

// Coordinates of one operand box: logical values per logical dim.
void coords(const std::vector<PDigit>& ds, const std::vector<int>& group,
            const std::vector<int64_t>& mult, const int64_t* lv, int32_t* out) {
  for (int d = 0; d < 5; ++d) out[d] = 0;
  for (size_t k = 0; k < ds.size(); ++k)
    out[group[k]] += static_cast<int32_t>(digit_of(ds[k], lv[ds[k].lj]) * mult[k]);
}

int64_t offset_of(const std::vector<PDigit>& ds, const int64_t* lv) {
  int64_t off = 0;
  for (const auto& d : ds) off += digit_of(d, lv[d.lj]) * d.stride;
  return off;
}

}  // namespace

// Output TMA-store view (OutStore): box = 16 columns (64-byte fp32 rows,
// SWIZZLE_64B) x the tile's rows. `yd` are the output's physical digits,
// `col_lj` its column (N / O) logical dim; `tile_lv[t]` the logical origin
// of tile t, `row_rel[r]` the logical offset of accumulator row r from the
// origin (`row_ok[r]` false: not an output row). The tile's rows must fill
// the box exactly (else no TMA store).
static void plan_out_store(const std::vector<PDigit>& yd, int nlog, int col_lj, int BN,
                           const std::vector<std::array<int64_t, 4>>& tile_lv,
                           const std::vector<std::array<int64_t, 4>>& row_rel,
                           const std::vector<bool>& row_ok, OutStore* o) {
  o->ok = false;
  if (BN % 16 || tile_lv.empty()) {
    o->why = "BN not a multiple of 16";
    return;
  }
  // The column digit: the innermost digit of the column index. When it is
  // not the innermost physical digit the box is "transposed": its inner
  // dims are row digits and each staged column is a plane of the box.
  const int nk = static_cast<int>(yd.size());
  int kc = -1;
  for (int k = 0; k < nk; ++k)
    if (yd[k].lj == col_lj && yd[k].div == 1) kc = k;
  if (kc < 0 || yd[kc].ext % 16) {
    o->why = "column digit not a multiple of 16";
    return;
  }
  const bool transposed = kc != nk - 1;
  auto dval = [&](const std::array<int64_t, 4>& lv, int k) { return digit_of(yd[k], lv[yd[k].lj]); };
  // Row digit ranges over the valid rows of tile 0.
  std::vector<int64_t> lo(nk, INT64_MAX), hi(nk, INT64_MIN);
  int nvalid = 0;
  for (int r = 0; r < 128; ++r) {
    if (!row_ok[r]) continue;
    ++nvalid;
    std::array<int64_t, 4> lv = tile_lv[0];
    for (int j = 0; j < nlog; ++j) lv[j] += row_rel[r][j];
    for (int k = 0; k < nk; ++k) {
      lo[k] = std::min(lo[k], dval(lv, k));
      hi[k] = std::max(hi[k], dval(lv, k));
    }
  }
  std::vector<VDim> v;
  int64_t cells = 1;
  for (const auto& lv : tile_lv)
    if (dval(lv, kc) + BN > yd[kc].ext) {
      o->why = "column tile crosses its digit";
      return;
    }
  for (int k = 0; k < nk; ++k) {
    // fp32 strides: merge_view counts bf16 elements, so doubled strides
    // give it fp32 bytes (and its 16-byte stride check applies to those).
    VDim d{yd[k].ext, yd[k].stride * 2, 1, 1};
    if (k == kc) d.box = 16;
    else if (yd[k].lj != col_lj) {
      if (dval(tile_lv[0], k) != lo[k]) {
        o->why = "tile origin is not the box corner";
        return;
      }
      d.box = hi[k] - lo[k] + 1;
      cells *= d.box;
    } else if (lo[k] != hi[k]) {
      o->why = "column tile spans an outer column digit";
      return;
    }
    v.push_back(d);
  }
  if (cells != nvalid) {
    o->why = "tile rows do not fill a box";
    return;
  }
  std::vector<int> grp;
  std::vector<int64_t> mult;
  std::string why;
  OperandView O;
  if (!merge_view(v, &O, &grp, &mult, &why)) {
    o->why = why;
    return;
  }
  O.elem_bytes = 4;
  O.swizzle = transposed ? 0 : 64;  // columns innermost: 16 fp32 = 64-byte box rows
  O.mn_major = 0;
  if (!umma_view_encodable(O, &why)) {
    o->why = why;
    return;
  }
  auto coord = [&](const std::array<int64_t, 4>& lv, int32_t* c) {
    for (int d = 0; d < 5; ++d) c[d] = 0;
    for (int k = 0; k < nk; ++k) c[grp[k]] += static_cast<int32_t>(dval(lv, k) * mult[k]);
  };
  // Row position inside the box (view dims >= 1, innermost first).
  int32_t c0[5];
  coord(tile_lv[0], c0);
  // Box element position of (row, column j): row_pos[row] + j * col_stride.
  const int cdim = grp[kc];
  int64_t col_stride = 1;
  for (int d = 0; d < cdim; ++d) col_stride *= O.box[d];
  col_stride *= mult[kc];
  if (transposed && (cdim == 0 || mult[kc] != 1)) {
    o->why = "column dim merged into a row dim";
    return;
  }
  o->row_pos.assign(128, -1);
  for (int r = 0; r < 128; ++r) {
    if (!row_ok[r]) continue;
    std::array<int64_t, 4> lv = tile_lv[0];
    for (int j = 0; j < nlog; ++j) lv[j] += row_rel[r][j];
    int32_t c[5];
    coord(lv, c);
    int64_t pos = 0, scale = 1;
    for (int d = 0; d < O.rank; ++d) {
      if (d == cdim) {
        if (c[d] != c0[d]) {
          o->why = "rows vary the column coordinate";
          return;
        }
        if (transposed) scale *= O.box[d];  // else row_pos counts 16-column rows
        continue;
      }
      const int64_t rel = c[d] - c0[d];
      if (rel < 0 || rel >= O.box[d]) {
        o->why = "row outside the box";
        return;
      }
      pos += rel * scale;
      scale *= O.box[d];
    }
    o->row_pos[r] = static_cast<int32_t>(pos);
  }
  o->box_rows = static_cast<int>(cells);
  o->tile_coords.assign(tile_lv.size() * 5, 0);
  for (size_t t = 0; t < tile_lv.size(); ++t) coord(tile_lv[t], &o->tile_coords[t * 5]);
  o->O = O;
  o->col_dim = cdim;
  o->col_stride = static_cast<int32_t>(transposed ? col_stride : 0);
  o->ok = true;
}

// ---------------------------------------------------------------------------
// GEMM: C[M,N] = A[M,K] B[K,N]   (interp.cpp:109-122)

bool umma_plan_gemm(const std::vector<Dim>& a_log, const Seq& a_seq, const std::vector<Dim>& b_log,
                    const Seq& b_seq, const std::vector<Dim>& c_log, const Seq& c_seq,
                    const lfgpu_sched& s, UmmaPlan* out, std::string* why, int RT) {
  // RT: logical rows per tile (<= 128). Below 128 the UMMA still computes
  // 128 rows; rows >= RT read stale SMEM and are never stored (the im2col
  // stem tiles one 112-pixel output row per tile).
  if (RT < 16 || RT > 128) {
    *why = "rows per tile out of range";
    return false;
  }
  // Loop point tile_second (tile of the M brick loop) picks the M tile:
  // 128 -> the 1-CTA kernel (BM = 128); otherwise the CTA-pair kernel
  // (BM = 256) when the shape and layouts allow it.
  if (RT == 128 && s.tile_second != 128 && !getenv("LFGPU_NO_PAIR")) {
    // The CTA-pair kernel (256-row tiles, cta_group::2) when the shape and
    // the layouts allow it; the 1-CTA kernel below otherwise.
    PairPlan pp;
    std::string pwhy;
    if (pair_plan_gemm(a_log, a_seq, b_log, b_seq, c_log, c_seq, s, &pp, &pwhy)) {
      UmmaPlan q;
      q.kind = UMMA_GEMM;
      q.BM = 256;
      q.BN = pp.BN;
      q.pipe = pp.pipe;
      q.summary = pp.summary;
      q.pair = std::make_shared<PairPlan>(pp);
      *out = q;
      return true;
    }
    if (getenv("LFGPU_DEBUG_PAIR")) fprintf(stderr, "pair GEMM rejected: %s\n", pwhy.c_str());
  }
  const int64_t M = a_log[0].extent, K = a_log[1].extent, N = b_log[1].extent;
  if (K % 64) {
    *why = "K must be a multiple of 64";
    return false;
  }
  std::vector<PDigit> cds;
  if (!analyze(c_log, c_seq, &cds)) {
    *why = "output layout is not a brick layout";
    return false;
  }
  UmmaPlan p;
  p.kind = UMMA_GEMM;
  p.BM = 128;
  p.KC = 64;
  // N tile: the schedule's innermost tile when legal, else the widest tile
  // that still fills most of the 148 SMs.
  std::vector<int> cands;
  if (s.tile_last >= 16 && s.tile_last <= 256 && s.tile_last % 16 == 0) cands.push_back(s.tile_last);
  const int64_t mtiles = (M + RT - 1) / RT;
  // Widest tile that still fills ~3/4 of the 148 SMs first, then the rest
  // from wide to narrow (legality may rule some out).
  for (int bn : {256, 128, 64, 32, 16})
    if (mtiles * ((N + bn - 1) / bn) >= 111) cands.push_back(bn);
  for (int bn : {64, 128, 256, 32, 16})
    if (mtiles * ((N + bn - 1) / bn) < 111) cands.push_back(bn);
  // K per stage: up to 256 (four 64-wide K slabs per TMA box) — a producer
  // warp sustains about one TMA request per ~800 cycles whatever its size
  // (DESIGN.md §4.3), so fewer, larger requests per K byte (cfg2 1024^3 at
  // BN 64: 11.9 / 10.4 / 9.3 us for 64 / 128 / 256, tools/kcs_probe.py);
  // smaller when the layouts (K bricks of 64 outside the M / N bricks) or
  // two stages of SMEM cannot take it. LFGPU_GEMM_KCS overrides.
  int kcs_pref = 256;
  if (const char* e = getenv("LFGPU_GEMM_KCS")) kcs_pref = atoi(e);
  if (kcs_pref != 64 && kcs_pref != 128 && kcs_pref != 256) kcs_pref = 64;
  std::string last_why;
  for (int BN : cands) {
    if (N % BN && N > BN) continue;
    std::vector<PDigit> ads, bds;
    std::vector<int64_t> abox, bbox;
    std::vector<int> ag, bg;
    std::vector<int64_t> am, bm;
    UmmaPlan q = p;
    q.BN = BN;
    // Candidate K stages, largest first; among the ones that divide K, a
    // stage count that is a multiple of 4 (then of 2) goes first so split-K
    // (<= 4 splits) deals equal stage counts (K = 768: 4 x 192, not 3 x 256).
    std::vector<int> kc_list;
    for (int c : {256, 192, 128, 64})
      if (c <= kcs_pref && K % c == 0) kc_list.push_back(c);
    if (getenv("LFGPU_GEMM_KCS")) kc_list.assign(1, kcs_pref);
    std::stable_sort(kc_list.begin(), kc_list.end(), [&](int x, int y) {
      auto rank = [&](int c) { return (K / c) % 4 == 0 ? 0 : (K / c) % 2 == 0 ? 1 : 2; };
      return rank(x) < rank(y);
    });
    if (kc_list.empty() || kc_list.back() != 64) kc_list.push_back(64);
    int kcs = 64;
    bool a_ok = false, b_ok = false;
    for (int kci = 0; kci < static_cast<int>(kc_list.size()); ++kci) {
      kcs = kc_list[kci];
      if (K % kcs || (kcs > 64 && RT != 128)) continue;
      std::string wa, wb;
      a_ok = gemm_operand(a_log, a_seq, 0, 1, RT, kcs, &q.A, &ads, &abox, &ag, &am, &wa);
      b_ok = a_ok && gemm_operand(b_log, b_seq, 1, 0, BN, kcs, &q.B, &bds, &bbox, &bg, &bm, &wb);
      if (a_ok && b_ok && kcs > 64) {
        // Two stages must fit beside the tables, and beside the epilogue
        // buffers unless every CTA gets one tile (they then alias the ring,
        // k_umma.cu layout_smem).
        OperandView ta = q.A, tb = q.B;
        finish_descriptor(&ta, 128);
        finish_descriptor(&tb, BN);
        const int per = ta.slot_bytes * ta.boxes + tb.slot_bytes * tb.boxes;
        const int64_t ntiles = mtiles * ((N + BN - 1) / BN);
        const int epi = ntiles <= 148 && !getenv("LFGPU_NO_EPI_ALIAS") ? 0 : kEpiSmemBytes;
        if (2 * per > 227 * 1024 - epi - 12 * 1024) {
          a_ok = b_ok = false;
          continue;
        }
      }
      if (a_ok && b_ok) break;
      if (kcs == 64) last_why = a_ok ? wb : wa;
    }
    if (!a_ok) {
      *why = "A: " + last_why;
      return false;
    }
    if (RT != 128 && q.A.mn_major) {
      *why = "A: partial row tiles need a K-major A";
      return false;
    }
    if (!b_ok) {
      last_why = "B: " + last_why;
      continue;
    }
    // Output digits must align with the tile (rows and columns).
    std::vector<int64_t> tmp;
    if (!cover(digits_of(cds, 0), RT, &tmp, &last_why) ||
        !cover(digits_of(cds, 1), BN, &tmp, &last_why)) {
      last_why = "C: " + last_why;
      continue;
    }
    finish_descriptor(&q.A, 128);
    finish_descriptor(&q.B, BN);
    // Multi-slab stages run as KC/64 UMMA groups ("taps") of 4 K-steps, tap t
    // reading slab t: K-major slabs are [rows][64] (rows x 128 B), MN-major
    // ones 64 K rows of 128 B inside each box.
    q.ntaps = kcs / 64;
    q.a_tap.clear();
    q.b_tapv.clear();
    for (int t = 0; t < q.ntaps; ++t) {
      q.a_tap.push_back(t * (q.A.mn_major ? 64 * 128 : 128 * 128));
      q.b_tapv.push_back(t * (q.B.mn_major ? 64 * 128 : BN * 128));
    }
    const int64_t ntile_n = (N + BN - 1) / BN;
    for (int64_t tm = 0; tm < mtiles; ++tm)
      for (int64_t tn = 0; tn < ntile_n; ++tn) {
        TileEntry te;
        std::memset(&te, 0, sizeof(te));
        for (int b = 0; b < q.A.boxes; ++b) {
          int64_t lv[2] = {tm * RT + (q.A.mn_major ? b * 64 : 0), 0};
          coords(ads, ag, am, lv, te.ca[b]);
        }
        for (int b = 0; b < q.B.boxes; ++b) {
          int64_t lv[2] = {0, tn * BN + (q.B.mn_major ? b * 64 : 0)};
          coords(bds, bg, bm, lv, te.cb[b]);
        }
        int64_t lv[2] = {tm * RT, tn * BN};
        te.out_base = offset_of(cds, lv);
        te.rows = static_cast<int32_t>(std::min<int64_t>(RT, M - tm * RT));
        te.cols = static_cast<int32_t>(std::min<int64_t>(BN, N - tn * BN));
        te.n_base = static_cast<int32_t>(tn * BN);
        q.tiles.push_back(te);
      }
    for (int64_t k0 = 0; k0 < K; k0 += kcs) {
      StageEntry se;
      std::memset(&se, 0, sizeof(se));
      int64_t la[2] = {0, k0}, lb[2] = {k0, 0};
      coords(ads, ag, am, la, se.sa);
      coords(bds, bg, bm, lb, se.sb);
      q.stages.push_back(se);
    }
    for (int r = 0; r < 128; ++r) {
      int64_t lv[2] = {r, 0};
      q.row_off.push_back(r < RT ? offset_of(cds, lv) : -1);
    }
    for (int c = 0; c < BN; ++c) {
      int64_t lv[2] = {0, c};
      q.col_off.push_back(offset_of(cds, lv));
    }
    {
      std::vector<std::array<int64_t, 4>> tl, rr(128);
      std::vector<bool> ok(128);
      for (int64_t tm = 0; tm < mtiles; ++tm)
        for (int64_t tn = 0; tn < ntile_n; ++tn) tl.push_back({tm * RT, tn * BN, 0, 0});
      for (int r = 0; r < 128; ++r) {
        rr[r] = {r, 0, 0, 0};
        ok[r] = r < M && r < RT;
      }
      bool full = M % RT == 0 && N % BN == 0;
      if (full) plan_out_store(cds, 2, 1, BN, tl, rr, ok, &q.ost);
    }
    q.pipe = pick_pipe(q);
    std::ostringstream os;
    os << "gemm BM=128" << (RT != 128 ? "(rows " + std::to_string(RT) + ")" : std::string()) << " BN=" << BN << " KC=" << kcs << " A=" << (q.A.mn_major ? "MN" : "K") << "-major B="
       << (q.B.mn_major ? "MN" : "K") << "-major tiles=" << q.tiles.size() << " pipe=" << q.pipe;
    q.summary = os.str();
    q.persistent = s.parallel;
    q.split_pref = s.order;
    q.tma_store = s.vectorize;
    *out = q;
    return true;
  }
  *why = last_why;
  return false;
}

// ---------------------------------------------------------------------------
// C2D: y[b,o,h,w] = sum_{i,rh,rw} x[b,i,V*h+rh,V*w+rw] * ker[o,i,rh,rw]
// (interp.cpp:70-89) as an implicit GEMM over the template layouts.

static bool plan_conv_halo_kc(const std::vector<Dim>& x_log, const std::vector<PDigit>& xd,
                              const std::vector<Dim>& k_log, const std::vector<PDigit>& kd,
                              const std::vector<Dim>& y_log, const std::vector<PDigit>& yd,
                              int64_t V, const lfgpu_sched& s, int64_t kc_cap, UmmaPlan* out,
                              std::string* why);

// The halo plan with the widest channel chunk whose stages fit SMEM (a
// chunk carries the weights of all KH*KW taps, so wide output tiles need
// narrower chunks).
static bool plan_conv_halo(const std::vector<Dim>& x_log, const std::vector<PDigit>& xd,
                           const std::vector<Dim>& k_log, const std::vector<PDigit>& kd,
                           const std::vector<Dim>& y_log, const std::vector<PDigit>& yd,
                           int64_t V, const lfgpu_sched& s, UmmaPlan* out, std::string* why) {
  for (int64_t cap : {64, 32, 16}) {
    if (plan_conv_halo_kc(x_log, xd, k_log, kd, y_log, yd, V, s, cap, out, why)) return true;
    if (why->find("exceed SMEM") == std::string::npos) return false;
  }
  return false;
}

// C2D with the overlapped input tile reused across taps ("halo" path).
//
// The template input brick xp[n][h0][w0][i0][B_h][B_w][i_t] already holds
// every pixel one output tile reads (B = (t-1)V + K, space.cpp:279-280). It
// is loaded ONCE per channel chunk (one TMA box, SWIZZLE_NONE, channel groups
// of 8 outermost: SMEM [group][pixel][8 ch]), and each tap (rh, rw) is a UMMA
// A operand starting rh*B_w + rw pixels into it: UMMA rows are pixels
// y*B_w + x of the tile computed on the B_w-wide grid (columns x >= w_t are
// discarded by the epilogue). The weights of the chunk for all KH*KW taps are
// one TMA box ([KH][KW][i'][o'] is contiguous in the template weight brick).
// Compared with one shifted input box per tap this cuts the input's L2->SMEM
// traffic by ~KH*KW.
static bool plan_conv_halo_kc(const std::vector<Dim>& x_log, const std::vector<PDigit>& xd,
                              const std::vector<Dim>& k_log, const std::vector<PDigit>& kd,
                              const std::vector<Dim>& y_log, const std::vector<PDigit>& yd,
                              int64_t V, const lfgpu_sched& s, int64_t kc_cap, UmmaPlan* out,
                              std::string* why) {
  const int64_t N = y_log[0].extent, O = y_log[1].extent, Ho = y_log[2].extent,
                Wo = y_log[3].extent, I = x_log[1].extent, KH = k_log[2].extent,
                KW = k_log[3].extent;
  if (V != 1 || KH * KW < 2 || KH * KW > kMaxTaps) {
    *why = "halo path: stride 1, 2..32 taps";
    return false;
  }
  auto yh = digits_of(yd, 2), yw = digits_of(yd, 3), yo = digits_of(yd, 1);
  if (yh.size() > 2 || yw.size() > 2 || yo.size() > 2 || digits_of(yd, 0).size() != 1) {
    *why = "halo path: output is not a one-level template layout";
    return false;
  }
  const int64_t h_t = yh[0]->ext, w_t = yw[0]->ext, o_t = yo[0]->ext;
  // Input: N, H0, W0, I0, Hoff, Woff, i_t (H/W either unfolded with S = t,
  // B = t + K - 1, or whole with extent = out + K - 1).
  struct Ax {
    int tile = -1, off = -1;
  } ah, aw;
  int an = -1, ai0 = -1, ai1 = -1;
  for (size_t k = 0; k < xd.size(); ++k) {
    const PDigit& d = xd[k];
    if (d.lj == 0) an = static_cast<int>(k);
    else if (d.lj == 1) (d.div == 1 ? ai1 : ai0) = static_cast<int>(k);
    else {
      Ax& a = d.lj == 2 ? ah : aw;
      if (d.kind == DG_TILE) a.tile = static_cast<int>(k);
      else a.off = static_cast<int>(k);  // DG_OFF, or the whole dim (DG_PART)
    }
  }
  const int nk = static_cast<int>(xd.size());
  if (ai1 != nk - 1 || ah.off < 0 || aw.off < 0 || xd[ai1].ext % 16 || !(ah.off < aw.off)) {
    *why = "halo path: input needs H outside W outside an innermost i_t brick";
    return false;
  }
  const int64_t i_t = xd[ai1].ext;
  const int64_t B_h = xd[ah.off].ext, B_w = xd[aw.off].ext;
  auto fits = [&](const Ax& a, int64_t t, int64_t out_ext, int64_t K, int64_t Bx) {
    const PDigit& o = xd[a.off];
    if (a.tile >= 0) return xd[a.tile].kind == DG_TILE && o.kind == DG_OFF && o.S == t && Bx == t + K - 1;
    return o.kind == DG_PART && o.div == 1 && t == out_ext && Bx == out_ext + K - 1;
  };
  if (!fits(ah, h_t, Ho, KH, B_h) || !fits(aw, w_t, Wo, KW, B_w)) {
    *why = "halo path: input tiles do not match the output tile";
    return false;
  }
  if (B_w > 128) {
    *why = "halo path: B_w > 128";
    return false;
  }
  // trans (schedule unroll = 2): output channels are the 128 UMMA rows and
  // the tile's pixels the N columns (up to 256) - for small spatial tiles
  // (deep layers, small batches) this puts 4-8x more work in every UMMA.
  const bool trans = s.unroll == 2;
  int64_t h_sub = std::min<int64_t>(h_t, (trans ? 256 : 128) / B_w);
  // Loop point tile_second (the second-innermost spatial tile, space.cpp:
  // 497-499) caps the output rows per UMMA tile: smaller tiles, more of them
  // (fills the SMs at small batch) at the cost of more halo re-reads.
  if (s.tile_second > 1 && s.tile_second < h_sub) h_sub = s.tile_second;
  if (trans || s.tile_second > 1)  // whole row chunks per tile: every tile has the same shape
    while (h_sub > 1 && h_t % h_sub) --h_sub;
  const int64_t rows_h = h_sub + KH - 1;
  // Weight: [..][KH][KW][i'][o'] (o' innermost: MN-major B) or, when the
  // template leaves O whole (o' == O), [O][I0][KH][KW][i'] (K-major B).
  if (kd.size() < 3) return false;
  const bool b_kmajor = kd.back().lj == 1;
  const size_t kbase = b_kmajor ? kd.size() - 3 : kd.size() - 4;  // index of the KH digit
  if (kd.size() < (b_kmajor ? 3u : 4u)) return false;
  const PDigit& kh_ = kd[kbase];
  const PDigit& kw_ = kd[kbase + 1];
  const PDigit& ki = kd[kbase + 2];
  if (kh_.lj != 2 || kw_.lj != 3 || kh_.ext != KH || kw_.ext != KW || ki.lj != 1 || ki.div != 1 ||
      ki.ext % 16) {
    *why = "halo path: weight brick must end [KH][KW][i'] or [KH][KW][i'][o']";
    return false;
  }
  int ko_outer = -1, ki_outer = -1;  // K-major: the whole-O digit and the I0 digit
  for (size_t k = 0; k < kbase; ++k) {
    if (kd[k].lj == 0) {
      if (ko_outer >= 0) return false;
      ko_outer = static_cast<int>(k);
    } else if (kd[k].lj == 1) {
      if (ki_outer >= 0) return false;
      ki_outer = static_cast<int>(k);
    } else {
      return false;
    }
  }
  if (!b_kmajor) {
    const PDigit& ko = kd.back();
    if (ko.lj != 0 || ko.div != 1 || ko.ext % 16) {
      *why = "halo path: weight o' brick";
      return false;
    }
  } else if (ko_outer < 0 || kd[ko_outer].div != 1 || kd[ko_outer].ext != O) {
    *why = "halo path: K-major weight needs O whole";
    return false;
  }
  const int64_t o2 = b_kmajor ? O : kd.back().ext, i2 = ki.ext;
  int64_t KC = std::gcd(i_t, i2);
  KC = std::min<int64_t>(KC, kc_cap);
  while (KC > 16 && (KC & (KC - 1))) KC /= 2;
  if (KC % 16) {
    *why = "halo path: channel chunk";
    return false;
  }
  int64_t BN = std::min<int64_t>({o_t, o2, 256});
  if (s.tile_last >= 16 && s.tile_last < BN && BN % s.tile_last == 0 && s.tile_last % 16 == 0)
    BN = s.tile_last;
  // MN-major weight boxes are 64 channels wide (128B swizzle), each inside
  // one o' brick; a K-major slab takes all BN rows in one box.
  if (trans) BN = 128;  // weight rows per tile
  const int64_t wbox = b_kmajor ? BN : std::min<int64_t>(BN, 64);
  if (o_t % BN || o2 % wbox || (!b_kmajor && BN > 64 && (BN % 64 || o2 % 64)) || BN % 16 ||
      (!trans && o2 % BN)) {
    *why = "halo path: channel tile";
    return false;
  }
  const int64_t nbw = b_kmajor ? BN : std::min<int64_t>(BN, 64);  // o per weight box
  const int64_t taps = KH * KW;

  UmmaPlan p;
  p.kind = UMMA_CONV;
  p.BM = 128;
  p.BN = static_cast<int>(BN);
  p.KC = static_cast<int>(KC);
  // --- A: box {KC of i_t, B_w (W offsets), rows_h (H offsets)} over the
  // physical digits (other digits box 1, merged into <= 5 TMA dims). SMEM
  // rows are pixels (h, w) of KC*2 bytes in the K-major swizzled canonical
  // layout (swizzle = row bytes), so a tap is a start-address shift of
  // (rh*B_w + rw) rows.
  if (rows_h > 256 || B_w > 256) {
    *why = "halo path: box too large";
    return false;
  }
  std::vector<VDim> xv;
  for (int k = 0; k < nk; ++k) {
    VDim v{xd[k].ext, xd[k].stride, 1, 1};
    if (k == ai1) v.box = KC;
    else if (k == aw.off) v.box = B_w;
    else if (k == ah.off) v.box = rows_h;
    xv.push_back(v);
  }
  std::vector<int> ag;
  std::vector<int64_t> am;
  if (!merge_view(xv, &p.A, &ag, &am, why)) {
    *why = "halo path: " + *why;
    return false;
  }
  // Coordinates of the A box: tile part (n, h0, w0, first H row) and stage
  // part (channel chunk c0: the i0 brick and the offset inside i_t).
  auto coord_a = [&](int64_t n, int64_t h0, int64_t w0, int64_t h1s, int64_t c0, bool tile_part,
                     int32_t* outc) {
    for (int d = 0; d < 5; ++d) outc[d] = 0;
    for (int k = 0; k < nk; ++k) {
      int64_t c = 0;
      if (k == an) c = tile_part ? n : 0;
      else if (k == ah.tile) c = tile_part ? h0 : 0;
      else if (k == aw.tile) c = tile_part ? w0 : 0;
      else if (k == ah.off) c = tile_part ? h1s : 0;
      else if (k == ai0) c = tile_part ? 0 : c0 / i_t;
      else if (k == ai1) c = tile_part ? 0 : c0 % i_t;
      outc[ag[k]] += static_cast<int32_t>(c * am[k]);
    }
  };
  p.A.swizzle = static_cast<int32_t>(KC * 2);
  p.A.mn_major = 0;
  p.A.boxes = 1;
  const int64_t npix = rows_h * B_w;
  const int64_t tapmax = (KH - 1) * B_w + (KW - 1);
  p.A.box_bytes = static_cast<int32_t>(npix * KC * 2);
  const int64_t a_need = std::max(npix, tapmax + 128) * KC * 2;
  p.A.slot_bytes = static_cast<int32_t>((a_need + 1023) / 1024 * 1024);
  p.A.sbo = static_cast<uint32_t>(8 * p.A.swizzle);
  p.A.lbo = 16;
  p.A.k_adv = 32;
  // --- B
  int64_t wbr = 1;
  for (size_t k = 0; k < kbase; ++k) wbr *= kd[k].ext;
  p.B.rank = 5;
  if (!b_kmajor) {
    // {o', i', KW, KH, outer bricks} box {nbw, KC, KW, KH, 1}: per tap a
    // [KC][nbw] MN-major tile.
    p.B.dims[0] = o2;
    p.B.dims[1] = i2;
    p.B.dims[2] = KW;
    p.B.dims[3] = KH;
    p.B.dims[4] = wbr;
    p.B.strides[1] = o2 * 2;
    p.B.strides[2] = i2 * o2 * 2;
    p.B.strides[3] = KW * i2 * o2 * 2;
    p.B.strides[4] = KH * KW * i2 * o2 * 2;
    p.B.box[0] = static_cast<uint32_t>(nbw);
    p.B.box[1] = static_cast<uint32_t>(KC);
    p.B.swizzle = static_cast<int32_t>(nbw * 2);
    p.B.mn_major = 1;
  } else {
    // {i', O, KW, KH, I0} box {KC, BN, KW, KH, 1}: per tap a [BN][KC] K-major
    // tile (the view permutes the O digit inside the taps).
    const int64_t ostride = kd[ko_outer].stride, istride = ki_outer >= 0 ? kd[ki_outer].stride : 0;
    p.B.dims[0] = i2;
    p.B.dims[1] = O;
    p.B.dims[2] = KW;
    p.B.dims[3] = KH;
    p.B.dims[4] = ki_outer >= 0 ? kd[ki_outer].ext : 1;
    p.B.strides[1] = ostride * 2;
    p.B.strides[2] = kw_.stride * 2;
    p.B.strides[3] = kh_.stride * 2;
    p.B.strides[4] = (ki_outer >= 0 ? istride : KH * KW * i2) * 2;
    p.B.box[0] = static_cast<uint32_t>(KC);
    p.B.box[1] = static_cast<uint32_t>(BN);
    p.B.swizzle = static_cast<int32_t>(KC * 2);
    p.B.mn_major = 0;
  }
  p.B.strides[0] = 2;
  p.B.box[2] = static_cast<uint32_t>(KW);
  p.B.box[3] = static_cast<uint32_t>(KH);
  p.B.box[4] = 1;
  for (int d = 1; d < 5; ++d)
    if (p.B.strides[d] % 16) {
      *why = "halo path: weight stride not 16-byte aligned";
      return false;
    }
  p.B.boxes = static_cast<int32_t>(BN / nbw);
  if (p.B.boxes > kMaxBoxes) {
    *why = "halo path: too many weight boxes";
    return false;
  }
  p.B.box_bytes = static_cast<int32_t>(nbw * KC * taps * 2);
  p.B.slot_bytes = (p.B.box_bytes + 1023) / 1024 * 1024;
  p.B.sbo = static_cast<uint32_t>(8 * p.B.swizzle);
  p.B.lbo = b_kmajor ? 16u : static_cast<uint32_t>(p.B.slot_bytes);
  p.B.k_adv = b_kmajor ? 32u : static_cast<uint32_t>(16 * p.B.swizzle);
  p.ntaps = static_cast<int>(taps);
  p.b_tap = static_cast<int>(KC * nbw * 2);
  p.a_tap.clear();
  for (int64_t rh = 0; rh < KH; ++rh)
    for (int64_t rw = 0; rw < KW; ++rw) p.a_tap.push_back(static_cast<int32_t>((rh * B_w + rw) * KC * 2));
  auto wbrick_of = [&](int64_t o, int64_t i) {  // o, i logical; digits outside [KH][KW][i'][o']
    int64_t b = 0;
    for (size_t k = 0; k < kbase; ++k) b = b * kd[k].ext + digit_of(kd[k], kd[k].lj == 0 ? o : i);
    return b;
  };
  auto y_off = [&](int64_t n, int64_t o, int64_t h, int64_t w) {
    int64_t lv[4] = {n, o, h, w};
    return offset_of(yd, lv);
  };
  const int64_t H0 = Ho / h_t, W0 = Wo / w_t, O0 = O / o_t;
  const int64_t hchunks = (h_t + h_sub - 1) / h_sub, ochunks = o_t / BN;
  std::vector<std::array<int64_t, 4>> tile_lv;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t h0 = 0; h0 < H0; ++h0)
      for (int64_t w0 = 0; w0 < W0; ++w0)
        for (int64_t hc = 0; hc < hchunks; ++hc)
          for (int64_t o0 = 0; o0 < O0; ++o0)
            for (int64_t oc = 0; oc < ochunks; ++oc) {
              TileEntry te;
              std::memset(&te, 0, sizeof(te));
              const int64_t h1s = hc * h_sub;
              coord_a(n, h0, w0, h1s, 0, true, te.ca[0]);
              const int64_t obase = o0 * o_t + oc * BN;
              for (int b = 0; b < p.B.boxes; ++b) {
                const int64_t o = obase + b * nbw;
                if (b_kmajor) {
                  te.cb[b][1] = static_cast<int32_t>(o);
                } else {
                  te.cb[b][0] = static_cast<int32_t>(o % o2);
                  te.cb[b][4] = static_cast<int32_t>(wbrick_of(o, 0));
                }
              }
              te.out_base = y_off(n, obase, h0 * h_t + h1s, w0 * w_t);
              tile_lv.push_back({n, obase, h0 * h_t + h1s, w0 * w_t});
              te.org[0] = static_cast<int32_t>(n);
              te.org[1] = static_cast<int32_t>(h0 * h_t + h1s);
              te.org[2] = static_cast<int32_t>(w0 * w_t);
              te.rows = static_cast<int32_t>(std::min<int64_t>(h_sub, h_t - h1s) * B_w);
              te.cols = static_cast<int32_t>(BN);
              te.n_base = static_cast<int32_t>(obase);
              p.tiles.push_back(te);
            }
  for (int64_t c0 = 0; c0 < I; c0 += KC) {
    StageEntry se;
    std::memset(&se, 0, sizeof(se));
    coord_a(0, 0, 0, 0, c0, false, se.sa);
    if (b_kmajor) {
      se.sb[0] = static_cast<int32_t>(c0 % i2);
      se.sb[4] = static_cast<int32_t>(c0 / i2);
    } else {
      se.sb[1] = static_cast<int32_t>(c0 % i2);
      se.sb[4] = static_cast<int32_t>(wbrick_of(0, c0) - wbrick_of(0, 0));
    }
    p.stages.push_back(se);
  }
  // Rows: UMMA row r = pixel (r / B_w, r % B_w) of the B_w-wide grid; columns
  // x >= w_t are not outputs (-1).
  const int64_t base0 = y_off(0, 0, 0, 0);
  for (int r = 0; r < 128; ++r) {
    const int64_t hh = r / B_w, ww = r % B_w;
    p.row_off.push_back(hh < h_sub && ww < w_t ? y_off(0, 0, hh, ww) - base0 : -1);
    p.row_rel.push_back(static_cast<int32_t>((hh << 16) | ww));
  }
  for (int c = 0; c < BN; ++c) p.col_off.push_back(y_off(0, c, 0, 0) - base0);
  if (h_t % h_sub == 0) {
    std::vector<std::array<int64_t, 4>> rr(128);
    std::vector<bool> ok(128);
    for (int r = 0; r < 128; ++r) {
      rr[r] = {0, 0, r / B_w, r % B_w};
      ok[r] = p.row_off[r] >= 0;
    }
    plan_out_store(yd, 4, 1, static_cast<int>(BN), tile_lv, rr, ok, &p.ost);
  }
  if (trans) {
    // Swap roles: A = the weight slabs (128 channel rows per tile), B = the
    // overlapped input tile (pixel rows, shifted per tap); the runtime binds
    // the operand buffers accordingly (swap_ab). The accumulator is
    // [channel][pixel]: rows = channels, columns = pixels of the B_w-wide
    // grid (x >= w_t and padding columns are not outputs).
    const int64_t npad = (h_sub * B_w + 15) / 16 * 16;
    const int64_t slab = p.b_tap;  // bytes of one tap's weight slab (per box)
    std::swap(p.A, p.B);
    p.swap_ab = 1;
    p.B.slot_bytes = static_cast<int32_t>(
        (std::max(npix, tapmax + npad) * KC * 2 + 1023) / 1024 * 1024);
    p.b_tapv = p.a_tap;
    p.a_tap.clear();
    for (int64_t t = 0; t < taps; ++t) p.a_tap.push_back(static_cast<int32_t>(t * slab));
    p.b_tap = 0;
    for (auto& te : p.tiles) {
      int32_t tmp[kMaxBoxes][5];
      std::memcpy(tmp, te.ca, sizeof(tmp));
      std::memcpy(te.ca, te.cb, sizeof(tmp));
      std::memcpy(te.cb, tmp, sizeof(tmp));
      te.rows = 128;
      te.cols = static_cast<int32_t>(npad);
    }
    for (auto& se : p.stages) {
      int32_t tmp[5];
      std::memcpy(tmp, se.sa, sizeof(tmp));
      std::memcpy(se.sa, se.sb, sizeof(tmp));
      std::memcpy(se.sb, tmp, sizeof(tmp));
    }
    p.row_off.clear();
    p.col_off.clear();
    p.row_rel.assign(128, 0);
    for (int r = 0; r < 128; ++r) p.row_off.push_back(y_off(0, r, 0, 0) - base0);
    for (int64_t c = 0; c < npad; ++c) {
      const int64_t hh = c / B_w, ww = c % B_w;
      p.col_off.push_back(hh < h_sub && ww < w_t ? y_off(0, 0, hh, ww) - base0 : -1);
    }
    p.BN = static_cast<int>(npad);
    p.trans = 1;
    p.ost = OutStore();
  }
  if (!umma_view_encodable(p.A, why) || !umma_view_encodable(p.B, why)) {
    *why = "halo path: " + *why;
    return false;
  }
  p.pipe = pick_pipe(p);
  {
    const int64_t need = 2LL * (p.A.boxes * p.A.slot_bytes + p.B.boxes * p.B.slot_bytes) + 1024 + 512 +
                         kEpiSmemBytes + sizeof(StageEntry) * p.stages.size() + 8 * BN + 8 * 128;
    if (need > 227 * 1024) {
      *why = "halo path: two stages exceed SMEM";
      return false;
    }
  }
  {
    // Weights resident when the layer has one output-channel tile and all
    // its chunks' slabs fit beside a >= 3-deep input ring.
    const int64_t wbytes = static_cast<int64_t>(p.stages.size()) * p.B.boxes * p.B.slot_bytes;
    const int64_t fixed = 1024 + 512 + kEpiSmemBytes + 8 * static_cast<int64_t>(p.stages.size()) * 6 +
                          static_cast<int64_t>(sizeof(StageEntry) * p.stages.size() + 8 * p.col_off.size() + 8 * 128);
    const int64_t budget = 227 * 1024 - fixed - wbytes;
    const char* e = getenv("LFGPU_NO_WRES");
    if (!trans && O0 * ochunks == 1 && !(e && atoi(e)) && budget >= 3 * p.A.slot_bytes) {
      p.wres = 1;
      p.pipe = static_cast<int>(std::min<int64_t>(8, budget / p.A.slot_bytes));
    }
  }
  p.persistent = s.parallel;
  p.split_pref = s.order;
  p.tma_store = s.vectorize;
  std::ostringstream os;
  os << (p.wres ? "conv-halo-wres" : trans ? "conv-halo-trans" : "conv-halo") << " h_t=" << h_t << " w_t=" << w_t << " o_t=" << o_t << " i_t=" << i_t << " i'=" << i2
     << " o'=" << o2 << " rows=" << h_sub << "x" << B_w << " BN=" << BN << " KC=" << KC
     << " taps=" << taps << " tiles=" << p.tiles.size() << " stages=" << p.stages.size()
     << " pipe=" << p.pipe;
  p.summary = os.str();
  *out = p;
  return true;
}

bool umma_plan_conv(const std::vector<Dim>& x_log, const Seq& x_seq, const std::vector<Dim>& k_log,
                    const Seq& k_seq, const std::vector<Dim>& y_log, const Seq& y_seq,
                    int64_t V, const lfgpu_sched& s, UmmaPlan* out, std::string* why) {
  const int64_t N = y_log[0].extent, O = y_log[1].extent, Ho = y_log[2].extent,
                Wo = y_log[3].extent, I = x_log[1].extent, KH = k_log[2].extent,
                KW = k_log[3].extent;
  std::vector<PDigit> xd, kd, yd;
  if (!analyze(x_log, x_seq, &xd) || !analyze(k_log, k_seq, &kd) || !analyze(y_log, y_seq, &yd)) {
    *why = "layouts are not template brick layouts";
    return false;
  }
  std::string halo_why;
  {
    const char* e = getenv("LFGPU_NO_HALO");
    std::string hwhy;
    if (!(e && atoi(e)) && s.unroll != 1 &&
        plan_conv_halo(x_log, xd, k_log, kd, y_log, yd, V, s, out, &hwhy))
      return true;
    halo_why = hwhy.empty() ? "off" : hwhy;
  }
  if (V > 8) {
    *why = "stride > 8 exceeds TMA traversal stride";
    return false;
  }
  // Output tiling: innermost digits of H, W, O.
  auto yh = digits_of(yd, 2), yw = digits_of(yd, 3), yo = digits_of(yd, 1);
  const int64_t h_t = yh[0]->ext, w_t = yw[0]->ext, o_t = yo[0]->ext;
  if (yh.size() > 2 || yw.size() > 2 || yo.size() > 2 || digits_of(yd, 0).size() != 1) {
    *why = "output is not a one-level template layout";
    return false;
  }
  for (const auto& d : yd)
    if (d.kind != DG_PART) {
      *why = "unfolded output";
      return false;
    }
  if (w_t > 128) {
    *why = "w_t > 128 rows";
    return false;
  }
  int64_t h_sub = std::min<int64_t>(h_t, 128 / w_t);
  if (s.tile_second > 1 && s.tile_second < h_sub) {  // loop point tile_second: rows per tile cap
    h_sub = s.tile_second;
    while (h_sub > 1 && h_t % h_sub) --h_sub;
  }
  if (h_sub * V > 256 || w_t * V > 256) {
    *why = "TMA box exceeds 256";
    return false;
  }
  // Input: innermost = I inner brick.
  const PDigit& xi = xd.back();
  if (xi.lj != 1 || xi.kind != DG_PART || xi.div != 1 || xi.ext % 16) {
    *why = "input channel brick i_t must be innermost and a multiple of 16";
    return false;
  }
  const int64_t i_t = xi.ext;
  // Weight: innermost = O inner brick (MN-major B, the template's o' when
  // o' < O) or the I inner brick (K-major B, when o' == O leaves O whole).
  const PDigit& ko = kd.back();
  const bool b_kmajor = ko.lj == 1;
  if ((ko.lj != 0 && ko.lj != 1) || ko.kind != DG_PART || ko.div != 1 || ko.ext % 16) {
    *why = "weight innermost brick must be o' or i' and a multiple of 16";
    return false;
  }
  const int64_t o2 = b_kmajor ? 64 : ko.ext;  // K-major: O rows, no swizzle constraint on N
  auto ki = digits_of(kd, 1);
  const int64_t i2 = ki[0]->ext;
  if (i2 % 16) {
    *why = "weight input-channel brick i' must be a multiple of 16";
    return false;
  }
  int64_t KC = std::gcd(i_t, i2);
  KC = std::min<int64_t>(KC, 64);
  while (KC > 16 && (KC & (KC - 1))) KC /= 2;
  if (KC != 16 && KC != 32 && KC != 64) {
    *why = "channel chunk not in {16,32,64}";
    return false;
  }
  // Channel tile of the CTA (UMMA N).
  int64_t BN = std::min<int64_t>(o_t, 256);
  if (s.tile_last >= 16 && s.tile_last < BN && o_t % s.tile_last == 0 && s.tile_last % 16 == 0)
    BN = s.tile_last;
  if (o_t % BN || BN % 16) {
    *why = "channel tile not a multiple of 16";
    return false;
  }
  const int64_t bn_sw = std::min<int64_t>(o2 * 2, 128);  // B swizzle bytes
  const int64_t nbox = bn_sw / 2;                       // n per B box
  if (BN % nbox) {
    *why = "channel tile does not align with the weight brick";
    return false;
  }

  UmmaPlan p;
  p.kind = UMMA_CONV;
  p.BM = 128;
  p.BN = static_cast<int>(BN);
  p.KC = static_cast<int>(KC);

  // --- A view (input): boxes and coordinate recipes per phys digit.
  std::vector<VDim> xv;
  for (const auto& d : xd) {
    VDim v{d.ext, d.stride, 1, 1};
    if (d.lj == 1 && d.div == 1 && &d == &xd.back()) v.box = KC;
    if ((d.lj == 2 || d.lj == 3) && (d.kind == DG_OFF || d.kind == DG_PART)) {
      if (d.kind == DG_PART && (d.div != 1 || d.ext != x_log[d.lj].extent)) {
        *why = "input H/W split without unfold";
        return false;
      }
      int64_t rows = d.lj == 2 ? h_sub : w_t;
      v.box = rows * V;
      v.estride = V;
    }
    if (d.kind == DG_TILE || d.kind == DG_OFF) {
      int64_t t = d.lj == 2 ? h_t : w_t;
      int64_t Bneed = (t - 1) * V + (d.lj == 2 ? KH : KW);
      if (d.S != t * V || (d.kind == DG_OFF && d.ext < Bneed)) {
        *why = "input unfold does not match the output tile";
        return false;
      }
    }
    xv.push_back(v);
  }
  // SMEM rows of the A box come out in the physical order of the H and W
  // row dims: (h, w) when H is outer (the template), (w, h) when an untiled
  // W dim sits outside the H tile (decode_layout with w_t == W).
  bool h_outer = true;
  {
    int hpos = -1, wpos = -1;
    for (size_t k = 0; k + 1 < xd.size(); ++k) {
      if (xv[k].box > 1 && xd[k].lj == 2) hpos = static_cast<int>(k);
      if (xv[k].box > 1 && xd[k].lj == 3) wpos = static_cast<int>(k);
    }
    if (hpos >= 0 && wpos >= 0 && hpos > wpos) h_outer = false;
    if (!h_outer && h_t % h_sub != 0) {
      *why = "W-outer input needs whole H chunks";
      return false;
    }
  }
  std::vector<int> ag;
  std::vector<int64_t> am;
  p.A.mn_major = 0;
  p.A.swizzle = static_cast<int32_t>(KC * 2);
  p.A.boxes = 1;
  if (!merge_view(xv, &p.A, &ag, &am, why)) return false;
  finish_descriptor(&p.A, 128);

  // --- B view (weight). MN-major: o' contiguous, k rows over i'.
  // K-major: i' contiguous (KC per box row), BN rows over the O digits.
  std::vector<VDim> kv;
  std::vector<int64_t> obox;
  if (b_kmajor) {
    auto od = digits_of(kd, 0);
    if (!cover(od, BN, &obox, why)) return false;
  }
  for (size_t k = 0; k < kd.size(); ++k) {
    const PDigit& d = kd[k];
    VDim v{d.ext, d.stride, 1, 1};
    if (!b_kmajor && k + 1 == kd.size()) v.box = nbox;
    if (d.lj == 1 && d.div == 1) {
      if (d.ext % KC) {
        *why = "weight channel brick";
        return false;
      }
      v.box = KC;
    }
    if (b_kmajor && d.lj == 0) {
      auto od = digits_of(kd, 0);
      for (size_t q = 0; q < od.size(); ++q)
        if (od[q] == &d) v.box = obox[q];
    }
    kv.push_back(v);
  }
  std::vector<int> bg;
  std::vector<int64_t> bm;
  p.B.mn_major = b_kmajor ? 0 : 1;
  p.B.swizzle = static_cast<int32_t>(b_kmajor ? KC * 2 : bn_sw);
  p.B.boxes = b_kmajor ? 1 : static_cast<int32_t>(BN / nbox);
  if (p.B.boxes > kMaxBoxes) {
    *why = "too many weight boxes";
    return false;
  }
  {
    // MN-major: exactly one row dim (i'); K-major: the O digits, in order.
    std::vector<int64_t> bx;
    int rows_dims = 0;
    for (size_t k = 0; k < kd.size(); ++k) {
      bx.push_back(kv[k].box);
      if (k + 1 < kd.size() && kv[k].box > 1) ++rows_dims;
    }
    if ((!b_kmajor && rows_dims != 1) || (b_kmajor && !rows_ordered(kd, bx))) {
      *why = "weight brick rows not contiguous";
      return false;
    }
  }
  if (!merge_view(kv, &p.B, &bg, &bm, why)) return false;
  finish_descriptor(&p.B, static_cast<int>(BN));

  // --- tiles
  const int64_t H0 = Ho / h_t, W0 = Wo / w_t, O0 = O / o_t;
  const int64_t hchunks = (h_t + h_sub - 1) / h_sub, ochunks = o_t / BN;
  auto coord_x = [&](int64_t n, int64_t h0, int64_t w0, int64_t h1s, int64_t c0, int64_t rh,
                     int64_t rw, bool tile_part, int32_t* outc) {
    for (int d = 0; d < 5; ++d) outc[d] = 0;
    for (size_t k = 0; k < xd.size(); ++k) {
      const PDigit& d = xd[k];
      int64_t c = 0;
      if (d.lj == 0) c = tile_part ? n : 0;
      else if (d.lj == 1) c = tile_part ? 0 : digit_of(d, c0);
      else {
        int64_t t0 = d.lj == 2 ? h0 : w0, s1 = d.lj == 2 ? h1s : 0, r = d.lj == 2 ? rh : rw;
        int64_t tt = d.lj == 2 ? h_t : w_t;
        if (d.kind == DG_TILE) c = tile_part ? t0 : 0;
        else if (d.kind == DG_OFF) c = tile_part ? V * s1 : r;
        else c = tile_part ? V * (t0 * tt + s1) : r;  // whole dim
      }
      outc[ag[k]] += static_cast<int32_t>(c * am[k]);
    }
  };
  auto coord_k = [&](int64_t o, int64_t c0, int64_t rh, int64_t rw, bool tile_part,
                     int32_t* outc) {
    for (int d = 0; d < 5; ++d) outc[d] = 0;
    for (size_t k = 0; k < kd.size(); ++k) {
      const PDigit& d = kd[k];
      int64_t c = 0;
      if (d.lj == 0) c = tile_part ? digit_of(d, o) : 0;
      else if (d.lj == 1) c = tile_part ? 0 : digit_of(d, c0);
      else if (d.lj == 2) c = tile_part ? 0 : digit_of(d, rh);
      else c = tile_part ? 0 : digit_of(d, rw);
      outc[bg[k]] += static_cast<int32_t>(c * bm[k]);
    }
  };
  auto y_off = [&](int64_t n, int64_t o, int64_t h, int64_t w) {
    int64_t lv[4] = {n, o, h, w};
    return offset_of(yd, lv);
  };
  std::vector<std::array<int64_t, 4>> tile_lv;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t h0 = 0; h0 < H0; ++h0)
      for (int64_t w0 = 0; w0 < W0; ++w0)
        for (int64_t hc = 0; hc < hchunks; ++hc)
          for (int64_t o0 = 0; o0 < O0; ++o0)
            for (int64_t oc = 0; oc < ochunks; ++oc) {
              TileEntry te;
              std::memset(&te, 0, sizeof(te));
              int64_t h1s = hc * h_sub;
              coord_x(n, h0, w0, h1s, 0, 0, 0, true, te.ca[0]);
              int64_t obase = o0 * o_t + oc * BN;
              for (int b = 0; b < p.B.boxes; ++b) coord_k(obase + b * nbox, 0, 0, 0, true, te.cb[b]);
              te.out_base = y_off(n, obase, h0 * h_t + h1s, w0 * w_t);
              tile_lv.push_back({n, obase, h0 * h_t + h1s, w0 * w_t});
              te.org[0] = static_cast<int32_t>(n);
              te.org[1] = static_cast<int32_t>(h0 * h_t + h1s);
              te.org[2] = static_cast<int32_t>(w0 * w_t);
              te.rows = static_cast<int32_t>(std::min<int64_t>(h_sub, h_t - h1s) * w_t);
              te.cols = static_cast<int32_t>(BN);
              te.n_base = static_cast<int32_t>(obase);
              p.tiles.push_back(te);
            }
  for (int64_t c0 = 0; c0 < I; c0 += KC)
    for (int64_t rh = 0; rh < KH; ++rh)
      for (int64_t rw = 0; rw < KW; ++rw) {
        StageEntry se;
        std::memset(&se, 0, sizeof(se));
        coord_x(0, 0, 0, 0, c0, rh, rw, false, se.sa);
        coord_k(0, c0, rh, rw, false, se.sb);
        p.stages.push_back(se);
      }
  // Rows: r -> (hh, ww) inside the tile; offsets relative to the tile base.
  const int64_t base0 = y_off(0, 0, 0, 0);
  for (int r = 0; r < 128; ++r) {
    int64_t hh = h_outer ? r / w_t : r % h_sub;
    int64_t ww = h_outer ? r % w_t : r / h_sub;
    if (hh >= h_sub || ww >= w_t) hh = 0, ww = 0;
    p.row_off.push_back(y_off(0, 0, hh, ww) - base0);
    p.row_rel.push_back(static_cast<int32_t>((hh << 16) | ww));
  }
  for (int c = 0; c < BN; ++c) p.col_off.push_back(y_off(0, c, 0, 0) - base0);
  if (h_t % h_sub == 0) {
    std::vector<std::array<int64_t, 4>> rr(128);
    std::vector<bool> ok(128);
    for (int r = 0; r < 128; ++r) {
      const int64_t hh = h_outer ? r / w_t : r % h_sub, ww = h_outer ? r % w_t : r / h_sub;
      rr[r] = {0, 0, hh, ww};
      ok[r] = r < h_sub * w_t;
    }
    plan_out_store(yd, 4, 1, static_cast<int>(BN), tile_lv, rr, ok, &p.ost);
  }
  p.pipe = pick_pipe(p);
  p.persistent = s.parallel;
  p.split_pref = s.order;
  p.tma_store = s.vectorize;
  std::ostringstream os;
  os << "conv h_t=" << h_t << " w_t=" << w_t << " o_t=" << o_t << " i_t=" << i_t << " i'=" << i2
     << " o'=" << o2 << " rows=" << h_sub * w_t << " BN=" << BN << " KC=" << KC
     << " tiles=" << p.tiles.size() << " stages=" << p.stages.size() << " pipe=" << p.pipe
     << " (halo: " << halo_why << ")";
  p.summary = os.str();
  *out = p;
  return true;
}

bool umma_scatter_desc(const std::vector<Dim>& xp_log, const Seq& xp_seq, int64_t pad,
                       ScatterDesc* sd, std::string* why) {
  std::vector<PDigit> ds;
  if (xp_log.size() != 4 || !analyze(xp_log, xp_seq, &ds)) {
    *why = "padded layout is not a brick layout";
    return false;
  }
  ScatterDesc d;
  d.pad = static_cast<int32_t>(pad);
  int nN = 0, nC = 0;
  for (const auto& g : ds) {
    switch (g.lj) {
      case 0:
        if (g.kind != DG_PART || g.div != 1) return *why = "N split", false;
        d.sN = g.stride;
        ++nN;
        break;
      case 1:
        if (g.kind != DG_PART) return *why = "C unfolded", false;
        if (g.div == 1) {
          d.sC1 = g.stride;
          d.ic = static_cast<int32_t>(g.ext);
        } else {
          d.sC0 = g.stride;
        }
        ++nC;
        break;
      default: {
        const bool h = g.lj == 2;
        const int64_t D = xp_log[g.lj].extent;
        if (g.kind == DG_PART) {
          if (g.div != 1 || g.ext != D) return *why = "H/W split without unfold", false;
          (h ? d.sHo : d.sWo) = g.stride;
        } else if (g.kind == DG_TILE) {
          (h ? d.sHt : d.sWt) = g.stride;
          (h ? d.Th : d.Tw) = static_cast<int32_t>(g.ext);
          (h ? d.Sh : d.Sw) = static_cast<int32_t>(g.S);
        } else {
          (h ? d.sHo : d.sWo) = g.stride;
          (h ? d.Bh : d.Bw) = static_cast<int32_t>(g.ext);
        }
      }
    }
  }
  if (nN != 1 || nC < 1 || nC > 2) return *why = "N/C digits", false;
  if (nC == 1 && d.sC1 == 0) return *why = "C digit", false;
  // Exact unfold tilings only (no clamped overhang duplicates).
  for (int k = 0; k < 2; ++k) {
    const int64_t D = xp_log[2 + k].extent;
    const int64_t T = k ? d.Tw : d.Th, B = k ? d.Bw : d.Bh, S = k ? d.Sw : d.Sh;
    if (T > 1 && (T - 1) * S + B != D) return *why = "unfold with overhang", false;
    if (T == 1 && B == 1) {  // whole dim: one 'tile' covering it
      if (k) d.Bw = static_cast<int32_t>(D);
      else d.Bh = static_cast<int32_t>(D);
    }
  }
  d.enabled = 1;
  *sd = d;
  return true;
}

// ---------------------------------------------------------------------------
// CTA-pair GEMM (k_pair.cu): 256 x BN tiles, cta_group::2, K splits in one
// cluster. Same brick analysis as umma_plan_gemm; A is viewed in 128-row
// boxes (one per CTA of the pair), B in BN/2-column boxes.

bool pair_plan_gemm(const std::vector<Dim>& a_log, const Seq& a_seq, const std::vector<Dim>& b_log,
                    const Seq& b_seq, const std::vector<Dim>& c_log, const Seq& c_seq,
                    const lfgpu_sched& s, PairPlan* out, std::string* why) {
  const int64_t M = a_log[0].extent, K = a_log[1].extent, N = b_log[1].extent;
  if (M % 256 || K % 64) {
    *why = "pair GEMM needs M % 256 == 0 and K % 64 == 0";
    return false;
  }
  std::vector<PDigit> cds;
  if (!analyze(c_log, c_seq, &cds)) {
    *why = "output layout is not a brick layout";
    return false;
  }
  const int sms = 148;
  // K per stage as in the 1-CTA kernel (umma_plan_gemm): several 64-wide K
  // slabs per TMA box when the layouts and two stages of SMEM allow.
  int kcs_pref = 256;
  if (const char* e = getenv("LFGPU_GEMM_KCS")) kcs_pref = atoi(e);
  if (kcs_pref != 64 && kcs_pref != 128 && kcs_pref != 256) kcs_pref = 64;
  int force_bn = 0, force_s = 0;
  if (const char* e = getenv("LFGPU_PAIR_BN")) force_bn = atoi(e);
  if (const char* e = getenv("LFGPU_PAIR_S")) force_s = atoi(e);
  if (!force_bn && (s.tile_last == 64 || s.tile_last == 128 || s.tile_last == 256)) force_bn = s.tile_last;
  struct Cand {
    int BN, S;
    double cost;
  };
  std::vector<Cand> cands;
  std::string last_why = "no legal pair tile";
  PairPlan best;
  double best_cost = 1e300;
  for (int BN : {256, 128, 64}) {
    if (force_bn && BN != force_bn) continue;
    if (N % BN) {
      last_why = "N not a multiple of the pair tile";
      continue;
    }
    // Multi-slab stages only for short K loops: deeper rings of 64-wide
    // stages win once the tensor pipe binds (2048^3 and up, measured).
    bool found = false;
    for (int kcs = K <= 1024 ? kcs_pref : 64; kcs >= 64 && !found; kcs /= 2) {
      if (K % kcs) continue;
      PairPlan q;
      q.BN = BN;
      std::vector<PDigit> ads, bds;
      std::vector<int64_t> abox, bbox, tmp;
      std::vector<int> ag, bg;
      std::vector<int64_t> am, bm;
      {
        std::string wa, wb;
        if (!gemm_operand(a_log, a_seq, 0, 1, 128, kcs, &q.A, &ads, &abox, &ag, &am, &wa)) {
          if (kcs == 64) {
            *why = "A: " + wa;
            return false;
          }
          continue;
        }
        if (!gemm_operand(b_log, b_seq, 1, 0, BN / 2, kcs, &q.B, &bds, &bbox, &bg, &bm, &wb)) {
          last_why = "B: " + wb;
          continue;
        }
      }
      const int KS = static_cast<int>(K / kcs);
      q.slabs = kcs / 64;
      q.a_slab = q.A.mn_major ? 64 * 128 : 128 * 128;
      q.b_slab = q.B.mn_major ? 64 * 128 : (BN / 2) * 128;
      if (!cover(digits_of(cds, 0), 128, &tmp, &last_why) ||
          !cover(digits_of(cds, 1), BN, &tmp, &last_why)) {
        last_why = "C: " + last_why;
        continue;
      }
      finish_descriptor(&q.A, 128);
      finish_descriptor(&q.B, BN / 2);
      q.MT = static_cast<int>(M / 128);
      q.NT = static_cast<int>(N / BN);
      q.KS = KS;
      for (int mi = 0; mi < q.MT; ++mi)
        for (int b = 0; b < q.A.boxes; ++b) {
          int64_t lv[2] = {mi * 128 + (q.A.mn_major ? b * 64 : 0), 0};
          int32_t c[5];
          coords(ads, ag, am, lv, c);
          q.a_crd.insert(q.a_crd.end(), c, c + 5);
        }
      for (int nb = 0; nb < 2 * q.NT; ++nb)
        for (int b = 0; b < q.B.boxes; ++b) {
          int64_t lv[2] = {0, static_cast<int64_t>(nb) * (BN / 2) + (q.B.mn_major ? b * 64 : 0)};
          int32_t c[5];
          coords(bds, bg, bm, lv, c);
          q.b_crd.insert(q.b_crd.end(), c, c + 5);
        }
      for (int64_t k0 = 0; k0 < K; k0 += kcs) {
        int64_t la[2] = {0, k0}, lb[2] = {k0, 0};
        int32_t ca[5], cb[5];
        coords(ads, ag, am, la, ca);
        coords(bds, bg, bm, lb, cb);
        q.s_crd.insert(q.s_crd.end(), ca, ca + 5);
        q.s_crd.insert(q.s_crd.end(), cb, cb + 5);
      }
      for (int mi = 0; mi < q.MT; ++mi) {
        int64_t lv[2] = {static_cast<int64_t>(mi) * 128, 0};
        q.out_r.push_back(offset_of(cds, lv));
      }
      for (int nj = 0; nj < q.NT; ++nj) {
        int64_t lv[2] = {0, static_cast<int64_t>(nj) * BN};
        q.out_c.push_back(offset_of(cds, lv));
      }
      for (int r = 0; r < 128; ++r) {
        int64_t lv[2] = {r, 0};
        q.row_off.push_back(offset_of(cds, lv));
      }
      for (int c = 0; c < BN; ++c) {
        int64_t lv[2] = {0, c};
        q.col_off.push_back(offset_of(cds, lv));
      }
      const int stage = q.A.slot_bytes * q.A.boxes + q.B.slot_bytes * q.B.boxes;
      // 227 KB minus alignment slack, 4 epilogue transpose buffers and barriers.
      if (q.MT + q.NT > 4096) {
        last_why = "pair GEMM output tables exceed SMEM";
        continue;
      }
      const int budget = 227 * 1024 - 1024 - 8 * 32 * 36 * 4 - 512 -
                         static_cast<int>(pair_table_bytes(KS, q.MT, q.NT, BN, q.A.boxes, q.B.boxes));
      const int tiles = q.MT / 2 * q.NT;
      for (int S : {1, 2, 4}) {
        // Split K with one tile per cluster exchanges partials over DSMEM: a
        // dedicated receive buffer of (S-1) x 128 x BN/S fp32 (the send
        // staging aliases the idle operand ring).
        const bool dsm0 = S > 1 && tiles <= sms / (2 * S) && !getenv("LFGPU_PAIR_NO_DSMEM");
        const int rx = (S - 1) * 128 * (BN / S) * 4;
        // send staging: each epilogue warp stages its chunks of the sibling
        // slices in the idle operand ring
        const int staging = ((BN / 64) * (S - 1) + S - 1) / S * 8 * 4096;
        constexpr int kEpi = 8 * 32 * 36 * 4;
        // Ring depth and exchange mode for a budget; with `al` the epilogue's
        // transpose buffers live in the idle ring behind the send staging
        // (one tile per cluster), freeing their 36 KB for the ring.
        auto layout = [&](bool al, int* pipe_o, bool* dsm_o) {
          const int bud = budget + (al ? kEpi : 0);
          bool d = dsm0;
          int pp = std::max(2, std::min(8, (bud - (d ? rx : 0)) / stage));
          if (d && pp * stage < staging) {
            d = false;
            pp = std::max(2, std::min(8, bud / stage));
          }
          if (al && pp * stage < (d ? staging : 0) + kEpi) return false;
          *pipe_o = pp;
          *dsm_o = d;
          return bud - (d ? rx : 0) >= 2 * stage;  // two stages must fit
        };
        bool dsm = false, fits = false;
        int pp = 2;
        q.epi_alias = 0;
        if (tiles <= sms / (2 * S) && !getenv("LFGPU_PAIR_NO_EPI_ALIAS") && layout(true, &pp, &dsm)) {
          q.epi_alias = 1;
          fits = true;
        } else {
          fits = layout(false, &pp, &dsm);
        }
        q.rx_bytes = dsm ? rx : 0;
        q.pipe = pp;
        if (const char* e = getenv("LFGPU_PAIR_PIPE")) q.pipe = std::max(2, std::min(q.pipe, atoi(e)));
        if (force_s && S != force_s) continue;
        if (!force_s && s.order == 1 && S > 1) continue;
        if (!force_s && s.order == 2 && S < 2) continue;
        if (KS % S || (BN / S) % 32) continue;
        // Measured: with S > 1 (clusters of 4-8 CTAs) a second TMA box per
        // operand in the second and later pairs of a cluster reads wrong data
        // (MN-major B with BN/2 = 128, tests/test_gpu_pair.py); the first pair
        // and K-major single-box operands are exact. Split only single-box tiles.
        if (S > 1 && (q.A.boxes > 1 || q.B.boxes > 1)) continue;
        if (S > 1 && KS / S < 2) continue;
        if (!fits) continue;
        found = true;
        // Cost model (cycles): waves x stages x max(MMA, ingest) + epilogue
        // + split reduction + fixed latency. Ingest assumed ~48 B/clk/SM.
        const int clusters = std::max(1, std::min(tiles, sms / (2 * S)));
        const int waves = (tiles + clusters - 1) / clusters;
        const double per_stage = std::max(2.0 * BN * q.slabs, stage / 48.0);
        const double epi = 128.0 * BN * 4 / 64.0;
        const double red = S == 1 ? 0.0
                           : dsm ? ((S - 1.0) * 128 * BN / S * 4) / 20.0
                                 : (2.0 * 128 * BN * 4 + (S + 1.0) * 128 * BN / S * 4) / 64.0;
        const double cost = waves * ((KS / S) * per_stage + epi + red) + 2500.0;
        if (cost < best_cost) {
          best_cost = cost;
          best = q;
          best.S = S;
        }
      }
    }  // kcs
  }
  if (best_cost >= 1e299) {
    *why = last_why;
    return false;
  }
  std::ostringstream os;
  os << "gemm-pair BM=256 BN=" << best.BN << " KC=" << 64 * best.slabs << " S=" << best.S << " A=" << (best.A.mn_major ? "MN" : "K")
     << "-major B=" << (best.B.mn_major ? "MN" : "K") << "-major tiles=" << best.MT / 2 * best.NT
     << " pipe=" << best.pipe;
  best.group = s.parallel ? 1 : 8;
  os << " raster=" << (best.group == 1 ? "rows" : "group8") << (best.epi_alias ? " epi-in-ring" : "");
  best.summary = os.str();
  *out = best;
  return true;
}

}  // namespace lfg
