// lf_core.hpp — host-side layout algebra and the index-map compiler of the
// B200 backend, plus the POD descriptors the CUDA kernels consume.
//
// The reference keeps layouts as primitive sequences and rewrites symbolic
// access expressions (proj/src/layout.cpp:186-335) that its interpreter
// re-evaluates per element (interp.cpp:348-363). Here a sequence is compiled
// ONCE on the host into one of two device descriptors:
//   * DigitMap — the affine "digit" form: the copy space is factored into
//     digits x_d, and dst offset, src offset, zero-predicates and unfold
//     clamps are all linear in the digits. Every layout the tuner emits
//     (split / reorder / unfold, space.cpp:211-401) and the Padding nest on
//     those layouts compile to this; the tiled/vectorised kernels run it.
//   * IxProgram — a general per-element program of split/fuse/perm/fold/
//     unfold/unpad steps, for hand-written sequences the digit form cannot
//     express (fuse across misaligned splits, pads inside splits, ...).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lfgpu.h"

namespace lfg {

constexpr int kMaxRank = LFGPU_MAX_RANK;
constexpr int kMaxDig = 16;    // digits of a DigitMap
constexpr int kMaxPred = 6;    // zero predicates of a DigitMap
constexpr int kMaxClamp = 4;   // unfold clamps of a DigitMap
constexpr int kMaxTab = 4;     // source offset-table terms of a DigitMap
constexpr int kMaxOps = 40;    // steps of an IxProgram

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

// ---------------------------------------------------------------------------
// Layout algebra (lf::apply_primitive_shape / derive_layout / invert_sequence)

struct Dim {
  std::string name;
  int64_t extent = 0;
};

using Prim = lfgpu_prim;
using Seq = std::vector<Prim>;

Prim make_split(int dim, const std::vector<int64_t>& factors);
Prim make_reorder(const std::vector<int>& perm);
Prim make_fuse(int dim, int span);
Prim make_unfold(int dim, int64_t tile, int64_t stride);
Prim make_fold(int dim, int64_t tile, int64_t stride, int64_t orig_extent);
Prim make_pad(int dim, int64_t pad);
Prim make_unpad(int dim, int64_t pad);

int64_t unfold_tiles(int64_t d, int64_t b, int64_t s);
std::vector<Dim> apply_shape(const std::vector<Dim>& dims, const Prim& p);
std::vector<Dim> derive(const std::vector<Dim>& dims, const Seq& seq);
std::vector<int64_t> extents(const std::vector<Dim>& dims);
int64_t numel(const std::vector<Dim>& dims);
Seq invert(const std::vector<Dim>& dims, const Seq& seq);
bool seq_equal(const Seq& a, const Seq& b);
std::string seq_str(const Seq& s);

// ---------------------------------------------------------------------------
// Device descriptors

// General per-element index program. Operates on an index vector.
enum IxKind : int32_t {
  IX_SPLIT = 0,   // v[dim] -> n digits by mixed radix a[0..n)         (split access)
  IX_FUSE = 1,    // v[dim..dim+n) -> one linear index, extents a[0..n)  (fuse access)
  IX_PERM = 2,    // new[j] = old[a[j]]                                  (reorder)
  IX_FOLD = 3,    // v[dim] = v[dim]*a[0] + v[dim+1]; clamp to a[1] if a[1] >= 0
  IX_UNFOLD = 4,  // t = min(v/a[0], a[1]-1), o = v - t*a[0]
  IX_BOUND = 5,   // predicate: a[0] <= v[dim] < a[1], else -> zero (flag 0) or error (flag 1)
  IX_SHIFT = 6    // v[dim] += a[0]
};

struct IxOp {
  int32_t kind;
  int32_t dim;
  int32_t n;
  int32_t flag;
  int32_t a[kMaxRank];
};

struct IxProgram {
  int32_t nops = 0;
  int32_t in_rank = 0;
  int32_t out_rank = 0;
  int32_t reserved = 0;
  int32_t in_ext[kMaxRank] = {};
  int32_t out_ext[kMaxRank] = {};
  IxOp ops[kMaxOps];
};

// The affine digit form. For every digit tuple x (x_d in [0, ext[d])):
//   dst[ sum_d dst_stride[d]*x_d ] =
//     all preds p: lo_p <= pcoef[p].x + pconst_p < hi_p
//       ? src[ src_base + sum_d src_stride[d]*x_d
//              + sum_c cstride_c * min(ccoef[c].x + cconst_c, cmax_c) ]
//       : 0
// When the source sequence is not affine in the digits (a split of a
// shifted / unfolded coordinate), each source logical coordinate l_t is kept
// as an affine (clamped) digit form and looked up in a per-dimension offset
// table: src offset += tab[toff_t + clamp(tcoef[t].x + tconst_t, 0, tmax_t)].
struct DigitMap {
  int32_t ndig = 0;
  int32_t npred = 0;
  int32_t nclamp = 0;
  int32_t ntab = 0;
  int64_t ext[kMaxDig] = {};
  int64_t dst_stride[kMaxDig] = {};
  int64_t src_stride[kMaxDig] = {};
  int64_t src_base = 0;
  int64_t pcoef[kMaxPred][kMaxDig] = {};
  int64_t pconst[kMaxPred] = {};
  int64_t plo[kMaxPred] = {};
  int64_t phi[kMaxPred] = {};
  int64_t ccoef[kMaxClamp][kMaxDig] = {};
  int64_t cconst[kMaxClamp] = {};
  int64_t cmax[kMaxClamp] = {};
  int64_t cstride[kMaxClamp] = {};
  int64_t tcoef[kMaxTab][kMaxDig] = {};
  int64_t tconst[kMaxTab] = {};
  int64_t tmax[kMaxTab] = {};
  int64_t toff[kMaxTab] = {};
  int64_t dst_numel = 0;
};

// How a copy between two layouts of the same logical tensor is described.
// `shift`/`lo`/`hi` express the Padding nest (lower.cpp:228-238): src logical
// j = dst logical j + shift[j], valid iff lo[j] <= dst logical j < hi[j].
struct LogicalMap {
  std::vector<Dim> dst_logical;
  std::vector<Dim> src_logical;
  std::vector<int64_t> shift, lo, hi;
  bool has_guard = false;
};

enum class FoldMode {
  Clamp,  // materialize_step semantics: overhang reads clamp to D-1 (interp.cpp:210-213)
  Nest    // loop-nest semantics: t*S+o unclamped (layout.cpp:296-303)
};

struct CopySpec {
  LogicalMap lmap;
  Seq dst_seq;  // layout written
  Seq src_seq;  // layout read
  FoldMode mode = FoldMode::Clamp;
};

// Compile to the affine digit form. Returns false when the sequences need
// the general program (the out-param is then unspecified). `oob` is set
// when some destination cell would read outside the source's logical range
// without a guard (the reference throws out-of-range there).
// With `tables` non-null, a non-affine source side falls back to offset
// tables (their int32 data is appended to *tables; the caller uploads it).
bool compile_digit_map(const CopySpec& spec, DigitMap* out, bool* oob,
                       std::vector<int32_t>* tables = nullptr);
// Compile to the general program pair: dst physical -> dst logical (+guard,
// +shift) -> src physical. Always succeeds for valid sequences.
void compile_ix_programs(const CopySpec& spec, IxProgram* dst_inv, IxProgram* src_fwd);

// Physical dims after `seq`, row-major strides.
std::vector<int64_t> row_strides(const std::vector<int64_t>& ext);

// Numeric forward access (logical index -> physical index) through a
// sequence: the value of lf::rewrite_access (layout.cpp:324-335) without
// window hints. Returns the physical flat offset.
int64_t forward_offset(const std::vector<Dim>& logical, const Seq& seq, const int64_t* idx);

// Per-logical-dimension offset tables: offset(l) = sum_j table[off[j] + l_j].
// Exists iff no primitive re-splits a value that mixes logical dims.
bool separable_tables(const std::vector<Dim>& logical, const Seq& seq,
                      std::vector<int64_t>* table, std::vector<int64_t>* off);

}  // namespace lfg
