// lf_rows.hpp — the BERT-encoder op-set extension (lfgpu.h LFGPU_OP_SOFTMAX,
// LAYERNORM, BMM_QK, BMM_PV): row reductions over the last logical dim and
// the per-head batched matmuls of attention. Every operand is read and
// written in its own physical layout through separable per-dim offset
// tables (split / reorder layouts, e.g. the GMM output bricks), so no
// layout conversion sits between these ops and the tcgen05 GEMMs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lfg {

enum RowsOp : int32_t { ROWS_SOFTMAX = 0, ROWS_LAYERNORM = 1 };

struct RowsParams {
  int32_t op = ROWS_SOFTMAX;
  int32_t d = 0;        // row length (last logical dim)
  int64_t rows = 0;     // product of the leading dims
  float eps = 1e-12f;   // LayerNorm
  const float* x = nullptr;
  float* y = nullptr;
  void* y_bf16 = nullptr;           // optional bf16 copy of y (tensor-core consumer), same layout
  const float* gb = nullptr;        // LayerNorm [2, d]: gamma, beta
  const int64_t* row_x = nullptr;   // rows: base offset of each row in x
  const int64_t* row_y = nullptr;
  const int64_t* col_x = nullptr;   // d: offset of column j
  const int64_t* col_y = nullptr;
  const int64_t* col_gb = nullptr;  // 2 x d: gamma then beta offsets in gb
};

// QK: s[h,i,j] = sum_d q[i, h*Dh+d] k[j, h*Dh+d]
// PV: o[i, h*Dh+d] = sum_j p[h,i,j] v[j, h*Dh+d]
struct BmmParams {
  int32_t mode = 0;  // 0 QK, 1 PV
  int32_t H = 0, T = 0, T2 = 0, Dh = 0;
  const float* a = nullptr;  // q (QK) / p (PV)
  const float* b = nullptr;  // k (QK) / v (PV)
  float* out = nullptr;      // s (QK) / o (PV)
  void* out_bf16 = nullptr;  // optional bf16 copy of out, same layout
  // separable tables: rank-2 operands [rows, H*Dh] use 2 tables, rank-3
  // [H, T, T2] use 3 (concatenated; *_off = start of each dim's table)
  const int64_t* ta = nullptr;
  const int64_t* tb = nullptr;
  const int64_t* to = nullptr;
  int64_t a_off[3] = {}, b_off[3] = {}, o_off[3] = {};
  // fused attention: every operand's head columns contiguous in 16-byte
  // aligned runs of 4 (16-byte gathers)
  int32_t vec = 0;
  // diagnostics (lfgpu_debug_umma_trace): 8 %globaltimer stamps per CTA
  unsigned long long* dbg = nullptr;
};

// LFGPU_PLAN_TC_SPLIT operand preparation: x = x0 + x1 + x2 (bf16 pieces);
// the K extent becomes kTerms*K with term t holding piece kPiece[side][t]
// (A: columns t*K + k, B: rows t*K + k), so one bf16 GEMM sums the six
// leading piece products, smallest first: x2y0 + x1y1 + x0y2 + x1y0 + x0y1 + x0y0.
constexpr int kSplitTerms = 6;
struct SplitParams {
  int32_t side = 0;  // 0: A [M, K] (K = columns), 1: B [K, N] (K = rows)
  int64_t R = 0, C = 0, K = 0;  // source logical extents; K = the contraction extent
  const float* src = nullptr;
  const int64_t* src_row = nullptr;  // R
  const int64_t* src_col = nullptr;  // C
  void* dst = nullptr;               // bf16
  const int64_t* dst_row = nullptr;  // A: R; B: kSplitTerms * R
  const int64_t* dst_col = nullptr;  // A: kSplitTerms * C; B: C
};
cudaError_t launch_split_bf16(const SplitParams& P, cudaStream_t stream);

cudaError_t launch_rows(const RowsParams& P, cudaStream_t stream);
cudaError_t launch_bmm(const BmmParams& P, bool exact, cudaStream_t stream);
// BmmQK -> Softmax -> BmmPV in one kernel (k_rows.cu attn_kernel): QK's q / k
// operands and PV's v operand and output; the scores stay in SMEM.
cudaError_t launch_attention(const BmmParams& QK, const BmmParams& PV, bool exact, cudaStream_t stream);

}  // namespace lfg
