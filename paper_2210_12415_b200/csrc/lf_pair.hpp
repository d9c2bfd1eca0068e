// lf_pair.hpp — the CTA-pair (cta_group::2) tcgen05 GEMM for GMM nodes on
// tuned brick layouts (K3, second generation).
//
// A pair of CTAs on one TPC computes a 256 x BN output tile with
// tcgen05.mma.cta_group::2: each CTA stages its own 128 rows of A and BN/2
// columns of B (the pair's tensor cores read both halves), so per-SM
// L2->SMEM traffic per MAC is half that of a 128 x BN single-CTA tile. K
// splits of one tile run in the same thread-block cluster (cluster = 2 x S
// CTAs): the S pairs publish fp32 partials to an L2 workspace, meet on a
// cluster-scope mbarrier and each reduces a column slice in split order
// (deterministic, no global spin: co-residency is the cluster's).
//
// Layout generality comes from the same brick analysis as the 1-CTA kernel
// (umma_plan.cpp): A coordinates depend only on the 128-row block, B
// coordinates only on the BN/2 column block, stage coordinates only on K.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "lf_umma.hpp"

namespace lfg {

struct PairPlan {
  int BN = 256;   // pair tile columns (each CTA stages BN/2 of B)
  int S = 1;      // K splits (cluster = 2*S CTAs)
  int MT = 0;     // 128-row blocks (even)
  int NT = 0;     // BN-column pair tiles
  int KS = 0;     // K stages of 64
  int pipe = 4;
  OperandView A, B;           // A: 128-row box, B: BN/2-column box
  std::vector<int32_t> a_crd; // MT x A.boxes x 5
  std::vector<int32_t> b_crd; // 2*NT x B.boxes x 5
  std::vector<int32_t> s_crd; // KS x 10 (A part, B part)
  std::vector<int64_t> out_r; // MT: output offset of row block origin
  std::vector<int64_t> out_c; // NT: output offset of column tile origin
  std::vector<int64_t> row_off, col_off;  // 128 / BN
  EpiOp epi[kMaxEpi];
  int epi_count = 0;
  const void* a = nullptr;
  const void* b = nullptr;
  float* out = nullptr;
  void* out_bf16 = nullptr;
  std::string summary;
};

struct PairLaunch {
  CUtensorMap tma_a, tma_b;
  std::shared_ptr<void> owner;  // device tables + workspace
  const int32_t* a_crd = nullptr;
  const int32_t* b_crd = nullptr;
  const int32_t* s_crd = nullptr;
  const int64_t* out_r = nullptr;
  const int64_t* out_c = nullptr;
  const int64_t* row_off = nullptr;
  const int64_t* col_off = nullptr;
  float* ws = nullptr;
  int BN = 0, S = 1, MT = 0, NT = 0, KS = 0, pipe = 0, group = 8;
  int a_boxes = 0, b_boxes = 0, a_slot = 0, b_slot = 0, stage_bytes = 0, tx_bytes = 0;
  uint64_t a_desc = 0, b_desc = 0;
  uint32_t a_kadv = 0, b_kadv = 0, idesc = 0, tmem_cols = 0;
  int ring_bytes = 0;
  int col_unit = 0;
  int epi_kinds[kMaxEpi] = {};
  const float* epi_ptr[kMaxEpi] = {};
  int epi_count = 0;
  float* out = nullptr;
  void* out_bf16 = nullptr;
  size_t smem = 0;
  int grid = 0;  // CTAs (multiple of 2*S)
};

// Plan the pair kernel for C[M,N] = A[M,K] B[K,N] on the given layouts.
// `bn` / `splits` force the tile width / K splits (0 = heuristic; the
// schedule's tile_last / order are honoured when legal).
bool pair_plan_gemm(const std::vector<Dim>& a_log, const Seq& a_seq, const std::vector<Dim>& b_log,
                    const Seq& b_seq, const std::vector<Dim>& c_log, const Seq& c_seq,
                    const lfgpu_sched& s, PairPlan* out, std::string* why);
PairLaunch pair_prepare(const PairPlan& p);
cudaError_t pair_launch(const PairLaunch& L, cudaStream_t stream);

}  // namespace lfg
