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

// The kernel's tables, one int32 blob copied to SMEM in a single pass at
// kernel start (one DRAM latency, before the PDL wait): stage coordinates,
// output row offsets, 32-column chunk offsets, row-block / column-tile
// origins, per-row-block A box coordinates, per-column-block B box
// coordinates. Sections start on 16-byte boundaries.
struct PairBlob {
  int stage = 0, row = 0, colc = 0, outr = 0, outc = 0, acrd = 0, bcrd = 0, total = 0;  // int32 offsets
};
inline PairBlob pair_blob_layout(int KS, int MT, int NT, int a_boxes, int b_boxes) {
  auto up4 = [](int x) { return (x + 3) / 4 * 4; };
  PairBlob b;
  int o = 0;
  b.stage = o;
  o += up4(10 * KS);
  b.row = o;
  o += 256;
  b.colc = o;
  o += 16;
  b.outr = o;
  o += up4(2 * MT);
  b.outc = o;
  o += up4(2 * NT);
  b.acrd = o;
  o += up4(MT * a_boxes * 5);
  b.bcrd = o;
  o += up4(2 * NT * b_boxes * 5);
  b.total = o;
  return b;
}
// SMEM bytes of the tables plus the double-buffered tile bias.
inline size_t pair_table_bytes(int KS, int MT, int NT, int BN, int a_boxes, int b_boxes) {
  return 4 * static_cast<size_t>(pair_blob_layout(KS, MT, NT, a_boxes, b_boxes).total) + 8 * static_cast<size_t>(BN);
}

struct PairPlan {
  int BN = 256;   // pair tile columns (each CTA stages BN/2 of B)
  int S = 1;      // K splits (cluster = 2*S CTAs)
  int MT = 0;     // 128-row blocks (even)
  int NT = 0;     // BN-column pair tiles
  int KS = 0;     // K stages of 64 * slabs
  int slabs = 1;  // 64-wide K slabs per stage (one TMA box each operand)
  int a_slab = 0, b_slab = 0;  // SMEM bytes between slabs inside a box
  int pipe = 4;
  int rx_bytes = 0;  // S > 1 with one tile per cluster: DSMEM receive buffer
  int epi_alias = 0; // one tile per cluster: the epilogue transpose buffers live in the idle ring
  int group = 8;     // tile rasterization: row pairs that sweep the column tiles together (loop point `parallel`)
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
  const int32_t* blob = nullptr;     // PairBlob-laid-out tables
  PairBlob lay;
  const int64_t* col_off = nullptr;  // full column table (generic epilogue)
  float* ws = nullptr;
  int BN = 0, S = 1, MT = 0, NT = 0, KS = 0, pipe = 0, group = 8;
  int nprod = 4;  // TMA producer warps
  int xmode = 0, rx_bytes = 0;  // split-K exchange over DSMEM
  int epi_alias = 0, epi_off = 0;  // epilogue buffers inside the ring at epi_off (one tile per cluster)
  int a_boxes = 0, b_boxes = 0, a_slot = 0, b_slot = 0, stage_bytes = 0, tx_bytes = 0;
  int a_box_bytes = 0;
  uint64_t a_desc = 0, b_desc = 0;
  uint32_t a_kadv = 0, b_kadv = 0, idesc = 0, tmem_cols = 0;
  int slabs = 1, a_slab = 0, b_slab = 0;
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
