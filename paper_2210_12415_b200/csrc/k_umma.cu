// k_umma.cu — K3/K4: the tcgen05 contraction kernel for sm_100a.
//
// Replaces the GMM and C2D loop nests of the reference (lower.cpp:196-227,
// evaluated by interp.cpp:381-411; oracle interp.cpp:70-122) on tuned
// layouts. One CTA computes a 128 x BN output tile:
//   warp 0 (one lane)  TMA producer: per K stage, box loads of the A and B
//                      bricks into a `pipe`-deep SMEM ring (mbarrier
//                      complete_tx), coordinates = tile part + stage part
//                      from host tables (umma_plan.cpp);
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//                      bf16 x bf16 -> fp32 accumulator in TMEM, K=16 per
//                      instruction; tcgen05.commit frees SMEM slots;
//   warps 2-5          epilogue: tcgen05.ld 32 columns at a time, fused
//                      BiasAdd / EwAdd / ReLU (lower.cpp:566-608 fusion
//                      groups), stores into the output's physical layout.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>

#include "lf_umma.hpp"

namespace lfg {

namespace {

struct UmmaParams {
  const TileEntry* tiles;
  const StageEntry* stages;
  const int64_t* row_off;
  const int64_t* col_off;
  float* out;
  const float* epi_ptr[kMaxEpi];
  int32_t epi_kind[kMaxEpi];
  int32_t epi_count;
  int32_t nstages, BN, ksteps, pipe;
  int32_t a_boxes, b_boxes, a_slot, b_slot, tx_bytes;
  int32_t a_rank, b_rank;
  uint64_t a_desc, b_desc;  // LBO/SBO/version/layout bits; start address added on device
  uint32_t a_kadv, b_kadv;
  uint32_t idesc;
  uint32_t tmem_cols;
  int32_t cols_unit;  // col_off[c] == col_off[0] + c
  int32_t rows_unit;  // row_off[r] == r
  int32_t ring_bytes; // pipeline ring (>= the epilogue's fp32 staging tile)
  unsigned long long* dbg;  // optional per-CTA %globaltimer checkpoints (8 per CTA)
  int32_t epi_mode;         // unused (diagnostics)
  int32_t epi_sig;          // EPI_SIG of a <= 3-op chain, -1 = generic
  // Split-K: CTA (tile, split) accumulates stages [split*n/S, (split+1)*n/S);
  // partial tiles go to `ws`, the last CTA of a tile (per-tile counter) sums
  // them in split order and runs the fused epilogue.
  int32_t splits;
  float* ws;
  int* counters;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_LOOP;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load(const CUtensorMap* map, int rank, uint32_t dst,
                                         uint32_t bar, const int32_t* c) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 1:
      asm volatile(
          "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0])
          : "memory");
      break;
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1])
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2])
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
          : "memory");
      break;
  }
}

__device__ __forceinline__ void tma_load5(const CUtensorMap* map, uint32_t dst, uint32_t bar,
                                          int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                          int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31},"
      " [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  // The registers are valid only after wait::ld; tie them to the wait so no
  // consumer is scheduled between the load and the wait.
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                 "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                 "+r"(v[30]), "+r"(v[31])::"memory");
}

#define EPI_SIG(a, b, c) ((a) | ((b) << 2) | ((c) << 4))

template <int K>
__device__ __forceinline__ float epi_op(float x, const float* __restrict__ p, int64_t addr,
                                        int n) {
  if (K == EPI_BIAS) return x + __ldg(p + n);
  if (K == EPI_RESIDUAL) return x + __ldg(p + addr);
  if (K == EPI_RELU) return fmaxf(x, 0.0f);
  return x;
}

// Row-contiguous output brick: each epilogue warp walks rows, lanes walk
// 4-column groups (16-byte SMEM reads and global stores when aligned).
template <int K0, int K1, int K2>
__device__ __forceinline__ void epi_rows(const float* __restrict__ stile, int ld, int rows, int cols,
                                         int64_t cbase, const int64_t* __restrict__ s_row,
                                         int n_base, float* __restrict__ out,
                                         const float* __restrict__ e0, const float* __restrict__ e1,
                                         const float* __restrict__ e2, int ew, int lane) {
  const int groups = (cols + 3) >> 2;
  for (int r = ew; r < rows; r += 4) {
    const int64_t rb = cbase + s_row[r];
    const bool vec = ((rb & 3) == 0) && ((cols & 3) == 0);
    for (int g = lane; g < groups; g += 32) {
      const int c = g << 2;
      float4 x = *reinterpret_cast<const float4*>(stile + r * ld + c);
      float v[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t a = rb + c + j;
        const int n = n_base + c + j;
        if (c + j < cols) {
          v[j] = epi_op<K0>(v[j], e0, a, n);
          v[j] = epi_op<K1>(v[j], e1, a, n);
          v[j] = epi_op<K2>(v[j], e2, a, n);
        }
      }
      if (vec) {
        *reinterpret_cast<float4*>(out + rb + c) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < cols) out[rb + c + j] = v[j];
      }
    }
  }
}

// Row-contiguous side (M-major output, e.g. NCHW or a (M/m_t) N m_t brick):
// each epilogue warp walks columns, lanes walk consecutive rows.
template <int K0, int K1, int K2>
__device__ __forceinline__ void epi_cols(const float* __restrict__ stile, int ld, int rows, int cols,
                                         int64_t rbase, const int64_t* __restrict__ s_col,
                                         int n_base, float* __restrict__ out,
                                         const float* __restrict__ e0, const float* __restrict__ e1,
                                         const float* __restrict__ e2, int ew, int lane) {
  for (int c = ew; c < cols; c += 4) {
    const int64_t cb = rbase + s_col[c];
    const int n = n_base + c;
    for (int r = lane; r < rows; r += 32) {
      float v = stile[r * ld + c];
      v = epi_op<K0>(v, e0, cb + r, n);
      v = epi_op<K1>(v, e1, cb + r, n);
      v = epi_op<K2>(v, e2, cb + r, n);
      out[cb + r] = v;
    }
  }
}

// Any output brick (e.g. M-contiguous C): lanes walk rows when the rows are
// the contiguous side, else columns; runtime op chain (rare shapes).
template <typename PT>
__device__ __noinline__ void epi_generic(const PT& P, const float* __restrict__ stile, int ld,
                                         int rows, int cols, int64_t obase,
                                         const int64_t* __restrict__ s_row,
                                         const int64_t* __restrict__ s_col, int n_base,
                                         float* __restrict__ out, int et) {
  int ek[kMaxEpi];
  const float* ep[kMaxEpi];
#pragma unroll
  for (int e = 0; e < kMaxEpi; ++e) {
    ek[e] = e < P.epi_count ? P.epi_kind[e] : EPI_NONE;
    ep[e] = P.epi_ptr[e];
  }
  const bool row_fast = P.rows_unit && !P.cols_unit;
  const int ew = et >> 5, lane = et & 31;
  const int outer = row_fast ? cols : rows, inner = row_fast ? rows : cols;
  for (int o = ew; o < outer; o += 4) {
    for (int i = lane; i < inner; i += 32) {
      const int r = row_fast ? i : o, c = row_fast ? o : i;
      const int64_t addr = obase + s_row[r] + s_col[c];
      float x = stile[r * ld + c];
#pragma unroll
      for (int e = 0; e < kMaxEpi; ++e) {
        if (ek[e] == EPI_BIAS) x += __ldg(ep[e] + n_base + c);
        else if (ek[e] == EPI_RESIDUAL) x += __ldg(ep[e] + addr);
        else if (ek[e] == EPI_RELU) x = fmaxf(x, 0.0f);
      }
      out[addr] = x;
    }
  }
}

constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    umma_kernel(const __grid_constant__ CUtensorMap tma_a,
                const __grid_constant__ CUtensorMap tma_b, const UmmaParams P) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B atoms) by offsetting the __shared__
  // array itself, so every derived pointer stays in the shared window.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stage_bytes = P.a_boxes * P.a_slot + P.b_boxes * P.b_slot;
  // The epilogue stages the fp32 tile (128 x (BN+1)) over the pipeline ring
  // once every MMA has retired; ring_bytes >= that (host-checked).
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.ring_bytes);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * P.pipe;
  const uint32_t accf = empty0 + 8 * P.pipe;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P.pipe + 1);
  // After the barriers: this tile's entry, the stage table and the epilogue's
  // row/column offsets, all copied from global memory once.
  TileEntry* s_tile = reinterpret_cast<TileEntry*>(bars + 2 * P.pipe + 2);
  StageEntry* s_stage = reinterpret_cast<StageEntry*>(s_tile + 1);
  int64_t* s_col = reinterpret_cast<int64_t*>(s_stage + P.nstages);
  int64_t* s_row = s_col + P.BN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int splits = P.splits;
  const int tile = blockIdx.x / splits, split = blockIdx.x - tile * splits;
  const int s_lo = split * P.nstages / splits, s_hi = (split + 1) * P.nstages / splits;
  int* s_flag = reinterpret_cast<int*>(s_row + 128);
  unsigned long long* dbg = P.dbg ? P.dbg + 8 * tile : nullptr;
  const int pipe = P.pipe;
  const int early = 0;

  if (threadIdx.x == 0) {
    if (dbg) {
      dbg[0] = gtimer();
      P.dbg[8 * gridDim.x + 2 * tile] = clock64();
    }
    for (int s = 0; s < pipe; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  {
    const int* g = reinterpret_cast<const int*>(P.tiles + tile);
    int* d = reinterpret_cast<int*>(s_tile);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(TileEntry) / 4); i += kThreads) d[i] = g[i];
    const int* gs = reinterpret_cast<const int*>(P.stages);
    int* ds = reinterpret_cast<int*>(s_stage);
    const int nst = P.nstages * static_cast<int>(sizeof(StageEntry) / 4);
    for (int i = threadIdx.x; i < nst; i += kThreads) ds[i] = gs[i];
    for (int i = threadIdx.x; i < P.BN; i += kThreads) s_col[i] = P.col_off[i];
    for (int i = threadIdx.x; i < 128; i += kThreads) s_row[i] = P.row_off[i];
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (dbg && threadIdx.x == 0) dbg[1] = gtimer();

  // ---- TMA producers. One thread's serial issue path (barrier wait +
  // expect_tx + UTMALDGs, ~450 cycles per stage measured) would cap a CTA at
  // ~one stage per 0.25 us, so warps 0 and 2-4 (the epilogue warps are idle
  // during the main loop) issue stages round-robin; each computes its own
  // ring slot / phase. Coordinates = tile part (registers) + stage part
  // (SMEM); views are always 5-D (host pads unit dims) so each load is one
  // straight-line UTMALDG.5D with no rank dispatch.
  constexpr int kProducers = 4;
  const int prod = warp == 0 ? 0 : (warp >= 2 && warp <= 4 ? warp - 1 : -1);
  if (prod >= 0) {
    int32_t ta[kMaxBoxes][5], tb[kMaxBoxes][5];
#pragma unroll
    for (int b = 0; b < kMaxBoxes; ++b)
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        ta[b][d] = s_tile->ca[b][d];
        tb[b][d] = s_tile->cb[b][d];
      }
    const int na = P.a_boxes, nb = P.b_boxes;
    const uint32_t tx = P.tx_bytes, a_slot = P.a_slot, b_slot = P.b_slot;
    const uint32_t ring0 = smem_u32(smem);
    const uint32_t b_off = na * a_slot;
    const bool leader = elect_one();
    for (int s = s_lo + prod; s < s_hi; s += kProducers) {
      if (leader) {
        const int it = s - s_lo;
        const int slot = it % pipe;
        const uint32_t phase = static_cast<uint32_t>(it / pipe) & 1u;
        const long long c_top = dbg ? clock64() : 0;
        mbar_wait(empty0 + 8 * slot, phase ^ 1);
        const long long c_wait = dbg ? clock64() : 0;
        const uint32_t bar = full0 + 8 * slot;
        mbar_expect_tx(bar, tx);
        const StageEntry se = s_stage[s];
        if (dbg && s < 32) P.dbg[10 * gridDim.x + 64 * tile + s] = gtimer();
        const uint32_t a_dst = ring0 + slot * stage_bytes;
        const long long c_issue = dbg ? clock64() : 0;
        if (dbg && it < 32) {
          P.dbg[106 * gridDim.x + 64 * tile + 2 * it] = c_wait - c_top;
          P.dbg[106 * gridDim.x + 64 * tile + 2 * it + 1] = c_issue - c_wait;
        }
#pragma unroll
        for (int b = 0; b < kMaxBoxes; ++b)
          if (b < na)
            tma_load5(&tma_a, a_dst + b * a_slot, bar, ta[b][0] + se.sa[0], ta[b][1] + se.sa[1],
                      ta[b][2] + se.sa[2], ta[b][3] + se.sa[3], ta[b][4] + se.sa[4]);
#pragma unroll
        for (int b = 0; b < kMaxBoxes; ++b)
          if (b < nb)
            tma_load5(&tma_b, a_dst + b_off + b * b_slot, bar, tb[b][0] + se.sb[0],
                      tb[b][1] + se.sb[1], tb[b][2] + se.sb[2], tb[b][3] + se.sb[3],
                      tb[b][4] + se.sb[4]);
        if (dbg && it < 32) P.dbg[74 * gridDim.x + 32 * tile + it] = clock64() - c_issue;
      }
    }
    __syncwarp();
    if (dbg && leader && prod == 0) dbg[2] = gtimer();
  }
  if (warp == 0) {
  } else if (warp == 1) {
    // ---- MMA issuer (whole warp loops; one elected lane issues tcgen05.mma)
    const uint64_t adesc = P.a_desc, bdesc = P.b_desc;
    const uint32_t idesc = P.idesc, akadv = P.a_kadv, bkadv = P.b_kadv;
    const int ksteps = P.ksteps;
    const uint32_t ring0 = smem_u32(smem);
    const uint32_t a_off_b = P.a_boxes * P.a_slot;
    const bool leader = elect_one();
    int slot = 0;
    uint32_t phase = 0;
    for (int s = s_lo; s < s_hi; ++s) {
      mbar_wait(full0 + 8 * slot, phase);
      if (dbg && leader && s == s_lo) dbg[3] = gtimer();
      if (dbg && leader && s < 32) P.dbg[10 * gridDim.x + 64 * tile + 32 + s] = gtimer();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (leader) {
        const uint32_t a_addr = ring0 + slot * stage_bytes;
        const uint32_t b_addr = a_addr + a_off_b;
        for (int k = 0; k < ksteps; ++k) {
          const uint64_t ad = adesc | (((a_addr + k * akadv) >> 4) & 0x3FFFull);
          const uint64_t bd = bdesc | (((b_addr + k * bkadv) >> 4) & 0x3FFFull);
          umma_bf16(tmem, ad, bd, idesc, (s != s_lo) || (k != 0));
        }
        umma_commit(empty0 + 8 * slot);
      }
      __syncwarp();
      if (++slot == pipe) {
        slot = 0;
        phase ^= 1;
      }
    }
    if (leader) umma_commit(accf);
    if (dbg && leader) dbg[4] = gtimer();
  } else if (warp >= 2) {
    // ---- epilogue (4 warps). Phase 1: TMEM -> SMEM tile (row r = TMEM lane r).
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    // SMEM row stride: 16-byte aligned rows for the float4 row pass, odd for
    // the column pass (conflict-free lane-per-row reads).
    const int ld = (P.cols_unit || !P.rows_unit) ? P.BN + 4 : P.BN + 1;
    float* stile = reinterpret_cast<float*>(smem);
    mbar_wait(accf, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (dbg && threadIdx.x == 64) dbg[5] = gtimer();
    if (splits == 1) {
      for (int c0 = 0; c0 < P.BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < P.BN) stile[row * ld + c0 + j] = __uint_as_float(v[j]);
      }
    } else {
      // Split-K: publish this split's partial tile, count arrivals; the last
      // CTA of the tile sums the partials in split order (deterministic).
      float* wrow = P.ws + ((static_cast<int64_t>(tile) * splits + split) * 128 + row) * P.BN;
      for (int c0 = 0; c0 < P.BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < P.BN) __stcg(wrow + c0 + j, __uint_as_float(v[j]));
      }
      __threadfence();
      epi_bar();
      if (threadIdx.x == 64) {
        const int prev = atomicAdd(P.counters + tile, 1);
        *s_flag = prev == splits - 1;
        if (prev == splits - 1) P.counters[tile] = 0;  // re-armed for the next launch
      }
      epi_bar();
      if (*s_flag) {
        __threadfence();
        const float* w0 = P.ws + (static_cast<int64_t>(tile) * splits * 128 + row) * P.BN;
        for (int c = 0; c < P.BN; ++c) {
          float acc = 0.f;
          for (int q = 0; q < splits; ++q) acc += __ldcg(w0 + static_cast<int64_t>(q) * 128 * P.BN + c);
          stile[row * ld + c] = acc;
        }
      }
    }
    epi_bar();
    if (splits == 1 || *s_flag) {
    if (dbg && threadIdx.x == 64) dbg[7] = gtimer();
    // Phase 2: cooperative, coalesced stores with the fused element-wise chain
    // (bias / residual / relu, lower.cpp:566-608). Lanes run along the
    // physically contiguous side of the output brick.
    const int et = threadIdx.x - 64;  // 0..127
    const int rows = s_tile->rows, cols = s_tile->cols, n_base = s_tile->n_base;
    const int64_t obase = s_tile->out_base;
    float* __restrict__ out = P.out;
    // The element-wise chain (<= 3 ops: bias / residual / relu) is resolved
    // once into a signature and each signature runs a specialised loop: no
    // per-element switch, no indirect branches, no param-buffer loads.
    const int sig = P.epi_sig;
    const float* e0 = P.epi_ptr[0];
    const float* e1 = P.epi_ptr[1];
    const float* e2 = P.epi_ptr[2];
    const int ew = et >> 5;  // epilogue warp 0..3
    if (P.cols_unit && (ld & 3) == 0) {
      const int64_t cbase = obase + s_col[0];
      switch (sig) {
        case EPI_SIG(0, 0, 0): epi_rows<0, 0, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 0, 0): epi_rows<1, 0, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 2, 0): epi_rows<1, 2, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 3, 0): epi_rows<1, 3, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 3, 2): epi_rows<1, 3, 2>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(2, 0, 0): epi_rows<2, 0, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(3, 0, 0): epi_rows<3, 0, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(3, 2, 0): epi_rows<3, 2, 0>(stile, ld, rows, cols, cbase, s_row, n_base, out, e0, e1, e2, ew, lane); break;
        default: epi_generic(P, stile, ld, rows, cols, obase, s_row, s_col, n_base, out, et); break;
      }
    } else if (P.rows_unit) {
      switch (sig) {
        case EPI_SIG(0, 0, 0): epi_cols<0, 0, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 0, 0): epi_cols<1, 0, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 2, 0): epi_cols<1, 2, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 3, 0): epi_cols<1, 3, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(1, 3, 2): epi_cols<1, 3, 2>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(2, 0, 0): epi_cols<2, 0, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(3, 0, 0): epi_cols<3, 0, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        case EPI_SIG(3, 2, 0): epi_cols<3, 2, 0>(stile, ld, rows, cols, obase, s_col, n_base, out, e0, e1, e2, ew, lane); break;
        default: epi_generic(P, stile, ld, rows, cols, obase, s_row, s_col, n_base, out, et); break;
      }
    } else {
      epi_generic(P, stile, ld, rows, cols, obase, s_row, s_col, n_base, out, et);
    }
    if (dbg && threadIdx.x == 64) {
      dbg[6] = gtimer();
      P.dbg[8 * gridDim.x + 2 * tile + 1] = clock64();
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(P.tmem_cols)
                 : "memory");
  }
}

// ---- host side ------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !p)
      fail(LFGPU_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

CUtensorMap encode(const OperandView& v, const void* base) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t dims[5], strides[5];
  cuuint32_t box[5], es[5];
  for (int d = 0; d < 5; ++d) {
    if (d < v.rank) {
      dims[d] = v.dims[d];
      strides[d] = v.strides[d];
      box[d] = v.box[d];
      es[d] = v.estride[d];
    } else {  // unit padding dims: the kernel always issues 5-D loads
      dims[d] = 1;
      strides[d] = d == 1 ? ((v.dims[0] * 2 + 15) / 16) * 16 : strides[d - 1] * dims[d - 1];
      box[d] = 1;
      es[d] = 1;
    }
  }
  CUtensorMapSwizzle sw = v.swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : v.swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base),
                           dims, strides + 1, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(LFGPU_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

uint64_t desc_bits(const OperandView& v) {
  uint64_t layout = v.swizzle == 128 ? 2 : v.swizzle == 64 ? 4 : 6;
  uint64_t d = 0;
  d |= static_cast<uint64_t>((v.lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((v.sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= layout << 61;
  return d;
}

uint32_t idesc_of(int M, int N, bool a_mn, bool b_mn) {
  uint32_t d = 0;
  d |= 1u << 4;   // D: F32
  d |= 1u << 7;   // A: BF16
  d |= 1u << 10;  // B: BF16
  d |= (a_mn ? 1u : 0u) << 15;
  d |= (b_mn ? 1u : 0u) << 16;
  d |= static_cast<uint32_t>(N >> 3) << 17;
  d |= static_cast<uint32_t>(M >> 4) << 24;
  return d;
}

struct Tables {
  void* p[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  ~Tables() {
    for (auto* q : p)
      if (q) cudaFree(q);
  }
};

template <typename T>
void* up(const std::vector<T>& v) {
  void* d = nullptr;
  size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
  if (cudaMalloc(&d, bytes) != cudaSuccess) fail(LFGPU_ECUDA, "cudaMalloc tables");
  if (!v.empty() && cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    fail(LFGPU_ECUDA, "cudaMemcpy tables");
  return d;
}

}  // namespace

static void* g_umma_dbg = nullptr;
void* umma_debug_buffer() { return g_umma_dbg; }
void umma_set_debug_buffer(void* p) { g_umma_dbg = p; }

UmmaLaunch umma_prepare(const UmmaPlan& p) {
  UmmaLaunch L;
  L.tma_a = encode(p.A, p.a);
  L.tma_b = encode(p.B, p.b);
  auto t = std::make_shared<Tables>();
  t->p[0] = up(p.tiles);
  t->p[1] = up(p.stages);
  t->p[2] = up(p.row_off);
  t->p[3] = up(p.col_off);
  L.d_tiles = t->p[0];
  L.d_stages = t->p[1];
  L.d_rows = t->p[2];
  L.d_cols = t->p[3];
  L.owner = t;
  L.ntiles = static_cast<int>(p.tiles.size());
  L.nstages = static_cast<int>(p.stages.size());
  L.BN = p.BN;
  L.KC = p.KC;
  L.pipe = p.pipe;
  int cols = 32;
  while (cols < p.BN) cols *= 2;
  L.tmem_cols = cols;
  L.a_boxes = p.A.boxes;
  L.b_boxes = p.B.boxes;
  L.a_slot = p.A.slot_bytes;
  L.b_slot = p.B.slot_bytes;
  L.a_bytes = p.A.box_bytes;
  L.b_bytes = p.B.box_bytes;
  L.a_desc = desc_bits(p.A);
  L.b_desc = desc_bits(p.B);
  L.a_kadv = p.A.k_adv;
  L.b_kadv = p.B.k_adv;
  L.idesc = idesc_of(p.BM, p.BN, p.A.mn_major, p.B.mn_major);
  L.epi_count = p.epi_count;
  for (int e = 0; e < p.epi_count; ++e) {
    L.epi_kinds[e] = p.epi[e].kind;
    L.epi_ptr[e] = p.epi[e].ptr;
  }
  L.out = p.out;
  const size_t ring = static_cast<size_t>(p.pipe) * (L.a_boxes * L.a_slot + L.b_boxes * L.b_slot);
  const size_t staging = static_cast<size_t>(128) * (p.BN + 4) * 4;
  L.ring_bytes = static_cast<int>((std::max(ring, staging) + 1023) / 1024 * 1024);
  L.smem = 1024 + L.ring_bytes + 8 * (2 * p.pipe + 2) + sizeof(TileEntry) +
           sizeof(StageEntry) * p.stages.size() + 8 * p.BN + 8 * 128 + 64;
  // Contiguity over the rows any tile actually stores.
  int max_rows = 0;
  for (const auto& t : p.tiles) max_rows = std::max(max_rows, static_cast<int>(t.rows));
  L.rows_unit = 1;
  for (int r = 0; r < max_rows && r < static_cast<int>(p.row_off.size()); ++r)
    if (p.row_off[r] != static_cast<int64_t>(r)) L.rows_unit = 0;
  L.cols_unit = 1;
  for (size_t c = 0; c < p.col_off.size(); ++c)
    if (p.col_off[c] != p.col_off[0] + static_cast<int64_t>(c)) L.cols_unit = 0;
  // Split-K when the tiles alone leave most of the 148 SMs idle and the
  // K loop is long: up to 8 splits of >= 4 stages each.
  L.splits = 1;
  if (L.ntiles * 2 <= 148 && L.nstages >= 8) {
    L.splits = std::min({148 / L.ntiles, L.nstages / 4, 8});
    if (L.splits < 2) L.splits = 1;
  }
  if (const char* e = getenv("LFGPU_SPLITK")) L.splits = std::max(1, std::min(atoi(e), L.nstages));
  if (L.splits > 1) {
    const size_t ws = sizeof(float) * static_cast<size_t>(L.ntiles) * L.splits * 128 * L.BN;
    if (cudaMalloc(&t->p[4], ws) != cudaSuccess) fail(LFGPU_ECUDA, "cudaMalloc split-K workspace");
    if (cudaMalloc(&t->p[5], sizeof(int) * L.ntiles) != cudaSuccess ||
        cudaMemset(t->p[5], 0, sizeof(int) * L.ntiles) != cudaSuccess)
      fail(LFGPU_ECUDA, "cudaMalloc split-K counters");
    L.ws = static_cast<float*>(t->p[4]);
    L.counters = static_cast<int*>(t->p[5]);
  }
  L.grid = L.ntiles * L.splits;
  L.a_rank_ = p.A.rank;
  L.b_rank_ = p.B.rank;
  static_assert(sizeof(TileEntry) == 192, "TileEntry layout");
  return L;
}

cudaError_t umma_launch(const UmmaLaunch& L, cudaStream_t stream) {
  if (L.ntiles == 0) return cudaSuccess;
  UmmaParams P;
  std::memset(&P, 0, sizeof(P));
  P.tiles = static_cast<const TileEntry*>(L.d_tiles);
  P.stages = static_cast<const StageEntry*>(L.d_stages);
  P.row_off = static_cast<const int64_t*>(L.d_rows);
  P.col_off = static_cast<const int64_t*>(L.d_cols);
  P.out = L.out;
  P.epi_count = L.epi_count;
  P.epi_sig = L.epi_count <= 3 ? 0 : -1;
  for (int e = 0; e < L.epi_count && e < 3; ++e) P.epi_sig |= L.epi_kinds[e] << (2 * e);
  for (int e = 0; e < L.epi_count; ++e) {
    P.epi_kind[e] = L.epi_kinds[e];
    P.epi_ptr[e] = L.epi_ptr[e];
  }
  P.nstages = L.nstages;
  P.BN = L.BN;
  P.ksteps = L.KC / 16;
  P.pipe = L.pipe;
  P.a_boxes = L.a_boxes;
  P.b_boxes = L.b_boxes;
  P.a_slot = L.a_slot;
  P.b_slot = L.b_slot;
  P.tx_bytes = L.a_boxes * L.a_bytes + L.b_boxes * L.b_bytes;
  // rank is encoded in the tensor map; keep our own copy for the PTX form
  P.a_desc = L.a_desc;
  P.b_desc = L.b_desc;
  P.a_kadv = L.a_kadv;
  P.b_kadv = L.b_kadv;
  P.idesc = L.idesc;
  P.tmem_cols = L.tmem_cols;
  P.a_rank = L.a_rank_;
  P.cols_unit = L.cols_unit;
  P.rows_unit = L.rows_unit;
  P.ring_bytes = L.ring_bytes;
  P.splits = L.splits;
  P.ws = L.ws;
  P.counters = L.counters;
  P.dbg = static_cast<unsigned long long*>(umma_debug_buffer());
  if (P.dbg) {
    const char* em = getenv("LFGPU_EPI_MODE");
    P.epi_mode = em ? atoi(em) : 0;
  }
  P.b_rank = L.b_rank_;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  umma_kernel<<<L.grid, kThreads, L.smem, stream>>>(L.tma_a, L.tma_b, P);
  return cudaGetLastError();
}

}  // namespace lfg
