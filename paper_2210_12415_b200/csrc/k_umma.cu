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

#include "lf_pair.hpp"
#include "lf_alloc.hpp"
#include "lf_umma.hpp"

namespace lfg {

namespace {

struct UmmaParams {
  const TileEntry* tiles;
  const StageEntry* stages;
  const int64_t* row_off;
  const int64_t* col_off;
  float* out;
  __nv_bfloat16* out_bf16;  // optional bf16 copy of the output (same layout)
  int32_t out_stream;       // final graph output: streaming (evict-first) stores
  const float* epi_ptr[kMaxEpi];
  int32_t epi_kind[kMaxEpi];
  int32_t epi_count;
  int32_t ntiles, nstages, BN, ksteps, pipe, nprod;
  int32_t dual;  // two MMA issuers: warp 1 takes even units, warp 3 odd ones
  int32_t blocked;  // loop point `parallel` = 1: contiguous unit chunks per CTA (static schedule), else cyclic
  int32_t xsplit;   // split-K partials exchanged over DSMEM: the S splits of a tile are one cluster, one unit per CTA
  int32_t a_boxes, b_boxes, a_slot, b_slot, tx_bytes;
  uint64_t a_desc, b_desc;  // LBO/SBO/version/layout bits; start address added on device
  uint32_t a_kadv, b_kadv;
  uint32_t idesc;
  uint32_t tmem_cols;       // >= 2*BN: two accumulators
  int32_t ring_bytes;       // SMEM pipeline ring
  int32_t table_ints;       // [stages | col_off | row_off] as one contiguous int array
  int32_t ntaps;            // halo C2D: tap t reads A at +a_tap[t], B at +b_tap[t] bytes
  int32_t bias_rows;        // BiasAdd indexed by accumulator row (channels-as-rows C2D)
  // Weights resident (halo C2D with one output-channel tile): every chunk's
  // B slab is loaded once per CTA into SMEM at w_off (w_chunk bytes apart,
  // barrier wfull[c]); the ring then carries A only.
  int32_t wres, w_off, w_chunk, w_tx;
  int32_t w_prewait;  // resident weights are constants no earlier kernel of this run writes: load before the PDL wait
  int32_t red_bytes;        // split-K: SMEM for the siblings' column slices
  // Store mode 2 (TMA store): staging buffers (2 x stg_f32 fp32 + 2 x stg_bf
  // bf16 bytes) at stg_off; per-tile box origins; row positions in the box
  // follow row_off in the SMEM table.
  int32_t stg_off, stg_f32, stg_bf;
  int32_t stg_nbuf;    // staging buffers per half (ring of bulk groups)
  int32_t epi_alias;   // epilogue region lives in the (idle) operand ring
  int32_t epi_region;  // bytes of the epilogue region (wbuf, or the mode-2 staging it aliases)
  int32_t stg_cstride, stg_cdim;  // >0: transposed box, column j at plane j * stg_cstride
  const int32_t* tile_coords;
  ScatterDesc sc;           // Padding absorbed into this epilogue (sc.enabled)
  int32_t a_tap[kMaxTaps];
  int32_t b_tap[kMaxTaps];
  int32_t store_mode;       // 1: row-contiguous, 16-byte aligned output rows; 0: generic
  int32_t diag;             // diagnostics (LFGPU_UMMA_DIAG, timing only): bit0 skips the
                            // epilogue's stores, 2 traces, 4 unshifted taps, 8 one tap
  int64_t col0;             // col_off[0] folded into the tile base in store mode 1
  unsigned long long* dbg;  // optional per-CTA %globaltimer checkpoints (8 per CTA)
  unsigned long long* cdbg;  // optional chain trace slot: [0] entry min, [1] wait min, [2] wait max,
                             // [3] first stage landed min, [4] exit max, [5] epilogue done max
  // Split-K: unit (tile, split) accumulates stages [split*n/S, (split+1)*n/S);
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

__device__ __forceinline__ void tma_load5(const CUtensorMap* map, uint32_t dst, uint32_t bar,
                                          int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                          int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// TMA store of one SMEM box (bulk-group completion).
__device__ __forceinline__ void tma_store5(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1,
                                           int32_t c2, int32_t c3, int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
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

// ---- kernel -----------------------------------------------------------------
//
// Persistent, warp-specialised (256 threads, one CTA per SM):
//   warps 0, 2, 3   TMA producers: the CTA's stage sequence (over all its work
//                   units) is dealt round-robin to them; one elected lane per
//                   warp waits the ring slot, arms expect_tx and issues the
//                   UTMALDG.5D boxes (tile part from the tile table + stage part
//                   from the SMEM stage table);
//   warp 1          MMA issuer: tcgen05.mma.cta_group::1.kind::f16 into one of
//                   two TMEM accumulators (columns [0,BN) / [BN,2BN)), commit
//                   frees the ring slot; the last stage of a unit commits the
//                   accumulator to the epilogue;
//   warps 4-7       epilogue: tcgen05.ld.32x32b (thread = tile row), the fused
//                   element-wise chain, stores; releases the accumulator so the
//                   MMA of the unit after next can reuse it. The epilogue of
//                   unit i overlaps the main loop of unit i+1.
// A work unit is (tile, K split). Split-K partials go to a workspace laid out
// [unit][col/4][row][4] (coalesced float4 per warp); the last CTA to finish a
// tile (per-tile counter) sums the partials in split order (deterministic) and
// runs the epilogue.

constexpr int kThreads = 384;
#ifndef LFGPU_UMMA_MINB
#define LFGPU_UMMA_MINB 1  // resident CTAs per SM the register allocation is bounded for
#endif
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, alternating 16-column chunks
constexpr int kEpiLd = 36;  // per-warp transpose buffer row stride (floats)
constexpr int kMaxSplits = 4;
static_assert(kEpiSmemBytes == kEpiWarps * 32 * kEpiLd * 4, "epilogue SMEM size");

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// One half of the epilogue (4 warps = the 128 TMEM lanes).
__device__ __forceinline__ void half_bar(int h) {
  asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory");
}

// Cluster helpers for the DSMEM split-K exchange (the K splits of a tile are
// the CTAs of one cluster).
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_arrive(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cl_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAITX:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAITX;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])::"memory");
}

template <int W>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float* f) {
  uint32_t* v = reinterpret_cast<uint32_t*>(f);
  if (W == 32) tmem_ld32(taddr, v);
  else tmem_ld16(taddr, v);
}

// The unit's accumulator columns [c, c + W): with split issue (dual == 2)
// the two issuers' partial accumulators (BN columns apart) summed.
template <int W>
__device__ __forceinline__ void acc_ld(int dual, int BN, uint32_t taddr, float* f) {
  tmem_ld<W>(taddr, f);
  if (dual == 2) {
    float g[W];
    tmem_ld<W>(taddr + static_cast<uint32_t>(BN), g);
#pragma unroll
    for (int j = 0; j < W; ++j) f[j] += g[j];
  }
}

// The fused element-wise chain (BiasAdd / EwAdd / ReLU, interp.cpp:137-165;
// fusion groups lower.cpp:566-608). Kinds are kernel parameters, so every
// branch is warp-uniform.
//
// Code size matters more than instruction count here: each SM runs the
// epilogue only a few times per launch, so straight-line (unrolled) code is
// fetched cold from L2 instruction by instruction (ncu: stall_no_inst
// dominated an unrolled version, ~12 us per tile). The loops below are kept
// rolled so one small body is fetched once and reused.
// Sum one W-column chunk over the split-K partials in split order (this
// split's own values `v` from TMEM; the siblings' slices were bulk-copied
// into SMEM `red`, laid out [other split][col/4][row] float4).
template <int W>
__device__ __forceinline__ void split_sum(const UmmaParams& P, float* v, const float4* red, int c0,
                                          int red_lo, int row, int split, int splits) {
    const int slice4 = P.BN / splits / 4;
    const float4* r0 = red + ((c0 - red_lo) / 4) * 128 + row;
    float4 part[kMaxSplits - 1][W / 4];
#pragma unroll
    for (int o = 0; o < kMaxSplits - 1; ++o) {
      if (o < splits - 1) {
#pragma unroll
        for (int j = 0; j < W / 4; ++j) part[o][j] = r0[(o * slice4 + j) * 128];
      }
    }
#pragma unroll
    for (int j = 0; j < W / 4; ++j) {
      // Terms in split order: the other splits' partials in order, with
      // this split's own values inserted at position `split`.
      const float4 mine = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int o = 0; o < kMaxSplits - 1; ++o) {
        if (o == split && split < splits - 1) {
          acc.x += mine.x;
          acc.y += mine.y;
          acc.z += mine.z;
          acc.w += mine.w;
        }
        if (o < splits - 1) {
          acc.x += part[o][j].x;
          acc.y += part[o][j].y;
          acc.z += part[o][j].z;
          acc.w += part[o][j].w;
        }
      }
      if (split == splits - 1) {
        acc.x += mine.x;
        acc.y += mine.y;
        acc.z += mine.z;
        acc.w += mine.w;
      }
      v[4 * j] = acc.x;
      v[4 * j + 1] = acc.y;
      v[4 * j + 2] = acc.z;
      v[4 * j + 3] = acc.w;
    }
}

// The absorbed Padding: 4 consecutive channels of output pixel (n, h, w)
// into every copy of (h+pad, w+pad) in the consumer's (unfolded) bf16 layout.
__device__ __forceinline__ void scatter4(const ScatterDesc& sc, int n, int c, int h, int w,
                                         float4 x) {
  const int hp = h + sc.pad, wp = w + sc.pad;
  const int64_t base = n * sc.sN + (c / sc.ic) * sc.sC0 + (c % sc.ic);
  __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(x.z, x.w);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  const int th0 = max(0, (hp - sc.Bh + sc.Sh) / sc.Sh), th1 = min(sc.Th - 1, hp / sc.Sh);
  const int tw0 = max(0, (wp - sc.Bw + sc.Sw) / sc.Sw), tw1 = min(sc.Tw - 1, wp / sc.Sw);
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(sc.dst);
  for (int th = th0; th <= th1; ++th)
    for (int tw = tw0; tw <= tw1; ++tw) {
      const int64_t off = base + th * sc.sHt + static_cast<int64_t>(hp - th * sc.Sh) * sc.sHo +
                          tw * sc.sWt + static_cast<int64_t>(wp - tw * sc.Sw) * sc.sWo;
      *reinterpret_cast<uint2*>(dst + off) = pk;
    }
}

// One W-column chunk of one unit's accumulator for the calling thread's row.
// mode 3 publishes a split-K partial; otherwise (after the split-K sum when
// splits > 1) the chunk goes through the per-warp SMEM buffer and is stored
// with mode 1 (row-contiguous output: float4 row segments, 8 lanes per
// 128 bytes) or mode 0 (generic: thread = row, coalesced when rows are the
// contiguous side).
template <int W>
__device__ __forceinline__ void epi_chunk(const UmmaParams& P, uint32_t taddr, int c0, int row,
                                       int lane, int q, float* wbuf, int rows, int cols,
                                       int n_base, int64_t obase, const int64_t* s_row,
                                       const int64_t* s_col, int mode, int split, int splits,
                                       int64_t ws_tile, const float4* red, int red_lo,
                                       bool release, uint32_t tempty, int3 org,
                                       const int32_t* s_rowrel, bool dry) {
  if (P.dbg && !dry && (P.diag & 2) && threadIdx.x == kEpiWarp0 * 32 && c0 == 0 &&
      P.dbg[32 * blockIdx.x + 30] == 0)
    P.dbg[32 * blockIdx.x + 30] = gtimer();
  float v[W];
  acc_ld<W>(P.dual, P.BN, taddr + c0, v);
  if (P.dbg && !dry && (P.diag & 2) && threadIdx.x == kEpiWarp0 * 32 && c0 == 0 &&
      P.dbg[32 * blockIdx.x + 28] == 0)
    P.dbg[32 * blockIdx.x + 28] = gtimer();

  if (release && !dry) {
    // Every TMEM read of this accumulator is complete: hand it back to the MMA.
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty);
  }
  const int64_t wstride = static_cast<int64_t>(P.BN / 4) * 128;
  if (mode == 3 && P.xsplit) {
    // DSMEM: straight into the receiving sibling's reduction buffer, laid out
    // [sender among its siblings][col/4 within its slice][row] float4.
    const int sl = P.BN / splits, r = c0 / sl, o = split < r ? split : split - 1;
    const uint32_t base = cl_mapa(smem_u32(red), static_cast<uint32_t>(r)) +
                          static_cast<uint32_t>(((o * (sl / 4) + (c0 - r * sl) / 4) * 128 + row) * 16);
#pragma unroll
    for (int j = 0; j < W / 4; ++j)
      asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(base + j * 128 * 16), "f"(v[4 * j]),
                   "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                   : "memory");
    return;
  }
  if (mode == 3) {  // publish this split's partial tile ([unit][col/4][row] float4)
    float4* w = reinterpret_cast<float4*>(P.ws) + (ws_tile + split) * wstride + (c0 / 4) * 128 + row;
#pragma unroll
    for (int j = 0; j < W / 4; ++j)
      __stcg(w + j * 128, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
    return;
  }
  if (splits > 1) split_sum<W>(P, v, red, c0, red_lo, row, split, splits);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < W / 4; ++j)
    *reinterpret_cast<float4*>(wbuf + lane * kEpiLd + 4 * j) =
        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();

  if (mode == 1) {
    // All SMEM reads and addresses first, then the op chain, then the
    // stores: independent instructions the SM can overlap (the previous
    // one-row-per-iteration loop was latency bound).
    constexpr int LPR = W / 4;     // lanes per row
    constexpr int RPI = 32 / LPR;  // rows per instruction
    constexpr int IT = 32 / RPI;
    const int cl = (lane % LPR) * 4;
    const int c = c0 + cl;
    float4 x[IT];
    int64_t addr[IT];
    bool ok[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int rr = it * RPI + lane / LPR;
      const int r = q * 32 + rr;
      ok[it] = r < rows && c < cols && s_row[r] >= 0;
      x[it] = *reinterpret_cast<const float4*>(wbuf + rr * kEpiLd + cl);
      addr[it] = obase + s_row[r] + c;
    }
#pragma unroll 1
    for (int e = 0; e < P.epi_count; ++e) {
      const int k = P.epi_kind[e];
      const float* ep = P.epi_ptr[e];
      if (k == EPI_RELU) {
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          x[it].x = fmaxf(x[it].x, 0.0f);
          x[it].y = fmaxf(x[it].y, 0.0f);
          x[it].z = fmaxf(x[it].z, 0.0f);
          x[it].w = fmaxf(x[it].w, 0.0f);
        }
      } else if (k == EPI_GELU) {
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          x[it].x = epi_gelu(x[it].x);
          x[it].y = epi_gelu(x[it].y);
          x[it].z = epi_gelu(x[it].z);
          x[it].w = epi_gelu(x[it].w);
        }
      } else if (k == EPI_BIAS) {
        const float* bp = ep + n_base + c;
        const float4 bb = c < cols ? make_float4(__ldg(bp), __ldg(bp + 1), __ldg(bp + 2), __ldg(bp + 3))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          x[it].x += bb.x;
          x[it].y += bb.y;
          x[it].z += bb.z;
          x[it].w += bb.w;
        }
      } else {  // EPI_RESIDUAL
        float4 rv[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it)
          rv[it] = ok[it] ? __ldg(reinterpret_cast<const float4*>(ep + addr[it]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          x[it].x += rv[it].x;
          x[it].y += rv[it].y;
          x[it].z += rv[it].z;
          x[it].w += rv[it].w;
        }
      }
    }
    if (dry || (P.diag & 1)) return;  // warm-up pass / timing knob: no side effects
#pragma unroll
    for (int it = 0; it < IT; ++it)
      if (ok[it]) {
        float4* o = reinterpret_cast<float4*>(P.out + addr[it]);
        if (P.out_stream)
          __stcs(o, x[it]);
        else
          *o = x[it];
      }
    if (P.sc.enabled) {
      // Unrolled: a rolled loop indexes x[] / ok[] dynamically and moves
      // them to local memory for the whole epilogue (ncu: STL.128 on the
      // store path of every mode-1 launch).
#pragma unroll
      for (int it = 0; it < IT; ++it)
        if (ok[it]) {
          const int rel = s_rowrel[q * 32 + it * RPI + lane / LPR];
          scatter4(P.sc, org.x, n_base + c, org.y + (rel >> 16), org.z + (rel & 0xFFFF), x[it]);
        }
    }
    if (P.out_bf16) {  // the tensor-core consumers' bf16 copy, same layout
#pragma unroll
      for (int it = 0; it < IT; ++it)
        if (ok[it]) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(x[it].x, x[it].y);
          __nv_bfloat162 hi = __floats2bfloat162_rn(x[it].z, x[it].w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(P.out_bf16 + addr[it]) = pk;
        }
    }
    return;
  }
  // Generic: thread = row, 8 columns per step (loads, ops, stores batched).
  if (dry || (P.diag & 1)) return;
  if (row < rows && s_row[row] >= 0) {
    const int64_t rb = obase + s_row[row];
    const float* mine = wbuf + lane * kEpiLd;
#pragma unroll 1
    for (int j0 = 0; j0 < W; j0 += 8) {
      float y[8];
      int64_t a[8];
      bool cv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        y[j] = mine[j0 + j];
        cv[j] = c0 + j0 + j < cols && s_col[c0 + j0 + j] >= 0;
        a[j] = rb + (cv[j] ? s_col[c0 + j0 + j] : 0);
      }
#pragma unroll 1
      for (int e = 0; e < P.epi_count; ++e) {  // one branch per op, loads batched
        const int k = P.epi_kind[e];
        const float* ep = P.epi_ptr[e];
        if (k == EPI_RELU) {
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = fmaxf(y[j], 0.0f);
        } else if (k == EPI_GELU) {
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = epi_gelu(y[j]);
        } else {
          float t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            t[j] = cv[j] ? __ldg(ep + (k == EPI_BIAS ? static_cast<int64_t>(n_base + (P.bias_rows ? row : c0 + j0 + j))
                                                     : a[j]))
                         : 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] += t[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (cv[j]) {
          if (P.out_stream)
            __stcs(P.out + a[j], y[j]);
          else
            P.out[a[j]] = y[j];
          if (P.out_bf16) P.out_bf16[a[j]] = __float2bfloat16_rn(y[j]);
        }
      if (P.sc.enabled && c0 + j0 + 8 <= cols) {
        const int rel = s_rowrel[row];
        const int hh = org.y + (rel >> 16), ww = org.z + (rel & 0xFFFF);
        scatter4(P.sc, org.x, n_base + c0 + j0, hh, ww, make_float4(y[0], y[1], y[2], y[3]));
        scatter4(P.sc, org.x, n_base + c0 + j0 + 4, hh, ww, make_float4(y[4], y[5], y[6], y[7]));
      }
    }
  }
}

// Instantiated per store mode and split-K (MODE, SPLITK): each instance
// carries only its epilogue path. The epilogue runs a few times per SM per
// launch, so its code is fetched cold; a smaller instance misses the
// instruction caches less (ncu: ~2300 L1i misses per SM on the
// all-paths kernel).
template <int MODE, bool SPLITK>
__global__ void __launch_bounds__(kThreads, LFGPU_UMMA_MINB)
    umma_kernel(const __grid_constant__ CUtensorMap tma_a,
                const __grid_constant__ CUtensorMap tma_b, const __grid_constant__ UmmaParams P,
                const __grid_constant__ CUtensorMap tma_o, const __grid_constant__ CUtensorMap tma_ob) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B atoms) by offsetting the __shared__
  // array itself, so every derived pointer stays in the shared window.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stage_bytes = P.a_boxes * P.a_slot + (P.wres ? 0 : P.b_boxes * P.b_slot);
  const int wbytes = P.wres ? P.nstages * P.w_chunk : 0;
  const int epi_own = P.epi_alias ? 0 : P.epi_region;  // bytes of a separate epilogue region
  float* s_epi = reinterpret_cast<float*>(P.epi_alias ? smem : smem + P.ring_bytes + wbytes);
  const float4* s_red = reinterpret_cast<const float4*>(smem + P.ring_bytes + wbytes + epi_own);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.ring_bytes + wbytes + epi_own + P.red_bytes);
  const int nw = P.wres ? P.nstages : 0;
  const int pipe = P.pipe;
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * pipe;
  const uint32_t tfull0 = empty0 + 8 * pipe;   // 2 accumulator-full barriers
  const uint32_t tempty0 = tfull0 + 16;        // 2 accumulator-empty barriers
  const uint32_t wfull0 = tempty0 + 16;        // nw resident-weight barriers
  const uint32_t redbar = wfull0 + 8 * nw;     // split-K sibling slices landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * pipe + 5 + nw);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);
  StageEntry* s_stage = reinterpret_cast<StageEntry*>(bars + 2 * pipe + 6 + nw);
  int64_t* s_col = reinterpret_cast<int64_t*>(s_stage + P.nstages);
  int64_t* s_row = s_col + P.BN;
  const int32_t* s_rowpos = reinterpret_cast<const int32_t*>(s_row + 128);  // store mode 2
  const int32_t* s_rowrel = s_rowpos + 128;                                   // C2D: (dh << 16) | dw

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int splits = SPLITK ? P.splits : 1;
  const int nunits = P.ntiles * splits;
  // This CTA's units: cyclic (u = blockIdx.x + k * gridDim.x) or, for loop
  // point parallel = 1 without split-K, one contiguous chunk (the outermost
  // loop's static-schedule parallelisation, space.cpp:569-575).
  const int uper = (nunits + gridDim.x - 1) / gridDim.x;
  const int u_first = P.blocked ? blockIdx.x * uper : blockIdx.x;
  const int u_end = P.blocked ? min(nunits, u_first + uper) : nunits;
  const int u_step = P.blocked ? 1 : gridDim.x;
  const int nst = P.nstages;
  unsigned long long* dbg = P.dbg ? P.dbg + 32 * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = gtimer();
  if (P.cdbg && threadIdx.x == 0) atomicMin(P.cdbg, gtimer());

  if (threadIdx.x == 0) {
    for (int s = 0; s < pipe; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, P.dual == 2 ? 2 : 1);  // split issue: both issuers release a stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, P.dual == 2 ? 2 : 1);
      mbar_init(tempty0 + 8 * b, kEpiWarps);  // one arrive per epilogue warp
    }
    for (int c = 0; c < nw; ++c) mbar_init(wfull0 + 8 * c, 1);
    mbar_init(redbar, P.xsplit ? (P.splits - 1) * kEpiWarps : 1);  // sibling warps' DSMEM arrivals / bulk copy
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    if (MODE == 2) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_o)) : "memory");
      if (P.stg_bf)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_ob)) : "memory");
    }
  }
  {  // plan tables (written once by the host, never by kernels: safe before
     // the PDL wait). One flat int array [stages | col_off | row_off]; all
     // loads of a thread are issued before any SMEM store (one DRAM latency).
    const int* src = reinterpret_cast<const int*>(P.stages);
    int* dst = reinterpret_cast<int*>(s_stage);
    const int n = P.table_ints;
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = threadIdx.x + k * kThreads;
      v[k] = i < n ? __ldg(src + i) : 0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = threadIdx.x + k * kThreads;
      if (i < n) dst[i] = v[k];
    }
    for (int i = threadIdx.x + 8 * kThreads; i < n; i += kThreads) dst[i] = __ldg(src + i);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (P.xsplit) cl_sync();  // siblings' barriers initialised before any DSMEM arrival
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // Resident weights that are plan constants can be loaded before the PDL
  // wait: no kernel of this run writes them and every kernel before this
  // one's predecessor has completed (the predecessor only released us after
  // its own wait). Their load then overlaps the previous kernel.
  const bool w_early = P.w_prewait && nw && warp == 0 && u_first < u_end;
  if (w_early && elect_one()) {
    const TileEntry* te = P.tiles + u_first / splits;
    const uint32_t ring0w = smem_u32(smem);
    for (int c = 0; c < nw; ++c) {
      const StageEntry se = s_stage[c];
      const uint32_t bar = wfull0 + 8 * c;
      mbar_expect_tx(bar, P.w_tx);
      for (int b = 0; b < P.b_boxes; ++b)
        tma_load5(&tma_b, ring0w + P.w_off + c * P.w_chunk + b * P.b_slot, bar, __ldg(&te->cb[b][0]) + se.sb[0],
                  __ldg(&te->cb[b][1]) + se.sb[1], __ldg(&te->cb[b][2]) + se.sb[2], __ldg(&te->cb[b][3]) + se.sb[3],
                  __ldg(&te->cb[b][4]) + se.sb[4]);
    }
  }
  __syncwarp();
  // Programmatic dependent launch: everything above overlapped the previous
  // kernel's tail; operands / outputs are touched only after this wait.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (dbg && threadIdx.x == 0) dbg[1] = gtimer();
  if (P.cdbg && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    atomicMin(P.cdbg + 1, t);
    atomicMax(P.cdbg + 2, t);
  }

  const int prod = warp == 0 ? 0 : (warp == 2 || warp == 3 ? warp - 1 : -1);
  if (prod >= 0 && prod < P.nprod) {
    // ---- TMA producers
    const int np = P.nprod;
    const uint32_t tx = P.tx_bytes, a_slot = P.a_slot, b_slot = P.b_slot;
    const uint32_t ring0 = smem_u32(smem);
    const uint32_t b_off = P.a_boxes * a_slot;
    const int na = P.a_boxes, nb = P.b_boxes;
    const bool leader = elect_one();
    if (nw && prod == 0 && leader && u_first < u_end && !w_early) {
      // Resident weights: every chunk's slab once, on its own barrier.
      const TileEntry* te = P.tiles + u_first / splits;
      for (int c = 0; c < nw; ++c) {
        const StageEntry se = s_stage[c];
        const uint32_t bar = wfull0 + 8 * c;
        mbar_expect_tx(bar, P.w_tx);
        for (int b = 0; b < nb; ++b)
          tma_load5(&tma_b, ring0 + P.w_off + c * P.w_chunk + b * b_slot, bar,
                    __ldg(&te->cb[b][0]) + se.sb[0], __ldg(&te->cb[b][1]) + se.sb[1],
                    __ldg(&te->cb[b][2]) + se.sb[2], __ldg(&te->cb[b][3]) + se.sb[3],
                    __ldg(&te->cb[b][4]) + se.sb[4]);
      }
    }
    const int nbs = nw ? 0 : nb;  // B boxes streamed per stage
    int g = 0;  // CTA-wide stage counter (ring slot / phase)
    for (int u = u_first; u < u_end; u += u_step) {
      const int tile = u / splits, split = u - tile * splits;
      const int s_lo = split * nst / splits, s_hi = (split + 1) * nst / splits;
      int s = s_lo + ((prod - g) % np + np) % np;
      g += s_hi - s_lo;
      if (s >= s_hi || !leader) continue;
      int32_t ta[kMaxBoxes][5], tb[kMaxBoxes][5];
      const TileEntry* te = P.tiles + tile;
#pragma unroll
      for (int b = 0; b < kMaxBoxes; ++b)
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          ta[b][d] = b < na ? __ldg(&te->ca[b][d]) : 0;
          tb[b][d] = b < nb ? __ldg(&te->cb[b][d]) : 0;
        }
      for (; s < s_hi; s += np) {
        const int it = g - (s_hi - s);  // CTA-wide index of stage s
        const int slot = it % pipe;
        const uint32_t phase = static_cast<uint32_t>(it / pipe) & 1u;
        mbar_wait(empty0 + 8 * slot, phase ^ 1);
        const uint32_t bar = full0 + 8 * slot;
        mbar_expect_tx(bar, tx);
        const StageEntry se = s_stage[s];
        const uint32_t a_dst = ring0 + slot * stage_bytes;
#pragma unroll
        for (int b = 0; b < kMaxBoxes; ++b)
          if (b < na)
            tma_load5(&tma_a, a_dst + b * a_slot, bar, ta[b][0] + se.sa[0], ta[b][1] + se.sa[1],
                      ta[b][2] + se.sa[2], ta[b][3] + se.sa[3], ta[b][4] + se.sa[4]);
#pragma unroll
        for (int b = 0; b < kMaxBoxes; ++b)
          if (b < nbs)
            tma_load5(&tma_b, a_dst + b_off + b * b_slot, bar, tb[b][0] + se.sb[0],
                      tb[b][1] + se.sb[1], tb[b][2] + se.sb[2], tb[b][3] + se.sb[3],
                      tb[b][4] + se.sb[4]);
      }
    }
    __syncwarp();
    if (dbg && prod == 0 && lane == 0) dbg[2] = gtimer();
  } else if (warp == 1 || (P.dual && warp == 3)) {
    // ---- MMA issuer (whole warp loops; one elected lane issues)
    const uint64_t adesc = P.a_desc, bdesc = P.b_desc;
    const uint32_t idesc = P.idesc, akadv16 = P.a_kadv >> 4, bkadv16 = P.b_kadv >> 4;
    const int ksteps = (P.diag & 128) ? 1 : P.ksteps;  // timing knob: one k-step per stage
    const uint32_t ring0 = smem_u32(smem);
    const uint32_t a_off_b = P.a_boxes * P.a_slot;
    const bool leader = elect_one();
    int slot = 0;
    uint32_t phase = 0;
    int i = 0;
    const int role = warp == 3 ? 1 : 0;
    for (int u = u_first; u < u_end; u += u_step, ++i) {
      const int split = u % splits;
      const int s_lo = split * nst / splits, s_hi = (split + 1) * nst / splits;
      if (P.dual == 1 && (i & 1) != role) {  // the other issuer's unit: step over its stages
        for (int s = s_lo; s < s_hi; ++s)
          if (++slot == pipe) {
            slot = 0;
            phase ^= 1;
          }
        continue;
      }
      const int b = i & 1;
      mbar_wait(tempty0 + 8 * b, (static_cast<uint32_t>(i >> 1) & 1u) ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // split issue (dual == 2): both issuers take every unit, alternate
      // MMAs of it, each into its own accumulator (summed by the epilogue)
      const bool split_issue = P.dual == 2;
      const uint32_t dtm = tmem + static_cast<uint32_t>((split_issue ? 2 * b + role : b) * P.BN);
      int mi = 0;  // this unit's MMA index (split issue: issuer `role` takes mi % 2 == role)
      for (int s = s_lo; s < s_hi; ++s) {
        mbar_wait(full0 + 8 * slot, phase);
        if (dbg && leader && i == 0 && s == s_lo) dbg[3] = gtimer();
        if (P.cdbg && leader && i == 0 && s == s_lo) atomicMin(P.cdbg + 3, gtimer());
        if (dbg && leader && (P.diag & 256) && i == 0 && s - s_lo < 16) dbg[16 + s - s_lo] = gtimer();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (nw) {
          mbar_wait(wfull0 + 8 * s, 0);  // completes once; later waits return at once
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (leader) {
          const uint32_t a_addr = ring0 + slot * stage_bytes;
          const uint32_t b_addr = nw ? ring0 + P.w_off + s * P.w_chunk : a_addr + a_off_b;
          // Descriptors are (address >> 4) in their low 14 bits: advance
          // them by 16-byte units directly (SMEM addresses < 256 KB never
          // carry out of the field).
          const uint64_t ad0 = adesc | (a_addr >> 4), bd0 = bdesc | (b_addr >> 4);
          const int ntaps = (P.diag & 8) ? 1 : P.ntaps;
          if (split_issue) {
            for (int t = 0; t < ntaps; ++t) {
              const uint64_t adt = ad0 + ((P.diag & 4) ? 0 : (P.a_tap[t] >> 4)), bdt = bd0 + (P.b_tap[t] >> 4);
              for (int k = 0; k < ksteps; ++k, ++mi)
                if ((mi & 1) == role)
                  umma_bf16(dtm, adt + k * akadv16, bdt + k * bkadv16, idesc, mi >= 2);
            }
          } else {
            for (int t = 0; t < ntaps; ++t) {
              const uint64_t adt = ad0 + ((P.diag & 4) ? 0 : (P.a_tap[t] >> 4)), bdt = bd0 + (P.b_tap[t] >> 4);
              for (int k = 0; k < ksteps; ++k)
                umma_bf16(dtm, adt + k * akadv16, bdt + k * bkadv16, idesc, (s != s_lo) | t | k);
            }
          }
          umma_commit(empty0 + 8 * slot);
        }
        __syncwarp();
        if (++slot == pipe) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (leader) umma_commit(tfull0 + 8 * b);
      __syncwarp();
    }
    if (dbg && leader) atomicMax(dbg + 4, gtimer());
  } else if (warp >= kEpiWarp0) {
    // ---- epilogue (8 warps; warp w reads TMEM lanes 32*(w%4)..+31; the
    // two halves take alternate 16-column chunks)
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    const int row = q * 32 + lane;
    float* wbuf = s_epi + (warp - kEpiWarp0) * 32 * kEpiLd;
    const bool half_leader = lane == 0 && q == 0;  // TMA-store issuer of this half
    const int BN = P.BN;
    uint32_t red_phase = 0;
    int i = 0;
    // Warm-up pass: the epilogue code is fetched cold (a few runs per SM per
    // launch), so the idle epilogue warps first run their path once over
    // the first unit with every side effect off (no accumulator wait, no
    // stores, no barrier arrivals) while the main loop fills TMEM; the real
    // pass then executes from a warm instruction cache.
    bool dry = !SPLITK && (P.diag & 64) && !P.epi_alias;  // opt-in (no measured gain)
    for (int u = u_first; u < u_end;) {
      const int tile = u / splits, split = u - tile * splits;
      const int b = i & 1;
      const uint32_t tempty = tempty0 + 8 * b;
      // The tile entry does not depend on the accumulator: load it before
      // waiting so its (possibly DRAM) latency hides under the main loop.
      const TileEntry* te = P.tiles + tile;
      const int rows = __ldg(&te->rows), cols = __ldg(&te->cols), n_base = __ldg(&te->n_base);
      const int3 org = make_int3(__ldg(&te->org[0]), __ldg(&te->org[1]), __ldg(&te->org[2]));
      const int64_t obase = __ldg(&te->out_base) + P.col0;
      int32_t tco[5] = {0, 0, 0, 0, 0};  // TMA-store box origin (mode 2 issuers)
      if (MODE == 2 && half_leader) {
#pragma unroll
        for (int d = 0; d < 5; ++d) tco[d] = __ldg(P.tile_coords + tile * 5 + d);
      }
      if (!dry) mbar_wait(tfull0 + 8 * b, static_cast<uint32_t>(i >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (dbg && !dry && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[5] = gtimer();
      if (dbg && !dry && (P.diag & 32) && i == 0 && lane == 0) dbg[24 + warp - kEpiWarp0] = gtimer();
      if (dbg && !dry && i < 4 && threadIdx.x == kEpiWarp0 * 32) dbg[8 + i] = gtimer();
      const uint32_t tbase =
          tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>((P.dual == 2 ? 2 * b : b) * BN);
      const int64_t ws_tile = static_cast<int64_t>(tile) * splits;
      const int red_lo = split * (BN / splits);
      constexpr int mode = MODE;
      // Items are 16-column chunks (one small inlined body: each SM runs the
      // epilogue only a few times per launch, so code size is paid in cold
      // instruction fetches): first (split-K only) the columns the sibling
      // splits reduce, published to the workspace; then this unit's own
      // columns [lo, hi), summed over the splits in split order (own partial
      // from TMEM) and stored with the fused chain.
      //   Split-K: split s reduces columns [s*BN/S, (s+1)*BN/S). The
      // siblings meet at a per-tile counter (they are co-resident: the grid
      // is a multiple of S and units are dealt in rounds), then bulk-copy
      // the siblings' slices of the reduced columns into SMEM.
      const int sl = BN / splits, lo = split * sl;
      const int npub = (BN - sl) / 16, nown = sl / 16;
      for (int it = half; it < npub; it += 2) {
        const int c0 = it * 16 < lo ? it * 16 : it * 16 + sl;
        epi_chunk<16>(P, tbase, c0, row, lane, q, wbuf, rows, cols, n_base, obase, s_row, s_col, 3,
                      split, splits, ws_tile, s_red, red_lo, false, tempty, org, s_rowrel, false);
      }
      if (splits > 1 && P.xsplit) {
        // Release this warp's DSMEM partials to every sibling (cluster
        // scope), then wait for theirs: no global round trip, no spin.
        if (dbg && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[16] = gtimer();
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        __syncwarp();
        if (lane == 0)
          for (int o2 = 0; o2 < splits; ++o2)
            if (o2 != split) cl_arrive(cl_mapa(redbar, static_cast<uint32_t>(o2)));
        cl_wait(redbar, red_phase);
        red_phase ^= 1;
        if (dbg && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[19] = gtimer();
      } else if (splits > 1) {
        if (dbg && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[16] = gtimer();
        __threadfence();
        epi_bar();
        if (dbg && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[17] = gtimer();
        if (threadIdx.x == kEpiWarp0 * 32) {
          atomicAdd(P.counters + tile, 1);
          int seen;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(P.counters + tile) : "memory");
            if (seen < splits) __nanosleep(64);
          } while (seen < splits);
          // generic-proxy writes of the siblings -> async-proxy bulk copies
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const uint32_t slice_bytes = static_cast<uint32_t>(sl) * 128 * 4;
          mbar_expect_tx(redbar, slice_bytes * (splits - 1));
          for (int o = 0; o < splits - 1; ++o) {
            const int sib = o < split ? o : o + 1;
            const float* src = P.ws + ((ws_tile + sib) * (BN / 4) + lo / 4) * 128 * 4;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(s_red) + o * slice_bytes),
                "l"(src), "r"(slice_bytes), "r"(redbar)
                : "memory");
          }
        }
        if (dbg && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[18] = gtimer();
        mbar_wait(redbar, red_phase);
        red_phase ^= 1;
        if (dbg && i == 0 && threadIdx.x == kEpiWarp0 * 32) dbg[19] = gtimer();
      }
      if (half >= nown && !dry) {  // nothing for this half: hand the accumulator back now
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
      for (int k = half; k < nown; k += 2) {
        const int c0 = lo + k * 16;
        const bool last = k + 2 >= nown;  // this warp's last TMEM read of the unit
        if (mode == 2) {
          // TMA-store epilogue: registers -> swizzled SMEM box -> one
          // cp.async.bulk.tensor per 16-column chunk; each half owns one
          // staging buffer and its own bulk group.
          const bool tr = dbg && !dry && (P.diag & 2) && i == ((P.diag & 16) ? 1 : 0) &&
                          threadIdx.x == kEpiWarp0 * 32;
          // Buffer ring per half: chunk n uses buffer n % nbuf, free once at
          // most nbuf-1 younger bulk groups are still reading.
          const int nbuf = P.stg_nbuf, bi = ((k - half) >> 1) % nbuf;
          if (half_leader) {
            if (nbuf == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          }
          half_bar(half);
          uint8_t* stf = smem + P.stg_off + (half * nbuf + bi) * P.stg_f32;
          uint8_t* stb = smem + P.stg_off + 2 * nbuf * P.stg_f32 + (half * nbuf + bi) * P.stg_bf;
          if (tr) dbg[k == half ? 24 : 29] = gtimer();
          float v[16];
          acc_ld<16>(P.dual, BN, tbase + c0, v);
          if (tr && k == half) dbg[25] = gtimer();
          if (last && !dry) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
          }
          if (splits > 1) split_sum<16>(P, v, s_red, c0, red_lo, row, split, splits);
          const int rp = row < rows ? s_rowpos[row] : -1;
          if (rp >= 0) {
            const int64_t addr = obase + s_row[row];
            const int cs = P.stg_cstride;
            // One branch per op, and a bias / residual op's 16 loads all
            // issued before the adds: a per-element branch kept each load
            // behind the previous add (16 serial L1/L2 latencies per chunk;
            // ncu: ~59 instructions and a long-scoreboard stall per element).
#pragma unroll 1
            for (int e = 0; e < P.epi_count; ++e) {
              const int kk = P.epi_kind[e];
              const float* ep = P.epi_ptr[e];
              if (kk == EPI_RELU) {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.0f);
              } else if (kk == EPI_GELU) {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = epi_gelu(v[j]);
              } else {
                float t[16];
                if (kk == EPI_BIAS) {
#pragma unroll
                  for (int j = 0; j < 16; ++j) t[j] = __ldg(ep + n_base + c0 + j);
                } else {
#pragma unroll
                  for (int j = 0; j < 16; ++j) t[j] = __ldg(ep + addr + (cs ? s_col[c0 + j] : c0 + j));
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] += t[j];
              }
            }
            if (cs) {
              // Transposed box: column j is the plane at j * cs; consecutive
              // rows of a warp are consecutive words (conflict-free).
              float* sf = reinterpret_cast<float*>(stf) + rp;
#pragma unroll
              for (int j = 0; j < 16; ++j) sf[j * cs] = v[j];
              if (P.stg_bf) {
                __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(stb) + rp;
#pragma unroll
                for (int j = 0; j < 16; ++j) sb[j * cs] = __float2bfloat16_rn(v[j]);
              }
            } else {
            // SWIZZLE_64B rows of 16 fp32: 16-byte chunk j at j ^ ((rp >> 1) & 3)
            uint8_t* sf = stf + rp * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<float4*>(sf + ((j ^ ((rp >> 1) & 3)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            if (P.stg_bf) {  // SWIZZLE_32B rows of 16 bf16: chunk j at j ^ ((rp >> 2) & 1)
              uint8_t* sb = stb + rp * 32;
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                uint4 pk;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]);
                __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
                __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
                pk.x = *reinterpret_cast<uint32_t*>(&h0);
                pk.y = *reinterpret_cast<uint32_t*>(&h1);
                pk.z = *reinterpret_cast<uint32_t*>(&h2);
                pk.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(sb + ((j ^ ((rp >> 2) & 1)) << 4)) = pk;
              }
            }
            }
          }
          if (tr && k == half) dbg[26] = gtimer();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          half_bar(half);
          if (tr && k == half) dbg[27] = gtimer();
          if (half_leader && !dry) {
            const int cd = P.stg_cdim;
            const int32_t x0 = tco[0] + (cd == 0 ? c0 : 0), x1 = tco[1] + (cd == 1 ? c0 : 0),
                          x2 = tco[2] + (cd == 2 ? c0 : 0), x3 = tco[3] + (cd == 3 ? c0 : 0),
                          x4 = tco[4] + (cd == 4 ? c0 : 0);
            tma_store5(&tma_o, smem_u32(stf), x0, x1, x2, x3, x4);
            if (P.stg_bf)
              tma_store5(&tma_ob, smem_u32(stb), x0, x1, x2, x3, x4);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {
          epi_chunk<16>(P, tbase, c0, row, lane, q, wbuf, rows, cols, n_base, obase, s_row, s_col,
                        mode, split, splits, ws_tile, s_red, red_lo, last, tempty, org, s_rowrel, dry);
        }
        if (dbg && !dry && !(P.diag & 256) && i == 0 && k < 8 && threadIdx.x == kEpiWarp0 * 32)
          dbg[20 + k] = gtimer();
      }
      if (splits > 1) {
        epi_bar();  // every warp is done with the SMEM slices of this unit
        if (threadIdx.x == kEpiWarp0 * 32) {
          // Last one out re-arms both counters for the next launch.
          if (atomicAdd(P.counters + P.ntiles + tile, 1) == splits - 1) {
            P.counters[tile] = 0;
            P.counters[P.ntiles + tile] = 0;
          }
        }
      }
      if (dbg && !dry && i < 4 && threadIdx.x == kEpiWarp0 * 32) dbg[12 + i] = gtimer();
      if (dry) {  // same unit again, for real
        dry = false;
        continue;
      }
      u += u_step;
      ++i;
    }
    if (half_leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (dbg && threadIdx.x == kEpiWarp0 * 32) dbg[6] = gtimer();
    if (P.cdbg && threadIdx.x == kEpiWarp0 * 32) atomicMax(P.cdbg + 5, gtimer());
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (P.xsplit) cl_sync();  // no CTA leaves while a sibling may still address its SMEM
  else __syncthreads();
  if (P.cdbg && threadIdx.x == 0) atomicMax(P.cdbg + 4, gtimer());
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
      strides[d] = d == 1 ? ((v.dims[0] * v.elem_bytes + 15) / 16) * 16 : strides[d - 1] * dims[d - 1];
      box[d] = 1;
      es[d] = 1;
    }
  }
  CUtensorMapSwizzle sw = v.swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : v.swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : v.swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  const CUtensorMapDataType dt =
      v.elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = encode_fn()(&m, dt, 5, const_cast<void*>(base),
                           dims, strides + 1, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // A view TMA cannot express is an illegal candidate, not a device fault.
  if (r != CUDA_SUCCESS)
    fail(LFGPU_EUNSUPPORTED, "TMA cannot express operand view (cuTensorMapEncodeTiled " +
                                 std::to_string(r) + ")");
  return m;
}

uint64_t desc_bits(const OperandView& v) {
  uint64_t layout = v.swizzle == 128 ? 2 : v.swizzle == 64 ? 4 : v.swizzle == 32 ? 6 : 0;
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
  void* p[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  ~Tables() {
    for (auto* q : p)
      if (q) dev_free(q);
  }
};

template <typename T>
void* up(const std::vector<T>& v) {
  void* d = nullptr;
  size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
  if (!(d = dev_alloc(bytes))) fail(LFGPU_ECUDA, "device allocation of tables");
  if (!v.empty() && cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    fail(LFGPU_ECUDA, "cudaMemcpy tables");
  return d;
}

}  // namespace

bool umma_view_encodable(const OperandView& v, std::string* why) {
  try {
    encode(v, reinterpret_cast<void*>(static_cast<uintptr_t>(1) << 20));
    return true;
  } catch (const Error& e) {
    *why = e.what();
    return false;
  }
}

CUtensorMap umma_encode(const OperandView& v, const void* base) { return encode(v, base); }
uint64_t umma_desc_bits(const OperandView& v) { return desc_bits(v); }
uint32_t umma_idesc(int M, int N, bool a_mn, bool b_mn) { return idesc_of(M, N, a_mn, b_mn); }

static void* g_umma_dbg = nullptr;
static unsigned long long* g_chain_dbg = nullptr;
void umma_set_chain_buffer(void* p) { g_chain_dbg = static_cast<unsigned long long*>(p); }
void* umma_debug_buffer() { return g_umma_dbg; }
void umma_set_debug_buffer(void* p) { g_umma_dbg = p; }

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

int umma_num_sms() { return num_sms(); }

const void* umma_kernel_fn(int mode, bool splitk);

UmmaLaunch umma_prepare(const UmmaPlan& p) {
  UmmaLaunch L;
  if (p.pair) {
    PairPlan q = *p.pair;
    q.a = p.a;
    q.b = p.b;
    q.out = p.out;
    q.out_bf16 = p.out_bf16;
    q.epi_count = p.epi_count;
    for (int e = 0; e < p.epi_count; ++e) q.epi[e] = p.epi[e];
    L.pair = std::make_shared<PairLaunch>(pair_prepare(q));
    L.ntiles = q.MT / 2 * q.NT;
    L.BN = q.BN;
    L.splits = L.pair->S;
    L.grid = L.pair->grid;
    L.pipe = L.pair->pipe;
    L.store_mode = L.pair->col_unit;
    return L;
  }
  std::memset(&L.tma_o, 0, sizeof(L.tma_o));
  std::memset(&L.tma_ob, 0, sizeof(L.tma_ob));
  L.tma_a = encode(p.A, p.a);
  L.tma_b = encode(p.B, p.b);
  auto t = std::make_shared<Tables>();
  t->p[0] = up(p.tiles);
  {  // [stages | col_off | row_off] contiguous: the kernel copies it to SMEM in one pass
    std::vector<int32_t> tab(p.stages.size() * sizeof(StageEntry) / 4 + 2 * (p.col_off.size() + 128) + 256);
    size_t o = 0;
    std::memcpy(tab.data(), p.stages.data(), p.stages.size() * sizeof(StageEntry));
    o += p.stages.size() * sizeof(StageEntry) / 4;
    std::memcpy(tab.data() + o, p.col_off.data(), p.col_off.size() * 8);
    o += p.col_off.size() * 2;
    std::vector<int64_t> rows(128, 0);
    for (size_t r = 0; r < 128 && r < p.row_off.size(); ++r) rows[r] = p.row_off[r];
    std::memcpy(tab.data() + o, rows.data(), 128 * 8);
    o += 256;
    for (int r = 0; r < 128; ++r) tab[o + r] = p.ost.ok ? p.ost.row_pos[r] : -1;
    o += 128;
    for (int r = 0; r < 128; ++r) tab[o + r] = r < static_cast<int>(p.row_rel.size()) ? p.row_rel[r] : 0;
    L.table_ints = static_cast<int>(tab.size());
    t->p[1] = up(tab);
  }
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
  while (cols < 2 * p.BN) cols *= 2;  // two accumulators (epilogue/main-loop overlap)
  if (cols > 512) fail(LFGPU_EUNSUPPORTED, "accumulators exceed 512 TMEM columns");
  L.tmem_cols = cols;  // split issue doubles it below
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
  L.out_bf16 = p.out_bf16;
  L.out_stream = p.out_stream;
  // Split-K (schedule `order`: 0 = heuristic, 1 = never, 2 = at least 2):
  // when the tiles alone leave most of the SMs idle and the K loop is long.
  const int sms = num_sms();
  L.splits = 1;
  // A halo C2D stage is KH*KW UMMA groups (heavy), so a split may be a
  // single stage there; a GEMM / per-tap stage is one K step (>= 4 each).
  const int min_stages = p.kind == UMMA_GEMM ? std::max(1, 4 / p.ntaps) : (p.ntaps > 1 ? 1 : 4);
  if (p.split_pref != 1 && L.ntiles * 2 <= sms && L.nstages >= 2 * min_stages) {
    L.splits = std::min({sms / L.ntiles, L.nstages / min_stages, 8});
    if (L.splits < 2) L.splits = 1;
  }
  if (p.split_pref == 2) L.splits = std::max(L.splits, std::min(2, L.nstages));
  if (const char* e = getenv("LFGPU_SPLITK")) L.splits = std::max(1, std::min(atoi(e), L.nstages));
  // Each split reduces a column slice: BN/S must be a multiple of 16, and
  // all S splits of a tile must fit in one round of the persistent grid.
  L.splits = std::min(L.splits, 4);  // kMaxSplits (k_umma.cu)
  while (L.splits > 1 && ((L.BN % L.splits) || (L.BN / L.splits) % 16 || L.splits > sms))
    --L.splits;
  L.red_bytes = L.splits > 1 ? (L.splits - 1) * 128 * (p.BN / L.splits) * 4 : 0;
  L.wres = p.wres;
  L.w_chunk = L.b_boxes * L.b_slot;
  L.w_tx = L.b_boxes * L.b_bytes;
  const size_t wbytes = p.wres ? static_cast<size_t>(p.stages.size()) * L.w_chunk : 0;
  // Store mode 1 (transposed, float4 row stores): output columns contiguous
  // and every stored row 16-byte aligned.
  int max_rows = 0;
  for (const auto& te : p.tiles) max_rows = std::max(max_rows, static_cast<int>(te.rows));
  bool cols_unit = !p.col_off.empty();
  for (size_t c = 0; c < p.col_off.size(); ++c)
    if (p.col_off[c] != p.col_off[0] + static_cast<int64_t>(c)) cols_unit = false;
  bool aligned = cols_unit && (p.col_off[0] % 4 == 0);
  for (int r = 0; aligned && r < max_rows && r < static_cast<int>(p.row_off.size()); ++r)
    if (p.row_off[r] >= 0 && p.row_off[r] % 4) aligned = false;
  for (const auto& te : p.tiles)
    if (te.out_base % 4 || te.cols % 4) aligned = false;
  L.store_mode = aligned ? 1 : 0;
  L.col0 = aligned ? p.col_off[0] : 0;
  // Store mode 2 (TMA store) when the output tile is a TMA box.
  bool full_cols = true;
  for (const auto& te : p.tiles)
    if (te.cols != p.BN) full_cols = false;
  const char* sm_env = getenv("LFGPU_STORE_MODE");
  // TMA store when the schedule asks (vectorize), and by default for
  // transposed boxes whose alternative is the generic scalar path (one
  // 4-byte store per element, ~3x slower epilogue on the cfg1 b16 conv).
  const bool auto_tma = p.ost.ok && p.ost.col_stride > 0 && !aligned;
  const bool want_tma = ((p.tma_store || auto_tma) && !(sm_env && atoi(sm_env) < 2)) ||
                        (sm_env && atoi(sm_env) == 2);
  // Transposed boxes (columns not innermost) stage each column as a plane
  // of the box, unswizzled; their bf16 twin must be encodable too.
  const bool tbox = p.ost.ok && p.ost.col_stride > 0;
  OperandView ob;
  bool ob_ok = true;
  if (p.ost.ok && p.out_bf16) {
    ob = p.ost.O;
    ob.elem_bytes = 2;
    ob.swizzle = tbox ? 0 : 32;
    for (int d = 1; d < ob.rank; ++d) ob.strides[d] /= 2;
    std::string why;
    ob_ok = umma_view_encodable(ob, &why);
  }
  if (p.ost.ok && (cols_unit || tbox) && ob_ok && full_cols && want_tma && !p.scatter.enabled) {
    L.store_mode = 2;
    L.col0 = tbox ? 0 : p.col_off[0];
    L.stg_cstride = tbox ? p.ost.col_stride : 0;
    L.stg_cdim = p.ost.col_dim;
    L.tma_o = encode(p.ost.O, p.out);
    L.stg_f32 = (p.ost.box_rows * 64 + 1023) / 1024 * 1024;
    if (p.out_bf16) {
      L.tma_ob = encode(ob, p.out_bf16);
      L.stg_bf = (p.ost.box_rows * 32 + 1023) / 1024 * 1024;
    }
    t->p[6] = up(p.ost.tile_coords);
    L.d_tcoords = t->p[6];
    L.stg_nbuf = (L.BN / L.splits / 16 + 1) / 2 >= 2 ? 2 : 1;
  }
  if (sm_env && atoi(sm_env) == 0) {  // diagnostics: force the generic path
    L.store_mode = 0;
    L.col0 = 0;
  }
  // SMEM: ring | resident weights | epilogue buffers | split-K slices |
  // barriers | tables. The ring gives up stages if the rest needs room.
  // When every CTA gets at most one unit, the epilogue runs only after the
  // unit's last MMA (the ring is idle: all loads landed and were consumed),
  // so its buffers alias the ring and the freed bytes become one more stage
  // in flight (L2->SMEM ingest is latency-bound: bytes in flight / ~1.4 us).
  const int64_t ntl = static_cast<int64_t>(p.tiles.size());
  auto layout_smem = [&]() {
    const size_t ring = static_cast<size_t>(L.pipe) *
                        (L.a_boxes * L.a_slot + (p.wres ? 0 : L.b_boxes * L.b_slot));
    L.ring_bytes = static_cast<int>((ring + 1023) / 1024 * 1024);
    // Mode 2 stages in the epilogue region (its transpose buffers are
    // unused then): two buffers per half when a half stores >= 2 chunks.
    L.epi_region = std::max(kEpiSmemBytes, 2 * L.stg_nbuf * (L.stg_f32 + L.stg_bf));
    L.epi_alias = !getenv("LFGPU_NO_EPI_ALIAS") && ntl * L.splits <= sms / L.splits * L.splits &&
                  L.ring_bytes >= L.epi_region;
    L.smem = 1024 + L.ring_bytes + wbytes + (L.epi_alias ? 0 : L.epi_region) + L.red_bytes +
             8 * (2 * L.pipe + 5 + (p.wres ? p.stages.size() : 0)) + 8 +
             sizeof(StageEntry) * p.stages.size() + 8 * p.BN + 8 * 128 + 8 * 128 + 64;
  };
  for (;;) {
    layout_smem();
    if (L.smem <= 227 * 1024) break;
    if (L.stg_nbuf > 1 && L.pipe <= 4) {
      L.stg_nbuf = 1;
    } else if (L.pipe > 2) {
      --L.pipe;
    } else if (L.splits > 1) {  // then give up split-K slices
      --L.splits;
      while (L.splits > 1 && ((L.BN % L.splits) || (L.BN / L.splits) % 16)) --L.splits;
      L.red_bytes = L.splits > 1 ? (L.splits - 1) * 128 * (p.BN / L.splits) * 4 : 0;
    } else {
      break;
    }
  }
  if (L.smem > 227 * 1024) fail(LFGPU_EUNSUPPORTED, "tcgen05 kernel SMEM exceeds 227 KB");
  if (L.epi_alias) {  // grow the ring into the freed bytes, up to one unit's stages
    const int spu = (L.nstages + L.splits - 1) / L.splits;
    while (L.pipe < spu && !getenv("LFGPU_MAX_PIPE")) {
      ++L.pipe;
      layout_smem();
      if (L.smem > 227 * 1024 || !L.epi_alias) {
        --L.pipe;
        layout_smem();
        break;
      }
    }
  }
  // One CTA per SM: the kernel's register budget (launch bounds 1, ~230
  // registers) leaves no room for a second; measured 2-per-SM variants
  // (launch bounds 2, <= 128 registers, <= 113 KB SMEM) were not faster.
  L.per_sm = 1;
  L.nprod = std::max(1, std::min(3, L.pipe - 1));
  L.ntaps = p.ntaps;
  L.scatter = p.scatter;
  if (L.scatter.enabled && (L.scatter.ic % 4 || p.BN % 8))
    fail(LFGPU_EINVAL, "umma: absorbed Padding needs 4-aligned channel bricks");
  for (int t = 0; t < p.ntaps; ++t)
    L.b_tapv[t] = t < static_cast<int>(p.b_tapv.size()) ? p.b_tapv[t] : t * p.b_tap;
  L.bias_rows = p.trans;
  if (p.ntaps > kMaxTaps || static_cast<int>(p.a_tap.size()) < p.ntaps)
    fail(LFGPU_EINVAL, "umma: tap table");
  for (int t = 0; t < p.ntaps; ++t) L.a_tap[t] = p.a_tap[t];
  if (L.splits > 1) {
    const size_t ws = sizeof(float) * static_cast<size_t>(L.ntiles) * L.splits * 128 * L.BN;
    if (!(t->p[4] = dev_alloc(ws))) fail(LFGPU_ECUDA, "device allocation of the split-K workspace");
    if (!(t->p[5] = dev_alloc(2 * sizeof(int) * L.ntiles)) ||
        cudaMemset(t->p[5], 0, 2 * sizeof(int) * L.ntiles) != cudaSuccess)
      fail(LFGPU_ECUDA, "cudaMalloc split-K counters");
    L.ws = static_cast<float*>(t->p[4]);
    L.counters = static_cast<int*>(t->p[5]);
  }
  // Persistent grid: one CTA per SM at most, units dealt round-robin.
  {
    // Fill both resident slots only when there is more than one wave of
    // units (then one CTA's epilogue overlaps the other's main loop).
    const char* e = getenv("LFGPU_GRID_PER_SM");  // diagnostics override
    int per = L.ntiles * L.splits > sms ? L.per_sm : 1;
    if (e) per = std::max(1, std::min(atoi(e), L.per_sm));
    L.grid = std::min(L.ntiles * L.splits, per * sms / L.splits * L.splits);
  }
  // Two MMA issuers. One thread issues a tcgen05.mma only every ~80 cycles
  // (tools/micro/mma_rate.cu: M=128 N<=128 tops out at 84 cycles per MMA
  // from one thread, while two issuing warps on different SM sub-partitions
  // reach 48 (N=64) and the dense peak (N=128)), so N <= 128 tiles are
  // issue-bound. Warp 3 becomes a second issuer taking every other unit
  // (own TMEM accumulator, the ring's stages in order), leaving two TMA
  // producers. Worth it when a CTA gets >= 2 units and two units' stages
  // fit in the ring together.
  {
    const int units = L.ntiles * L.splits;
    const int spu = (L.nstages + L.splits - 1) / L.splits;
    L.dual = p.BN <= 128 && units >= 2 * L.grid && 2 * spu <= L.pipe;
    if (const char* e = getenv("LFGPU_DUAL_MMA")) L.dual = atoi(e) != 0;
    L.blocked = p.persistent && L.splits == 1 ? 1 : 0;
  }
  // DSMEM split-K: when every CTA gets exactly one unit, the S splits of a
  // tile run as one cluster of S CTAs and exchange partials through their
  // SMEM (the workspace protocol stays for the multi-unit case).
  {
    const int units = L.ntiles * L.splits;
    // Measured (tools/xsplit_check.py): under a cluster launch an operand
    // loaded as two or more TMA boxes per stage (MN-major B wider than 64
    // bf16) reads wrong data — the same failure the CTA-pair kernel shows
    // (lf_pair.hpp); single-box operands are exact. Cluster exchange only then.
    L.xsplit = L.splits > 1 && units == L.grid && !L.dual && L.a_boxes == 1 && L.b_boxes == 1 &&
                       !getenv("LFGPU_NO_XSPLIT")
                   ? 1
                   : 0;
    if (L.xsplit) {
      cudaLaunchConfig_t cfg;
      std::memset(&cfg, 0, sizeof(cfg));
      cfg.gridDim = dim3(L.grid);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = L.smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = L.splits;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      const void* f = umma_kernel_fn(L.store_mode, true);
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (cudaOccupancyMaxActiveClusters(&n, f, &cfg) != cudaSuccess || n * L.splits < L.grid) L.xsplit = 0;
      cudaGetLastError();
    }
    // Split issue (dual = 2, opt-in with LFGPU_DUAL_MMA=2): both issuers take
    // every unit and alternate its MMAs into two accumulators the epilogue
    // sums. Measured on the cfg1 b16 conv it does not beat one issuer (MMA
    // phase 10.6 vs 10.1 us; the alternate-unit issuers 7.5 us): the two
    // accumulators' MMAs do not overlap in the tensor pipe the way two
    // units' do. Kept as a diagnostic, covered by the parity tests.
    const int dual_units = L.dual;
    if (const char* e = getenv("LFGPU_DUAL_MMA")) L.dual = std::max(0, std::min(2, atoi(e)));
    if (L.dual == 2) {
      if (L.tmem_cols * 2 > 512 || L.xsplit) L.dual = dual_units;
      else L.tmem_cols *= 2;
    }
    if (L.dual) L.nprod = std::min(L.nprod, 2);
  }
  static_assert(sizeof(TileEntry) == 192, "TileEntry layout");
  return L;
}

// The kernel instance for (store mode, split-K).
const void* umma_kernel_fn(int mode, bool splitk) {
  using KernelFn = void (*)(CUtensorMap, CUtensorMap, UmmaParams, CUtensorMap, CUtensorMap);
  static const KernelFn fns[3][2] = {{umma_kernel<0, false>, umma_kernel<0, true>},
                                     {umma_kernel<1, false>, umma_kernel<1, true>},
                                     {umma_kernel<2, false>, umma_kernel<2, true>}};
  return reinterpret_cast<const void*>(fns[std::min(std::max(mode, 0), 2)][splitk ? 1 : 0]);
}

cudaError_t umma_launch(const UmmaLaunch& L, cudaStream_t stream) {
  if (L.ntiles == 0) return cudaSuccess;
  if (L.pair) return pair_launch(*L.pair, stream);
  UmmaParams P;
  std::memset(&P, 0, sizeof(P));
  P.tiles = static_cast<const TileEntry*>(L.d_tiles);
  P.stages = static_cast<const StageEntry*>(L.d_stages);
  P.row_off = static_cast<const int64_t*>(L.d_rows);
  P.col_off = static_cast<const int64_t*>(L.d_cols);
  P.out = L.out;
  P.out_bf16 = static_cast<__nv_bfloat16*>(L.out_bf16);
  P.out_stream = L.out_stream;
  P.epi_count = L.epi_count;
  for (int e = 0; e < L.epi_count; ++e) {
    P.epi_kind[e] = L.epi_kinds[e];
    P.epi_ptr[e] = L.epi_ptr[e];
  }
  P.ntiles = L.ntiles;
  P.nstages = L.nstages;
  P.BN = L.BN;
  P.ksteps = L.KC / 16;
  P.pipe = L.pipe;
  P.nprod = L.nprod;
  P.dual = L.dual;
  P.blocked = L.blocked;
  P.xsplit = L.xsplit;
  P.a_boxes = L.a_boxes;
  P.b_boxes = L.b_boxes;
  P.a_slot = L.a_slot;
  P.b_slot = L.b_slot;
  P.tx_bytes = L.a_boxes * L.a_bytes + (L.wres ? 0 : L.b_boxes * L.b_bytes);
  P.wres = L.wres;
  P.w_prewait = L.w_prewait;
  P.w_off = L.ring_bytes;
  P.w_chunk = L.w_chunk;
  P.w_tx = L.w_tx;
  P.red_bytes = L.red_bytes;
  P.stg_f32 = L.stg_f32;
  P.stg_off = L.epi_alias ? 0 : L.ring_bytes + (L.wres ? L.nstages * L.w_chunk : 0);
  P.epi_alias = L.epi_alias;
  P.stg_nbuf = L.stg_nbuf;
  P.epi_region = L.epi_region;
  P.stg_bf = L.stg_bf;
  P.tile_coords = static_cast<const int32_t*>(L.d_tcoords);
  P.sc = L.scatter;

  P.a_desc = L.a_desc;
  P.b_desc = L.b_desc;
  P.a_kadv = L.a_kadv;
  P.b_kadv = L.b_kadv;
  P.idesc = L.idesc;
  P.tmem_cols = L.tmem_cols;
  P.ring_bytes = L.ring_bytes;
  P.table_ints = L.table_ints;
  P.ntaps = L.ntaps;
  for (int t = 0; t < kMaxTaps; ++t) P.b_tap[t] = L.b_tapv[t];
  P.bias_rows = L.bias_rows;
  for (int t = 0; t < kMaxTaps; ++t) P.a_tap[t] = L.a_tap[t];
  P.store_mode = L.store_mode;
  P.diag = getenv("LFGPU_UMMA_DIAG") ? atoi(getenv("LFGPU_UMMA_DIAG")) : 0;
  P.col0 = L.col0;
  P.stg_cstride = L.stg_cstride;
  P.stg_cdim = L.stg_cdim;
  P.splits = L.splits;
  P.ws = L.ws;
  P.counters = L.counters;
  P.dbg = static_cast<unsigned long long*>(umma_debug_buffer());
  P.cdbg = g_chain_dbg && L.chain_slot >= 0 ? g_chain_dbg + 8 * L.chain_slot : nullptr;
  using KernelFn = void (*)(CUtensorMap, CUtensorMap, UmmaParams, CUtensorMap, CUtensorMap);
  static const KernelFn fns[3][2] = {{umma_kernel<0, false>, umma_kernel<0, true>},
                                     {umma_kernel<1, false>, umma_kernel<1, true>},
                                     {umma_kernel<2, false>, umma_kernel<2, true>}};
  static bool attr_set = false;
  if (!attr_set) {
    for (auto& row : fns)
      for (auto f : row)
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const KernelFn fn = fns[std::min(std::max(L.store_mode, 0), 2)][L.splits > 1 ? 1 : 0];
  // Programmatic dependent launch: the prologue (barriers, TMEM, tables)
  // overlaps the previous kernel; the kernel waits (griddepcontrol.wait)
  // before touching operands or outputs.
  static const bool pdl = [] {
    const char* e = getenv("LFGPU_PDL");
    return !(e && atoi(e) == 0);
  }();
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (L.xsplit) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = L.splits;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, fn, L.tma_a, L.tma_b, P, L.tma_o, L.tma_ob);
}

}  // namespace lfg
