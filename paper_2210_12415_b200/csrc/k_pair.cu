// k_pair.cu — K3 (second generation): the CTA-pair tcgen05 GEMM for sm_100a.
//
// Replaces the GMM loop nest of the reference (lower.cpp:221-227, evaluated
// by interp.cpp:381-411; oracle interp.cpp:109-122) on the GMM template
// bricks (space.cpp:388-412) when M is a multiple of 256.
//
// One cluster = S CTA pairs working on the same 256 x BN output tile; pair p
// accumulates K stages [p*KS/S, (p+1)*KS/S). Per CTA (256 threads):
//   warp 0      TMA producer (one lane): A rows [128*r, +128) and B columns
//               [BN/2*r, +BN/2) of the pair tile for each K stage into a
//               `pipe`-deep ring; completion bytes land on the pair leader's
//               barrier (cp.async.bulk.tensor .cta_group::2);
//   warp 1      (pair leader only) MMA issuer: tcgen05.mma.cta_group::2
//               M=256 N=BN K=16, bf16 x bf16 -> fp32 into one of two TMEM
//               accumulators of BN columns; tcgen05.commit multicasts the
//               ring-slot release and the accumulator-ready signal to both
//               CTAs of the pair;
//   warp 2      TMEM allocation (cta_group::2, both CTAs);
//   warps 4-7   epilogue: tcgen05.ld (thread = accumulator row), fused
//               BiasAdd / EwAdd / ReLU chain (lower.cpp:566-608 fusion
//               groups), 128-byte row-segment stores through a per-warp
//               SMEM transpose; the accumulator is released to the leader's
//               MMA (remote mbarrier arrive) as soon as it has been read, so
//               the next tile's main loop overlaps this epilogue.
// With S > 1 every CTA publishes its fp32 partial rows to an L2 workspace,
// arrives (release, cluster scope) on the reduction barrier of the S CTAs
// holding the same rows, waits for theirs, and reduces the column slice
// [p*BN/S, (p+1)*BN/S) summing partials in split order: the result does not
// depend on arrival order, and no CTA spins on global memory (the cluster
// guarantees the S pairs are co-resident).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>

#include "lf_pair.hpp"
#include "lf_alloc.hpp"
#include "lf_ptx.hpp"

namespace lfg {

namespace {

using namespace ptx;

constexpr int kThreads = 448;  // 12 role warps + 2 extra producer warps
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, alternating 32-column chunks
constexpr int kLd = 36;       // transpose buffer row stride (floats)
constexpr int kEpiBytes = kEpiWarps * 32 * kLd * 4;

struct PairParams {
  const int4* blob;          // tables (PairBlob layout), copied to SMEM at entry
  PairBlob lay;
  const int64_t* col_off;    // generic epilogue only
  float* out;
  __nv_bfloat16* out_bf16;
  float* ws;
  const float* epi_ptr[kMaxEpi];
  int32_t epi_kind[kMaxEpi];
  int32_t epi_count;
  int32_t MT2, NT, KS, S, ntiles, group;
  int32_t a_boxes, b_boxes, a_slot, b_slot, stage_bytes, tx_bytes, pipe, BN;
  uint64_t a_desc, b_desc;
  uint32_t a_kadv, b_kadv, idesc, tmem_cols;
  int32_t slabs, a_slab16, b_slab16;  // multi-slab stages: slab offsets in 16-byte units
  int32_t ring_bytes;
  int32_t col_unit;
  // Diagnostics (lfgpu_debug_umma_trace): 256 %globaltimer stamps per CTA:
  // [0,64) producer slot acquired per stage, [64,128) leader full-wait done
  // per stage, [128,192) epilogue accumulator ready per tile, [192,256)
  // epilogue done per tile (first 64 of each).
  unsigned long long* dbg;
  int32_t dbg_split;  // diagnostics: >= 0 keeps only that split's partial in the reduction
  int32_t diag;       // diagnostics (LFGPU_PAIR_DIAG, timing only): bit0 skips the epilogue's global stores
  int32_t nprod;      // TMA producer warps (1..5)
  int32_t a_tx;       // bytes of the A boxes of one stage (diagnostics)
  int32_t xmode;      // split-K exchange: 0 L2 workspace, 1 DSMEM push (one tile per cluster)
  int32_t rx_bytes;   // DSMEM receive buffer bytes ((S-1) x 128 x BN/S fp32)
  int32_t epi_alias, epi_off;  // one tile per cluster: epilogue buffers inside the idle ring at epi_off
};

#ifdef LFG_PAIR_CLOCK_STAMPS
// diagnostics build: SM cycle counter scaled to ns at 1.965 GHz (per-SM, not
// comparable across SMs) instead of %globaltimer
__device__ __forceinline__ unsigned long long gtime() { return static_cast<unsigned long long>(clock64() / 1.965); }
#else
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// Grouped rasterisation: `group` row tiles sweep the column tiles together
// so concurrently running clusters share A row blocks and B column blocks in L2.
__device__ __forceinline__ void tile_coords(const PairParams& P, int t, int* Mi, int* Nj) {
  const int per = P.group * P.NT;
  const int g = t / per, first = g * P.group;
  const int gs = min(P.MT2 - first, P.group);
  const int r = t - g * per;
  *Mi = first + r % gs;
  *Nj = r / gs;
}

// SMEM tables of one CTA (after the barriers): stage coordinates, output
// row / column-chunk offsets, row-block / column-tile origins, the tile's bias.
struct Smem {
  int32_t* stage;   // KS x 10
  int64_t* row;     // 128
  int64_t* colc;    // BN / 32 (offset of each 32-column chunk)
  int64_t* outr;    // MT
  int64_t* outc;    // NT
  int32_t* acrd;    // MT x a_boxes x 5
  int32_t* bcrd;    // 2 NT x b_boxes x 5
  float* bias;      // 2 x BN (double-buffered by tile parity)
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Store 32 accumulator columns [c0, c0+32) of the calling thread's row
// (v[j] = column c0 + j). Row-segment path: a per-warp SMEM transpose so each
// store instruction writes four 128-byte row segments; every table lives in
// SMEM (an L2 round trip per chunk would pace the epilogue), residual loads
// are all issued before they are consumed.
template <bool UNIT>
__device__ __forceinline__ void store_chunk(const PairParams& P, const Smem& T, const float* v, float* wbuf,
                                            int q, int lane, int c0, int64_t obase, const float* bias) {
  if constexpr (UNIT) {
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(wbuf + lane * kLd + 4 * j) =
          make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    __syncwarp();
    const int cl = (lane & 7) * 4;
    const int64_t cb = obase + T.colc[c0 >> 5] + cl;
    float4 x[8];
    int64_t addr[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int rr = it * 4 + (lane >> 3);
      x[it] = *reinterpret_cast<const float4*>(wbuf + rr * kLd + cl);
      addr[it] = cb + T.row[q * 32 + rr];
    }
#pragma unroll 1
    for (int e = 0; e < P.epi_count; ++e) {
      const int k = P.epi_kind[e];
      if (k == EPI_RELU) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          x[it].x = fmaxf(x[it].x, 0.f);
          x[it].y = fmaxf(x[it].y, 0.f);
          x[it].z = fmaxf(x[it].z, 0.f);
          x[it].w = fmaxf(x[it].w, 0.f);
        }
      } else if (k == EPI_GELU) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          x[it].x = epi_gelu(x[it].x);
          x[it].y = epi_gelu(x[it].y);
          x[it].z = epi_gelu(x[it].z);
          x[it].w = epi_gelu(x[it].w);
        }
      } else if (k == EPI_BIAS) {
        const float4 b = *reinterpret_cast<const float4*>(bias + c0 + cl);
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          x[it].x += b.x;
          x[it].y += b.y;
          x[it].z += b.z;
          x[it].w += b.w;
        }
      } else {  // EPI_RESIDUAL: same physical layout as the output
        float4 r[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) r[it] = __ldg(reinterpret_cast<const float4*>(P.epi_ptr[e] + addr[it]));
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          x[it].x += r[it].x;
          x[it].y += r[it].y;
          x[it].z += r[it].z;
          x[it].w += r[it].w;
        }
      }
    }
    if (P.diag & 1) return;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      *reinterpret_cast<float4*>(P.out + addr[it]) = x[it];
      if (P.out_bf16) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(x[it].x, x[it].y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(x[it].z, x[it].w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(P.out_bf16 + addr[it]) = pk;
      }
    }
  } else {
    // Generic layouts: thread = row, one element at a time (column offsets
    // from the global table, L1-resident after the first tile).
    // 8 columns per step: addresses, then one branch per fused op with its
    // loads batched (a per-element branch serialises the loads), then stores.
    const int64_t rb = obase + T.row[q * 32 + lane];
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += 8) {  // unrolled: v[] stays in registers
      int64_t addr[8];
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        addr[j] = rb + __ldg(P.col_off + c0 + j0 + j);
        y[j] = v[j0 + j];
      }
#pragma unroll 1
      for (int e = 0; e < P.epi_count; ++e) {
        const int k = P.epi_kind[e];
        if (k == EPI_RELU) {
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = fmaxf(y[j], 0.f);
        } else if (k == EPI_GELU) {
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = epi_gelu(y[j]);
        } else if (k == EPI_BIAS) {
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] += bias[c0 + j0 + j];
        } else {
          float t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) t[j] = __ldg(P.epi_ptr[e] + addr[j]);
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] += t[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        P.out[addr[j]] = y[j];
        if (P.out_bf16) P.out_bf16[addr[j]] = __float2bfloat16_rn(y[j]);
      }
    }
  }
}

// SPLIT: K splits reduce through the L2 workspace (S > 1); UNIT: row-segment
// stores (contiguous 32-column output chunks). One instance per combination
// keeps each kernel's code within the SM's instruction cache.
template <bool SPLIT, bool UNIT, bool MULTI>
__global__ void __launch_bounds__(kThreads, 1)
    pair_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const __grid_constant__ PairParams P) {
  if (P.dbg && threadIdx.x == 0) P.dbg[512 * blockIdx.x + 320] = gtime();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int epi_bytes = P.epi_alias ? 0 : kEpiBytes;
  float* s_epi = reinterpret_cast<float*>(smem + (P.epi_alias ? P.epi_off : P.ring_bytes));
  float* s_rx = reinterpret_cast<float*>(smem + P.ring_bytes + epi_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.ring_bytes + epi_bytes + P.rx_bytes);
  const int pipe = P.pipe;
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * pipe;
  const uint32_t tfull0 = empty0 + 8 * pipe;  // 2 accumulator-ready barriers
  const uint32_t tempty0 = tfull0 + 16;       // 2 accumulator-free barriers (leader)
  const uint32_t red0 = tempty0 + 16;         // 2 split-reduction barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * pipe + 6);
  int32_t* blob = reinterpret_cast<int32_t*>(bars + 2 * pipe + 8);  // 16-byte aligned
  Smem T;
  T.stage = blob + P.lay.stage;
  T.row = reinterpret_cast<int64_t*>(blob + P.lay.row);
  T.colc = reinterpret_cast<int64_t*>(blob + P.lay.colc);
  T.outr = reinterpret_cast<int64_t*>(blob + P.lay.outr);
  T.outc = reinterpret_cast<int64_t*>(blob + P.lay.outc);
  T.acrd = blob + P.lay.acrd;
  T.bcrd = blob + P.lay.bcrd;
  T.bias = reinterpret_cast<float*>(blob + P.lay.total);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    // Touch every 32-byte sector of the parameter block once, in parallel:
    // a role warp's first read of a cold constant line after the PDL wait
    // costs a serial L2 round trip each (~1 us before the first TMA issue).
    const uint32_t np32 = static_cast<uint32_t>(sizeof(PairParams) / 32);
    if (threadIdx.x < np32) {
      const uint32_t x = reinterpret_cast<const uint32_t*>(&P)[threadIdx.x * 8];
      asm volatile("" ::"r"(x));
    }
  }
  const uint32_t crank = cluster_ctarank();
  const int pr = static_cast<int>(crank & 1u);     // rank inside the pair
  const int split = static_cast<int>(crank >> 1);  // pair index = K split
  const uint32_t lead = crank & ~1u;
  const uint16_t pair_mask = static_cast<uint16_t>(3u << lead);
  const int S = P.S;
  const int cid = static_cast<int>(cluster_id_x()), ncl = static_cast<int>(nclusters_x());

  if (threadIdx.x == 0) {
    for (int s = 0; s < pipe; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);  // the pair's MMA commit (both producer warps wait on it)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, 2 * kEpiWarps);  // both CTAs' epilogue warps
      mbar_init(red0 + 8 * b, P.xmode ? 1 : (S - 1) * kEpiWarps);  // sibling splits' epilogue warps / rx bytes
    }
    // DSMEM exchange: the receive buffer's expected bytes, armed before the
    // cluster barrier so no sibling's push can precede it.
    if (P.xmode) mbar_expect_tx(red0, static_cast<uint32_t>(P.rx_bytes));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  // Plan tables (host-written once, never by kernels: safe before the PDL wait).
  {  // one pass, all loads of a thread in flight together
    const int n4 = P.lay.total / 4;
    int4* dst = reinterpret_cast<int4*>(blob);
    int i0 = threadIdx.x;
    for (; i0 + 3 * kThreads < n4; i0 += 4 * kThreads) {
      int4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldg(P.blob + i0 + k * kThreads);
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[i0 + k * kThreads] = v[k];
    }
    for (; i0 < n4; i0 += kThreads) dst[i0] = __ldg(P.blob + i0);
  }
  if (P.dbg && threadIdx.x == 0) P.dbg[512 * blockIdx.x + 324] = gtime();
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    if (P.dbg && lane == 0) P.dbg[512 * blockIdx.x + 325] = gtime();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (P.dbg && threadIdx.x == 0) P.dbg[512 * blockIdx.x + 321] = gtime();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (P.dbg && threadIdx.x == 0) P.dbg[512 * blockIdx.x + 322] = gtime();

  const int s_lo = split * P.KS / S, s_hi = (split + 1) * P.KS / S;
  const uint32_t ring0 = smem_u32(smem);

  const int np = P.nprod;
  const int prod = warp == 0 ? 0 : warp == 3 ? 1 : warp == 2 ? 2 : warp >= kEpiWarp0 + kEpiWarps ? 3 + warp - (kEpiWarp0 + kEpiWarps) : -1;
  if (prod >= 0 && prod < np) {
    // ---- TMA producers (both CTAs of the pair). One issuing warp keeps
    // about one request in flight (tools/micro/tma_ingest.cu: ~800 cycles
    // per request per warp, independent of its size, while the SM takes
    // 80-100 B/clk from several warps), so the stages are dealt round-robin
    // to `np` producer warps; each issues the A and B boxes of its stages
    // (in the pair leader it also arms the stage's expected bytes for both
    // CTAs). Coordinates never come from global memory inside the loop: the
    // tile part is loaded into registers once per tile, the stage part
    // lives in SMEM.
    if (elect_one()) {
      if (P.dbg && prod == 0) P.dbg[512 * blockIdx.x + 326] = gtime();
      const uint32_t lead_full0 = mapa(full0, lead);
      const uint32_t b_off = P.a_boxes * P.a_slot;
      int g = 0;
      for (int t = cid; t < P.ntiles; t += ncl) {
        int Mi, Nj;
        tile_coords(P, t, &Mi, &Nj);
        int32_t ta[kMaxBoxes][5], tb[kMaxBoxes][5];
        const int32_t* ca = T.acrd + (2 * Mi + pr) * P.a_boxes * 5;
        const int32_t* cb = T.bcrd + (2 * Nj + pr) * P.b_boxes * 5;
#pragma unroll
        for (int b = 0; b < kMaxBoxes; ++b)
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            ta[b][d] = b < P.a_boxes ? ca[b * 5 + d] : 0;
            tb[b][d] = b < P.b_boxes ? cb[b * 5 + d] : 0;
          }
        if (P.dbg && prod == 0 && g == 0) P.dbg[512 * blockIdx.x + 327] = gtime();
        for (int s = s_lo; s < s_hi; ++s, ++g) {
          if (g % np != prod) continue;
          const int slot = g % pipe;
          const uint32_t ph = static_cast<uint32_t>(g / pipe) & 1u;
          const int32_t* sc = T.stage + s * 10;
          int32_t c[5];
          if (P.dbg && g == 0) P.dbg[512 * blockIdx.x + 328] = gtime();
          mbar_wait(empty0 + 8 * slot, ph ^ 1u);
          if (P.dbg && g < 64) P.dbg[512 * blockIdx.x + g] = gtime();
          if (pr == 0) mbar_expect_tx(full0 + 8 * slot, (P.diag & 4) ? 2 * P.a_tx : 2 * P.tx_bytes);
          const uint32_t bar = lead_full0 + 8 * slot;
          const uint32_t dst = ring0 + slot * P.stage_bytes;
#pragma unroll
          for (int b = 0; b < kMaxBoxes; ++b)
            if (b < P.a_boxes) {
#pragma unroll
              for (int d = 0; d < 5; ++d) c[d] = ta[b][d] + sc[d];
              tma_load5_pair(&tma_a, dst + b * P.a_slot, bar, c);
            }
#pragma unroll
          for (int b = 0; b < kMaxBoxes; ++b)
            if (b < P.b_boxes && !(P.diag & 4)) {  // diag bit 2: A operand only (ingest probe)
#pragma unroll
              for (int d = 0; d < 5; ++d) c[d] = tb[b][d] + sc[5 + d];
              tma_load5_pair(&tma_b, dst + b_off + b * P.b_slot, bar, c);
            }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1 && pr == 0) {
    // ---- MMA issuer (pair leader)
    const uint32_t akadv = P.a_kadv >> 4, bkadv = P.b_kadv >> 4;
    const uint32_t b_off = P.a_boxes * P.a_slot;
    const bool issuer = elect_one();
    int g = 0, i = 0;
    for (int t = cid; t < P.ntiles; t += ncl, ++i) {
      const int acc = i & 1;
      mbar_wait_cluster(tempty0 + 8 * acc, (static_cast<uint32_t>(i >> 1) & 1u) ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + static_cast<uint32_t>(acc * P.BN);
      for (int s = s_lo; s < s_hi; ++s, ++g) {
        const int slot = g % pipe;
        mbar_wait(full0 + 8 * slot, static_cast<uint32_t>(g / pipe) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (P.dbg && issuer && g < 64) P.dbg[512 * blockIdx.x + 64 + g] = gtime();
        if (issuer) {
          const uint32_t a_addr = ring0 + slot * P.stage_bytes;
          const uint64_t ad = P.a_desc | (a_addr >> 4), bd = P.b_desc | ((a_addr + b_off) >> 4);
          if constexpr (MULTI) {  // several 64-wide K slabs per stage
            if (!(P.diag & 2))
              for (int sl = 0; sl < P.slabs; ++sl)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  umma2_bf16(d, ad + sl * P.a_slab16 + k * akadv, bd + sl * P.b_slab16 + k * bkadv, P.idesc,
                             (s != s_lo) | sl | k);
          } else {
            if (!(P.diag & 2))  // diag bit 1: no MMAs (ingest probe; results are garbage)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma2_bf16(d, ad + k * akadv, bd + k * bkadv, P.idesc, (s != s_lo) | k);
          }
          umma2_commit_mc(empty0 + 8 * slot, pair_mask);
        }
        __syncwarp();
      }
      if (issuer) umma2_commit_mc(tfull0 + 8 * acc, pair_mask);
      __syncwarp();
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    // ---- epilogue (both CTAs): warp w reads TMEM lanes 32*(w%4)..+31; the
    // two warps of a lane quadrant take alternate 32-column chunks
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    const int row = q * 32 + lane;
    const int etid = (warp - kEpiWarp0) * 32 + lane;
    float* wbuf = s_epi + (warp - kEpiWarp0) * 32 * kLd;
    const uint32_t lead_tempty0 = mapa(tempty0, lead);
    bool has_bias = false;
    const float* bias_ptr = nullptr;
    for (int e = 0; e < P.epi_count; ++e)
      if (P.epi_kind[e] == EPI_BIAS) {
        has_bias = true;
        bias_ptr = P.epi_ptr[e];
      }
    int i = 0;
    for (int t = cid; t < P.ntiles; t += ncl, ++i) {
      int Mi, Nj;
      tile_coords(P, t, &Mi, &Nj);
      const int acc = i & 1;
      const int mi = 2 * Mi + pr;
      const int64_t obase = T.outr[mi] + T.outc[Nj];
      const int n0 = Nj * P.BN;
      float* bias = T.bias + acc * P.BN;
      if (has_bias) {  // the tile's bias slice, before waiting for the accumulator
        for (int c = etid; c < P.BN; c += 32 * kEpiWarps) bias[c] = __ldg(bias_ptr + n0 + c);
        epi_bar();
      }
      mbar_wait(tfull0 + 8 * acc, static_cast<uint32_t>(i >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (P.dbg && etid == 0 && i < 64) P.dbg[512 * blockIdx.x + 128 + i] = gtime();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * P.BN);
      float v[32];
      if constexpr (!SPLIT) {
        for (int c0 = 32 * half; c0 < P.BN; c0 += 64) {
          tmem_ld32(taddr + c0, v);
          if (P.dbg && etid == 0 && i == 0 && c0 < 32 * 32) P.dbg[512 * blockIdx.x + 256 + c0 / 16] = gtime();
          if (c0 + 64 >= P.BN) {  // this warp's last read of the accumulator: hand it back
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed_cluster(lead_tempty0 + 8 * acc);
          }
          store_chunk<UNIT>(P, T, v, wbuf, q, lane, c0, obase, bias);
          if (P.dbg && etid == 0 && i == 0 && c0 < 32 * 32) P.dbg[512 * blockIdx.x + 257 + c0 / 16] = gtime();
        }
        if (P.dbg && etid == 0 && i < 64) P.dbg[512 * blockIdx.x + 192 + i] = gtime();
      } else {
      const int W = P.BN / S;
      if (P.xmode) {
        // Split K over DSMEM (one tile per cluster): each 32x32 block of a
        // sibling's column slice is staged in the idle operand ring as
        // [col][row] and pushed into the sibling's receive buffer with one
        // bulk copy that completes on the sibling's barrier; no global
        // round trip, no fence. Receive layout: [sender][chunk][quadrant][32 col][32 row].
        const int blk = 32 * 32 * 4;
        uint8_t* stage_base = smem + (warp - kEpiWarp0) * (((P.BN / 64) * (S - 1) + S - 1) / S) * blk;
        int nb = 0;
        for (int c0 = 32 * half; c0 < P.BN; c0 += 64) {
          const int p = c0 / W;
          if (p == split) continue;
          tmem_ld32(taddr + c0, v);
          float* st = reinterpret_cast<float*>(stage_base + (nb++) * blk);
#pragma unroll
          for (int j = 0; j < 32; ++j) st[j * 32 + lane] = v[j];
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int sidx = split < p ? split : split - 1;
            const uint32_t off = static_cast<uint32_t>(((sidx * (W / 32) + (c0 - p * W) / 32) * 4 + q) * blk);
            const uint32_t dst = mapa(smem_u32(s_rx) + off, 2 * p + pr);
            const uint32_t rb = mapa(red0, 2 * p + pr);
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "r"(smem_u32(st)), "r"(blk), "r"(rb)
                : "memory");
          }
        }
        if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 256] = gtime();
        mbar_wait_cluster(red0, 0);
        if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 258] = gtime();
        for (int c0 = split * W + 32 * half; c0 < (split + 1) * W; c0 += 64) {
          float own[32];
          tmem_ld32(taddr + c0, own);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
          for (int p = 0; p < S; ++p) {  // split order: deterministic sums
            if (p == split) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += own[j];
              continue;
            }
            const int sidx = p < split ? p : p - 1;
            const float* rx = s_rx + ((sidx * (W / 32) + (c0 - split * W) / 32) * 4 + q) * 1024;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += rx[j * 32 + lane];
          }
          store_chunk<UNIT>(P, T, v, wbuf, q, lane, c0, obase, bias);
          if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 259 + (c0 - split * W) / 64] = gtime();
        }
      } else {
      // Split K through L2: publish the column slices the sibling splits
      // reduce ([col/4][row] float4, coalesced); this split's own slice
      // stays in TMEM until its reduction.
      const size_t tile_floats = static_cast<size_t>(128) * P.BN;
      float4* mine = reinterpret_cast<float4*>(P.ws + ((static_cast<size_t>(t) * S + split) * 2 + pr) * tile_floats);
      for (int c0 = 32 * half; c0 < P.BN; c0 += 64) {
        if (c0 >= split * W && c0 < (split + 1) * W) continue;
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          __stcg(mine + (c0 / 4 + j) * 128 + row, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
      }
      if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 256] = gtime();
      // Release the partial at cluster scope (every reader is in this cluster).
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      __syncwarp();
      if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 257] = gtime();
      if (lane == 0)
        for (int p = 0; p < S; ++p)
          if (p != split) mbar_arrive_cluster(mapa(red0 + 8 * acc, 2 * p + pr));
      mbar_wait_cluster(red0 + 8 * acc, static_cast<uint32_t>(i >> 1) & 1u);
      if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 258] = gtime();
      for (int c0 = split * W + 32 * half; c0 < (split + 1) * W; c0 += 64) {
        float own[32];
        tmem_ld32(taddr + c0, own);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
        for (int p = 0; p < S; ++p) {  // split order: deterministic sums
          if (P.dbg_split >= 0 && p != P.dbg_split) continue;
          if (p == split) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += own[j];
            continue;
          }
          const float4* src =
              reinterpret_cast<const float4*>(P.ws + ((static_cast<size_t>(t) * S + p) * 2 + pr) * tile_floats);
          float4 x[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = __ldcg(src + (c0 / 4 + j) * 128 + row);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v[4 * j] += x[j].x;
            v[4 * j + 1] += x[j].y;
            v[4 * j + 2] += x[j].z;
            v[4 * j + 3] += x[j].w;
          }
        }
        store_chunk<UNIT>(P, T, v, wbuf, q, lane, c0, obase, bias);
        if (P.dbg && etid == 0 && i == 0) P.dbg[512 * blockIdx.x + 259 + (c0 - split * W) / 64] = gtime();
      }
      }
      // The accumulator has been read completely: hand it back to the MMA.
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed_cluster(lead_tempty0 + 8 * acc);
      if (P.dbg && etid == 0 && i < 64) P.dbg[512 * blockIdx.x + 192 + i] = gtime();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (P.dbg && threadIdx.x == 0) P.dbg[512 * blockIdx.x + 323] = gtime();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols)
                 : "memory");
  }
}

struct PairTables {
  void* p[8] = {};
  ~PairTables() {
    for (auto* q : p)
      if (q) dev_free(q);
  }
};

template <typename T>
void* upload(const std::vector<T>& v) {
  void* d = nullptr;
  const size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
  if (!(d = dev_alloc(bytes))) fail(LFGPU_ECUDA, "device allocation of pair tables");
  if (!v.empty() && cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    fail(LFGPU_ECUDA, "cudaMemcpy pair tables");
  return d;
}

// The kernel instance for (split-K, row-segment stores, multi-slab stages),
// with its dynamic SMEM limit raised once.
const void* pair_instance(bool split, bool unit, bool multi) {
  static const void* k[8] = {
      reinterpret_cast<const void*>(pair_kernel<false, false, false>),
      reinterpret_cast<const void*>(pair_kernel<false, true, false>),
      reinterpret_cast<const void*>(pair_kernel<true, false, false>),
      reinterpret_cast<const void*>(pair_kernel<true, true, false>),
      reinterpret_cast<const void*>(pair_kernel<false, false, true>),
      reinterpret_cast<const void*>(pair_kernel<false, true, true>),
      reinterpret_cast<const void*>(pair_kernel<true, false, true>),
      reinterpret_cast<const void*>(pair_kernel<true, true, true>)};
  static bool attr_set = [] {
    for (const void* f : k) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    return true;
  }();
  (void)attr_set;
  return k[(multi ? 4 : 0) + (split ? 2 : 0) + (unit ? 1 : 0)];
}

}  // namespace

PairLaunch pair_prepare(const PairPlan& p) {
  PairLaunch L;
  L.tma_a = umma_encode(p.A, p.a);
  L.tma_b = umma_encode(p.B, p.b);
  auto t = std::make_shared<PairTables>();
  L.lay = pair_blob_layout(p.KS, p.MT, p.NT, p.A.boxes, p.B.boxes);
  {
    std::vector<int32_t> blob(L.lay.total, 0);
    std::memcpy(blob.data() + L.lay.stage, p.s_crd.data(), 4 * p.s_crd.size());
    std::memcpy(blob.data() + L.lay.row, p.row_off.data(), 8 * std::min<size_t>(128, p.row_off.size()));
    for (int c = 0; c < p.BN / 32; ++c) std::memcpy(blob.data() + L.lay.colc + 2 * c, &p.col_off[32 * c], 8);
    std::memcpy(blob.data() + L.lay.outr, p.out_r.data(), 8 * p.out_r.size());
    std::memcpy(blob.data() + L.lay.outc, p.out_c.data(), 8 * p.out_c.size());
    std::memcpy(blob.data() + L.lay.acrd, p.a_crd.data(), 4 * p.a_crd.size());
    std::memcpy(blob.data() + L.lay.bcrd, p.b_crd.data(), 4 * p.b_crd.size());
    t->p[0] = upload(blob);
  }
  t->p[1] = upload(p.col_off);
  L.blob = static_cast<const int32_t*>(t->p[0]);
  L.col_off = static_cast<const int64_t*>(t->p[1]);
  L.BN = p.BN;
  L.S = p.S;
  L.MT = p.MT;
  L.NT = p.NT;
  L.KS = p.KS;
  L.pipe = p.pipe;
  L.a_boxes = p.A.boxes;
  L.b_boxes = p.B.boxes;
  L.a_slot = p.A.slot_bytes;
  L.b_slot = p.B.slot_bytes;
  L.stage_bytes = L.a_boxes * L.a_slot + L.b_boxes * L.b_slot;
  L.tx_bytes = L.a_boxes * p.A.box_bytes + L.b_boxes * p.B.box_bytes;
  L.a_box_bytes = p.A.box_bytes;
  L.a_desc = umma_desc_bits(p.A);
  L.b_desc = umma_desc_bits(p.B);
  L.a_kadv = p.A.k_adv;
  L.b_kadv = p.B.k_adv;
  L.slabs = p.slabs;
  L.a_slab = p.a_slab;
  L.b_slab = p.b_slab;
  L.idesc = umma_idesc(256, p.BN, p.A.mn_major, p.B.mn_major);
  int cols = 32;
  while (cols < 2 * p.BN) cols *= 2;
  L.tmem_cols = cols;
  L.ring_bytes = L.pipe * L.stage_bytes;
  L.rx_bytes = p.rx_bytes;
  L.xmode = p.rx_bytes > 0 ? 1 : 0;
  // Epilogue buffers inside the ring (planner: one tile per cluster), behind
  // the DSMEM send staging of the split-K exchange.
  L.epi_alias = p.epi_alias;
  L.epi_off = L.xmode ? ((p.BN / 64) * (p.S - 1) + p.S - 1) / p.S * 8 * 4096 : 0;
  if (L.epi_alias && L.epi_off + kEpiBytes > L.ring_bytes) L.epi_alias = 0;
  L.smem = 1024 + L.ring_bytes + (L.epi_alias ? 0 : kEpiBytes) + L.rx_bytes + 8 * (2 * L.pipe + 8) +
           pair_table_bytes(p.KS, p.MT, p.NT, p.BN, p.A.boxes, p.B.boxes);
  if (L.smem > 227 * 1024) fail(LFGPU_EUNSUPPORTED, "pair kernel SMEM exceeds 227 KB");
  // Row-segment stores need contiguous output columns and 16-byte aligned rows.
  bool unit = true;
  for (size_t c = 0; c < p.col_off.size(); c += 32)
    for (size_t j = 1; j < 32 && c + j < p.col_off.size(); ++j)
      if (p.col_off[c + j] != p.col_off[c] + static_cast<int64_t>(j)) unit = false;
  for (size_t c = 0; c < p.col_off.size(); c += 32)
    if (p.col_off[c] % 4) unit = false;
  for (auto v : p.row_off)
    if (v % 4) unit = false;
  for (auto v : p.out_r)
    if (v % 4) unit = false;
  for (auto v : p.out_c)
    if (v % 4) unit = false;
  for (int e = 0; e < p.epi_count; ++e)
    if (reinterpret_cast<uintptr_t>(p.epi[e].ptr) % 16) unit = false;
  L.col_unit = unit ? 1 : 0;
  L.epi_count = p.epi_count;
  for (int e = 0; e < p.epi_count; ++e) {
    L.epi_kinds[e] = p.epi[e].kind;
    L.epi_ptr[e] = p.epi[e].ptr;
  }
  L.out = p.out;
  L.out_bf16 = p.out_bf16;
  const int ntiles = p.MT / 2 * p.NT;
  if (L.S > 1) {  // L2 workspace (also the fallback when the DSMEM exchange cannot be used)
    const size_t ws = sizeof(float) * static_cast<size_t>(ntiles) * L.S * 256 * L.BN;
    if (!(t->p[7] = dev_alloc(ws))) fail(LFGPU_ECUDA, "device allocation of the pair split-K workspace");
    L.ws = static_cast<float*>(t->p[7]);
  }
  L.owner = t;
  L.group = p.group;
  if (const char* e = getenv("LFGPU_PAIR_GROUP")) L.group = std::max(1, atoi(e));
  if (const char* e = getenv("LFGPU_PAIR_NP")) L.nprod = std::max(1, std::min(5, atoi(e)));
  // A producer may run at most `pipe` stages ahead of the oldest unreleased
  // one, or the parity wait on a ring slot two phases behind passes early.
  L.nprod = std::min(L.nprod, L.pipe);
  // Persistent grid: as many clusters as can be co-resident, at most one per tile.
  const void* kfn = pair_instance(L.S > 1, L.col_unit != 0, L.slabs > 1);
  const int csize = 2 * L.S;
  int max_cl = umma_num_sms() / csize;
  {
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(csize * max_cl);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kfn, &cfg) == cudaSuccess && n > 0)
      max_cl = std::min(max_cl, n);
    cudaGetLastError();
  }
  if (L.xmode && max_cl < ntiles) L.xmode = 0;  // the DSMEM exchange needs one tile per cluster
  if (L.epi_alias && max_cl < ntiles)  // several tiles per cluster: the ring is not idle in the epilogue
    fail(LFGPU_EUNSUPPORTED, "pair kernel: epilogue-in-ring needs one tile per cluster");
  L.grid = csize * std::max(1, std::min(ntiles, max_cl));
  return L;
}

cudaError_t pair_launch(const PairLaunch& L, cudaStream_t stream) {
  PairParams P;
  std::memset(&P, 0, sizeof(P));
  P.blob = reinterpret_cast<const int4*>(L.blob);
  P.lay = L.lay;
  P.col_off = L.col_off;
  P.out = L.out;
  P.out_bf16 = static_cast<__nv_bfloat16*>(L.out_bf16);
  P.ws = L.ws;
  P.epi_count = L.epi_count;
  for (int e = 0; e < L.epi_count; ++e) {
    P.epi_kind[e] = L.epi_kinds[e];
    P.epi_ptr[e] = L.epi_ptr[e];
  }
  P.MT2 = L.MT / 2;
  P.NT = L.NT;
  P.KS = L.KS;
  P.S = L.S;
  P.ntiles = L.MT / 2 * L.NT;
  P.group = L.group;
  P.a_boxes = L.a_boxes;
  P.b_boxes = L.b_boxes;
  P.a_slot = L.a_slot;
  P.b_slot = L.b_slot;
  P.stage_bytes = L.stage_bytes;
  P.tx_bytes = L.tx_bytes;
  P.pipe = L.pipe;
  P.BN = L.BN;
  P.a_desc = L.a_desc;
  P.b_desc = L.b_desc;
  P.a_kadv = L.a_kadv;
  P.b_kadv = L.b_kadv;
  P.slabs = L.slabs;
  P.a_slab16 = L.a_slab >> 4;
  P.b_slab16 = L.b_slab >> 4;
  P.idesc = L.idesc;
  P.tmem_cols = L.tmem_cols;
  P.ring_bytes = L.ring_bytes;
  P.col_unit = L.col_unit;
  P.dbg = static_cast<unsigned long long*>(umma_debug_buffer());
  P.dbg_split = getenv("LFGPU_PAIR_DBG_SPLIT") ? atoi(getenv("LFGPU_PAIR_DBG_SPLIT")) : -1;
  P.diag = getenv("LFGPU_PAIR_DIAG") ? atoi(getenv("LFGPU_PAIR_DIAG")) : 0;
  P.nprod = L.nprod;
  P.a_tx = L.a_boxes * L.a_box_bytes;
  P.xmode = L.xmode;
  P.rx_bytes = L.rx_bytes;
  P.epi_alias = L.epi_alias;
  P.epi_off = L.epi_off;
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
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * L.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  void* args[] = {const_cast<CUtensorMap*>(&L.tma_a), const_cast<CUtensorMap*>(&L.tma_b), &P};
  return cudaLaunchKernelExC(&cfg, pair_instance(L.S > 1, L.col_unit != 0, L.slabs > 1), args);
}

}  // namespace lfg
