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
};

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
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr int kThreads = 192;

__global__ void __launch_bounds__(kThreads, 1)
    umma_kernel(const __grid_constant__ CUtensorMap tma_a,
                const __grid_constant__ CUtensorMap tma_b, const UmmaParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int stage_bytes = P.a_boxes * P.a_slot + P.b_boxes * P.b_slot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.pipe * stage_bytes);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * P.pipe;
  const uint32_t accf = empty0 + 8 * P.pipe;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P.pipe + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.pipe; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
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
  const int tile = blockIdx.x;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    const TileEntry& te = P.tiles[tile];
    for (int s = 0; s < P.nstages; ++s) {
      const int slot = s % P.pipe;
      const uint32_t ph = (s / P.pipe) & 1;
      mbar_wait(empty0 + 8 * slot, ph ^ 1);
      const uint32_t bar = full0 + 8 * slot;
      mbar_expect_tx(bar, P.tx_bytes);
      const StageEntry& se = P.stages[s];
      const uint32_t a_dst = smem_u32(smem + slot * stage_bytes);
      const uint32_t b_dst = a_dst + P.a_boxes * P.a_slot;
      int32_t c[5];
      for (int b = 0; b < P.a_boxes; ++b) {
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = te.ca[b][d] + se.sa[d];
        tma_load(&tma_a, P.a_rank, a_dst + b * P.a_slot, bar, c);
      }
      for (int b = 0; b < P.b_boxes; ++b) {
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = te.cb[b][d] + se.sb[d];
        tma_load(&tma_b, P.b_rank, b_dst + b * P.b_slot, bar, c);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    for (int s = 0; s < P.nstages; ++s) {
      const int slot = s % P.pipe;
      const uint32_t ph = (s / P.pipe) & 1;
      mbar_wait(full0 + 8 * slot, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_addr = smem_u32(smem + slot * stage_bytes);
      const uint32_t b_addr = a_addr + P.a_boxes * P.a_slot;
      for (int k = 0; k < P.ksteps; ++k) {
        const uint64_t ad = P.a_desc | (((a_addr + k * P.a_kadv) >> 4) & 0x3FFFull);
        const uint64_t bd = P.b_desc | (((b_addr + k * P.b_kadv) >> 4) & 0x3FFFull);
        umma_bf16(tmem, ad, bd, P.idesc, (s | k) != 0);
      }
      umma_commit(empty0 + 8 * slot);
    }
    umma_commit(accf);
  } else if (warp >= 2) {
    // ---- epilogue: TMEM -> registers -> fused element-wise -> global
    mbar_wait(accf, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const TileEntry& te = P.tiles[tile];
    const bool live = row < te.rows;
    const int64_t rbase = te.out_base + (live ? P.row_off[row] : 0);
    for (int c0 = 0; c0 < P.BN; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0, v);
      if (!live) continue;
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const int c = c0 + j;
        if (c >= te.cols) break;
        const int64_t addr = rbase + P.col_off[c];
        float x = __uint_as_float(v[j]);
        for (int e = 0; e < P.epi_count; ++e) {
          if (P.epi_kind[e] == EPI_BIAS) x += __ldg(P.epi_ptr[e] + te.n_base + c);
          else if (P.epi_kind[e] == EPI_RESIDUAL) x += __ldg(P.epi_ptr[e] + addr);
          else x = fmaxf(x, 0.0f);
        }
        P.out[addr] = x;
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
  for (int d = 0; d < v.rank; ++d) {
    dims[d] = v.dims[d];
    strides[d] = v.strides[d];
    box[d] = v.box[d];
    es[d] = v.estride[d];
  }
  CUtensorMapSwizzle sw = v.swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : v.swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, v.rank, const_cast<void*>(base),
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
  void* p[4] = {nullptr, nullptr, nullptr, nullptr};
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
  L.smem = 1024 + static_cast<size_t>(p.pipe) * (L.a_boxes * L.a_slot + L.b_boxes * L.b_slot) +
           8 * (2 * p.pipe + 2) + 16;
  L.grid = L.ntiles;
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
