// k_direct.cu — CUDA-core direct convolution for small input-channel counts.
//
// The C2D of interp.cpp:70-89 on logical (row-major NCHW / OIHW) fp32
// operands when I*KH*KW is small (ResNet's 3-channel 7x7 stem): tcgen05
// needs K-chunks of 16 bf16 channels, and the generic table-walking
// contraction (k_generic.cu) re-reads two offset tables per MAC. Here a CTA
// stages its input patch and a 16-channel weight slab in shared memory and
// each thread accumulates one output pixel x 16 channels (float4 broadcast
// weight reads, one patch read per 16 FMAs). The fused element-wise chain
// (BiasAdd / EwAdd / ReLU, lower.cpp:566-608) is applied before the store,
// which goes through the output's separable offset tables, so the output may
// carry any propagated layout.
#include <cuda_runtime.h>

#include <algorithm>

#include "lf_direct.hpp"
#include "lf_pdl.hpp"

namespace lfg {

constexpr int kDTW = 16, kDTH = 8, kDThreads = kDTW * kDTH, kDOC = 16;

__global__ void __launch_bounds__(kDThreads)
    c2d_direct(const DirectConv P) {
  LFG_PDL_ENTRY();
  extern __shared__ __align__(16) float sm[];
  const int R = P.I * P.KH * P.KW;
  const int PH = (kDTH - 1) * P.V + P.KH, PW = (kDTW - 1) * P.V + P.KW;
  float* wsm = sm;                          // [R][16] weights of this channel chunk
  float* xsm = sm + R * kDOC;               // [I][PH][PW] input patch
  const int oc_chunks = P.O / kDOC;
  const int b = blockIdx.z / oc_chunks, oc0 = (blockIdx.z % oc_chunks) * kDOC;
  const int h0 = blockIdx.y * kDTH, w0 = blockIdx.x * kDTW;
  const int tid = threadIdx.x;
  // weights: logical ker[o][i][rh][rw] -> wsm[r][o - oc0]
  for (int e = tid; e < R * kDOC; e += kDThreads) {
    const int o = e / R, r = e - o * R;
    wsm[r * kDOC + o] = P.w[static_cast<int64_t>(oc0 + o) * R + r];
  }
  // input patch rows [h0*V, h0*V + PH) x cols [w0*V, w0*V + PW), zero outside
  const int64_t img = static_cast<int64_t>(b) * P.I * P.H * P.W;
  for (int e = tid; e < P.I * PH * PW; e += kDThreads) {
    const int i = e / (PH * PW), rem = e - i * PH * PW, y = rem / PW, x = rem - y * PW;
    const int hy = h0 * P.V + y, wx = w0 * P.V + x;
    xsm[e] = hy < P.H && wx < P.W ? P.x[img + (static_cast<int64_t>(i) * P.H + hy) * P.W + wx] : 0.f;
  }
  __syncthreads();
  const int ty = tid / kDTW, tx = tid - ty * kDTW;
  const int ho = h0 + ty, wo = w0 + tx;
  float acc[kDOC];
#pragma unroll
  for (int j = 0; j < kDOC; ++j) acc[j] = 0.f;
  const float* xp = xsm + ty * P.V * PW + tx * P.V;
  const float4* wp = reinterpret_cast<const float4*>(wsm);
  for (int i = 0; i < P.I; ++i) {
    for (int rh = 0; rh < P.KH; ++rh) {
      const float* xr = xp + (i * PH + rh) * PW;
      for (int rw = 0; rw < P.KW; ++rw) {
        const float xv = xr[rw];
        const float4 a = wp[0], c = wp[1], d = wp[2], e = wp[3];
        wp += 4;
        acc[0] += xv * a.x, acc[1] += xv * a.y, acc[2] += xv * a.z, acc[3] += xv * a.w;
        acc[4] += xv * c.x, acc[5] += xv * c.y, acc[6] += xv * c.z, acc[7] += xv * c.w;
        acc[8] += xv * d.x, acc[9] += xv * d.y, acc[10] += xv * d.z, acc[11] += xv * d.w;
        acc[12] += xv * e.x, acc[13] += xv * e.y, acc[14] += xv * e.z, acc[15] += xv * e.w;
      }
    }
  }
  if (ho >= P.Ho || wo >= P.Wo) return;
  const int64_t base = P.tab[P.tab_off[0] + b] + P.tab[P.tab_off[2] + ho] + P.tab[P.tab_off[3] + wo];
#pragma unroll
  for (int j = 0; j < kDOC; ++j) {
    const int o = oc0 + j;
    const int64_t off = base + P.tab[P.tab_off[1] + o];
    float v = acc[j];
    for (int k = 0; k < P.nepi; ++k) {
      if (P.epi_kind[k] == DIRECT_EPI_BIAS) v += P.epi_ptr[k][o];
      else if (P.epi_kind[k] == DIRECT_EPI_RESIDUAL) v += P.epi_ptr[k][off];
      else v = v > 0.f ? v : 0.f;
    }
    P.out[off] = v;
  }
}

bool direct_conv_applies(int64_t I, int64_t KH, int64_t KW, int64_t O) {
  return I * KH * KW <= 512 && I < 16 && O % kDOC == 0;
}

size_t direct_conv_smem(const DirectConv& P) {
  const int R = static_cast<int>(P.I * P.KH * P.KW);
  const int PH = (kDTH - 1) * P.V + P.KH, PW = (kDTW - 1) * P.V + P.KW;
  return sizeof(float) * (static_cast<size_t>(R) * kDOC + static_cast<size_t>(P.I) * PH * PW);
}

cudaError_t launch_c2d_direct(const DirectConv& P, cudaStream_t stream) {
  const size_t smem = direct_conv_smem(P);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(c2d_direct, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(static_cast<unsigned>((P.Wo + kDTW - 1) / kDTW),
            static_cast<unsigned>((P.Ho + kDTH - 1) / kDTH),
            static_cast<unsigned>(P.N * (P.O / kDOC)));
  launch_pdl(c2d_direct, grid, dim3(kDThreads), smem, stream, P);
  return cudaGetLastError();
}

}  // namespace lfg
