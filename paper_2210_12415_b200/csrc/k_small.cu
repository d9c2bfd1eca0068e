// k_small.cu — MaxPool / GlobalAvgPool and the small-M GMM on sm_100a CUDA
// cores (lf_small.hpp). Each replaces a generic interpreted-index kernel
// (k_generic.cu) on the ResNet-18 tail and stem: offsets come from separable
// per-dim tables, threads walk the output in logical order.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "lf_pdl.hpp"
#include "lf_small.hpp"
#include "lf_umma.hpp"

namespace lfg {

namespace {

// MaxPool: one thread per output (n, c, oh, ow), ow fastest.
__global__ void __launch_bounds__(256) maxpool_kernel(const PoolParams P) {
  LFG_PDL_ENTRY();
  const int64_t total = static_cast<int64_t>(P.N) * P.C * P.Ho * P.Wo;
  for (int64_t e = blockIdx.x * 256ll + threadIdx.x; e < total; e += static_cast<int64_t>(gridDim.x) * 256) {
    int64_t r = e;
    const int ow = static_cast<int>(r % P.Wo);
    r /= P.Wo;
    const int oh = static_cast<int>(r % P.Ho);
    r /= P.Ho;
    const int c = static_cast<int>(r % P.C);
    const int n = static_cast<int>(r / P.C);
    const int64_t base = __ldg(P.xt + P.x_off[0] + n) + __ldg(P.xt + P.x_off[1] + c);
    float m = -INFINITY;
    if (P.pad == 0) {
      for (int kh = 0; kh < P.K; ++kh) {
        const int64_t hb = base + __ldg(P.xt + P.x_off[2] + oh * P.V + kh);
        for (int kw = 0; kw < P.K; ++kw) m = fmaxf(m, __ldg(P.x + hb + __ldg(P.xt + P.x_off[3] + ow * P.V + kw)));
      }
    } else {  // the absorbed Padding: its zeros take part in the max
      for (int kh = 0; kh < P.K; ++kh) {
        const int ih = oh * P.V + kh - P.pad;
        const bool hin = ih >= 0 && ih < P.H;
        const int64_t hb = hin ? base + __ldg(P.xt + P.x_off[2] + ih) : 0;
        for (int kw = 0; kw < P.K; ++kw) {
          const int iw = ow * P.V + kw - P.pad;
          m = fmaxf(m, hin && iw >= 0 && iw < P.W ? __ldg(P.x + hb + __ldg(P.xt + P.x_off[3] + iw)) : 0.f);
        }
      }
    }
    const int64_t o = __ldg(P.ot + P.o_off[0] + n) + __ldg(P.ot + P.o_off[1] + c) + __ldg(P.ot + P.o_off[2] + oh) +
                      __ldg(P.ot + P.o_off[3] + ow);
    P.out[o] = m;
    if (P.out_bf16) static_cast<__nv_bfloat16*>(P.out_bf16)[o] = __float2bfloat16_rn(m);
  }
}

// GlobalAvgPool: one warp per (n, c); lanes stride over the H*W pixels.
__global__ void __launch_bounds__(256) gap_kernel(const PoolParams P) {
  LFG_PDL_ENTRY();
  const int64_t nc = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (nc >= static_cast<int64_t>(P.N) * P.C) return;
  const int n = static_cast<int>(nc / P.C), c = static_cast<int>(nc % P.C);
  const int64_t base = __ldg(P.xt + P.x_off[0] + n) + __ldg(P.xt + P.x_off[1] + c);
  const int hw = P.H * P.W;
  float s = 0.f;
  for (int p = lane; p < hw; p += 32) {
    const int h = p / P.W, w = p - h * P.W;
    s += __ldg(P.x + base + __ldg(P.xt + P.x_off[2] + h) + __ldg(P.xt + P.x_off[3] + w));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const float y = s / static_cast<float>(hw);
    const int64_t o = __ldg(P.ot + P.o_off[0] + n) + __ldg(P.ot + P.o_off[1] + c);
    P.out[o] = y;
    if (P.out_bf16) static_cast<__nv_bfloat16*>(P.out_bf16)[o] = __float2bfloat16_rn(y);
  }
}

constexpr int kGemvCols = 32, kGemvSlices = 8;

__global__ void __launch_bounds__(256) gemv_kernel(const GemvParams P) {
  LFG_PDL_ENTRY();
  __shared__ float red[kGemvSlices][kGemvCols];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = blockIdx.x * kGemvCols + lane, m = blockIdx.y;
  const int k0 = w * P.K / kGemvSlices, k1 = (w + 1) * P.K / kGemvSlices;
  float acc = 0.f;
  if (n < P.N) {
    const float* arow = P.a + __ldg(P.at + P.a_off[0] + m);
    const int64_t bn = __ldg(P.bt + P.b_off[1] + n);
    for (int k = k0; k < k1; ++k)
      acc = fmaf(__ldg(arow + __ldg(P.at + P.a_off[1] + k)), __ldg(P.b + __ldg(P.bt + P.b_off[0] + k) + bn), acc);
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w != 0 || n >= P.N) return;
  float y = red[0][lane];
#pragma unroll
  for (int s = 1; s < kGemvSlices; ++s) y += red[s][lane];
  const int64_t o = __ldg(P.ot + P.o_off[0] + m) + __ldg(P.ot + P.o_off[1] + n);
  for (int e = 0; e < P.nepi; ++e) {
    const int kd = P.epi_kind[e];
    if (kd == EPI_RELU) y = fmaxf(y, 0.f);
    else if (kd == EPI_GELU) y = epi_gelu(y);
    else if (kd == EPI_BIAS) y += __ldg(P.epi_ptr[e] + n);
    else y += __ldg(P.epi_ptr[e] + o);
  }
  P.out[o] = y;
  if (P.out_bf16) static_cast<__nv_bfloat16*>(P.out_bf16)[o] = __float2bfloat16_rn(y);
}

}  // namespace

cudaError_t launch_pool(const PoolParams& P, cudaStream_t stream) {
  if (P.op == 0) {
    const int64_t total = static_cast<int64_t>(P.N) * P.C * P.Ho * P.Wo;
    if (total == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    return launch_pdl(maxpool_kernel, dim3(blocks), dim3(256), 0, stream, P);
  }
  const int64_t nc = static_cast<int64_t>(P.N) * P.C;
  if (nc == 0) return cudaSuccess;
  return launch_pdl(gap_kernel, dim3(static_cast<unsigned>((nc + 7) / 8)), dim3(256), 0, stream, P);
}

cudaError_t launch_gemv(const GemvParams& P, cudaStream_t stream) {
  if (P.M == 0 || P.N == 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((P.N + kGemvCols - 1) / kGemvCols), static_cast<unsigned>(P.M));
  return launch_pdl(gemv_kernel, grid, dim3(256), 0, stream, P);
}

}  // namespace lfg
