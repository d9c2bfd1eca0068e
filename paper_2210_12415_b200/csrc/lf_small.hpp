// lf_small.hpp — CUDA-core kernels for the small operators at the ends of
// ResNet-18 (k_small.cu): MaxPool / GlobalAvgPool through separable offset
// tables, and the small-M GMM (batch-1 classifier) with its element-wise
// epilogue fused. Semantics: lfgpu.h (LFGPU_OP_MAXPOOL, _GLOBAL_AVGPOOL) and
// lf::interp (interp.cpp:109-122 for GMM); fp32 arithmetic (the exact-mode
// plans keep the fp64-accumulating generic kernels).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lfg {

struct PoolParams {
  int32_t op = 0;  // 0 MaxPool (window K, stride V), 1 GlobalAvgPool
  int32_t N = 0, C = 0, H = 0, W = 0, Ho = 0, Wo = 0, K = 1, V = 1;
  int32_t pad = 0;  // MaxPool reading an absorbed Padding's input: zeros outside [0, H) x [0, W)
  const float* x = nullptr;
  const int64_t* xt = nullptr;  // input tables (n, c, h, w)
  int64_t x_off[4] = {};
  float* out = nullptr;
  void* out_bf16 = nullptr;     // optional bf16 copy, same layout
  const int64_t* ot = nullptr;  // output tables (n, c[, h, w])
  int64_t o_off[4] = {};
};
cudaError_t launch_pool(const PoolParams& P, cudaStream_t stream);

// C[M, N] = A[M, K] B[K, N] for small M, then the fused chain (bias over N,
// residual in C's layout, ReLU, GELU); 32 columns x 8 K-slices per CTA, the
// slices summed in a fixed order.
struct GemvParams {
  int32_t M = 0, K = 0, N = 0;
  const float* a = nullptr;
  const int64_t* at = nullptr;
  int64_t a_off[2] = {};
  const float* b = nullptr;
  const int64_t* bt = nullptr;
  int64_t b_off[2] = {};
  float* out = nullptr;
  void* out_bf16 = nullptr;
  const int64_t* ot = nullptr;
  int64_t o_off[2] = {};
  int32_t nepi = 0;
  int32_t epi_kind[4] = {};     // EPI_* (lf_umma.hpp)
  const float* epi_ptr[4] = {};
};
cudaError_t launch_gemv(const GemvParams& P, cudaStream_t stream);

}  // namespace lfg
