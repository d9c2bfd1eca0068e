// lf_direct.hpp — CUDA-core direct convolution for small I (k_direct.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lf_core.hpp"

namespace lfg {

enum { DIRECT_EPI_BIAS = 1, DIRECT_EPI_RELU = 2, DIRECT_EPI_RESIDUAL = 3 };

struct DirectConv {
  int32_t N = 0, I = 0, H = 0, W = 0;  // logical (padded) input extents
  int32_t O = 0, KH = 0, KW = 0, V = 1;
  int32_t Ho = 0, Wo = 0;
  const float* x = nullptr;            // logical NCHW input
  const float* w = nullptr;            // logical OIHW weights
  float* out = nullptr;
  const int64_t* tab = nullptr;        // output separable offset tables
  int64_t tab_off[4] = {};
  int32_t nepi = 0;
  int32_t epi_kind[4] = {};
  const float* epi_ptr[4] = {};        // bias: logical [O]; residual: output layout
};

bool direct_conv_applies(int64_t I, int64_t KH, int64_t KW, int64_t O);
size_t direct_conv_smem(const DirectConv& P);
cudaError_t launch_c2d_direct(const DirectConv& P, cudaStream_t stream);

}  // namespace lfg
