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

// K6: depthwise C2D (DEP, interp.cpp:90-108) on tuned layouts. Every
// operand is addressed through per-logical-dim offset tables (the layout
// must be separable: split / reorder / fuse / unfold / pad), one thread
// per output element, threads ordered so that `fast` — the output's
// unit-stride logical dim (C for channel bricks, W for NCHW) — varies
// fastest: loads and stores coalesce. Accumulates in fp32 in the
// reference's (rh, rw) order; the fused element-wise chain runs before
// the store.
struct DirectDep {
  int32_t N = 0, C = 0, Ho = 0, Wo = 0, KH = 0, KW = 0, V = 1;
  int32_t fast = 1;                    // 1: C fastest, 3: W fastest
  int32_t vec4 = 0;                    // float4 over 4 channels (dep_direct4)
  const float* x = nullptr;            // padded input, its own layout
  const int64_t* xt = nullptr;         // input tables (n, c, h, w)
  int64_t x_off[4] = {};
  const float* w = nullptr;            // weights [C][KH][KW], their own layout
  const int64_t* wt = nullptr;
  int64_t w_off[3] = {};
  float* out = nullptr;
  const int64_t* ot = nullptr;         // output tables (n, c, h, w)
  int64_t o_off[4] = {};
  int32_t nepi = 0;
  int32_t epi_kind[4] = {};
  const float* epi_ptr[4] = {};        // bias: logical [C]; residual: output layout
};

cudaError_t launch_dep_direct(const DirectDep& P, cudaStream_t stream);

// Small-I C2D on tensor cores (the ResNet stem): im2col into K-major
// [M/RT][Kp/64][RT][64] bf16 bricks (RT = whole output rows per tile) (M = N*Ho*Wo pixels, K = I*KH*KW
// zero-padded to Kp) plus the weights as [1][Kp/64][O][64] bf16, then the
// tcgen05 GEMM writes the conv output layout directly. One launch prepares
// both operands.
struct Im2col {
  const float* x = nullptr;  // logical (padded) NCHW input
  const float* w = nullptr;  // logical OIHW weights
  void* a = nullptr;         // bf16 A bricks
  void* b = nullptr;         // bf16 B bricks
  int32_t N = 0, I = 0, H = 0, W = 0, KH = 0, KW = 0, V = 1, Ho = 0, Wo = 0, O = 0, K = 0, Kp = 0;
  int32_t RT = 128;          // rows (pixels) per A brick = per GEMM tile
  int32_t pad = 0;           // absorbed Padding: x is the unpadded input
};

cudaError_t launch_im2col(const Im2col& Q, cudaStream_t stream);

bool direct_conv_applies(int64_t I, int64_t KH, int64_t KW, int64_t O);
size_t direct_conv_smem(const DirectConv& P);
cudaError_t launch_c2d_direct(const DirectConv& P, cudaStream_t stream);

}  // namespace lfg
