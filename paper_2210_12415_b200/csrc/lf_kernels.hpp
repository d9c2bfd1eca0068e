// lf_kernels.hpp — host launchers of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lf_core.hpp"

namespace lfg {

struct KernelInfo {
  const char* name = "";
  int64_t grid = 0;
};

int elem_size(int elem);

// K1/K2 (k_copy.cu)
// d_tab: the DigitMap's source offset tables in device memory (ntab > 0).
cudaError_t launch_digit_copy(const DigitMap& m, int src_elem, int dst_elem, const void* src,
                              void* dst, cudaStream_t stream, KernelInfo* info,
                              const int32_t* d_tab = nullptr);
// Stream-read a > L2 buffer (measurement hygiene after the flush write).
cudaError_t launch_l2_touch(const void* buf, size_t bytes, int* sink, cudaStream_t stream);
// d_progs: two IxPrograms (dst inverse, src forward) in device memory.
cudaError_t launch_ix_copy(const IxProgram* d_progs, int64_t n, int src_elem, int dst_elem,
                           const void* src, void* dst, int* d_err, cudaStream_t stream,
                           KernelInfo* info);

// ---------------------------------------------------------------------------
// K3/K4: tcgen05 contractions (k_umma.cu)

// A 5-D view of a bf16 operand for TMA: dims innermost-first, strides in
// elements for dims 1..4 (dim 0 is contiguous).
struct TmaView {
  int32_t rank = 0;
  int64_t dims[5] = {};
  int64_t strides[5] = {};  // elements; strides[0] unused (1)
  int32_t box[5] = {};
  int32_t elem_strides[5] = {1, 1, 1, 1, 1};
};

// Epilogue operations fused after the accumulator (lower.cpp:566-608
// fusion groups): out = relu?( acc + bias[n] + residual[m,n] ).
struct Epilogue {
  const float* bias = nullptr;      // indexed by the logical N coordinate
  const float* residual = nullptr;  // same physical layout as the output
  int relu = 0;
};

// Output addressing of the accumulator tile: physical offset of logical
// (m, n) = m_part(m) + n_part(n), each a sum over <= 4 mixed-radix digits.
struct OutMap {
  int32_t nm = 0, nn = 0;
  int64_t m_ext[4] = {}, m_stride[4] = {};  // innermost last
  int64_t n_ext[4] = {}, n_stride[4] = {};
};

struct UmmaGemmDesc {
  int64_t M = 0, N = 0, K = 0;
  int32_t BM = 128, BN = 128, BK = 64;
  int32_t stages = 4;
  int32_t a_mn_major = 0;  // 1: A is M-contiguous (MN-major operand)
  int32_t b_mn_major = 1;  // 1: B is N-contiguous (MN-major operand)
  TmaView a, b;            // boxes are one K-stage of the CTA tile
  // how TMA coordinates advance: coordinate of (m, k) and (k, n) tiles
  int32_t a_m_dims[5] = {}, a_k_dims[5] = {};  // per view dim: 1 if it carries m/k digits
  OutMap out;
  Epilogue epi;
  int32_t persistent = 0;
};

struct UmmaConvDesc {
  // logical problem
  int64_t N = 0, I = 0, O = 0, Ho = 0, Wo = 0, KH = 0, KW = 0, V = 1;
  // template factors (space.cpp:279-280; decode_layout)
  int64_t h_t = 0, w_t = 0, o_t = 0, i_t = 0;
  int32_t stages = 4;
};

}  // namespace lfg
