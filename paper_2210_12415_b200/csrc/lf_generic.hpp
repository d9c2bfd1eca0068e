// lf_generic.hpp — parameters of the layout-agnostic kernels (k_generic.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lf_core.hpp"

namespace lfg {

enum GenOp : int32_t {
  GEN_COPY = 0,
  GEN_RELU = 1,
  GEN_BIASADD = 2,
  GEN_EWADD = 3,
  GEN_C2D = 4,
  GEN_DEP = 5,
  GEN_GMM = 6,
  GEN_MAXPOOL = 7,         // window max (KH = KW = window, stride V); b unused
  GEN_GLOBAL_AVGPOOL = 8,  // [N,C,H,W] -> [N,C]: sum over (h, w) / (H*W); b unused
  GEN_GELU = 9             // element-wise 0.5 x (1 + erf(x / sqrt 2))
};

// Element-wise node: out physical element f -> logical l (out_prog), then
// operand offsets through separable tables (tab*[tab_off[j] + l_j]).
struct GenEltwise {
  int32_t op = GEN_COPY;
  int32_t rank = 0;
  int32_t bias_dim = 1;
  int32_t reserved = 0;
  int64_t n = 0;
  const void* in0 = nullptr;
  const void* in1 = nullptr;
  const int64_t* tab0 = nullptr;
  const int64_t* tab1 = nullptr;  // EwAdd: same shape as tab0; BiasAdd: 1-D
  int64_t tab_off[kMaxRank] = {};
};

struct GenContract {
  int32_t op = GEN_C2D;
  int32_t reserved = 0;
  int64_t n = 0;  // output physical elements
  int64_t I = 0, KH = 0, KW = 0, V = 1, K = 0;
  int64_t H = 0, W = 0;  // GEN_GLOBAL_AVGPOOL input extents
  const void* a = nullptr;
  const void* b = nullptr;
  const int64_t* ta = nullptr;
  const int64_t* tb = nullptr;
  int64_t a_off[4] = {};
  int64_t b_off[4] = {};
};

cudaError_t launch_gen_eltwise(const IxProgram* d_prog, const GenEltwise& P, int elem, void* out,
                               int* d_err, cudaStream_t stream);
cudaError_t launch_gen_contract(const IxProgram* d_prog, const GenContract& P, int elem,
                                bool exact, void* out, cudaStream_t stream);

}  // namespace lfg
