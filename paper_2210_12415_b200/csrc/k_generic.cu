// k_generic.cu — layout-agnostic element-wise and contraction kernels.
//
// These execute any node of a lowered graph on any legal layout, the way the
// reference's interpreter does (proj/src/interp.cpp:341-411), but with the
// index arithmetic precompiled: the output is walked in its physical order
// through the inverse IxProgram (like build_loop_nest's loops over the
// transformed output dims, lower.cpp:164-179), and each operand read goes
// through a per-logical-dimension offset table. Every sequence the tuner
// emits is separable per logical dimension (split/reorder/unfold/pad/fuse
// without a later re-split), so offset(l) = sum_j table_j[l_j].
//
// Contractions here are the CUDA-core path: used for layouts tcgen05 cannot
// consume (e.g. the 1-element channel tiles of the reference's fuzz tests)
// and for LFGPU_PLAN_EXACT, which accumulates in fp64 like reference_eval
// (interp.cpp:70-122).
#include <cuda_runtime.h>

#include <algorithm>

#include "lf_core.hpp"
#include "lf_generic.hpp"
#include "lf_pdl.hpp"

namespace lfg {

struct IxState {
  int32_t v[kMaxRank];
  int32_t r;
};

// Local copy of the program interpreter (k_copy.cu has the same semantics;
// separate compilation units keep their own inline copy).
__device__ __forceinline__ int ix_exec(const IxProgram& p, IxState& s) {
  int status = 0;
  for (int k = 0; k < p.nops; ++k) {
    const IxOp& o = p.ops[k];
    switch (o.kind) {
      case IX_SPLIT: {
        int32_t e = s.v[o.dim];
        int32_t tmp[kMaxRank];
        for (int j = o.n - 1; j >= 0; --j) {
          tmp[j] = e % o.a[j];
          e /= o.a[j];
        }
        tmp[0] += e * o.a[0];
        for (int j = s.r - 1; j > o.dim; --j) s.v[j + o.n - 1] = s.v[j];
        for (int j = 0; j < o.n; ++j) s.v[o.dim + j] = tmp[j];
        s.r += o.n - 1;
        break;
      }
      case IX_FUSE: {
        int32_t acc = 0;
        for (int j = 0; j < o.n; ++j) acc = acc * o.a[j] + s.v[o.dim + j];
        s.v[o.dim] = acc;
        for (int j = o.dim + 1; j + o.n - 1 < s.r; ++j) s.v[j] = s.v[j + o.n - 1];
        s.r -= o.n - 1;
        break;
      }
      case IX_PERM: {
        int32_t tmp[kMaxRank];
        for (int j = 0; j < o.n; ++j) tmp[j] = s.v[o.a[j]];
        for (int j = 0; j < o.n; ++j) s.v[j] = tmp[j];
        break;
      }
      case IX_FOLD: {
        int32_t x = s.v[o.dim] * o.a[0] + s.v[o.dim + 1];
        if (o.a[1] >= 0) x = min(x, o.a[1]);
        s.v[o.dim] = x;
        for (int j = o.dim + 1; j + 1 < s.r; ++j) s.v[j] = s.v[j + 1];
        s.r -= 1;
        break;
      }
      case IX_UNFOLD: {
        int32_t e = s.v[o.dim];
        int32_t tt = min(e / o.a[0], o.a[1] - 1);
        for (int j = s.r - 1; j > o.dim; --j) s.v[j + 1] = s.v[j];
        s.v[o.dim] = tt;
        s.v[o.dim + 1] = e - tt * o.a[0];
        s.r += 1;
        break;
      }
      case IX_BOUND: {
        int32_t x = s.v[o.dim];
        if (x < o.a[0] || x >= o.a[1]) {
          if (o.flag) status = 2;
          else return 1;
        }
        break;
      }
      case IX_SHIFT:
        s.v[o.dim] += o.a[0];
        break;
    }
  }
  return status;
}

__device__ __forceinline__ void decode_phys(const IxProgram& p, int64_t f, IxState& s) {
  s.r = p.in_rank;
  for (int k = p.in_rank - 1; k >= 0; --k) {
    s.v[k] = static_cast<int32_t>(f % p.in_ext[k]);
    f /= p.in_ext[k];
  }
}

template <typename T>
__device__ __forceinline__ double ld(const T* p, int64_t off) {
  return static_cast<double>(p[off]);
}

template <typename T>
__global__ void __launch_bounds__(256)
    gen_eltwise(const IxProgram* __restrict__ out_prog, GenEltwise P, T* __restrict__ out,
                int* err) {
  LFG_PDL_ENTRY();
  __shared__ IxProgram sp;
  {
    const int* g = reinterpret_cast<const int*>(out_prog);
    int* s = reinterpret_cast<int*>(&sp);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(IxProgram) / 4); i += blockDim.x)
      s[i] = g[i];
  }
  __syncthreads();
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < P.n;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    IxState s;
    decode_phys(sp, f, s);
    int st = ix_exec(sp, s);
    if (st != 0) {
      if (st == 2 && err) atomicOr(err, 1);
      out[f] = T(0);
      continue;
    }
    double x = 0, y = 0;
    int64_t o0 = 0, o1 = 0;
    for (int j = 0; j < P.rank; ++j) o0 += P.tab0[P.tab_off[j] + s.v[j]];
    x = ld(static_cast<const T*>(P.in0), o0);
    if (P.op == GEN_BIASADD) {
      o1 = P.tab1[s.v[P.bias_dim]];
      y = ld(static_cast<const T*>(P.in1), o1);
    } else if (P.op == GEN_EWADD) {
      for (int j = 0; j < P.rank; ++j) o1 += P.tab1[P.tab_off[j] + s.v[j]];
      y = ld(static_cast<const T*>(P.in1), o1);
    }
    double r;
    switch (P.op) {
      case GEN_RELU: r = x > 0.0 ? x : 0.0; break;
      case GEN_GELU: r = 0.5 * x * (1.0 + erf(x * 0.70710678118654752440)); break;
      case GEN_BIASADD:
      case GEN_EWADD: r = x + y; break;
      default: r = x; break;
    }
    out[f] = static_cast<T>(r);
  }
}

template <typename T, typename Acc>
__global__ void __launch_bounds__(256)
    gen_contract(const IxProgram* __restrict__ out_prog, GenContract P, T* __restrict__ out) {
  LFG_PDL_ENTRY();
  __shared__ IxProgram sp;
  {
    const int* g = reinterpret_cast<const int*>(out_prog);
    int* s = reinterpret_cast<int*>(&sp);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(IxProgram) / 4); i += blockDim.x)
      s[i] = g[i];
  }
  __syncthreads();
  const T* A = static_cast<const T*>(P.a);
  const T* B = static_cast<const T*>(P.b);
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < P.n;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    IxState s;
    decode_phys(sp, f, s);
    ix_exec(sp, s);
    Acc acc = 0;
    if (P.op == GEN_MAXPOOL) {
      // max over the window of A(b, c, V*h+rh, V*w+rw) on a padded input
      const int64_t* ta = P.ta;
      const int64_t a1 = ta[P.a_off[0] + s.v[0]] + ta[P.a_off[1] + s.v[1]];
      const int h = s.v[2], w = s.v[3];
      Acc m = static_cast<Acc>(A[a1 + ta[P.a_off[2] + P.V * h] + ta[P.a_off[3] + P.V * w]]);
      for (int64_t rh = 0; rh < P.KH; ++rh) {
        const int64_t a2 = a1 + ta[P.a_off[2] + P.V * h + rh];
        for (int64_t rw = 0; rw < P.KW; ++rw) {
          const Acc x = static_cast<Acc>(A[a2 + ta[P.a_off[3] + P.V * w + rw]]);
          m = x > m ? x : m;
        }
      }
      out[f] = static_cast<T>(m);
      continue;
    }
    if (P.op == GEN_GLOBAL_AVGPOOL) {
      const int64_t* ta = P.ta;
      const int64_t a1 = ta[P.a_off[0] + s.v[0]] + ta[P.a_off[1] + s.v[1]];
      for (int64_t h = 0; h < P.H; ++h) {
        const int64_t a2 = a1 + ta[P.a_off[2] + h];
        for (int64_t w = 0; w < P.W; ++w) acc += static_cast<Acc>(A[a2 + ta[P.a_off[3] + w]]);
      }
      out[f] = static_cast<T>(acc / static_cast<Acc>(P.H * P.W));
      continue;
    }
    if (P.op == GEN_GMM) {
      const int64_t* ta = P.ta;
      const int64_t* tb = P.tb;
      int64_t am = ta[P.a_off[0] + s.v[0]];
      int64_t bn = tb[P.b_off[1] + s.v[1]];
      for (int64_t k = 0; k < P.K; ++k)
        acc += static_cast<Acc>(A[am + ta[P.a_off[1] + k]]) *
               static_cast<Acc>(B[tb[P.b_off[0] + k] + bn]);
    } else {
      // C2D: A(b, i, V*h+rh, V*w+rw) * B(o, i, rh, rw)   (interp.cpp:70-89)
      // DEP: A(b, c, V*h+rh, V*w+rw) * B(c, rh, rw)      (interp.cpp:90-108)
      const int64_t* ta = P.ta;
      const int64_t* tb = P.tb;
      int b = s.v[0], o = s.v[1], h = s.v[2], w = s.v[3];
      int64_t a0 = ta[P.a_off[0] + b];
      if (P.op == GEN_C2D) {
        int64_t b0 = tb[P.b_off[0] + o];
        for (int64_t i = 0; i < P.I; ++i) {
          int64_t a1 = a0 + ta[P.a_off[1] + i];
          int64_t b1 = b0 + tb[P.b_off[1] + i];
          for (int64_t rh = 0; rh < P.KH; ++rh) {
            int64_t a2 = a1 + ta[P.a_off[2] + P.V * h + rh];
            int64_t b2 = b1 + tb[P.b_off[2] + rh];
            for (int64_t rw = 0; rw < P.KW; ++rw)
              acc += static_cast<Acc>(A[a2 + ta[P.a_off[3] + P.V * w + rw]]) *
                     static_cast<Acc>(B[b2 + tb[P.b_off[3] + rw]]);
          }
        }
      } else {
        int64_t a1 = a0 + ta[P.a_off[1] + o];
        int64_t b0 = tb[P.b_off[0] + o];
        for (int64_t rh = 0; rh < P.KH; ++rh) {
          int64_t a2 = a1 + ta[P.a_off[2] + P.V * h + rh];
          int64_t b1 = b0 + tb[P.b_off[1] + rh];
          for (int64_t rw = 0; rw < P.KW; ++rw)
            acc += static_cast<Acc>(A[a2 + ta[P.a_off[3] + P.V * w + rw]]) *
                   static_cast<Acc>(B[b1 + tb[P.b_off[2] + rw]]);
        }
      }
    }
    out[f] = static_cast<T>(acc);
  }
}

// Few outputs, long reductions (FC at small batch, GlobalAvgPool, a
// downsample conv on a layout tcgen05 cannot consume): one warp per output
// element, lanes split the flattened reduction index r and combine with
// shuffles. Same operand tables as gen_contract.
template <typename T, typename Acc>
__global__ void __launch_bounds__(256)
    gen_contract_warp(const IxProgram* __restrict__ out_prog, GenContract P, T* __restrict__ out) {
  LFG_PDL_ENTRY();
  __shared__ IxProgram sp;
  {
    const int* g = reinterpret_cast<const int*>(out_prog);
    int* s = reinterpret_cast<int*>(&sp);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(IxProgram) / 4); i += blockDim.x)
      s[i] = g[i];
  }
  __syncthreads();
  const T* A = static_cast<const T*>(P.a);
  const T* B = static_cast<const T*>(P.b);
  const int64_t* ta = P.ta;
  const int64_t* tb = P.tb;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const bool is_max = P.op == GEN_MAXPOOL;
  int64_t R;
  switch (P.op) {
    case GEN_GMM: R = P.K; break;
    case GEN_C2D: R = P.I * P.KH * P.KW; break;
    case GEN_GLOBAL_AVGPOOL: R = P.H * P.W; break;
    default: R = P.KH * P.KW; break;  // DEP, MaxPool
  }
  const int64_t khw = P.KH * P.KW;
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); f < P.n;
       f += warps) {
    IxState s;
    decode_phys(sp, f, s);
    ix_exec(sp, s);
    Acc acc = 0;
    bool any = false;
    for (int64_t r = lane; r < R; r += 32) {
      Acc x;
      if (P.op == GEN_GMM) {
        x = static_cast<Acc>(A[ta[P.a_off[0] + s.v[0]] + ta[P.a_off[1] + r]]) *
            static_cast<Acc>(B[tb[P.b_off[0] + r] + tb[P.b_off[1] + s.v[1]]]);
      } else if (P.op == GEN_GLOBAL_AVGPOOL) {
        const int64_t h = r / P.W, w = r - h * P.W;
        x = static_cast<Acc>(A[ta[P.a_off[0] + s.v[0]] + ta[P.a_off[1] + s.v[1]] +
                               ta[P.a_off[2] + h] + ta[P.a_off[3] + w]]);
      } else if (P.op == GEN_C2D) {
        const int64_t i = r / khw, rr = r - i * khw, rh = rr / P.KW, rw = rr - rh * P.KW;
        x = static_cast<Acc>(A[ta[P.a_off[0] + s.v[0]] + ta[P.a_off[1] + i] +
                               ta[P.a_off[2] + P.V * s.v[2] + rh] +
                               ta[P.a_off[3] + P.V * s.v[3] + rw]]) *
            static_cast<Acc>(B[tb[P.b_off[0] + s.v[1]] + tb[P.b_off[1] + i] +
                               tb[P.b_off[2] + rh] + tb[P.b_off[3] + rw]]);
      } else {  // DEP / MaxPool window element
        const int64_t rh = r / P.KW, rw = r - rh * P.KW;
        const int64_t ao = ta[P.a_off[0] + s.v[0]] + ta[P.a_off[1] + s.v[1]] +
                           ta[P.a_off[2] + P.V * s.v[2] + rh] + ta[P.a_off[3] + P.V * s.v[3] + rw];
        x = static_cast<Acc>(A[ao]);
        if (P.op == GEN_DEP)
          x *= static_cast<Acc>(B[tb[P.b_off[0] + s.v[1]] + tb[P.b_off[1] + rh] + tb[P.b_off[2] + rw]]);
      }
      if (is_max) acc = any ? (x > acc ? x : acc) : x;
      else acc += x;
      any = true;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Acc y = __shfl_xor_sync(0xffffffffu, acc, o);
      const int ay = __shfl_xor_sync(0xffffffffu, any ? 1 : 0, o);
      if (is_max) {
        if (ay && (!any || y > acc)) acc = y;
        any = any || ay;
      } else {
        acc += y;
      }
    }
    if (lane == 0) {
      if (P.op == GEN_GLOBAL_AVGPOOL) acc = acc / static_cast<Acc>(P.H * P.W);
      out[f] = static_cast<T>(acc);
    }
  }
}

static int64_t grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32;
}

cudaError_t launch_gen_eltwise(const IxProgram* d_prog, const GenEltwise& P, int elem, void* out,
                               int* d_err, cudaStream_t stream) {
  if (P.n == 0) return cudaSuccess;
  unsigned g = static_cast<unsigned>(grid_for(P.n));
  if (elem == LFGPU_ELEM_I32)
    launch_pdl(gen_eltwise<int32_t>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<int32_t*>(out), d_err);
  else
    launch_pdl(gen_eltwise<float>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<float*>(out), d_err);
  return cudaGetLastError();
}

cudaError_t launch_gen_contract(const IxProgram* d_prog, const GenContract& P, int elem,
                                bool exact, void* out, cudaStream_t stream) {
  if (P.n == 0) return cudaSuccess;
  int64_t R;
  switch (P.op) {
    case GEN_GMM: R = P.K; break;
    case GEN_C2D: R = P.I * P.KH * P.KW; break;
    case GEN_GLOBAL_AVGPOOL: R = P.H * P.W; break;
    default: R = P.KH * P.KW; break;
  }
  // Warp per output when the outputs alone cannot fill the GPU with long
  // serial reductions (148 SMs x 2048 threads).
  if (R >= 32 && P.n * 8 <= 148 * 2048) {
    const int64_t warps = std::min<int64_t>(P.n, 148 * 64);
    const unsigned g = static_cast<unsigned>((warps + 7) / 8);
    if (elem == LFGPU_ELEM_I32)
      launch_pdl(gen_contract_warp<int32_t, long long>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<int32_t*>(out));
    else if (exact)
      launch_pdl(gen_contract_warp<float, double>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<float*>(out));
    else
      launch_pdl(gen_contract_warp<float, float>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<float*>(out));
    return cudaGetLastError();
  }
  unsigned g = static_cast<unsigned>(grid_for(P.n));
  if (elem == LFGPU_ELEM_I32)
    launch_pdl(gen_contract<int32_t, long long>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<int32_t*>(out));
  else if (exact)
    launch_pdl(gen_contract<float, double>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<float*>(out));
  else
    launch_pdl(gen_contract<float, float>, dim3(g), dim3(256), 0, stream, d_prog, P, static_cast<float*>(out));
  return cudaGetLastError();
}

}  // namespace lfg
