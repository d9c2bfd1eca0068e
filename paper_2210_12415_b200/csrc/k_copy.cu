// k_copy.cu — K1 layout conversion and K2 pad-convert kernels (sm_100a).
//
// Replaces the per-element materialization of the reference
// (lf::materialize_step, proj/src/interp.cpp:181-264; the LayoutConvert and
// Padding nests, lower.cpp:228-243) with two kernels:
//   * digit_copy: runs a DigitMap (lf_core.hpp). The copy space is tiled on
//     two digits: `a` = the destination-contiguous digit and `b` = the
//     source-contiguous digit when they differ (SMEM-staged transpose with a
//     padded tile so both global sides are coalesced), else the next digit
//     out (direct coalesced copy). Remaining digits are decoded once per CTA.
//     Zero predicates (pad / Padding guard) and unfold clamps are linear in
//     the digits, so per element they cost a few integer FMAs.
//   * ix_copy: runs the general IxProgram pair per element.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "lf_core.hpp"
#include "lf_kernels.hpp"

namespace lfg {

// ---------------------------------------------------------------------------
// element conversion

template <typename T>
struct Elem;
template <>
struct Elem<float> {
  __device__ static float to_f(float v) { return v; }
  __device__ static double to_d(float v) { return v; }
  __device__ static float from_d(double v) { return static_cast<float>(v); }
  __device__ static float from_f(float v) { return v; }
};
template <>
struct Elem<int32_t> {
  __device__ static float to_f(int32_t v) { return static_cast<float>(v); }
  __device__ static double to_d(int32_t v) { return v; }
  __device__ static int32_t from_d(double v) { return static_cast<int32_t>(v); }
  __device__ static int32_t from_f(float v) { return static_cast<int32_t>(v); }
};
template <>
struct Elem<__nv_bfloat16> {
  __device__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static double to_d(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static __nv_bfloat16 from_d(double v) {
    return __float2bfloat16_rn(static_cast<float>(v));
  }
  __device__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <>
struct Elem<double> {
  __device__ static float to_f(double v) { return static_cast<float>(v); }
  __device__ static double to_d(double v) { return v; }
  __device__ static double from_d(double v) { return v; }
  __device__ static double from_f(float v) { return v; }
};

// Exact conversion path: go through double unless both sides are 32-bit
// float/bf16 (float is exact for bf16).
template <typename TS, typename TD>
__device__ __forceinline__ TD convert(TS v) {
  return Elem<TD>::from_d(Elem<TS>::to_d(v));
}
template <>
__device__ __forceinline__ float convert<float, float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 convert<float, __nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ float convert<__nv_bfloat16, float>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 convert<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 v) {
  return v;
}

template <typename T>
__device__ __forceinline__ T zero_of() {
  return Elem<T>::from_f(0.0f);
}

// ---------------------------------------------------------------------------
// digit_copy

constexpr int kCopyThreads = 256;

struct DCParams {
  int32_t nout;
  int32_t npred, nclamp;
  int32_t ta, tb;          // tile sizes along a, b
  int32_t tiles_a, tiles_b;
  int32_t transpose;       // 1: SMEM-staged (src-contiguous digit b)
  int64_t oext[kMaxDig];
  int64_t odst[kMaxDig], osrc[kMaxDig];
  int64_t opred[kMaxPred][kMaxDig];
  int64_t oclamp[kMaxClamp][kMaxDig];
  int64_t ea, eb;
  int64_t dst_a, dst_b, src_a, src_b;
  int64_t pa[kMaxPred], pb[kMaxPred], pconst[kMaxPred], plo[kMaxPred], phi[kMaxPred];
  int64_t ca[kMaxClamp], cb[kMaxClamp], cconst[kMaxClamp], cmax[kMaxClamp],
      cstride[kMaxClamp];
  int64_t src_base;
};

template <typename TS, typename TD>
__global__ void __launch_bounds__(kCopyThreads)
    digit_copy(const DCParams P, const TS* __restrict__ src, TD* __restrict__ dst) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TS* tile = reinterpret_cast<TS*>(smem_raw);

  // Decode this CTA's tile and outer digits once.
  int64_t t = blockIdx.x;
  const int64_t ia0 = (t % P.tiles_a) * P.ta;
  t /= P.tiles_a;
  const int64_t ib0 = (t % P.tiles_b) * P.tb;
  t /= P.tiles_b;
  int64_t dbase = 0, sbase = P.src_base;
  int64_t pv[kMaxPred], cv[kMaxClamp];
#pragma unroll
  for (int p = 0; p < kMaxPred; ++p) pv[p] = P.pconst[p];
#pragma unroll
  for (int c = 0; c < kMaxClamp; ++c) cv[c] = P.cconst[c];
  for (int d = P.nout - 1; d >= 0; --d) {
    int64_t x = t % P.oext[d];
    t /= P.oext[d];
    dbase += x * P.odst[d];
    sbase += x * P.osrc[d];
    for (int p = 0; p < P.npred; ++p) pv[p] += x * P.opred[p][d];
    for (int c = 0; c < P.nclamp; ++c) cv[c] += x * P.oclamp[c][d];
  }
  // Fold the tile origin into the bases.
  dbase += ia0 * P.dst_a + ib0 * P.dst_b;
  sbase += ia0 * P.src_a + ib0 * P.src_b;
  for (int p = 0; p < P.npred; ++p) pv[p] += ia0 * P.pa[p] + ib0 * P.pb[p];
  for (int c = 0; c < P.nclamp; ++c) cv[c] += ia0 * P.ca[c] + ib0 * P.cb[c];
  const int ta = static_cast<int>(min(static_cast<int64_t>(P.ta), P.ea - ia0));
  const int tb = static_cast<int>(min(static_cast<int64_t>(P.tb), P.eb - ib0));
  const int n = ta * tb;

  auto load = [&](int ia, int ib, bool& valid) -> TS {
    valid = true;
    for (int p = 0; p < P.npred; ++p) {
      int64_t v = pv[p] + ia * P.pa[p] + ib * P.pb[p];
      valid = valid && v >= P.plo[p] && v < P.phi[p];
    }
    int64_t off = sbase + ia * P.src_a + ib * P.src_b;
    for (int c = 0; c < P.nclamp; ++c) {
      int64_t v = cv[c] + ia * P.ca[c] + ib * P.cb[c];
      off += min(v, P.cmax[c]) * P.cstride[c];
    }
    return valid ? __ldg(src + off) : zero_of<TS>();
  };

  if (P.transpose) {
    const int ld = P.tb + 1;  // padded row: conflict-free column walk
    // Read phase: b (source-contiguous) fastest.
    for (int i = threadIdx.x; i < n; i += kCopyThreads) {
      int ib = i % tb, ia = i / tb;
      bool ok;
      tile[ia * ld + ib] = load(ia, ib, ok);
    }
    __syncthreads();
    // Write phase: a (destination-contiguous) fastest.
    for (int i = threadIdx.x; i < n; i += kCopyThreads) {
      int ia = i % ta, ib = i / ta;
      dst[dbase + ia * P.dst_a + ib * P.dst_b] = convert<TS, TD>(tile[ia * ld + ib]);
    }
  } else {
    // Direct: a fastest on both sides; 4 independent loads in flight.
    constexpr int U = 4;
    for (int i0 = threadIdx.x; i0 < n; i0 += kCopyThreads * U) {
      TS v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int i = i0 + u * kCopyThreads;
        if (i < n) {
          bool ok;
          v[u] = load(i % ta, i / ta, ok);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int i = i0 + u * kCopyThreads;
        if (i < n) {
          int ia = i % ta, ib = i / ta;
          dst[dbase + ia * P.dst_a + ib * P.dst_b] = convert<TS, TD>(v[u]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ix_copy: the general per-element program

struct IxState {
  int32_t v[kMaxRank];
  int32_t r;
};

// Returns 0 ok, 1 zero (guard/pad), 2 error (out-of-range access).
__device__ int ix_run(const IxProgram& p, IxState& s) {
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
        // the leading component takes the remaining quotient (no mod)
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
        int32_t tt = e >= 0 ? e / o.a[0] : -((-e + o.a[0] - 1) / o.a[0]);
        tt = min(tt, o.a[1] - 1);
        for (int j = s.r - 1; j > o.dim; --j) s.v[j + 1] = s.v[j];
        s.v[o.dim] = tt;
        s.v[o.dim + 1] = e - tt * o.a[0];
        s.r += 1;
        break;
      }
      case IX_BOUND: {
        int32_t x = s.v[o.dim];
        if (x < o.a[0] || x >= o.a[1]) {
          if (o.flag) status = status == 1 ? 1 : 2;
          else return 1;  // zero cell: guard wins over any later error
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

template <typename TS, typename TD>
__global__ void __launch_bounds__(kCopyThreads)
    ix_copy(const IxProgram* __restrict__ progs, int64_t n, const TS* __restrict__ src,
            TD* __restrict__ dst, int* err) {
  __shared__ IxProgram sp[2];
  {
    const int* g = reinterpret_cast<const int*>(progs);
    int* s = reinterpret_cast<int*>(sp);
    for (int i = threadIdx.x; i < static_cast<int>(2 * sizeof(IxProgram) / 4); i += blockDim.x)
      s[i] = g[i];
  }
  __syncthreads();
  const IxProgram& pd = sp[0];
  const IxProgram& ps = sp[1];
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    IxState s;
    s.r = pd.in_rank;
    int64_t rem = f;
    for (int k = pd.in_rank - 1; k >= 0; --k) {
      s.v[k] = static_cast<int32_t>(rem % pd.in_ext[k]);
      rem /= pd.in_ext[k];
    }
    int st = ix_run(pd, s);
    if (st == 0) st = ix_run(ps, s);
    if (st == 0) {
      int64_t off = 0;
      for (int k = 0; k < ps.out_rank; ++k) {
        if (s.v[k] < 0 || s.v[k] >= ps.out_ext[k]) st = 2;
        off = off * ps.out_ext[k] + s.v[k];
      }
      if (st == 0) {
        dst[f] = convert<TS, TD>(src[off]);
        continue;
      }
    }
    if (st == 2 && err) atomicOr(err, 1);
    dst[f] = zero_of<TD>();
  }
}

// ---------------------------------------------------------------------------
// host launchers

namespace {

template <template <typename, typename> class K, typename F>
cudaError_t dispatch(int se, int de, F&& f) {
  auto inner = [&](auto s_tag) -> cudaError_t {
    using TS = decltype(s_tag);
    switch (de) {
      case LFGPU_ELEM_F32: return f(TS{}, float{});
      case LFGPU_ELEM_I32: return f(TS{}, int32_t{});
      case LFGPU_ELEM_BF16: return f(TS{}, __nv_bfloat16{});
      case LFGPU_ELEM_F64: return f(TS{}, double{});
    }
    return cudaErrorInvalidValue;
  };
  switch (se) {
    case LFGPU_ELEM_F32: return inner(float{});
    case LFGPU_ELEM_I32: return inner(int32_t{});
    case LFGPU_ELEM_BF16: return inner(__nv_bfloat16{});
    case LFGPU_ELEM_F64: return inner(double{});
  }
  return cudaErrorInvalidValue;
}

template <typename, typename>
struct Unused {};

}  // namespace

int elem_size(int elem) {
  switch (elem) {
    case LFGPU_ELEM_F32:
    case LFGPU_ELEM_I32: return 4;
    case LFGPU_ELEM_BF16: return 2;
    case LFGPU_ELEM_F64: return 8;
  }
  return 0;
}

// Tile selection for a DigitMap (see file comment).
static DCParams make_params(const DigitMap& m, int src_elem) {
  DCParams P;
  std::memset(&P, 0, sizeof(P));
  int nd = m.ndig;
  int a = nd - 1;  // innermost destination digit (dst stride 1)
  int b = -1;
  bool transpose = false;
  if (nd >= 2) {
    if (m.src_stride[a] != 1) {
      for (int d = 0; d < nd - 1; ++d)
        if (m.src_stride[d] == 1) b = d;
      transpose = b >= 0;
    }
    if (b < 0) b = nd - 2;
  }
  const int64_t ea = nd ? m.ext[a] : 1;
  const int64_t eb = b >= 0 ? m.ext[b] : 1;
  int ta, tb;
  if (transpose) {
    // Square-ish tile within a 48 KB SMEM budget, both sides >= 32 B runs.
    int es = std::max(elem_size(src_elem), 1);
    int cap = std::max(1024, 32768 / es);
    ta = static_cast<int>(std::min<int64_t>(ea, 64));
    tb = static_cast<int>(std::min<int64_t>(eb, std::max<int64_t>(64, cap / ta - 1)));
    tb = static_cast<int>(std::min<int64_t>(tb, 256));
  } else {
    ta = static_cast<int>(std::min<int64_t>(ea, 4096));
    tb = static_cast<int>(std::min<int64_t>(eb, std::max<int64_t>(1, 4096 / ta)));
  }
  P.transpose = transpose ? 1 : 0;
  P.ta = std::max(ta, 1);
  P.tb = std::max(tb, 1);
  P.ea = ea;
  P.eb = eb;
  P.tiles_a = static_cast<int32_t>((ea + P.ta - 1) / P.ta);
  P.tiles_b = static_cast<int32_t>((eb + P.tb - 1) / P.tb);
  P.npred = m.npred;
  P.nclamp = m.nclamp;
  P.src_base = m.src_base;
  if (nd) {
    P.dst_a = m.dst_stride[a];
    P.src_a = m.src_stride[a];
    for (int p = 0; p < m.npred; ++p) P.pa[p] = m.pcoef[p][a];
    for (int c = 0; c < m.nclamp; ++c) P.ca[c] = m.ccoef[c][a];
  }
  if (b >= 0) {
    P.dst_b = m.dst_stride[b];
    P.src_b = m.src_stride[b];
    for (int p = 0; p < m.npred; ++p) P.pb[p] = m.pcoef[p][b];
    for (int c = 0; c < m.nclamp; ++c) P.cb[c] = m.ccoef[c][b];
  }
  for (int p = 0; p < m.npred; ++p) {
    P.pconst[p] = m.pconst[p];
    P.plo[p] = m.plo[p];
    P.phi[p] = m.phi[p];
  }
  for (int c = 0; c < m.nclamp; ++c) {
    P.cconst[c] = m.cconst[c];
    P.cmax[c] = m.cmax[c];
    P.cstride[c] = m.cstride[c];
  }
  int k = 0;
  for (int d = 0; d < nd; ++d) {
    if (d == a || d == b) continue;
    P.oext[k] = m.ext[d];
    P.odst[k] = m.dst_stride[d];
    P.osrc[k] = m.src_stride[d];
    for (int p = 0; p < m.npred; ++p) P.opred[p][k] = m.pcoef[p][d];
    for (int c = 0; c < m.nclamp; ++c) P.oclamp[c][k] = m.ccoef[c][d];
    ++k;
  }
  P.nout = k;
  return P;
}

cudaError_t launch_digit_copy(const DigitMap& m, int src_elem, int dst_elem, const void* src,
                              void* dst, cudaStream_t stream, KernelInfo* info) {
  if (m.dst_numel == 0) return cudaSuccess;
  DCParams P = make_params(m, src_elem);
  int64_t outer = 1;
  for (int d = 0; d < P.nout; ++d) outer *= P.oext[d];
  int64_t grid = outer * P.tiles_a * P.tiles_b;
  size_t smem = P.transpose ? static_cast<size_t>(P.ta) * (P.tb + 1) * elem_size(src_elem) : 0;
  if (info) {
    info->name = P.transpose ? "digit_copy_transpose" : "digit_copy_direct";
    info->grid = grid;
  }
  return dispatch<Unused>(src_elem, dst_elem, [&](auto s, auto d) -> cudaError_t {
    using TS = decltype(s);
    using TD = decltype(d);
    auto kern = digit_copy<TS, TD>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    kern<<<static_cast<unsigned>(grid), kCopyThreads, smem, stream>>>(
        P, static_cast<const TS*>(src), static_cast<TD*>(dst));
    return cudaGetLastError();
  });
}

cudaError_t launch_ix_copy(const IxProgram* d_progs, int64_t n, int src_elem, int dst_elem,
                           const void* src, void* dst, int* d_err, cudaStream_t stream,
                           KernelInfo* info) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = std::min<int64_t>((n + kCopyThreads - 1) / kCopyThreads, 148 * 16);
  if (info) {
    info->name = "ix_copy";
    info->grid = blocks;
  }
  return dispatch<Unused>(src_elem, dst_elem, [&](auto s, auto d) -> cudaError_t {
    using TS = decltype(s);
    using TD = decltype(d);
    ix_copy<TS, TD><<<static_cast<unsigned>(blocks), kCopyThreads, 0, stream>>>(
        d_progs, n, static_cast<const TS*>(src), static_cast<TD*>(dst), d_err);
    return cudaGetLastError();
  });
}

}  // namespace lfg
