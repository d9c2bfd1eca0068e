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
#include <climits>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "lf_core.hpp"
#include "lf_kernels.hpp"
#include "lf_pdl.hpp"

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

// Division by a runtime constant as a multiply-high (Granlund-Montgomery):
// for n, d < 2^31, q = (umulhi(n, m) + n) >> l with l = ceil(log2 d).
struct FastDiv {
  uint32_t d, m, l;
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.l;
}

// Tiles are powers of two (TA = 1 << la along the destination-contiguous
// digit a, TB = 1 << lb along digit b) so per-element indexing is shifts and
// masks; each CTA walks tiles grid-stride and decodes the outer digits once
// per tile with multiply-high division. All offsets are 32-bit (tensors
// above 2^31 elements take the general path).
struct DCParams {
  int32_t nout;
  int32_t npred, nclamp;
  int32_t la, lb;  // log2 tile sizes along a, b
  int32_t lg;      // log2 tiles packed per CTA batch
  int32_t transpose;
  int32_t ntiles;
  FastDiv ftiles_a, ftiles_b;
  FastDiv fext[kMaxDig];
  int32_t odst[kMaxDig], osrc[kMaxDig];
  int32_t opred[kMaxPred][kMaxDig];
  int32_t oclamp[kMaxClamp][kMaxDig];
  int32_t ea, eb;
  int32_t dst_a, dst_b, src_a, src_b;
  int32_t pa[kMaxPred], pb[kMaxPred], pconst[kMaxPred], plo[kMaxPred], phi[kMaxPred];
  int32_t ca[kMaxClamp], cb[kMaxClamp], cconst[kMaxClamp], cmax[kMaxClamp],
      cstride[kMaxClamp];
  int32_t src_base;
  int32_t vec;     // 1: the 16-B vector kernels apply; 2: vector stores only
  int32_t rowinv;  // guards/clamps independent of digit a; tables depend on a or b only
  int32_t ntab;
  int32_t ta[kMaxTab], tb[kMaxTab], tconst[kMaxTab], tmax[kMaxTab], toff[kMaxTab];
  int32_t otab[kMaxTab][kMaxDig];
  const int32_t* tab;  // source offset tables (DigitMap::toff), device memory
};

struct TileOrigin {
  int32_t dbase, sbase;
  int32_t pv[kMaxPred], cv[kMaxClamp], tv[kMaxTab];
  int32_t ta, tb;  // valid extents of this tile
};

__device__ __forceinline__ int32_t tab_at(const DCParams& P, int t, int32_t v) {
  return __ldg(P.tab + P.toff[t] + min(max(v, 0), P.tmax[t]));
}

// Param arrays are only ever indexed with compile-time indices (unrolled,
// guarded loops): a runtime index would make nvcc address the parameter
// buffer through a generic pointer, i.e. a global-latency load per access.
// NP / NC: compile-time bounds on the guard / clamp counts (P.npred <= NP,
// P.nclamp <= NC); the unrolled per-digit terms cost NP + NC IMADs each.
template <int NP, int NC, int NT = 0>
__device__ __forceinline__ void decode_tile(const DCParams& P, uint32_t t, TileOrigin& o) {
  constexpr bool PC = NP + NC + NT > 0;
  uint32_t q = fdiv(t, P.ftiles_a);
  const int32_t ia0 = static_cast<int32_t>(t - q * P.ftiles_a.d) << P.la;
  t = q;
  q = fdiv(t, P.ftiles_b);
  const int32_t ib0 = static_cast<int32_t>(t - q * P.ftiles_b.d) << P.lb;
  t = q;
  o.dbase = 0;
  o.sbase = P.src_base;
  if (PC) {
#pragma unroll
    for (int p = 0; p < NP; ++p) o.pv[p] = P.pconst[p] + ia0 * P.pa[p] + ib0 * P.pb[p];
#pragma unroll
    for (int c = 0; c < NC; ++c) o.cv[c] = P.cconst[c] + ia0 * P.ca[c] + ib0 * P.cb[c];
#pragma unroll
    for (int k = 0; k < NT; ++k) o.tv[k] = P.tconst[k] + ia0 * P.ta[k] + ib0 * P.tb[k];
  }
#pragma unroll
  for (int d = kMaxDig - 1; d >= 0; --d) {
    if (d < P.nout) {
      const uint32_t qq = fdiv(t, P.fext[d]);
      const int32_t x = static_cast<int32_t>(t - qq * P.fext[d].d);
      t = qq;
      o.dbase += x * P.odst[d];
      o.sbase += x * P.osrc[d];
      if (PC) {
#pragma unroll
        for (int p = 0; p < NP; ++p) o.pv[p] += x * P.opred[p][d];
#pragma unroll
        for (int c = 0; c < NC; ++c) o.cv[c] += x * P.oclamp[c][d];
#pragma unroll
        for (int k = 0; k < NT; ++k) o.tv[k] += x * P.otab[k][d];
      }
    }
  }
  o.dbase += ia0 * P.dst_a + ib0 * P.dst_b;
  o.sbase += ia0 * P.src_a + ib0 * P.src_b;
  o.ta = min(1 << P.la, P.ea - ia0);
  o.tb = min(1 << P.lb, P.eb - ib0);
}

template <int NP, int NC, int NT, typename TS>
__device__ __forceinline__ TS load_elem(const DCParams& P, const TileOrigin& o,
                                        const TS* __restrict__ src, int ia, int ib) {
  int32_t off = o.sbase + ia * P.src_a + ib * P.src_b;
  if (NP + NC + NT == 0) return __ldg(src + off);
#pragma unroll
  for (int k = 0; k < NT; ++k)
    if (k < P.ntab) off += tab_at(P, k, o.tv[k] + ia * P.ta[k] + ib * P.tb[k]);
  bool valid = true;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int32_t v = o.pv[p] + ia * P.pa[p] + ib * P.pb[p];
    valid = valid && (p >= P.npred || (v >= P.plo[p] && v < P.phi[p]));
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int32_t v = o.cv[c] + ia * P.ca[c] + ib * P.cb[c];
    if (c < P.nclamp) off += min(v, P.cmax[c]) * P.cstride[c];
  }
  return valid ? __ldg(src + off) : zero_of<TS>();
}

// Load phase of the SMEM-staged transposes: tile[ia][ib] for the tile's
// valid extents. When every guard and clamp is independent of digit a
// (P.rowinv: K2's Padding guards and unfold clamps live on the spatial
// digits, a is the channel brick) and a thread's column ib is fixed across
// its iterations (tpt a multiple of TB), the guard/clamp terms are
// evaluated once per tile and each element costs one guarded load.
template <int NP, int NC, int NT, typename TS>
__device__ __forceinline__ void load_tile(const DCParams& P, const TileOrigin& o,
                                          const TS* __restrict__ src, TS* tile, int ld, int lt,
                                          int tpt) {
  const int lb = P.lb, TB = 1 << lb, n = (1 << P.la) * TB;
  if (NP + NC + NT > 0 && P.rowinv && (tpt & (TB - 1)) == 0) {
    const int ib = lt & (TB - 1);
    if (ib >= o.tb) return;
    int32_t off = o.sbase + ib * P.src_b;
    bool valid = true;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int32_t v = o.pv[p] + ib * P.pb[p];
      valid = valid && (p >= P.npred || (v >= P.plo[p] && v < P.phi[p]));
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < P.nclamp) off += min(o.cv[c] + ib * P.cb[c], P.cmax[c]) * P.cstride[c];
    // table terms on the column (b) side here, on the row (a) side per element
#pragma unroll
    for (int k = 0; k < NT; ++k)
      if (k < P.ntab && P.ta[k] == 0) off += tab_at(P, k, o.tv[k] + ib * P.tb[k]);
    const int step = tpt >> lb;
#pragma unroll 4
    for (int ia = lt >> lb; ia < o.ta; ia += step) {
      int32_t e = off + ia * P.src_a;
#pragma unroll
      for (int k = 0; k < NT; ++k)
        if (k < P.ntab && P.ta[k] != 0) e += tab_at(P, k, o.tv[k] + ia * P.ta[k]);
      tile[ia * ld + ib] = valid ? __ldg(src + e) : zero_of<TS>();
    }
    return;
  }
#pragma unroll 4
  for (int idx = lt; idx < n; idx += tpt) {
    const int ia = idx >> lb, ib = idx & (TB - 1);
    if (ia < o.ta && ib < o.tb) tile[ia * ld + ib] = load_elem<NP, NC, NT>(P, o, src, ia, ib);
  }
}

// SMEM-staged transpose: read along b (source-contiguous), write along a
// (destination-contiguous); padded rows keep the column walk conflict-free.
// Tiles are sized to the digit extents; G = 1 << lg small tiles are packed
// per CTA batch (TPT = 256 >> lg threads each) so short unfolded rows
// (e.g. B_w = 10) do not leave most threads idle.
template <typename TS, typename TD, int NP, int NC, int NT>
__global__ void __launch_bounds__(kCopyThreads)
    digit_transpose(const DCParams P, const TS* __restrict__ src, TD* __restrict__ dst) {
  LFG_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int la = P.la, lb = P.lb, lg = P.lg;
  const int TA = 1 << la, TB = 1 << lb, ld = TB + 1, n = TA * TB;
  const int tpt = kCopyThreads >> lg;
  const int q = threadIdx.x >> (8 - lg), lt = threadIdx.x & (tpt - 1);
  TS* tile = reinterpret_cast<TS*>(smem_raw) + q * TA * ld;
  for (int base = blockIdx.x << lg; base < P.ntiles; base += gridDim.x << lg) {
    const int t = base + q;
    TileOrigin o;
    const bool ok = t < P.ntiles;
    if (ok) {
      decode_tile<NP, NC, NT>(P, static_cast<uint32_t>(t), o);
      load_tile<NP, NC, NT>(P, o, src, tile, ld, lt, tpt);
    }
    __syncthreads();
    if (ok) {
#pragma unroll 4
      for (int idx = lt; idx < n; idx += tpt) {
        const int ia = idx & (TA - 1), ib = idx >> la;
        if (ia < o.ta && ib < o.tb)
          dst[o.dbase + ia * P.dst_a + ib * P.dst_b] = convert<TS, TD>(tile[ia * ld + ib]);
      }
    }
    __syncthreads();
  }
}

// Direct copy: a fastest on both sides (coalesced destination; the source is
// coalesced too when its a-stride is 1). Same tile packing as above.
template <typename TS, typename TD, int NP, int NC, int NT>
__global__ void __launch_bounds__(kCopyThreads)
    digit_direct(const DCParams P, const TS* __restrict__ src, TD* __restrict__ dst) {
  LFG_PDL_ENTRY();
  const int la = P.la, lb = P.lb, lg = P.lg;
  const int TA = 1 << la, n = TA << lb;
  const int tpt = kCopyThreads >> lg;
  const int q = threadIdx.x >> (8 - lg), lt = threadIdx.x & (tpt - 1);
  for (int base = blockIdx.x << lg; base < P.ntiles; base += gridDim.x << lg) {
    const int t = base + q;
    if (t >= P.ntiles) continue;
    TileOrigin o;
    decode_tile<NP, NC, NT>(P, static_cast<uint32_t>(t), o);
    constexpr int U = 4;
    for (int i0 = lt; i0 < n; i0 += tpt * U) {
      TS v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * tpt;
        const int a = idx & (TA - 1), b = idx >> la;
        if (idx < n && a < o.ta && b < o.tb) v[u] = load_elem<NP, NC, NT>(P, o, src, a, b);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * tpt;
        const int a = idx & (TA - 1), b = idx >> la;
        if (idx < n && a < o.ta && b < o.tb)
          dst[o.dbase + a * P.dst_a + b * P.dst_b] = convert<TS, TD>(v[u]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Vectorised variants (no predicates / clamps): every global access is 16 B.
// V = 16 / min(sizeof(TS), sizeof(TD)) elements per vector, so both sides
// move whole multiples of 16 B (fp32->bf16: two LDG.128 + one STG.128).
// The host only picks these when V divides the vector digit's extent and
// every other stride on that side, and the base pointers are 16-B aligned.

template <typename TS, typename TD>
struct VecW {
  static constexpr int V = 16 / (sizeof(TS) < sizeof(TD) ? sizeof(TS) : sizeof(TD));
};

template <typename T, int V>
__device__ __forceinline__ void ld_vec(const T* __restrict__ p, T (&v)[V]) {
  static_assert((V * sizeof(T)) % 16 == 0, "vector must be whole 16-B words");
  constexpr int W = V * sizeof(T) / 16;
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const uint4 x = __ldg(q + w);
    memcpy(reinterpret_cast<unsigned char*>(v) + 16 * w, &x, 16);
  }
}

template <typename T, int V>
__device__ __forceinline__ void st_vec(T* __restrict__ p, const T (&v)[V]) {
  constexpr int W = V * sizeof(T) / 16;
  uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint4 x;
    memcpy(&x, reinterpret_cast<const unsigned char*>(v) + 16 * w, 16);
    q[w] = x;
  }
}

// Transpose: loads are V-vectors along b (source-contiguous), stores are
// V-vectors along a (destination-contiguous). The SMEM tile is [TA][TB + V]
// (rows 16-B aligned for vector SMEM stores on the load side; the column
// reads of the store side are scalar).
template <typename TS, typename TD>
__global__ void __launch_bounds__(kCopyThreads)
    digit_transpose_vec(const DCParams P, const TS* __restrict__ src, TD* __restrict__ dst) {
  LFG_PDL_ENTRY();
  constexpr int V = VecW<TS, TD>::V;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int la = P.la, lb = P.lb, lg = P.lg;
  const int TA = 1 << la, TB = 1 << lb, ld = TB + V;
  const int lbv = lb - __ffs(V) + 1, lav = la - __ffs(V) + 1;  // log2(T / V)
  const int nv = (TA * TB) / V;
  const int tpt = kCopyThreads >> lg;
  const int q = threadIdx.x >> (8 - lg), lt = threadIdx.x & (tpt - 1);
  TS* tile = reinterpret_cast<TS*>(smem_raw) + q * TA * ld;
  for (int base = blockIdx.x << lg; base < P.ntiles; base += gridDim.x << lg) {
    const int t = base + q;
    TileOrigin o;
    const bool ok = t < P.ntiles;
    if (ok) {
      decode_tile<0, 0, 0>(P, static_cast<uint32_t>(t), o);
      const int tbv = o.tb / V;
#pragma unroll 2
      for (int idx = lt; idx < nv; idx += tpt) {
        const int ia = idx >> lbv, ibv = idx & ((TB / V) - 1);
        if (ia < o.ta && ibv < tbv) {
          TS v[V];
          ld_vec<TS, V>(src + o.sbase + ia * P.src_a + ibv * V, v);
          st_vec<TS, V>(tile + ia * ld + ibv * V, v);
        }
      }
    }
    __syncthreads();
    if (ok) {
      const int tav = o.ta / V;
#pragma unroll 2
      for (int idx = lt; idx < nv; idx += tpt) {
        const int iav = idx & ((TA / V) - 1), ib = idx >> lav;
        if (iav < tav && ib < o.tb) {
          TD v[V];
#pragma unroll
          for (int j = 0; j < V; ++j) v[j] = convert<TS, TD>(tile[(iav * V + j) * ld + ib]);
          st_vec<TD, V>(dst + o.dbase + iav * V + ib * P.dst_b, v);
        }
      }
    }
    __syncthreads();
  }
}

// Transpose with guarded/clamped scalar loads (K2: Padding guards, unfold
// overhang clamps, unaligned source rows) and 16-B vector stores along a.
template <typename TS, typename TD, int NP, int NC, int NT>
__global__ void __launch_bounds__(kCopyThreads)
    digit_transpose_vst(const DCParams P, const TS* __restrict__ src, TD* __restrict__ dst) {
  LFG_PDL_ENTRY();
  constexpr int V = 16 / sizeof(TD);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int la = P.la, lb = P.lb, lg = P.lg;
  const int TA = 1 << la, TB = 1 << lb, ld = TB + 1, n = TA * TB;
  const int lav = la - __ffs(V) + 1;
  const int tpt = kCopyThreads >> lg;
  const int q = threadIdx.x >> (8 - lg), lt = threadIdx.x & (tpt - 1);
  TS* tile = reinterpret_cast<TS*>(smem_raw) + q * TA * ld;
  for (int base = blockIdx.x << lg; base < P.ntiles; base += gridDim.x << lg) {
    const int t = base + q;
    TileOrigin o;
    const bool ok = t < P.ntiles;
    if (ok) {
      decode_tile<NP, NC, NT>(P, static_cast<uint32_t>(t), o);
      load_tile<NP, NC, NT>(P, o, src, tile, ld, lt, tpt);
    }
    __syncthreads();
    if (ok) {
      const int tav = o.ta / V;
#pragma unroll 2
      for (int idx = lt; idx < n / V; idx += tpt) {
        const int iav = idx & ((TA / V) - 1), ib = idx >> lav;
        if (iav < tav && ib < o.tb) {
          TD v[V];
#pragma unroll
          for (int j = 0; j < V; ++j) v[j] = convert<TS, TD>(tile[(iav * V + j) * ld + ib]);
          st_vec<TD, V>(dst + o.dbase + iav * V + ib * P.dst_b, v);
        }
      }
    }
    __syncthreads();
  }
}

// Direct: a is contiguous on both sides; V-vectors along a.
template <typename TS, typename TD>
__global__ void __launch_bounds__(kCopyThreads)
    digit_direct_vec(const DCParams P, const TS* __restrict__ src, TD* __restrict__ dst) {
  LFG_PDL_ENTRY();
  constexpr int V = VecW<TS, TD>::V;
  const int la = P.la, lb = P.lb, lg = P.lg;
  const int lav = la - __ffs(V) + 1;
  const int nv = (1 << (la + lb)) / V;
  const int tpt = kCopyThreads >> lg;
  const int q = threadIdx.x >> (8 - lg), lt = threadIdx.x & (tpt - 1);
  for (int base = blockIdx.x << lg; base < P.ntiles; base += gridDim.x << lg) {
    const int t = base + q;
    if (t >= P.ntiles) continue;
    TileOrigin o;
    decode_tile<0, 0, 0>(P, static_cast<uint32_t>(t), o);
    const int tav = o.ta / V;
    constexpr int U = 4;
    for (int i0 = lt; i0 < nv; i0 += tpt * U) {
      TS v[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * tpt;
        const int av = idx & ((1 << lav) - 1), b = idx >> lav;
        if (idx < nv && av < tav && b < o.tb)
          ld_vec<TS, V>(src + o.sbase + av * V + b * P.src_b, v[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * tpt;
        const int av = idx & ((1 << lav) - 1), b = idx >> lav;
        if (idx < nv && av < tav && b < o.tb) {
          TD w[V];
#pragma unroll
          for (int j = 0; j < V; ++j) w[j] = convert<TS, TD>(v[u][j]);
          st_vec<TD, V>(dst + o.dbase + av * V + b * P.dst_b, w);
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
  LFG_PDL_ENTRY();
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

static int log2_ceil(int64_t v) {
  int l = 0;
  while ((static_cast<int64_t>(1) << l) < v) ++l;
  return l;
}

static FastDiv make_fastdiv(int64_t d) {
  FastDiv f;
  f.d = static_cast<uint32_t>(d);
  f.l = static_cast<uint32_t>(log2_ceil(d));
  f.m = static_cast<uint32_t>(((static_cast<uint64_t>(1) << 32) *
                               ((static_cast<uint64_t>(1) << f.l) - static_cast<uint64_t>(d))) /
                                  static_cast<uint64_t>(d) +
                              1);
  return f;
}

static int32_t i32(int64_t v) {
  if (v > INT32_MAX || v < INT32_MIN) fail(LFGPU_EUNSUPPORTED, "digit map offset exceeds 32 bits");
  return static_cast<int32_t>(v);
}

// Tile selection for a DigitMap (see file comment).
static DCParams make_params(const DigitMap& m, int src_elem, int dst_elem) {
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
  // Tiles fit the digit extents (<= 32 x 256 transposed, <= 4096 direct),
  // shrink while the grid would underfill 148 SMs x 8 CTAs, and small tiles
  // are packed 1 << lg per CTA batch (~2K elements per batch).
  int64_t outer_ext = 1;
  for (int d = 0; d < nd; ++d)
    if (d != a && d != b) outer_ext *= m.ext[d];
  // 16-B vectors: V elements along a (and along b when transposing) when V
  // divides the vector digits' extents and every other stride on that side.
  const int V = 16 / std::min(elem_size(src_elem), elem_size(dst_elem));
  const int lv = log2_ceil(V);
  bool vec = nd >= 1 && m.npred == 0 && m.nclamp == 0 && m.ntab == 0 && m.dst_stride[a] == 1 &&
             ea % V == 0 &&
             m.src_base % V == 0;
  if (vec) {
    const int sv = transpose ? b : a;  // the source digit read as vectors
    if (m.src_stride[sv] != 1 || (transpose && eb % V != 0)) vec = false;
    for (int d = 0; d < nd && vec; ++d) {
      if (d != a && m.dst_stride[d] % V != 0) vec = false;
      if (d != sv && m.src_stride[d] % V != 0) vec = false;
    }
  }
  int la, lb;
  if (transpose) {
    la = std::min(std::max(log2_ceil(ea), 1), 5);
    lb = std::min(std::max(log2_ceil(eb), 1), 8);
  } else {
    la = std::min(log2_ceil(ea), 12);
    lb = std::max(0, std::min(12 - la, log2_ceil(std::max<int64_t>(eb, 1))));
  }
  // Otherwise a transpose can still store 16-B vectors along a (K2 with
  // guards/clamps or an unaligned source): VS = 16 / sizeof(dst) elements.
  const int VS = 16 / elem_size(dst_elem);
  const int lvs = log2_ceil(VS);
  bool vst = !vec && transpose && m.dst_stride[a] == 1 && ea % VS == 0 && lvs <= 5;
  for (int d = 0; d < nd && vst; ++d)
    if (d != a && m.dst_stride[d] % VS != 0) vst = false;
  if (vec) {
    la = std::max(la, lv);
    if (transpose) lb = std::max(lb, lv);
  }
  if (vst) la = std::max(la, lvs);
  const int min_la = vec ? lv : (vst ? lvs : 1),
            min_lb = vec && transpose ? lv : (transpose ? 1 : 0);
  auto ntiles_for = [&](int x, int y) {
    return outer_ext * ((ea + (int64_t(1) << x) - 1) >> x) * ((eb + (int64_t(1) << y) - 1) >> y);
  };
  while (la + lb > 8 && ntiles_for(la, lb) < 148 * 8) {
    if (lb >= la && lb > min_lb) --lb;
    else if (la > min_la) --la;
    else break;
  }
  P.vec = vec ? 1 : (vst ? 2 : 0);
  // ~16 elements per thread per tile for transposes (one warp per 512-element
  // tile amortises the per-tile digit decode), ~8 for direct copies.
  P.lg = std::max(0, std::min(5, (transpose ? 12 : 11) - la - lb));
  P.transpose = transpose ? 1 : 0;
  P.la = la;
  P.lb = lb;
  P.ea = i32(ea);
  P.eb = i32(eb);
  const int64_t tiles_a = (ea + (1 << la) - 1) >> la, tiles_b = (eb + (1 << lb) - 1) >> lb;
  P.ftiles_a = make_fastdiv(tiles_a);
  P.ftiles_b = make_fastdiv(tiles_b);
  P.npred = m.npred;
  P.nclamp = m.nclamp;
  P.rowinv = 1;
  for (int p = 0; p < m.npred && nd; ++p)
    if (m.pcoef[p][a] != 0) P.rowinv = 0;
  for (int c = 0; c < m.nclamp && nd; ++c)
    if (m.ccoef[c][a] != 0) P.rowinv = 0;
  P.ntab = m.ntab;
  for (int t = 0; t < m.ntab; ++t) {
    const int64_t ca_ = nd ? m.tcoef[t][a] : 0, cb_ = b >= 0 ? m.tcoef[t][b] : 0;
    if (ca_ != 0 && cb_ != 0) P.rowinv = 0;
    P.ta[t] = i32(ca_);
    P.tb[t] = i32(cb_);
    P.tconst[t] = i32(m.tconst[t]);
    P.tmax[t] = i32(m.tmax[t]);
    P.toff[t] = i32(m.toff[t]);
  }
  P.src_base = i32(m.src_base);
  if (nd) {
    P.dst_a = i32(m.dst_stride[a]);
    P.src_a = i32(m.src_stride[a]);
    for (int p = 0; p < m.npred; ++p) P.pa[p] = i32(m.pcoef[p][a]);
    for (int c = 0; c < m.nclamp; ++c) P.ca[c] = i32(m.ccoef[c][a]);
  }
  if (b >= 0) {
    P.dst_b = i32(m.dst_stride[b]);
    P.src_b = i32(m.src_stride[b]);
    for (int p = 0; p < m.npred; ++p) P.pb[p] = i32(m.pcoef[p][b]);
    for (int c = 0; c < m.nclamp; ++c) P.cb[c] = i32(m.ccoef[c][b]);
  }
  for (int p = 0; p < m.npred; ++p) {
    P.pconst[p] = i32(m.pconst[p]);
    P.plo[p] = i32(m.plo[p]);
    P.phi[p] = i32(m.phi[p]);
  }
  for (int c = 0; c < m.nclamp; ++c) {
    P.cconst[c] = i32(m.cconst[c]);
    P.cmax[c] = i32(m.cmax[c]);
    P.cstride[c] = i32(m.cstride[c]);
  }
  int k = 0;
  int64_t outer = 1;
  for (int d = 0; d < nd; ++d) {
    if (d == a || d == b) continue;
    P.fext[k] = make_fastdiv(m.ext[d]);
    P.odst[k] = i32(m.dst_stride[d]);
    P.osrc[k] = i32(m.src_stride[d]);
    for (int p = 0; p < m.npred; ++p) P.opred[p][k] = i32(m.pcoef[p][d]);
    for (int c = 0; c < m.nclamp; ++c) P.oclamp[c][k] = i32(m.ccoef[c][d]);
    for (int t = 0; t < m.ntab; ++t) P.otab[t][k] = i32(m.tcoef[t][d]);
    outer *= m.ext[d];
    ++k;
  }
  P.nout = k;
  P.ntiles = i32(outer * tiles_a * tiles_b);
  return P;
}

cudaError_t launch_digit_copy(const DigitMap& m, int src_elem, int dst_elem, const void* src,
                              void* dst, cudaStream_t stream, KernelInfo* info,
                              const int32_t* d_tab) {
  if (m.dst_numel == 0) return cudaSuccess;
  if (m.ntab > 0 && (!d_tab || src_elem != LFGPU_ELEM_F32)) return cudaErrorInvalidValue;
  DCParams P = make_params(m, src_elem, dst_elem);
  P.tab = d_tab;
  if (P.vec == 1 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15))
    P.vec = 0;
  if (P.vec == 2 && (reinterpret_cast<uintptr_t>(dst) & 15)) P.vec = 0;
  const int V = 16 / std::min(elem_size(src_elem), elem_size(dst_elem));
  size_t smem = P.transpose ? (static_cast<size_t>(1) << P.lg) * (1 << P.la) *
                                  ((1 << P.lb) + (P.vec == 1 ? V : 1)) * elem_size(src_elem)
                            : 0;
  const int64_t batches = (P.ntiles + (1 << P.lg) - 1) >> P.lg;
  if (info)
    info->name = P.transpose ? (P.vec == 1   ? "digit_copy_transpose_v16"
                                : P.vec == 2 ? "digit_copy_transpose_st16"
                                             : "digit_copy_transpose")
                             : (P.vec ? "digit_copy_direct_v16" : "digit_copy_direct");
  return dispatch<Unused>(src_elem, dst_elem, [&](auto s, auto d) -> cudaError_t {
    using TS = decltype(s);
    using TD = decltype(d);
    using Kern = void (*)(const DCParams, const TS* __restrict__, TD* __restrict__);
    // guard/clamp mode: none, small (<= 2 + <= 2: 2-D Padding + unfold),
    // general, general + source tables (fp32 sources only)
    const int mode = P.ntab > 0 ? 3
                     : P.npred == 0 && P.nclamp == 0 ? 0
                     : (P.npred <= 2 && P.nclamp <= 2 ? 1 : 2);
    Kern k = nullptr;
    if (mode == 3) {
      if constexpr (std::is_same_v<TS, float>) {
        if (P.vec == 2) k = digit_transpose_vst<TS, TD, kMaxPred, kMaxClamp, kMaxTab>;
        else if (P.transpose) k = digit_transpose<TS, TD, kMaxPred, kMaxClamp, kMaxTab>;
        else k = digit_direct<TS, TD, kMaxPred, kMaxClamp, kMaxTab>;
      } else {
        return cudaErrorInvalidValue;
      }
    } else if (P.vec == 2)
      k = mode == 0   ? digit_transpose_vst<TS, TD, 0, 0, 0>
          : mode == 1 ? digit_transpose_vst<TS, TD, 2, 2, 0>
                      : digit_transpose_vst<TS, TD, kMaxPred, kMaxClamp, 0>;
    else if (P.vec) k = P.transpose ? digit_transpose_vec<TS, TD> : digit_direct_vec<TS, TD>;
    else if (P.transpose)
      k = mode == 0   ? digit_transpose<TS, TD, 0, 0, 0>
          : mode == 1 ? digit_transpose<TS, TD, 2, 2, 0>
                      : digit_transpose<TS, TD, kMaxPred, kMaxClamp, 0>;
    else
      k = mode == 0   ? digit_direct<TS, TD, 0, 0, 0>
          : mode == 1 ? digit_direct<TS, TD, 2, 2, 0>
                      : digit_direct<TS, TD, kMaxPred, kMaxClamp, 0>;
    // One full wave of resident CTAs (occupancy-derived), each walking tile
    // batches grid-stride: no partial second wave.
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kCopyThreads, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(batches, int64_t(nsm) * per_sm));
    if (info) info->grid = grid;
    cudaError_t le = launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(kCopyThreads), smem, stream,
                                P, static_cast<const TS*>(src), static_cast<TD*>(dst));
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
  });
}

// L2 scrub for measurements: read `bytes` (> L2) with the normal L2 policy,
// so the next timed kernel starts with a cold and clean L2 (dirty lines of
// the previous execution are written back during the scrub).
__global__ void __launch_bounds__(256) l2_touch(const int4* __restrict__ p, int64_t n, int* sink) {
  int acc = 0;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += gridDim.x * 256ll) {
    int4 v = __ldcg(p + i);  // normal L2 policy: displaces resident lines
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

cudaError_t launch_l2_touch(const void* buf, size_t bytes, int* sink, cudaStream_t stream) {
  l2_touch<<<148 * 8, 256, 0, stream>>>(static_cast<const int4*>(buf),
                                         static_cast<int64_t>(bytes / 16), sink);
  return cudaGetLastError();
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
    launch_pdl(ix_copy<TS, TD>, dim3(static_cast<unsigned>(blocks)), dim3(kCopyThreads), 0, stream,
        d_progs, n, static_cast<const TS*>(src), static_cast<TD*>(dst), d_err);
    return cudaGetLastError();
  });
}

}  // namespace lfg
