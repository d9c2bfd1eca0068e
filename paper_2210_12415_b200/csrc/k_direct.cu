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
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

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

// ---- K6: depthwise (DEP) -----------------------------------------------
// K > 0: square KxK window unrolled with its offsets in registers; K == 0:
// any window through the tables.
template <int K>
__global__ void __launch_bounds__(256) dep_direct(const DirectDep P) {
  LFG_PDL_ENTRY();
  const int64_t total = static_cast<int64_t>(P.N) * P.C * P.Ho * P.Wo;
  const int64_t* xt = P.xt;
  const int64_t* wt = P.wt;
  const int64_t* ot = P.ot;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e;
    int n, c, h, w;
    if (P.fast == 1) {  // (c, w, h, n) from fastest to slowest
      c = static_cast<int>(r % P.C), r /= P.C;
      w = static_cast<int>(r % P.Wo), r /= P.Wo;
      h = static_cast<int>(r % P.Ho), n = static_cast<int>(r / P.Ho);
    } else {  // (w, h, c, n)
      w = static_cast<int>(r % P.Wo), r /= P.Wo;
      h = static_cast<int>(r % P.Ho), r /= P.Ho;
      c = static_cast<int>(r % P.C), n = static_cast<int>(r / P.C);
    }
    const int64_t xb = __ldg(xt + P.x_off[0] + n) + __ldg(xt + P.x_off[1] + c);
    const int64_t wb = __ldg(wt + P.w_off[0] + c);
    const int64_t* xh = xt + P.x_off[2] + static_cast<int64_t>(P.V) * h;
    const int64_t* xw = xt + P.x_off[3] + static_cast<int64_t>(P.V) * w;
    float acc = 0.f;
    if constexpr (K > 0) {
      int64_t ow[K], kw[K];
#pragma unroll
      for (int j = 0; j < K; ++j) ow[j] = __ldg(xw + j), kw[j] = __ldg(wt + P.w_off[2] + j);
#pragma unroll
      for (int rh = 0; rh < K; ++rh) {
        const int64_t oh = xb + __ldg(xh + rh), kh = wb + __ldg(wt + P.w_off[1] + rh);
#pragma unroll
        for (int rw = 0; rw < K; ++rw) acc = fmaf(__ldg(P.x + oh + ow[rw]), __ldg(P.w + kh + kw[rw]), acc);
      }
    } else {
      for (int rh = 0; rh < P.KH; ++rh) {
        const int64_t oh = xb + __ldg(xh + rh), kh = wb + __ldg(wt + P.w_off[1] + rh);
        for (int rw = 0; rw < P.KW; ++rw)
          acc = fmaf(__ldg(P.x + oh + __ldg(xw + rw)), __ldg(P.w + kh + __ldg(wt + P.w_off[2] + rw)), acc);
      }
    }
    const int64_t off = __ldg(ot + P.o_off[0] + n) + __ldg(ot + P.o_off[1] + c) +
                        __ldg(ot + P.o_off[2] + h) + __ldg(ot + P.o_off[3] + w);
    for (int k = 0; k < P.nepi; ++k) {
      if (P.epi_kind[k] == DIRECT_EPI_BIAS) acc += __ldg(P.epi_ptr[k] + c);
      else if (P.epi_kind[k] == DIRECT_EPI_RESIDUAL) acc += __ldg(P.epi_ptr[k] + off);
      else acc = acc > 0.f ? acc : 0.f;
    }
    P.out[off] = acc;
  }
}

// Channel-vectorised K6: four consecutive channels per thread as float4
// (channel-brick layouts: C is unit-stride in 4-aligned groups in the input,
// the weights and the output, every other table entry a multiple of 4), and
// a strip of WS outputs along W per thread so each input column and each
// table entry is loaded once per strip instead of once per tap.
template <int K, int V, int WS>
__global__ void __launch_bounds__(256, (K == 3 ? 3 : 2)) dep_direct4(const DirectDep P) {
  LFG_PDL_ENTRY();
  constexpr int NC = (WS - 1) * V + K;  // input columns a strip touches
  const int C4 = P.C >> 2, WSN = (P.Wo + WS - 1) / WS;
  const int64_t total = static_cast<int64_t>(P.N) * C4 * P.Ho * WSN;
  const int64_t* xt = P.xt;
  const int64_t* wt = P.wt;
  const int64_t* ot = P.ot;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e;
    const int c = static_cast<int>(r % C4) * 4;
    r /= C4;
    const int w0 = static_cast<int>(r % WSN) * WS;
    r /= WSN;
    const int h = static_cast<int>(r % P.Ho), n = static_cast<int>(r / P.Ho);
    const int64_t xb = __ldg(xt + P.x_off[0] + n) + __ldg(xt + P.x_off[1] + c);
    const int64_t wb = __ldg(wt + P.w_off[0] + c);
    const int64_t* xh = xt + P.x_off[2] + static_cast<int64_t>(V) * h;
    // Columns past the padded input (a ragged last strip) read column 0:
    // their outputs are not stored.
    const int Wi = (P.Wo - 1) * V + K;
    int64_t oc[NC], kw[K];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int col = w0 * V + j;
      oc[j] = __ldg(xt + P.x_off[3] + (col < Wi ? col : 0));
    }
#pragma unroll
    for (int j = 0; j < K; ++j) kw[j] = __ldg(wt + P.w_off[2] + j);
    float4 acc[WS];
#pragma unroll
    for (int o = 0; o < WS; ++o) acc[o] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int rh = 0; rh < K; ++rh) {
      const int64_t oh = xb + __ldg(xh + rh), kh = wb + __ldg(wt + P.w_off[1] + rh);
      float4 wv[K];
#pragma unroll
      for (int rw = 0; rw < K; ++rw) wv[rw] = __ldg(reinterpret_cast<const float4*>(P.w + kh + kw[rw]));
      float4 xv[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) xv[j] = __ldg(reinterpret_cast<const float4*>(P.x + oh + oc[j]));
      // (rh, rw) order per output, as interp.cpp:90-108 accumulates.
#pragma unroll
      for (int o = 0; o < WS; ++o)
#pragma unroll
        for (int rw = 0; rw < K; ++rw) {
          const float4 a = xv[o * V + rw], b = wv[rw];
          acc[o].x = fmaf(a.x, b.x, acc[o].x);
          acc[o].y = fmaf(a.y, b.y, acc[o].y);
          acc[o].z = fmaf(a.z, b.z, acc[o].z);
          acc[o].w = fmaf(a.w, b.w, acc[o].w);
        }
    }
    const int64_t ob = __ldg(ot + P.o_off[0] + n) + __ldg(ot + P.o_off[1] + c) + __ldg(ot + P.o_off[2] + h);
#pragma unroll
    for (int o = 0; o < WS; ++o) {
      const bool live = w0 + o < P.Wo;
      const int64_t off = ob + __ldg(ot + P.o_off[3] + (live ? w0 + o : 0));
      float4 v = acc[o];
      for (int k = 0; k < P.nepi; ++k) {
        if (P.epi_kind[k] == DIRECT_EPI_RELU) {
          v.x = fmaxf(v.x, 0.f), v.y = fmaxf(v.y, 0.f), v.z = fmaxf(v.z, 0.f), v.w = fmaxf(v.w, 0.f);
        } else {
          const float* ep = P.epi_ptr[k];
          const float4 b = P.epi_kind[k] == DIRECT_EPI_BIAS
                               ? make_float4(__ldg(ep + c), __ldg(ep + c + 1), __ldg(ep + c + 2), __ldg(ep + c + 3))
                               : __ldg(reinterpret_cast<const float4*>(ep + off));
          v.x += b.x, v.y += b.y, v.z += b.z, v.w += b.w;
        }
      }
      if (live) *reinterpret_cast<float4*>(P.out + off) = v;
    }
  }
}

// K6 with a rolling window over TR output rows per thread (K = 3): each
// input row of the strip is loaded once and feeds every output row whose
// window covers it, so a thread reads (TR-1)*V+K input rows for TR output
// rows instead of K per row. Per output the FMAs run rh-major, rw-minor,
// exactly as dep_direct4 and interp.cpp:90-108 — bit-identical results.
template <int K, int V, int WS, int TR, int MINB>
__global__ void __launch_bounds__(256, MINB) dep_direct4_rows(const DirectDep P) {
  constexpr int NC = (WS - 1) * V + K;
  constexpr int NR = (TR - 1) * V + K;  // input rows a task touches
  const int C4 = P.C >> 2, WSN = (P.Wo + WS - 1) / WS, HB = (P.Ho + TR - 1) / TR;
  const int64_t total = static_cast<int64_t>(P.N) * C4 * HB * WSN;
  const int64_t* xt = P.xt;
  const int64_t* wt = P.wt;
  const int64_t* ot = P.ot;
  const int Wi = (P.Wo - 1) * V + K, Hi = (P.Ho - 1) * V + K;
  LFG_PDL_ENTRY();
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e;
    const int c = static_cast<int>(r % C4) * 4;
    r /= C4;
    const int w0 = static_cast<int>(r % WSN) * WS;
    r /= WSN;
    const int h0 = static_cast<int>(r % HB) * TR, n = static_cast<int>(r / HB);
    const int64_t xb = __ldg(xt + P.x_off[0] + n) + __ldg(xt + P.x_off[1] + c);
    const int64_t wb = __ldg(wt + P.w_off[0] + c);
    int64_t oc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int col = w0 * V + j;
      oc[j] = __ldg(xt + P.x_off[3] + (col < Wi ? col : 0));
    }
    float4 wv[K][K];
#pragma unroll
    for (int rh = 0; rh < K; ++rh) {
      const int64_t kh = wb + __ldg(wt + P.w_off[1] + rh);
#pragma unroll
      for (int rw = 0; rw < K; ++rw) wv[rh][rw] = __ldg(reinterpret_cast<const float4*>(P.w + kh + __ldg(wt + P.w_off[2] + rw)));
    }
    float4 acc[TR][WS];
#pragma unroll
    for (int o = 0; o < TR; ++o)
#pragma unroll
      for (int q = 0; q < WS; ++q) acc[o][q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int ir = 0; ir < NR; ++ir) {
      const int row = h0 * V + ir;
      const int64_t oh = xb + __ldg(xt + P.x_off[2] + (row < Hi ? row : 0));
      float4 xv[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) xv[j] = __ldg(reinterpret_cast<const float4*>(P.x + oh + oc[j]));
#pragma unroll
      for (int o = 0; o < TR; ++o) {
        const int rh = ir - o * V;
        if (rh < 0 || rh >= K) continue;  // resolved at compile time (unrolled)
#pragma unroll
        for (int q = 0; q < WS; ++q)
#pragma unroll
          for (int rw = 0; rw < K; ++rw) {
            const float4 a = xv[q * V + rw], b = wv[rh][rw];
            acc[o][q].x = fmaf(a.x, b.x, acc[o][q].x);
            acc[o][q].y = fmaf(a.y, b.y, acc[o][q].y);
            acc[o][q].z = fmaf(a.z, b.z, acc[o][q].z);
            acc[o][q].w = fmaf(a.w, b.w, acc[o][q].w);
          }
      }
    }
#pragma unroll
    for (int o = 0; o < TR; ++o) {
      const int h = h0 + o;
      if (h >= P.Ho) continue;
      const int64_t ob = __ldg(ot + P.o_off[0] + n) + __ldg(ot + P.o_off[1] + c) + __ldg(ot + P.o_off[2] + h);
#pragma unroll
      for (int q = 0; q < WS; ++q) {
        const bool live = w0 + q < P.Wo;
        const int64_t off = ob + __ldg(ot + P.o_off[3] + (live ? w0 + q : 0));
        float4 v = acc[o][q];
        for (int k = 0; k < P.nepi; ++k) {
          if (P.epi_kind[k] == DIRECT_EPI_RELU) {
            v.x = fmaxf(v.x, 0.f), v.y = fmaxf(v.y, 0.f), v.z = fmaxf(v.z, 0.f), v.w = fmaxf(v.w, 0.f);
          } else {
            const float* ep = P.epi_ptr[k];
            const float4 b = P.epi_kind[k] == DIRECT_EPI_BIAS
                                 ? make_float4(__ldg(ep + c), __ldg(ep + c + 1), __ldg(ep + c + 2), __ldg(ep + c + 3))
                                 : __ldg(reinterpret_cast<const float4*>(ep + off));
            v.x += b.x, v.y += b.y, v.z += b.z, v.w += b.w;
          }
        }
        if (live) *reinterpret_cast<float4*>(P.out + off) = v;
      }
    }
  }
}

template <int K, int V>
static void launch_dep4(const DirectDep& P, unsigned grid, cudaStream_t stream) {
  launch_pdl(dep_direct4<K, V, 2>, dim3(grid), dim3(256), 0, stream, P);
}

cudaError_t launch_dep_direct(const DirectDep& P, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(P.N) * P.C * P.Ho * P.Wo;
  if (total == 0) return cudaSuccess;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  }
  // Grid: enough 256-thread blocks for one output each, capped at 8 waves
  // of 148 SMs x 8 resident blocks (grid-stride beyond).
  const int64_t want = (total + 255) / 256;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(sms) * 8 * 8));
  const bool sq = P.KH == P.KW;
  if (P.vec4 && sq && (P.KH == 3 || P.KH == 5 || P.KH == 7) && (P.V == 1 || P.V == 2)) {
    const int ws = 2;
    const int64_t strips = static_cast<int64_t>(P.N) * (P.C / 4) * P.Ho * ((P.Wo + ws - 1) / ws);
    const unsigned g4 = static_cast<unsigned>(std::min<int64_t>((strips + 255) / 256,
                                                                static_cast<int64_t>(sms) * 64));
    static const int tr = getenv("LFGPU_DEP_ROWS") ? atoi(getenv("LFGPU_DEP_ROWS")) : 8;
    if (P.KH == 3 && tr > 1) {  // rolling window over output rows
      const int wq = 2;
      const int64_t tasks = static_cast<int64_t>(P.N) * (P.C / 4) * ((P.Ho + tr - 1) / tr) * ((P.Wo + wq - 1) / wq);
      const unsigned gt = static_cast<unsigned>(std::min<int64_t>((tasks + 255) / 256, static_cast<int64_t>(sms) * 64));
      if (P.V == 1) {
        if (tr >= 8) launch_pdl(dep_direct4_rows<3, 1, 2, 8, 2>, dim3(gt), dim3(256), 0, stream, P);
        else launch_pdl(dep_direct4_rows<3, 1, 2, 4, 2>, dim3(gt), dim3(256), 0, stream, P);
      } else {
        launch_pdl(dep_direct4_rows<3, 2, 2, 4, 2>, dim3(gt), dim3(256), 0, stream, P);
      }
      return cudaGetLastError();
    }
    if (P.V == 1) {
      if (P.KH == 3) launch_dep4<3, 1>(P, g4, stream);
      else if (P.KH == 5) launch_dep4<5, 1>(P, g4, stream);
      else launch_dep4<7, 1>(P, g4, stream);
    } else {
      if (P.KH == 3) launch_dep4<3, 2>(P, g4, stream);
      else if (P.KH == 5) launch_dep4<5, 2>(P, g4, stream);
      else launch_dep4<7, 2>(P, g4, stream);
    }
    return cudaGetLastError();
  }
  if (sq && P.KH == 3) launch_pdl(dep_direct<3>, dim3(grid), dim3(256), 0, stream, P);
  else if (sq && P.KH == 5) launch_pdl(dep_direct<5>, dim3(grid), dim3(256), 0, stream, P);
  else if (sq && P.KH == 7) launch_pdl(dep_direct<7>, dim3(grid), dim3(256), 0, stream, P);
  else launch_pdl(dep_direct<0>, dim3(grid), dim3(256), 0, stream, P);
  return cudaGetLastError();
}

// ---- im2col for the tensor-core stem ----------------------------------------
// One thread per (pixel m, 64-wide k block): lanes take consecutive pixels,
// so each x read of a warp is one strided run of a row (coalesced), and the
// thread writes its pixel's whole 128-byte brick row as eight 16-byte
// stores. (k -> (i, rh, rw) is stepped incrementally, no divisions.)
__global__ void __launch_bounds__(256) im2col_stem(const Im2col Q) {
  LFG_PDL_ENTRY();
  const int kb_n = Q.Kp / 64, hw = Q.Ho * Q.Wo;
  const int64_t M = static_cast<int64_t>(Q.N) * hw;
  const int64_t na = M * kb_n, nb = static_cast<int64_t>(Q.O) * (Q.Kp / 8);
  __nv_bfloat16* A = static_cast<__nv_bfloat16*>(Q.a);
  __nv_bfloat16* B = static_cast<__nv_bfloat16*>(Q.b);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < na + nb;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    __align__(16) __nv_bfloat16 v[8];
    if (e < na) {
      const int kb = static_cast<int>(e / M);
      const int64_t m = e - static_cast<int64_t>(kb) * M;
      const int n = static_cast<int>(m / hw), rem = static_cast<int>(m - static_cast<int64_t>(n) * hw);
      const int ho = rem / Q.Wo, wo = rem - ho * Q.Wo;
      // Window origin in x; with an absorbed Padding (Q.pad > 0) taps
      // outside x read as zero (interp.cpp:123-136).
      const int y0 = ho * Q.V - Q.pad, x0 = wo * Q.V - Q.pad;
      const float* xb = Q.x + static_cast<int64_t>(n) * Q.I * Q.H * Q.W;
      int k = kb * 64;
      int i = k / (Q.KH * Q.KW), r = k - i * Q.KH * Q.KW, rh = r / Q.KW, rw = r - rh * Q.KW;
      const int64_t mt = m / Q.RT;
      __nv_bfloat16* dst = A + (mt * kb_n + kb) * (static_cast<int64_t>(Q.RT) * 64) + (m - mt * Q.RT) * 64;
#pragma unroll 1
      for (int g = 0; g < 8; ++g) {
#pragma unroll
        for (int j = 0; j < 8; ++j, ++k) {
          float x = 0.f;
          const int yy = y0 + rh, xx = x0 + rw;
          if (k < Q.K && yy >= 0 && yy < Q.H && xx >= 0 && xx < Q.W)
            x = __ldg(xb + (static_cast<int64_t>(i) * Q.H + yy) * Q.W + xx);
          v[j] = __float2bfloat16_rn(x);
          if (++rw == Q.KW) {
            rw = 0;
            if (++rh == Q.KH) rh = 0, ++i;
          }
        }
        reinterpret_cast<uint4*>(dst)[g] = *reinterpret_cast<const uint4*>(v);
      }
    } else {  // B[o][k0..k0+8) as [K0][O][64]
      const int64_t f = e - na;
      const int o = static_cast<int>(f / (Q.Kp / 8)), k0 = static_cast<int>(f - static_cast<int64_t>(o) * (Q.Kp / 8)) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j;
        v[j] = __float2bfloat16_rn(k < Q.K ? __ldg(Q.w + static_cast<int64_t>(o) * Q.K + k) : 0.f);
      }
      *reinterpret_cast<uint4*>(B + (static_cast<int64_t>(k0 >> 6) * Q.O + o) * 64 + (k0 & 63)) =
          *reinterpret_cast<const uint4*>(v);
    }
  }
}

// im2col by tiles: one CTA per A brick of RT pixels = RT / Wo whole output
// rows. The input rows the tile's windows touch (zero-padded) are staged in
// SMEM with coalesced loads, a per-k offset table maps k -> (i, rh, rw), and
// the brick is written as consecutive 16-byte chunks (a warp stores 512
// contiguous bytes). The trailing CTAs convert the weights as before.
// Same values as im2col_stem (bf16 of the same fp32 element, zeros outside).
__global__ void __launch_bounds__(256) im2col_tiles(const Im2col Q, int tiles) {
  extern __shared__ __align__(16) float xs[];  // [I][rows][Wp], then int koff[Kp]
  const int r = Q.RT / Q.Wo, rows = (r - 1) * Q.V + Q.KH, Wp = Q.W + 2 * Q.pad;
  int* koff = reinterpret_cast<int*>(xs + static_cast<size_t>(Q.I) * rows * Wp);
  const int kb_n = Q.Kp / 64;
  if (static_cast<int>(blockIdx.x) >= tiles) {  // weights: B[o][k0..k0+8) as [K0][O][64]
    LFG_PDL_ENTRY();
    __nv_bfloat16* B = static_cast<__nv_bfloat16*>(Q.b);
    const int64_t nb = static_cast<int64_t>(Q.O) * (Q.Kp / 8);
    for (int64_t f = (blockIdx.x - tiles) * 256ll + threadIdx.x; f < nb; f += (gridDim.x - tiles) * 256ll) {
      __align__(16) __nv_bfloat16 v[8];
      const int o = static_cast<int>(f / (Q.Kp / 8)), k0 = static_cast<int>(f - static_cast<int64_t>(o) * (Q.Kp / 8)) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j;
        v[j] = __float2bfloat16_rn(k < Q.K ? __ldg(Q.w + static_cast<int64_t>(o) * Q.K + k) : 0.f);
      }
      *reinterpret_cast<uint4*>(B + (static_cast<int64_t>(k0 >> 6) * Q.O + o) * 64 + (k0 & 63)) =
          *reinterpret_cast<const uint4*>(v);
    }
    return;
  }
  const int mt = blockIdx.x;  // tile: pixels [mt*RT, (mt+1)*RT) = output rows of image n
  const int64_t m0 = static_cast<int64_t>(mt) * Q.RT;
  const int n = static_cast<int>(m0 / (static_cast<int64_t>(Q.Ho) * Q.Wo));
  const int ho0 = static_cast<int>((m0 - static_cast<int64_t>(n) * Q.Ho * Q.Wo) / Q.Wo);
  const int y0 = ho0 * Q.V - Q.pad;  // first input row staged
  for (int k = threadIdx.x; k < Q.Kp; k += 256) {  // k -> (i, rh, rw) offset in xs
    if (k < Q.K) {
      const int i = k / (Q.KH * Q.KW), rr = k - i * Q.KH * Q.KW, rh = rr / Q.KW, rw = rr - rh * Q.KW;
      koff[k] = (i * rows + rh) * Wp + rw;
    } else {
      koff[k] = -1;
    }
  }
  LFG_PDL_ENTRY();
  const float* xb = Q.x + static_cast<int64_t>(n) * Q.I * Q.H * Q.W;
  // stage the input rows: warp w takes lines (channel, row) w, w + 8, ...,
  // its lanes the columns, all of a line's loads in flight before the stores
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ir = warp; ir < Q.I * rows; ir += 8) {
    const int i = ir / rows, yy = y0 + ir - i * rows;
    float* line = xs + static_cast<size_t>(ir) * Wp;
    const bool yin = yy >= 0 && yy < Q.H;
    const float* src = xb + (static_cast<int64_t>(i) * Q.H + (yin ? yy : 0)) * Q.W - Q.pad;
    constexpr int kQ = 8;  // 256 columns per pass
    for (int c0 = 0; c0 < Wp; c0 += 32 * kQ) {
      float v[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int cc = c0 + lane + 32 * q, xx = cc - Q.pad;
        v[q] = yin && cc < Wp && xx >= 0 && xx < Q.W ? __ldg(src + cc) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        if (c0 + lane + 32 * q < Wp) line[c0 + lane + 32 * q] = v[q];
    }
  }
  __syncthreads();
  // thread: 16-byte chunk c8 of pixels p, p + 32, ...; per K brick the
  // warp's stores cover 4 pixels x 128 contiguous bytes
  __nv_bfloat16* A = static_cast<__nv_bfloat16*>(Q.a) + static_cast<int64_t>(mt) * kb_n * Q.RT * 64;
  const int c8 = threadIdx.x & 7;
  for (int kb = 0; kb < kb_n; ++kb) {
    int ko[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ko[j] = koff[kb * 64 + c8 * 8 + j];
    uint4* dst = reinterpret_cast<uint4*>(A + static_cast<int64_t>(kb) * Q.RT * 64) + c8;
    int pr = (threadIdx.x >> 3) / Q.Wo, pc = (threadIdx.x >> 3) - pr * Q.Wo;  // pixel p -> (row, col), stepped
    for (int p = threadIdx.x >> 3; p < Q.RT; p += 32) {
      const float* b = xs + pr * Q.V * Wp + pc * Q.V;
      pc += 32;
      while (pc >= Q.Wo) pc -= Q.Wo, ++pr;
      __align__(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __float2bfloat16_rn(ko[j] >= 0 ? b[ko[j]] : 0.f);
      dst[p * 8] = *reinterpret_cast<const uint4*>(v);
    }
  }
}

cudaError_t launch_im2col(const Im2col& Q, cudaStream_t stream) {
  if (Q.RT % Q.Wo == 0 && !getenv("LFGPU_IM2COL_FLAT")) {
    const int r = Q.RT / Q.Wo, rows = (r - 1) * Q.V + Q.KH, Wp = Q.W + 2 * Q.pad;
    const size_t smem = sizeof(float) * static_cast<size_t>(Q.I) * rows * Wp + sizeof(int) * Q.Kp;
    if (smem <= 200 * 1024) {
      static bool attr_set = false;
      if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(im2col_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
      }
      const int64_t tiles = static_cast<int64_t>(Q.N) * Q.Ho * Q.Wo / Q.RT;
      const int64_t nb = static_cast<int64_t>(Q.O) * (Q.Kp / 8);
      const int bblocks = static_cast<int>(std::min<int64_t>((nb + 255) / 256, 64));
      launch_pdl(im2col_tiles, dim3(static_cast<unsigned>(tiles + bblocks)), dim3(256), smem, stream, Q,
                 static_cast<int>(tiles));
      return cudaGetLastError();
    }
  }
  const int64_t total = static_cast<int64_t>(Q.N) * Q.Ho * Q.Wo * (Q.Kp / 64) + static_cast<int64_t>(Q.O) * (Q.Kp / 8);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 64));
  launch_pdl(im2col_stem, dim3(grid), dim3(256), 0, stream, Q);
  return cudaGetLastError();
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
