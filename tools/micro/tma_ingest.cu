// Microbenchmark (diagnostics only): per-SM L2->SMEM ingest rate as a
// function of request size, requests per slot and ring depth, for 1-D bulk
// copies and 3-D tensor boxes {64 bf16 (128 B, SWIZZLE_128B), rows, kdepth}
// — the K-major UMMA operand format with `kdepth` 64-element K slabs per box.
// One CTA per SM (grid = argv), one issuing thread, an `slots`-deep ring; the
// source is a 16 MB L2-resident buffer. Prints B/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ingest tma_ingest.cu -lcuda
//   ./tma_ingest
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar),
               "r"(ph)
               : "memory");
}

// mode 0: bulk 1-D; mode 1: tensor 3-D box {64, rows, kd}
__global__ void __launch_bounds__(256, 1) ingest(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                                size_t src_bytes, int mode, int chunk, int nreq, int slots, int kd,
                                                int iters, int nprod, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w >= nprod) return;
  const int req = chunk / nreq;           // bytes per request
  const int rows = req / (128 * kd);      // tensor rows per request
  const size_t nchunks = src_bytes / chunk;
  long long t0 = 0;
  for (int it = w; it < iters + slots; it += nprod) {
    if (t0 == 0 && it >= slots) t0 = clock64();
    const int s = it % slots;
    const uint32_t bar = smem_u32(&bars[s]);
    if (it >= slots) wait(bar, ((it - slots) / slots) & 1);
    if (it < iters) {
      const size_t c = (blockIdx.x * 7 + it) % nchunks;
      const uint32_t dst = smem_u32(smem + s * chunk);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk) : "memory");
      for (int q = 0; q < nreq; ++q) {
        if (mode == 0) {
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + q * req),
              "l"(src + c * chunk + q * req), "r"(req), "r"(bar)
              : "memory");
        } else if (mode == 2) {
          const int y = static_cast<int>((c * nreq + q) * rows % (1 << 14));
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                  dst + q * req),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(y), "r"(0), "r"(0), "r"(0), "r"(bar)
              : "memory");
        } else {
          // tensor dims {64, R, KS}: element (k1, r, k0); chunk c covers rows [c*rows*nreq ...)
          const int y = static_cast<int>((c * nreq + q) * rows % (1 << 14));
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  dst + q * req),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(y), "r"(0), "r"(bar)
              : "memory");
        }
      }
    }
  }
  if (w == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = 16 << 20;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  // 16 MB as [KS=4][R=16384][64] bf16 -> dims {64, 16384, 4}
  struct Case {
    int mode, chunk, nreq, slots, kd, grid, nprod;
  };
  std::vector<Case> cases;
  for (int mode : {1, 2})
    for (int chunk : {16384, 24576, 32768})
      for (int slots : {4, 7})
        for (int nprod : {1, 2, 3})
          for (int nreq : {1, 2}) {
            if (chunk * slots > 200 * 1024) continue;
            if ((chunk / nreq) % 128 || chunk / nreq / 128 > 256) continue;
            cases.push_back({mode, chunk, nreq, slots, 1, 24, nprod});
          }
  printf("grid mode kd chunk nreq slots nprod inflight_KB  B/clk/SM  cyc/slot\n");
  for (const Case& c : cases) {
    CUtensorMap map;
    const int rows = c.chunk / c.nreq / (128 * c.kd);
    cuuint64_t dims[5] = {64, 16384, 4, 1, 1};
    cuuint64_t strides[4] = {128, 128ull * 16384, 128ull * 16384 * 4, 128ull * 16384 * 4};
    cuuint32_t box[5] = {64, static_cast<cuuint32_t>(rows), static_cast<cuuint32_t>(c.kd), 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, c.mode == 2 ? 5 : 3, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      continue;
    }
    const int iters = 256;
    for (int rep = 0; rep < 2; ++rep)
      ingest<<<c.grid, 256, c.chunk * c.slots + 1024>>>(map, src, bytes, c.mode, c.chunk, c.nreq, c.slots, c.kd, iters,
                                                       c.nprod, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<long long> h(c.grid);
    cudaMemcpy(h.data(), out, c.grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += v;
    mean /= c.grid;
    printf("%4d %4d %2d %6d %4d %5d %5d %8d %9.1f %9.0f\n", c.grid, c.mode, c.kd, c.chunk, c.nreq, c.slots, c.nprod,
           c.chunk * c.slots / 1024, static_cast<double>(c.chunk) * iters / mean, mean / iters);
  }
  return 0;
}
