// Microbenchmark (diagnostics only): per-SM SM->L2 write rate of the three
// epilogue store paths — st.global.v4 from 8 warps, 1-D bulk copies
// (cp.async.bulk.global.shared::cta) and 2-D tensor stores
// (cp.async.bulk.tensor.2d.global.shared::cta) — one CTA per SM, each CTA
// writing its own `chunk`-byte region `iters` times. Prints B/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_rate store_rate.cu -lcuda && ./store_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256, 1) store(const __grid_constant__ CUtensorMap map, float* dst, int mode,
                                               int chunk, int nreq, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < chunk / 16; i += 256) reinterpret_cast<float4*>(smem)[i] = make_float4(1, 2, 3, 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  float* my = dst + static_cast<size_t>(blockIdx.x) * chunk / 4;
  long long t0 = clock64();
  if (mode == 0) {
    const float4 v = make_float4(threadIdx.x, 1, 2, 3);
    for (int it = 0; it < iters; ++it)
      for (int i = threadIdx.x; i < chunk / 16; i += 256) reinterpret_cast<float4*>(my)[i] = v;
    __syncthreads();
  } else if (threadIdx.x < 32 * nreq && (threadIdx.x & 31) == 0) {
    // nreq issuing warps, each writing 1/nreq of the chunk per iteration
    const int w = threadIdx.x >> 5;
    const int part = chunk / nreq;
    for (int it = 0; it < iters; ++it) {
      if (mode == 1) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<char*>(my) + w * part),
                     "r"(smem_u32(smem + w * part)), "r"(part)
                     : "memory");
      } else {
        // map: [rows][32 floats] 128-byte rows, box {32, part/128}
        const int y = (blockIdx.x * chunk + w * part) / 128;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                         reinterpret_cast<uint64_t>(&map)),
                     "r"(0), "r"(y), "r"(smem_u32(smem + w * part))
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int grid = 148;
  const size_t maxchunk = 64 << 10;
  float* dst;
  cudaMalloc(&dst, grid * maxchunk);
  long long* out;
  cudaMalloc(&out, grid * sizeof(long long));
  cudaFuncSetAttribute(store, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  printf("mode(0 stg,1 bulk,2 tensor) chunk nreq grid  B/clk/SM\n");
  for (int g : {148, 32})
    for (int mode : {0, 1, 2})
      for (int chunk : {16384, 32768, 65536})
        for (int nreq : {1, 2, 4}) {
          if (mode == 0 && nreq > 1) continue;
          CUtensorMap map;
          cuuint64_t dims[2] = {32, grid * maxchunk / 128};
          cuuint64_t strides[1] = {128};
          cuuint32_t box[2] = {32, static_cast<cuuint32_t>(std::min<int>(256, chunk / nreq / 128))};
          cuuint32_t es[2] = {1, 1};
          if (mode == 2 && chunk / nreq / 128 > 256) continue;
          enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dst, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          const int iters = 64;
          for (int rep = 0; rep < 2; ++rep) store<<<g, 256, chunk + 1024>>>(map, dst, mode, chunk, nreq, iters, out);
          if (cudaDeviceSynchronize() != cudaSuccess) {
            printf("error\n");
            return 1;
          }
          std::vector<long long> h(g);
          cudaMemcpy(h.data(), out, g * sizeof(long long), cudaMemcpyDeviceToHost);
          double mean = 0;
          for (auto v : h) mean += v;
          mean /= g;
          printf("%d %6d %d %4d %8.1f\n", mode, chunk, nreq, g, static_cast<double>(chunk) * iters / mean);
        }
  return 0;
}
