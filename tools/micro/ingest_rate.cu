// Microbenchmark: per-SM L2->SMEM ingest with 1-D bulk copies
// (cp.async.bulk, contiguous chunks) versus 2-D tensor TMA boxes of
// 128-byte rows (SWIZZLE_128B, the UMMA K-major operand format), one box or
// three boxes per slot. One CTA per SM streams a 4 MB L2-resident buffer
// through an 8-slot ring of CHUNK bytes. Diagnostics only; see DESIGN.md
// §4.3 for the readings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ingest_rate ingest_rate.cu -lcuda && ./ingest_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ int g_spin;  // 1: mbarrier.test_wait busy poll, 0: try_wait
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  if (false)
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar), "r"(ph) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}

template <int MODE>  // 0: bulk 1-D, 1: tensor 2-D box {64 bf16, rows}
__global__ void __launch_bounds__(32, 1) ingest(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                                size_t src_bytes, int chunk, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8];
  const int slots = 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const int rows = chunk / 128;
  const int nbox = g_spin ? 3 : 1;  // read once: a per-iteration global load would serialise issue
  const size_t nchunks = src_bytes / chunk;
  long long t0 = clock64();
  for (int it = 0; it < iters + slots; ++it) {
    const int s = it % slots;
    const uint32_t bar = smem_u32(&bars[s]);
    if (it >= slots) wait(bar, ((it - slots) / slots) & 1);
    if (it < iters) {
      const size_t c = (blockIdx.x * 7 + it) % nchunks;
      const uint32_t dst = smem_u32(smem + s * chunk);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk) : "memory");
      if (MODE == 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(src + c * chunk), "r"(chunk), "r"(bar)
                     : "memory");
      } else {
        // g_spin: the slot as three boxes of rows/3 (the GEMM's 2 A + 1 B boxes)
        const int r = rows / nbox;
        for (int q = 0; q < nbox; ++q) {
          const int y = static_cast<int>(c * rows) + q * r;
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + q * r * 128),
                       "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(y), "r"(bar)
                       : "memory");
        }
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x] = t1 - t0;
}

int main() {
  const size_t bytes = 4 << 20;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  for (int spin = 0; spin < 2; ++spin) {
  cudaMemcpyToSymbol(g_spin, &spin, sizeof(int));
  printf("-- %s\n", spin ? "tensor: three boxes per slot" : "one box per slot");
  for (int chunk : {24576}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {64, bytes / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(chunk / 128 / (spin ? 3 : 1))}, es[2] = {1, 1};
    if (chunk / 128 > 256) continue;
    ((Enc)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 0; mode < 2; ++mode)
      for (int grid : {148}) {
        const int iters = 512;
        auto k = mode == 0 ? ingest<0> : ingest<1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int rep = 0; rep < 2; ++rep) k<<<grid, 32, 8 * chunk>>>(map, src, bytes, chunk, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < grid; ++i) avg += h[i];
        avg /= grid;
        printf("%s chunk=%5d grid=%3d: %.1f B/clk/SM  %s\n", mode == 0 ? "bulk  " : "tensor", chunk, grid,
               static_cast<double>(iters) * chunk / avg, cudaGetErrorString(e));
      }
  }
  }
  return 0;
}
