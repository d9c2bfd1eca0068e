// Microbenchmark: latency of tcgen05.ld (32x32b.x16) from one warp while
// another thread keeps the tensor pipe busy with queued tcgen05.mma (M=128,
// N=64) into a disjoint TMEM region. Diagnostics only (garbage data).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ld_latency ld_latency.cu && ./ld_latency
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256, 1) ld_latency(int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ volatile int go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) go = 0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const int N = 64;
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t base = (1ull << 46) | (2ull << 61) | ((uint64_t)((1024 >> 4) & 0x3FFF) << 32) | ((uint64_t)((16 >> 4) & 0x3FFF) << 16);
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 64 * 1024;
    for (int i = 0; i < nmma; ++i) {
      const uint64_t ad = base | (((a0 + (i % 4) * 32) >> 4) & 0x3FFF), bd = base | (((b0 + (i % 4) * 32) >> 4) & 0x3FFF);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(i));
      if (i == 7) go = 1;  // let the reader start once a few MMAs are queued
    }
    if (nmma < 8) go = 1;
  }
  if (warp == 4) {
    while (go == 0) {
    }
    long long t0 = clock64();
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + 256));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    long long t1 = clock64();
    uint32_t x = 0;
    for (int j = 0; j < 16; ++j) x ^= v[j];
    if (lane == 0) out[blockIdx.x * 2] = t1 - t0;
    if (lane == 0) out[blockIdx.x * 2 + 1] = x;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * 8);
  cudaFuncSetAttribute(ld_latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int nmma : {0, 8, 16, 32, 64, 128}) {
    ld_latency<<<1, 256, 160 * 1024>>>(nmma, d);
    ld_latency<<<1, 256, 160 * 1024>>>(nmma, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("MMAs issued (N=64): %4d  tcgen05.ld x16 latency: %lld cycles  %s\n", nmma, h[0], cudaGetErrorString(e));
  }
  return 0;
}
