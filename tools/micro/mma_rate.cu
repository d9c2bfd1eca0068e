// Microbenchmark: tcgen05.mma issue/execute rate for M=128, N in {32..256},
// bf16 SS mode (both operands from SMEM), SWIZZLE_128B K-major descriptors.
// One CTA per SM issues `iters` MMAs into one TMEM accumulator; garbage
// data (timing only). Prints cycles per MMA. Diagnostics only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(128, 1) mma_rate(int N, int iters, int stride_kb, int swz,
                                                   unsigned long long* out, int nissue = 1, int M = 128) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[2];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot + (threadIdx.x == 32 ? 128 : 0);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0 || (threadIdx.x == 32 && nissue == 2)) {
    const uint64_t bar = reinterpret_cast<uint64_t>(&bars[threadIdx.x / 32]);
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t layout = swz == 128 ? 2 : swz == 64 ? 4 : swz == 32 ? 6 : 0;
    const uint64_t sbo = swz == 0 ? 128 : 8 * swz;
    const uint64_t lbo = swz == 0 ? 128 * 16 : 16;
    uint64_t base = (1ull << 46) | (layout << 61) | (((sbo >> 4) & 0x3FFF) << 32) | (((lbo >> 4) & 0x3FFF) << 16);
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 64 * 1024;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ao = a0 + (i % 4) * 32 + ((i / 4) % stride_kb) * 1024;
      const uint32_t bo = b0 + (i % 4) * 32;
      const uint64_t ad = base | ((ao >> 4) & 0x3FFF), bd = base | ((bo >> 4) & 0x3FFF);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(reinterpret_cast<void*>(bar))));
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(reinterpret_cast<void*>(bar))));
    t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int cfg = 0; cfg < 3; ++cfg) {
    const int nissue = cfg == 1 ? 2 : 1, M = cfg == 2 ? 64 : 128, swz = 128;
    printf("-- %d issuing thread(s), M=%d\n", nissue, M);
    for (int N : {32, 64, 128, 256}) {
      if (nissue == 2 && N > 128) continue;
      for (int grid : {1}) {
        const int iters = 4096;
        mma_rate<<<grid, 128, 200 * 1024>>>(N, iters, 8, swz, d, nissue, M);
        mma_rate<<<grid, 128, 200 * 1024>>>(N, iters, 8, swz, d, nissue, M);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < grid; ++i) avg += h[i];
        avg /= grid;
        printf("swz=%3d M=%d N=%3d grid=%3d: %.1f cycles/MMA per issuer (%.0f MAC/cycle/SM) %s\n", swz, M, N,
               grid, avg / iters, nissue * (double)M * N * 16 / (avg / iters), cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
