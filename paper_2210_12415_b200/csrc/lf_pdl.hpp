// lf_pdl.hpp — programmatic dependent launch for every kernel of a plan.
//
// A plan is a chain of dependent kernels on one stream (captured into a CUDA
// graph for measurement). Each kernel is launched with programmatic stream
// serialization and, at entry, waits for its predecessor to complete
// (griddepcontrol.wait) and lets its successor launch
// (griddepcontrol.launch_dependents). The successor's launch processing and
// CTA rasterization then overlap this kernel's tail instead of following it;
// memory visibility is unchanged (the wait returns only after the
// predecessor grid completed and flushed). LFGPU_PDL=0 turns it off.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <utility>

namespace lfg {

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("LFGPU_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

#ifdef __CUDACC__
#define LFG_PDL_ENTRY()                                         \
  do {                                                          \
    asm volatile("griddepcontrol.wait;" ::: "memory");          \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

}  // namespace lfg
