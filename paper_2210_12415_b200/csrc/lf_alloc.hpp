// lf_alloc.hpp — the plans' device memory: a caching allocator over
// cudaMalloc. Tuning builds and destroys a plan per candidate; a cudaMalloc /
// cudaFree pair per buffer (cudaFree synchronises the device) cost ~10 ms per
// cfg2 candidate (tools/tuner_overhead.py), more than measuring it. Freed
// blocks are kept per exact rounded size and handed to the next plan.
#pragma once

#include <cstddef>

namespace lfg {

// Device memory of at least `bytes` (256-byte aligned); nullptr on failure.
void* dev_alloc(size_t bytes);
// Return a dev_alloc block to the cache. The caller guarantees no device
// work still uses it (plans synchronise their stream before releasing).
void dev_free(void* p);
// Bytes currently held in the cache (diagnostics).
size_t dev_cached_bytes();

}  // namespace lfg
