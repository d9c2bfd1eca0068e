// lf_alloc.cpp — see lf_alloc.hpp.
#include "lf_alloc.hpp"

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace lfg {

namespace {

constexpr size_t kCacheCap = size_t(8) << 30;  // beyond this, blocks go back to the driver

struct Cache {
  std::mutex m;
  std::map<std::pair<int, size_t>, std::vector<void*>> free;  // (device, size) -> blocks
  std::unordered_map<void*, std::pair<int, size_t>> live;     // block -> (device, size)
  size_t cached = 0;
};

Cache& cache() {
  static Cache* c = new Cache();  // never destroyed: blocks may outlive static teardown
  return *c;
}

size_t round_size(size_t b) {
  if (b < (size_t(1) << 20)) return (b + 255) & ~size_t(255);
  return (b + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1);
}

}  // namespace

void* dev_alloc(size_t bytes) {
  const size_t sz = round_size(bytes ? bytes : 1);
  int dev = 0;
  cudaGetDevice(&dev);
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> lk(c.m);
    auto it = c.free.find({dev, sz});
    if (it != c.free.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      c.cached -= sz;
      c.live[p] = {dev, sz};
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, sz) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(c.m);
  c.live[p] = {dev, sz};
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  Cache& c = cache();
  std::unique_lock<std::mutex> lk(c.m);
  auto it = c.live.find(p);
  if (it == c.live.end()) {  // not ours
    lk.unlock();
    cudaFree(p);
    return;
  }
  const auto key = it->second;
  c.live.erase(it);
  if (c.cached + key.second > kCacheCap) {
    lk.unlock();
    cudaFree(p);
    return;
  }
  c.free[key].push_back(p);
  c.cached += key.second;
}

size_t dev_cached_bytes() {
  std::lock_guard<std::mutex> lk(cache().m);
  return cache().cached;
}

}  // namespace lfg
