// lp_launch.cpp — host-side launch helpers shared by the kernel files.
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

#include "lp_launch.h"

namespace lp {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) costs a driver call per
// use; a re-plan issues tens of histogram launches, so the opt-in is raised
// once per (device, kernel) to the largest size seen and never lowered (the
// attribute is a permission — occupancy follows the size passed at launch).
cudaError_t smem_optin(const void* fn, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  struct Key {
    int dev;
    const void* fn;
    bool operator==(const Key& o) const { return dev == o.dev && fn == o.fn; }
  };
  struct Hash {
    size_t operator()(const Key& k) const { return std::hash<const void*>()(k.fn) ^ (size_t)k.dev * 0x9e3779b97f4a7c15ull; }
  };
  static std::mutex mu;
  static std::unordered_map<Key, size_t, Hash> set;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = set[Key{dev, fn}];
  if (smem <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) cur = smem;
  return e;
}

void preload_kernels() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static std::mutex mu;
  static std::unordered_map<int, bool> done;
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return;
  done[dev] = true;
  preload_rows();
  preload_bits();
  preload_hist();
  preload_dp();
}

}  // namespace lp
