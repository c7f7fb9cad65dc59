// launch.cuh -- per-device launch-configuration cache for the persistent kernels.
// cudaFuncSetAttribute and the occupancy query are per device context, so the
// cache is indexed by the current device (a process may drive several GPUs).
#pragma once
#include <cuda_runtime.h>

namespace rpl {

constexpr int kMaxDevices = 64;

// Resident CTAs per SM of `kernel` with `threads` threads and `smem` bytes of
// dynamic shared memory (at least 1); sets the smem attribute on first use.
template <typename K>
inline int resident_ctas(K kernel, int threads, size_t smem, int* cache) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  if (!cache[dev]) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem);
    cache[dev] = v < 1 ? 1 : v;
  }
  return cache[dev];
}

inline int sm_count() {
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

}  // namespace rpl
