// launch.cuh -- per-device launch-configuration cache for the persistent kernels.
// cudaFuncSetAttribute and the occupancy query are per device context, so the
// cache is indexed by the current device (a process may drive several GPUs).
#pragma once
#include <stdlib.h>
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

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its stream predecessor finishes; it must execute
// `griddepcontrol.wait` before reading anything the predecessor wrote.
// RPL_PDL=0 disables it (plain stream order).
template <typename K, typename... Args>
inline cudaError_t launch_pdl(K kernel, int grid, int block, size_t smem, cudaStream_t s,
                              Args... args) {
  static const bool on = [] {
    const char* e = getenv("RPL_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

inline int sm_count() {
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

}  // namespace rpl
