// Microbenchmark: cost of CTA vs cluster barriers and of DSMEM reads on this GPU
// (inputs for the cluster-pair tile design in DESIGN.md "Next").
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_bench tools/cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cta(long long* out, int iters) {
  __shared__ int s[256];
  s[threadIdx.x] = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void __cluster_dims__(2, 1, 1) k_cluster2(long long* out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void __cluster_dims__(4, 1, 1) k_cluster4(long long* out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// dependent DSMEM reads (pointer chase in the peer CTA's shared memory)
__global__ void __cluster_dims__(2, 1, 1) k_dsmem(long long* out, int iters) {
  __shared__ int buf[1024];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 33) & 1023;
  cl.sync();
  int* peer = cl.map_shared_rank(buf, cl.block_rank() ^ 1);
  int j = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) j = peer[j];
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) + (j == -1);
}

int main() {
  long long* d;
  long long h[296];
  cudaMalloc(&d, sizeof(h));
  const int it = 10000;
  auto run = [&](const char* name, void (*k)(long long*, int), int grid, int block) {
    k<<<grid, block>>>(d, it);
    k<<<grid, block>>>(d, it);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < grid; ++i) m += h[i];
    printf("%-28s grid %4d block %4d: %.1f cycles per iteration (%s)\n", name, grid, block,
           m / grid / it, cudaGetErrorString(cudaGetLastError()));
  };
  run("__syncthreads 256", k_cta, 148, 256);
  run("__syncthreads 512", k_cta, 148, 512);
  run("cluster(2) arrive+wait 256", k_cluster2, 148, 256);
  run("cluster(4) arrive+wait 256", k_cluster4, 148, 256);
  run("cluster(2) arrive+wait 512", k_cluster2, 148, 512);
  run("DSMEM dependent load", k_dsmem, 148, 32);
  return 0;
}
