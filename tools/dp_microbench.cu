// FP64 / FP32 pipe microbenchmark on the B200 (sm_100a): throughput with many
// independent FMA chains, latency with one dependent chain, and the cost of the
// rcp.approx.f64 + Newton sequence used by the scheme.  Used to set the "alu"
// roofline in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int ILP>
__global__ void fma_tp(T* out, int iters, T a, T b) {
  T acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = (T)(threadIdx.x + i);
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == (T)-1) out[threadIdx.x] = s;
}

// packed FP32 (sm_100a FFMA2): two lanes' worth of FMA per issued instruction
template <int ILP>
__global__ void fma2_tp(float* out, int iters, float a, float b) {
  unsigned long long acc[ILP];
  const float2 av = make_float2(a, a), bv = make_float2(b, b);
  const unsigned long long A = *reinterpret_cast<const unsigned long long*>(&av);
  const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    const float2 v = make_float2((float)(threadIdx.x + i), (float)i);
    acc[i] = *reinterpret_cast<const unsigned long long*>(&v);
  }
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    const float2 v = *reinterpret_cast<const float2*>(&acc[i]);
    s += v.x + v.y;
  }
  if (s == -1.0f) out[threadIdx.x] = s;
}

__global__ void rcp_tp(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i]));
      double e = fma(-x[i], r, 1.0);
      x[i] = fma(r, fma(e, e, e), r) + 1.0;
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == -1) out[threadIdx.x] = s;
}

template <typename T>
__global__ void fma_lat(T* out, int iters, long long* cyc, T a, T b) {
  T x = (T)threadIdx.x;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == (T)-1) out[0] = x;
}

int main() {
  double* d;
  float* f;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&f, 1 << 20);
  cudaMalloc(&c, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    fma_tp<double, 8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * iters * 8;
    if (rep) printf("fp64 FMA: %.1f TFLOP/s  (%.2f lane-FMA/clk/SM at 1.965 GHz)\n", flops / ms / 1e9,
                    flops / 2 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0);
    fma_tp<float, 8><<<blocks, threads>>>(f, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("fp32 FMA: %.1f TFLOP/s  (%.2f lane-FMA/clk/SM)\n", flops / ms / 1e9,
                    flops / 2 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0);
    fma2_tp<8><<<blocks, threads>>>(f, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("fp32x2 FFMA2: %.1f TFLOP/s  (%.2f lane-FMA/clk/SM, %.2f FFMA2 warp-instr/clk/SM)\n",
                    2 * flops / ms / 1e9, flops / (ms * 1e-3) / sms / 1.965e9,
                    flops / (ms * 1e-3) / sms / 1.965e9 / 64);
    cudaEventRecord(e0);
    rcp_tp<<<blocks, threads>>>(d, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double nrcp = 1.0 * blocks * threads * (iters / 4) * 8;
    if (rep) printf("rcp64 (MUFU+3 DFMA+DADD): %.2f G/s  (%.2f per clk per SM)\n", nrcp / ms / 1e6,
                    nrcp / (ms * 1e-3) / sms / 1.965e9);
  }
  long long h;
  fma_lat<double><<<1, 32>>>(d, 4096, c, 1.0000001, 1e-9);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 DFMA dependent latency: %.2f cycles\n", h / 4096.0);
  fma_lat<float><<<1, 32>>>(f, 4096, c, 1.0000001f, 1e-9f);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp32 FFMA dependent latency: %.2f cycles\n", h / 4096.0);
  return 0;
}
