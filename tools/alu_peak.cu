// alu_peak.cu — measured FP64 / FP32 FMA throughput on the current GPU (roofline denominators for
// the ALU-bound raster kernels).  Many independent FMA chains per thread, grid of
// 8 CTAs/SM x 256 threads; prints lane-FMA/s and FLOP/s.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/alu_peak.cu -o /tmp/alu_peak && /tmp/alu_peak
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void k_fma(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)-1.2345) out[0] = s;
}

template <typename T>
double run(int nsm) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  constexpr int CH = 8;
  k_fma<T, CH><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_fma<T, CH><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double fmas = 5.0 * blocks * threads * (double)iters * CH;
  return fmas / (ms * 1e-3);
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double f64 = run<double>(nsm), f32 = run<float>(nsm);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"fp64_fma_per_s\": %.4e, \"fp32_fma_per_s\": %.4e, "
         "\"fp64_lanes_per_sm_clk\": %.1f, \"fp32_lanes_per_sm_clk\": %.1f}\n",
         nsm, clk, f64, f32, f64 / (nsm * clk * 1e3), f32 / (nsm * clk * 1e3));
  return 0;
}
