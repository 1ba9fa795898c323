// Measures, on the GPU, the accuracy of the fp64 value-path helpers of contract.cuh (exp64,
// rcp64) against libdevice exp() and IEEE division, over dense grids of their input ranges.
// Build/run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2602_23040_b200/csrc \
//            tools/value_path_check.cu -o /tmp/vpc && /tmp/vpc
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "contract.cuh"

using namespace puv;

__global__ void k_check(long long n, double lo, double hi, double ylo, double yhi, unsigned long long* out) {
  __shared__ double tab[kExpTab];
  exp64_table_fill(tab);
  __syncthreads();
  double emax = 0.0, rmax = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double t = (double)i / (double)(n - 1);
    const double x = lo + (hi - lo) * t;
    const double e = exp64(x, tab), ref = exp(x);
    emax = fmax(emax, fabs(e / ref - 1.0));
    const double y = ylo + (yhi - ylo) * t;
    const double r = rcp64(y);
    rmax = fmax(rmax, fabs(r * y - 1.0));
  }
  atomicMax(out + 0, __double_as_longlong(emax));   // non-negative doubles order like their bits
  atomicMax(out + 1, __double_as_longlong(rmax));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const double ranges[2][2] = {{-6.0, 0.0}, {-700.0, 0.0}};
  for (int k = 0; k < 2; ++k) {
    cudaMemset(d, 0, 16);
    k_check<<<148 * 8, 256>>>(1LL << 30, ranges[k][0], ranges[k][1], 0.01, 1.0, d);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    double e, r;
    memcpy(&e, &h[0], 8);
    memcpy(&r, &h[1], 8);
    printf("{\"exp64_range\": [%g, %g], \"exp64_max_rel_err\": %.3e, \"rcp64_range\": [0.01, 1], "
           "\"rcp64_max_rel_err\": %.3e, \"points\": %lld}\n", ranges[k][0], ranges[k][1], e, r, 1LL << 30);
  }
  return cudaGetLastError() != cudaSuccess;
}
