// K14: low-precision optimisation (LPO, NEXT-2).
//
// The renderer consumes a uniformly quantised K-bit proxy theta~ of the fp32 master planes theta
// (16 bits for the position planes, 8 for scale / rotation / opacity / colour);
// gradients pass straight through (STE): the backward of the proxy render IS the master gradient.
//   k_qfit_*   per-plane (min, max) over occupied texels: per-CTA reduction,
//              one ordered-key atomicMin/atomicMax per CTA and plane (exact, order independent).
//   k_quantize per texel and plane, in the fp32 contract (DESIGN.md §13 Q1-Q3):
//              t = ((x - min) / (max - min)) * L clamped to [0, L], code = roundf(t) (half away),
//              proxy = min + (code / L) * (max - min); writes the codes (uint8 / uint16 planes,
//              the storage format) and/or the fp32 proxy planes.
#include <cuda_fp16.h>

#include "contract.cuh"
#include "internal.cuh"

namespace puv {

namespace {

PUV_DEV uint32_t fkey(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
PUV_DEV float keyf(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }

__global__ void k_qfit_init(uint32_t* __restrict__ keys, int D) {
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    keys[2 * d] = 0xffffffffu;   // min key
    keys[2 * d + 1] = 0u;        // max key
  }
}

__global__ void __launch_bounds__(256) k_qfit(PlaneTab P, const uint8_t* __restrict__ occ, int64_t N,
                                              uint32_t* __restrict__ keys, bool vec) {
  const int d = blockIdx.y;
  const float* x = P.p[d];
  if (!x) return;
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = vec ? N / 4 : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
    const uchar4 o = occ ? reinterpret_cast<const uchar4*>(occ)[i] : make_uchar4(1, 1, 1, 1);
    const float e[4] = {v.x, v.y, v.z, v.w};
    const unsigned char f[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!f[j]) continue;
      const uint32_t k = fkey(e[j]);
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    if (occ && !occ[i]) continue;
    const uint32_t k = fkey(__ldg(x + i));
    kmin = min(kmin, k);
    kmax = max(kmax, k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  __shared__ uint32_t smin[8], smax[8];
  if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = kmin; smax[threadIdx.x >> 5] = kmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) { kmin = min(kmin, smin[w]); kmax = max(kmax, smax[w]); }
    if (kmin != 0xffffffffu) atomicMin(keys + 2 * d, kmin);
    if (kmax != 0u) atomicMax(keys + 2 * d + 1, kmax);
  }
}

__global__ void k_qfit_fin(uint32_t* __restrict__ keys, int D) {
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const uint32_t a = keys[2 * d], b = keys[2 * d + 1];
    const bool empty = a == 0xffffffffu && b == 0u;
    float* f = reinterpret_cast<float*>(keys);
    f[2 * d] = empty ? 0.f : keyf(a);
    f[2 * d + 1] = empty ? 0.f : keyf(b);
  }
}

struct QPlanes {
  const float* x[kMaxPlanes];
  float* proxy[kMaxPlanes];
  void* code[kMaxPlanes];
  int8_t bits[kMaxPlanes];   // 0: plane not quantised (rho mode's unused planes 1, 2); -1: binary16
};

// 4 texels per thread (float4 / uchar4 / ushort4 accesses); N % 4 == 0 and 16-byte aligned planes.
__global__ void __launch_bounds__(256) k_quantize4(QPlanes Q, int D, const float* __restrict__ spec,
                                                   const uint8_t* __restrict__ occ, int64_t n4) {
  __shared__ float smn[kMaxPlanes], smx[kMaxPlanes];
  for (int d = threadIdx.x; d < D; d += blockDim.x) { smn[d] = spec[2 * d]; smx[d] = spec[2 * d + 1]; }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const uchar4 o = occ ? reinterpret_cast<const uchar4*>(occ)[i] : make_uchar4(1, 1, 1, 1);
    const unsigned char f[4] = {o.x, o.y, o.z, o.w};
#pragma unroll 2
    for (int d = 0; d < D; ++d) {
      const int bits = Q.bits[d];
      if (bits == 0) continue;
      const float4 v = __ldcs(reinterpret_cast<const float4*>(Q.x[d]) + i);
      const float e[4] = {v.x, v.y, v.z, v.w};
      uint32_t c[4];
      float p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (f[j]) quant1(e[j], smn[d], smx[d], bits, c[j], p[j]);
        else { c[j] = 0; p[j] = 0.f; }
      }
      if (Q.proxy[d]) __stcs(reinterpret_cast<float4*>(Q.proxy[d]) + i, make_float4(p[0], p[1], p[2], p[3]));
      if (Q.code[d]) {
        if (bits > 8 || bits < 0)
          reinterpret_cast<ushort4*>(Q.code[d])[i] = make_ushort4(c[0], c[1], c[2], c[3]);
        else
          reinterpret_cast<uchar4*>(Q.code[d])[i] = make_uchar4(c[0], c[1], c[2], c[3]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_quantize(QPlanes Q, int D, const float* __restrict__ spec,
                                                  const uint8_t* __restrict__ occ, int64_t N) {
  __shared__ float smn[kMaxPlanes], smx[kMaxPlanes];
  for (int d = threadIdx.x; d < D; d += blockDim.x) { smn[d] = spec[2 * d]; smx[d] = spec[2 * d + 1]; }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const bool on = !occ || occ[i];
    for (int d = 0; d < D; ++d) {
      const int bits = Q.bits[d];
      if (bits == 0) continue;
      uint32_t code = 0;
      float prox = 0.f;
      if (on) quant1(__ldcs(Q.x[d] + i), smn[d], smx[d], bits, code, prox);
      if (Q.proxy[d]) Q.proxy[d][i] = prox;
      if (Q.code[d]) {
        if (bits > 8 || bits < 0) static_cast<uint16_t*>(Q.code[d])[i] = (uint16_t)code;
        else static_cast<uint8_t*>(Q.code[d])[i] = (uint8_t)code;
      }
    }
  }
}

}  // namespace

void launch_quant_fit(const PlaneTab& P, int D, const uint8_t* occ, int64_t N, float* spec, cudaStream_t s) {
  uint32_t* keys = reinterpret_cast<uint32_t*>(spec);
  k_qfit_init<<<1, 64, 0, s>>>(keys, D);
  bool vec = ((uintptr_t)occ % 4) == 0;
  for (int d = 0; d < D; ++d) vec = vec && ((uintptr_t)P.p[d] % 16) == 0;
  const int64_t want = (N / 4 + 255) / 256;
  const int bx = (int)(want < 32 ? (want > 0 ? want : 1) : 32);
  k_qfit<<<dim3(bx, D), 256, 0, s>>>(P, occ, N, keys, vec);
  k_qfit_fin<<<1, 64, 0, s>>>(keys, D);
  count_launches(3);
}

void launch_quantize(const float* const* x, float* const* proxy, void* const* code, const int8_t* bits, int D,
                     const float* spec, const uint8_t* occ, int64_t N, cudaStream_t s) {
  QPlanes Q{};
  for (int d = 0; d < D; ++d) {
    Q.x[d] = x[d];
    Q.proxy[d] = proxy ? proxy[d] : nullptr;
    Q.code[d] = code ? code[d] : nullptr;
    Q.bits[d] = bits[d];
  }
  bool vec = N % 4 == 0 && ((uintptr_t)occ % 4) == 0;
  for (int d = 0; d < D; ++d)
    vec = vec && ((uintptr_t)Q.x[d] % 16) == 0 && ((uintptr_t)Q.proxy[d] % 16) == 0 && ((uintptr_t)Q.code[d] % 8) == 0;
  if (vec) {
    const int64_t want = (N / 4 + 255) / 256;
    const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
    k_quantize4<<<blocks, 256, 0, s>>>(Q, D, spec, occ, N / 4);
  } else {
    const int64_t want = (N + 255) / 256;
    const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
    k_quantize<<<blocks, 256, 0, s>>>(Q, D, spec, occ, N);
  }
  count_launches(1);
}

}  // namespace puv
