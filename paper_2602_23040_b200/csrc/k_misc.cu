// K9 pack/unpack of atlas levels (R15) and K10 the L2 loss gradient (R11).
#include "contract.cuh"
#include "internal.cuh"

namespace puv {

struct LevelPtrs { const float* p[kMaxPlanes]; };
struct AtlasPtrs { float* p[kMaxPlanes]; };

__global__ void k_pack_level(LevelPtrs src, const uint8_t* __restrict__ socc, AtlasPtrs dst, uint8_t* __restrict__ docc,
                             int D, int rows, int cols, int x, int y, int rot, int WA) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int r = idx / cols, c = idx - r * cols;
  const int ay = rot ? y + cols - 1 - c : y + r;
  const int ax = rot ? x + r : x + c;
  const size_t o = (size_t)ay * WA + ax;
  for (int d = 0; d < D; ++d) dst.p[d][o] = src.p[d][idx];
  docc[o] = socc ? socc[idx] : (uint8_t)1;
}

__global__ void k_unpack_level(AtlasPtrs dstlv /*level planes*/, LevelPtrs src /*atlas planes*/, int D, int rows,
                               int cols, int x, int y, int rot, int WA) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int r = idx / cols, c = idx - r * cols;
  const int ay = rot ? y + cols - 1 - c : y + r;
  const int ax = rot ? x + r : x + c;
  const size_t o = (size_t)ay * WA + ax;
  for (int d = 0; d < D; ++d) dstlv.p[d][idx] = src.p[d][o];
}

void launch_pack(const puv_layout& L, const float* const* level_planes, const uint8_t* const* level_occ,
                 float* const* atlas_planes, uint8_t* atlas_occ, cudaStream_t s) {
  const size_t NA = (size_t)L.atlas_w * L.atlas_h;
  for (int d = 0; d < L.planes; ++d) cudaMemsetAsync(atlas_planes[d], 0, NA * 4, s);
  cudaMemsetAsync(atlas_occ, 0, NA, s);
  AtlasPtrs dst{};
  for (int d = 0; d < L.planes; ++d) dst.p[d] = atlas_planes[d];
  for (int k = 0; k < L.num_levels; ++k) {
    const puv_placement& pl = L.level[k];
    LevelPtrs src{};
    for (int d = 0; d < L.planes; ++d) src.p[d] = level_planes[(size_t)k * L.planes + d];
    const int n = pl.rows * pl.cols;
    k_pack_level<<<(n + 255) / 256, 256, 0, s>>>(src, level_occ ? level_occ[k] : nullptr, dst, atlas_occ, L.planes,
                                                 pl.rows, pl.cols, pl.x, pl.y, pl.rot90ccw, L.atlas_w);
  }
  count_launches(L.num_levels);
}

void launch_unpack(const puv_layout& L, const float* const* atlas_planes, float* const* level_planes, cudaStream_t s) {
  LevelPtrs src{};
  for (int d = 0; d < L.planes; ++d) src.p[d] = atlas_planes[d];
  for (int k = 0; k < L.num_levels; ++k) {
    const puv_placement& pl = L.level[k];
    AtlasPtrs dst{};
    for (int d = 0; d < L.planes; ++d) dst.p[d] = level_planes[(size_t)k * L.planes + d];
    const int n = pl.rows * pl.cols;
    k_unpack_level<<<(n + 255) / 256, 256, 0, s>>>(dst, src, L.planes, pl.rows, pl.cols, pl.x, pl.y, pl.rot90ccw,
                                                   L.atlas_w);
  }
  count_launches(L.num_levels);
}

// L = 1/2 sum (img - tgt)^2 ; dl = img - tgt.  float4 vectorised, fp64 partial sums.
__global__ void __launch_bounds__(256) k_l2_loss(int64_t n, const float* __restrict__ img,
                                                 const float* __restrict__ tgt, float* __restrict__ dl,
                                                 double* __restrict__ loss, bool vec) {
  __shared__ double sh[8];
  double acc = 0.0;
  const int64_t n4 = vec ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4* i4 = reinterpret_cast<const float4*>(img);
  const float4* t4 = reinterpret_cast<const float4*>(tgt);
  float4* d4 = reinterpret_cast<float4*>(dl);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 a = __ldcs(i4 + i), b = __ldcs(t4 + i);
    const float4 d = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
    d4[i] = d;
    acc += (double)(d.x * d.x + d.y * d.y) + (double)(d.z * d.z + d.w * d.w);
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float d = img[i] - tgt[i];
    dl[i] = d;
    acc += (double)d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sh[w];
    atomicAdd(loss, 0.5 * s);
  }
}

void launch_l2_loss(int64_t n, const float* img, const float* tgt, float* dl, double* loss, cudaStream_t s,
                    bool accumulate) {
  if (!accumulate) cudaMemsetAsync(loss, 0, sizeof(double), s);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n / 4 + 255) / 256;
  const int blocks = (int)(want < 4 * nsm ? (want > 0 ? want : 1) : 4 * nsm);
  const bool vec = ((uintptr_t)img % 16 == 0) && ((uintptr_t)tgt % 16 == 0) && ((uintptr_t)dl % 16 == 0);
  k_l2_loss<<<blocks, 256, 0, s>>>(n, img, tgt, dl, loss, vec);
  count_launches(1);
}

__global__ void k_contract(int op, const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = op == 0 ? exp_c(in[i]) : log_c(in[i]);
}

void launch_contract(int op, const float* in, float* out, int64_t n, cudaStream_t s) {
  k_contract<<<1184, 256, 0, s>>>(op, in, out, n);
  count_launches(1);
}

__global__ void k_begin_call(CallHdr* call, uint64_t cap, uint32_t n_views) {
  call->n_views = n_views;
  call->arena_used = 0;
  call->arena_need = 0;
  call->overflow_any = 0;
  call->arena_cap = cap;
}

void launch_begin_call(const Plan& p, const Views& v, uint64_t arena_cap, cudaStream_t s) {
  k_begin_call<<<1, 1, 0, s>>>(v.call, arena_cap, (uint32_t)p.n_views);
  count_launches(1);
}

// flag |= overflow of the last render call on this state; need = max(need, its arena bytes)
__global__ void k_overflow_acc(const CallHdr* call, uint32_t* flag, uint64_t* need) {
  *flag |= call->overflow_any;
  const uint64_t b = 4 * call->arena_need;
  if (b > *need) *need = b;
}

void launch_overflow_acc(const void* state, uint32_t* flag, uint64_t* need, cudaStream_t s) {
  k_overflow_acc<<<1, 1, 0, s>>>(reinterpret_cast<const CallHdr*>(state), flag, need);   // CallHdr at offset 0
  count_launches(1);
}

}  // namespace puv
