// K5 k_raster_fwd — per-tile front-to-back compositing (row a5).
//
// One 256-thread block per 16x16 tile, one pixel per thread (PAPER.md:195
// "tile-based rasterizer"; semantics R9).  The tile's sorted Gaussian list is
// consumed in batches of 256: each thread gathers one record into shared
// memory (float4 x3 per entry, LDS.128 broadcast on use).  A warp stops
// walking a batch as soon as all its pixels have terminated (ballot), the
// block stops fetching batches once all 256 pixels have (syncthreads_count).
// The skip test, alpha, cap and termination use the fp32 contract (R1, R14),
// so the per-pixel composited set, T_final and n_contrib match the oracle bit
// for bit.  The backward replays each pixel's list in reverse, recovers
// T_k = T_{k+1} / (1 - alpha_k), reduces the 9 per-pair gradients of each entry
// across the warp with a transposing butterfly (16 shuffles instead of 45)
// and issues one global atomic per value and warp.
#include "contract.cuh"
#include "internal.cuh"

namespace puv {

constexpr int kRasterThreads = kTile * kTile;

__global__ void __launch_bounds__(kRasterThreads) k_raster_fwd(const uint32_t* __restrict__ arena, Views v, int view,
                                                              int N, int W, int H, int gx, int ntiles, float bg0,
                                                              float bg1, float bg2, float* __restrict__ image) {
  __shared__ float4 sA[kRasterThreads], sB[kRasterThreads], sC[kRasterThreads];
  const int tile = blockIdx.x;
  const int tx = tile % gx, ty = tile / gx;
  const int px = tx * kTile + (threadIdx.x & (kTile - 1));
  const int py = ty * kTile + (threadIdx.x / kTile);
  const bool inside = px < W && py < H;
  const ViewHdr& hdr = v.hdr[view];
  uint32_t start = 0, end = 0;
  if (!hdr.overflow) {
    start = v.tstart[(size_t)view * ntiles + tile];
    end = v.tend[(size_t)view * ntiles + tile];
  }
  const uint32_t* list = arena + hdr.list_base;
  const float4* rec = v.rec + (size_t)view * N * 3;
  const float fi = (float)px, fj = (float)py;
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  uint32_t last = 0, n_exam = 0, n_comp = 0;
  bool done = !inside;
  for (uint32_t b0 = start; b0 < end; b0 += kRasterThreads) {
    if (__syncthreads_count(done) == kRasterThreads) break;
    const uint32_t idx = b0 + threadIdx.x;
    if (idx < end) {
      const uint32_t g = list[idx];
      sA[threadIdx.x] = rec[3 * (size_t)g + 0];
      sB[threadIdx.x] = rec[3 * (size_t)g + 1];
      sC[threadIdx.x] = rec[3 * (size_t)g + 2];
    }
    __syncthreads();
    const int n = (int)min((uint32_t)kRasterThreads, end - b0);
    for (int j = 0; j < n; ++j) {
      if (__all_sync(0xffffffffu, done)) break;
      if (done) continue;
      const float4 A = sA[j];
      const float4 B = sB[j];
      const float power = pair_power(A.x, A.y, A.z, A.w, B.x, fi, fj);
      ++n_exam;
      if (power > 0.0f || power < B.y) continue;
      const float ao = mul(B.z, exp_c(power));
      const float alpha = ao < 0.99f ? ao : 0.99f;
      const float Tn = mul(T, sub(1.0f, alpha));
      if (Tn < 1e-4f) { done = true; continue; }
      const float4 Cc = sC[j];
      const float w = alpha * T;
      C0 = fmaf(Cc.x, w, C0);
      C1 = fmaf(Cc.y, w, C1);
      C2 = fmaf(Cc.z, w, C2);
      T = Tn;
      last = b0 + j + 1 - start;
      ++n_comp;
    }
  }
  {  // pair statistics (one atomic per warp)
    const uint32_t we = __reduce_add_sync(0xffffffffu, n_exam), wc = __reduce_add_sync(0xffffffffu, n_comp);
    if ((threadIdx.x & 31) == 0 && (we | wc)) {
      atomicAdd((unsigned long long*)&v.hdr[view].examined, (unsigned long long)we);
      atomicAdd((unsigned long long*)&v.hdr[view].composited, (unsigned long long)wc);
    }
  }
  if (inside) {
    const size_t HW = (size_t)W * H, p = (size_t)py * W + px;
    image[p] = fmaf(T, bg0, C0);
    image[HW + p] = fmaf(T, bg1, C1);
    image[2 * HW + p] = fmaf(T, bg2, C2);
    v.tfinal[(size_t)view * HW + p] = T;
    v.ncontrib[(size_t)view * HW + p] = last;
  }
}


void launch_raster_fwd(const Plan& p, const Views& v, const uint32_t* arena, float* image, int view,
                       const float bg[3], cudaStream_t s) {
  k_raster_fwd<<<p.ntiles, kRasterThreads, 0, s>>>(arena, v, view, p.N, p.W, p.H, p.gx, p.ntiles, bg[0], bg[1], bg[2],
                                                   image);
  count_launches(1);
}

}  // namespace puv
