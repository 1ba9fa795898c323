// K5 k_raster_fwd — per-tile front-to-back compositing (row a5).
//
// One 256-thread block per 16x16 tile, one pixel per thread (PAPER.md:195
// "tile-based rasterizer"; semantics R9).  The tile's sorted Gaussian list is
// consumed in batches of 256: each thread gathers one entry into shared
// memory (contract record A, B and the fp64 value record; LDS broadcast on
// use).  A warp stops walking a batch as soon as all its pixels have
// terminated (vote), the block stops fetching batches once all 256 pixels have
// (syncthreads_count).
// Decisions — skip test, alpha cap, termination — use the fp32 contract (R1,
// R14), so the composited set, T_final and n_contrib match the oracle bit for
// bit.  The composited VALUES are carried in fp64: the image is
// the fp64 colour rounded once, and the pixel's full colour
// C = sum c_k a_k T_k + T_final bg is kept for the single-pass backward (K6).
#include "contract.cuh"
#include "internal.cuh"

namespace puv {

constexpr int kRasterThreads = kTile * kTile;

__global__ void __launch_bounds__(kRasterThreads) k_raster_fwd(const uint32_t* __restrict__ arena, Views v, int view,
                                                              int N, int W, int H, int gx, int ntiles, float bg0,
                                                              float bg1, float bg2, float* __restrict__ image) {
  __shared__ float4 sA[kRasterThreads], sB[kRasterThreads];
  __shared__ double2 sD[5][kRasterThreads];
  __shared__ double sExp[64];
  exp64_table_fill(sExp);
  const int tile = blockIdx.x;
  const int tx = tile % gx, ty = tile / gx;
  // compact 8x4 warp footprint: warp w covers columns 8(w&1).. and rows 4(w>>1)..
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
  const int py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
  const bool inside = px < W && py < H;
  const ViewHdr& hdr = v.hdr[view];
  uint32_t start = 0, end = 0;
  if (!hdr.overflow) {
    start = v.tstart[(size_t)view * ntiles + tile];
    end = v.tend[(size_t)view * ntiles + tile];
  }
  const uint32_t* list = arena + hdr.list_base;
  const float4* rec = v.rec + (size_t)view * N * 3;
  const double2* rec64 = v.rec64 + (size_t)view * N * 5;
  const float fi = (float)px, fj = (float)py;
  const double di = px, dj = py;
  float T = 1.0f;
  double T64 = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
  uint32_t last = 0, n_exam = 0, n_comp = 0;
  bool done = !inside;
  for (uint32_t b0 = start; b0 < end; b0 += kRasterThreads) {
    if (__syncthreads_count(done) == kRasterThreads) break;
    const uint32_t idx = b0 + threadIdx.x;
    if (idx < end) {
      const uint32_t g = list[idx];
      sA[threadIdx.x] = rec[3 * (size_t)g + 0];
      sB[threadIdx.x] = rec[3 * (size_t)g + 1];
#pragma unroll
      for (int k = 0; k < 5; ++k) sD[k][threadIdx.x] = rec64[5 * (size_t)g + k];
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
      const bool capped = !(ao < 0.99f);
      const float alpha = capped ? 0.99f : ao;
      const float Tn = mul(T, sub(1.0f, alpha));
      if (Tn < 1e-4f) { done = true; continue; }
      T = Tn;
      last = b0 + j + 1 - start;
      ++n_comp;
      // fp64 value of the composited pair
      const double2 d0 = sD[0][j], d1 = sD[1][j], d2 = sD[2][j], d3 = sD[3][j];
      const double d4x = sD[4][j].x;
      const double dx = d0.x - di, dy = d0.y - dj;
      const double a64 = capped ? 0.99 : d2.y * exp64(fma(d1.x * dx, dx, fma(d1.y * dx, dy, d2.x * dy * dy)), sExp);
      const double w = a64 * T64;
      C0 = fma(d3.x, w, C0);
      C1 = fma(d3.y, w, C1);
      C2 = fma(d4x, w, C2);
      T64 -= w;   // T64 * (1 - a64)
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
    C0 = fma(T64, (double)bg0, C0);
    C1 = fma(T64, (double)bg1, C1);
    C2 = fma(T64, (double)bg2, C2);
    image[p] = (float)C0;
    image[HW + p] = (float)C1;
    image[2 * HW + p] = (float)C2;
    double* cf = v.cfull + 3 * ((size_t)view * HW + p);
    cf[0] = C0;
    cf[1] = C1;
    cf[2] = C2;
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
