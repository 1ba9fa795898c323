// K5 k_raster_fwd — per-tile front-to-back compositing (row a5).
//
// One block per 16x16 tile, PPT pixels per thread in one column ("tile-based
// rasterizer"; semantics R9).  Warp w owns the 8-column block 8(w&1) of rows 4 PPT (w>>1) ..;
// lane l owns column l & 7 and rows (l >> 3) + 4k, k < PPT (the layout of K6).  The tile's
// sorted Gaussian list is consumed in batches of 128 entries gathered into shared memory
// (contract record A, B and the fp64 value record; LDS broadcast on use), so one set of record
// loads and one loop step serve all pixels of a thread.  Every lane runs the skip test of both its pixels;
// the composite runs under a per-pixel predicate and only when some pixel of the warp composites.
// A warp stops walking a batch as soon as all its pixels have terminated (vote), the block stops
// fetching batches once all 256 pixels have (syncthreads_count).
// Decisions — skip test, alpha cap, termination — use the fp32 contract (R1, R14), so the
// composited set, T_final and n_contrib match the oracle bit for bit.  The composited VALUES are
// carried in fp64: the image is the fp64 colour rounded once, and the pixel's full
// colour C = sum c_k a_k T_k + T_final bg is kept for the single-pass backward (K6).
#include <type_traits>

#include "contract.cuh"
#include "feed.cuh"
#include "internal.cuh"

namespace puv {

#ifndef PUV_FWD_PPT
#define PUV_FWD_PPT 2
#endif
constexpr int kFwdPPT = PUV_FWD_PPT;                     // pixels per thread (one column, rows r + 4k)
constexpr int kRasterThreads = kTile * kTile / kFwdPPT;  // 128 (PPT 2) or 64 (PPT 4)
#ifndef PUV_FWD_MINB
#define PUV_FWD_MINB 7
#endif
#if PUV_FWD_MINB > 0
#define PUV_FWD_BOUNDS __launch_bounds__(kTile * kTile / PUV_FWD_PPT, PUV_FWD_MINB)
#else
#define PUV_FWD_BOUNDS __launch_bounds__(kTile * kTile / PUV_FWD_PPT)
#endif
#ifndef PUV_FWD_BATCH
#define PUV_FWD_BATCH 128
#endif
constexpr int kFwdBatch = PUV_FWD_BATCH;                 // entries staged per batch

#ifndef PUV_FWD_POPCNT
#define PUV_FWD_POPCNT 0
#endif
#ifndef PUV_FWD_BRANCHFREE
#define PUV_FWD_BRANCHFREE 0
#endif
#ifndef PUV_FWD_CULL
#define PUV_FWD_CULL 1
#endif

template <int P>
__device__ __forceinline__ bool all_of(const bool (&b)[P]) {
  bool r = true;
#pragma unroll
  for (int k = 0; k < P; ++k) r = r && b[k];
  return r;
}
template <int P>
__device__ __forceinline__ bool any_of(const bool (&b)[P]) {
  bool r = false;
#pragma unroll
  for (int k = 0; k < P; ++k) r = r || b[k];
  return r;
}

__global__ void PUV_FWD_BOUNDS k_raster_fwd(const uint32_t* __restrict__ arena, Views v, int view0,
                                                              int N, int W, int H, int gx, int ntiles, float bg0,
                                                              float bg1, float bg2, float* __restrict__ images) {
  __shared__ float4 sA[kFwdBatch], sB[kFwdBatch];
  __shared__ double2 sD[5][kFwdBatch];
  __shared__ double sExp[kExpTab];
  exp64_table_fill(sExp);
  const int tile = blockIdx.x;
  const int tx = tile % gx, ty = tile / gx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
  const int py0 = ty * kTile + (warp >> 1) * 4 * kFwdPPT + (lane >> 3);
  const int view = view0 + blockIdx.y;   // grid.y: consecutive views launched together
  float* image = images + (size_t)blockIdx.y * 3 * W * H;
  const ViewHdr& hdr = v.hdr[view];
  uint32_t start = 0, end = 0;
#if PUV_DIRECT
  // the tile's entries: its super-tile's level-1 rank range, filtered by rect (feed.cuh)
  __shared__ uint32_t sGid[2 * kFwdBatch], sFeedCnt[kRasterThreads / 32 + 1];
  TileFeed<kRasterThreads, kFwdBatch> feed;
  {
    const int st = (ty / kSup) * v.sgx + (tx / kSup);
    const ViewHdr& l1 = v.l1[view];
    if (!hdr.overflow && !l1.overflow) {
      start = v.sst[(size_t)view * (v.nst + 1) + st];
      end = v.sen[(size_t)view * (v.nst + 1) + st];
    }
    feed.init(sGid, sFeedCnt, start, end);
  }
  const uint32_t* list1 = arena + v.l1[view].list_base;
  const uint32_t* sorted_v = v.sorted + (size_t)view * N;
  const uint2* rect_v = v.rect + (size_t)view * N;
  uint32_t ebase = 0;   // tile-list entries before the current batch
#else
  if (!hdr.overflow) {
    start = v.tstart[(size_t)view * ntiles + tile];
    end = v.tend[(size_t)view * ntiles + tile];
  }
  const uint32_t* list = arena + hdr.list_base;
#endif
  const float4* rec = v.rec + (size_t)view * N * 2;
  const double2* rec64 = v.rec64 + (size_t)view * N * 5;
  const float fi = (float)px;
  const double di = px;
  float fj[kFwdPPT], T[kFwdPPT];
  double dj[kFwdPPT], T64[kFwdPPT], C[kFwdPPT][3];
  uint32_t last[kFwdPPT];
  bool done[kFwdPPT];
#pragma unroll
  for (int k = 0; k < kFwdPPT; ++k) {
    fj[k] = (float)(py0 + 4 * k);
    dj[k] = py0 + 4 * k;
    T[k] = 1.0f;
    T64[k] = 1.0;
    C[k][0] = C[k][1] = C[k][2] = 0.0;
    last[k] = 0;
    done[k] = !(px < W && py0 + 4 * k < H);
  }
  // examined pairs of a pixel = entries walked until it terminated (inclusive) or the list ended
  uint32_t exam[kFwdPPT], n_comp = 0;
  static_assert(!kMaskFill || PUV_FWD_CULL, "the mask fill relies on the filtered walk's stop");
  // composited-pixel bits for K6 (8 words per entry, K6 order: K6 warp, row group), for each of the
  // tile's first kMaskCap entries.  PPT 2: this warp's two words (K6 warp (w & 1), row groups
  // 2 (w >> 1) + k'); PPT 4: the warp IS a K6 warp (8 x 16 pixels), its four words
  static_assert(kFwdPPT == 2 || kFwdPPT == 4, "the K6 mask layout takes 2 or 4 pixels per K5 thread");
  using MaskW = std::conditional_t<kFwdPPT == 4, uint4, uint2>;
  constexpr int kMaskStride = kFwdPPT == 4 ? 2 : 4;   // MaskW units per entry (8 words)
  MaskW* dmask = kMaskCap > 0 ? reinterpret_cast<MaskW*>(v.dmask + ((size_t)view * ntiles + tile) * kMaskCap * 8 +
                                                           (kFwdPPT == 4 ? warp * 4 : (warp & 1) * 4 + 2 * (warp >> 1)))
                              : nullptr;
#pragma unroll
  for (int k = 0; k < kFwdPPT; ++k) exam[k] = 0;
#if PUV_DIRECT
  for (;;) {
    if (__syncthreads_count(all_of(done)) == kRasterThreads) break;
    const int nb = feed.next(list1, sorted_v, rect_v, tx, ty);
    if (nb == 0) break;
#pragma unroll
    for (int i = threadIdx.x; i < kFwdBatch; i += kRasterThreads) {
      if (i < nb) {
        const uint32_t g = sGid[i];
        PUV_CHECK(g < (uint32_t)N);
        sA[i] = rec[2 * (size_t)g + 0];
        sB[i] = rec[2 * (size_t)g + 1];
#pragma unroll
        for (int k = 0; k < 5; ++k) sD[k][i] = rec64[5 * (size_t)g + k];
      }
    }
    __syncthreads();
    const int n = __all_sync(0xffffffffu, all_of(done)) ? 0 : nb;
    const uint32_t b0 = ebase + start;   // so that b0 + j - start is the entry index below
#else
  for (uint32_t b0 = start; b0 < end; b0 += kFwdBatch) {
    if (__syncthreads_count(all_of(done)) == kRasterThreads) break;
#pragma unroll
    for (int i = threadIdx.x; i < kFwdBatch; i += kRasterThreads) {
      const uint32_t idx = b0 + i;
      if (idx < end) {
        const uint32_t g = list[idx];
        PUV_CHECK(g < (uint32_t)N && idx < hdr.K);
        sA[i] = rec[2 * (size_t)g + 0];
        sB[i] = rec[2 * (size_t)g + 1];
#pragma unroll
        for (int k = 0; k < 5; ++k) sD[k][i] = rec64[5 * (size_t)g + k];
      }
    }
    __syncthreads();
    const int n = __all_sync(0xffffffffu, all_of(done)) ? 0 : (int)min((uint32_t)kFwdBatch, end - b0);
#endif
#if PUV_FWD_CULL
    // per-warp filter: one box test per staged entry (lanes split the batch), ballots -> the
    // entries whose ellipse can reach this warp's 8x8 block; the walk visits only those (the
    // skipped ones get their all-zero K6 mask words here)
    static_assert(kFwdBatch % 32 == 0 && kFwdBatch <= 128, "batch = 1..4 words of entry bits");
    uint32_t mwords[kFwdBatch / 32];
    {
      const float bx0 = (float)(tx * kTile + (warp & 1) * 8), by0 = (float)(ty * kTile + (warp >> 1) * 4 * kFwdPPT);
#pragma unroll
      for (int q = 0; q < kFwdBatch / 32; ++q) {
        const int j = 32 * q + lane;
        bool may = false;
        if (j < n) {
          const float4 A = sA[j];
          const float4 B = sB[j];
          may = block_may_hit(A.x, A.y, A.z, A.w, B.x, B.y, bx0, by0, 7.f, (float)(4 * kFwdPPT - 1));
          const uint32_t e = b0 + j - start;
          if (!may && kMaskCap > 0 && e < (uint32_t)kMaskCap) dmask[(size_t)e * kMaskStride] = MaskW{};
        }
        mwords[q] = __ballot_sync(0xffffffffu, may);
      }
    }
    bool stop = false;
    for (int q = 0; q < kFwdBatch / 32 && !stop; ++q)
    for (uint32_t bits = mwords[q]; bits; bits &= bits - 1) {
      const int j = 32 * q + __ffs(bits) - 1;
#else
    for (int j = 0; j < n; ++j) {
#endif
      const float4 A = sA[j];
      const float4 B = sB[j];
      bool hit[kFwdPPT];
      float power[kFwdPPT];
#pragma unroll
      for (int k = 0; k < kFwdPPT; ++k) {
        power[k] = pair_power(A.x, A.y, A.z, A.w, B.x, fi, fj[k]);
        hit[k] = !done[k] && !(power[k] > 0.0f || power[k] < B.y);
      }
      const uint32_t e = b0 + j - start;   // entry index in the tile list
      if (!__any_sync(0xffffffffu, any_of(hit))) {
        if (kMaskCap > 0 && lane == 0 && e < (uint32_t)kMaskCap) dmask[(size_t)e * kMaskStride] = MaskW{};
        continue;
      }
      bool comp[kFwdPPT] = {};
      // fp64 record and the column terms shared by both pixels (same px): dx, ha dx^2, nb dx
      const double2 d0 = sD[0][j], d1 = sD[1][j], d2 = sD[2][j], d3 = sD[3][j];
      const double d4x = sD[4][j].x;
      const double dx = d0.x - di;
      // kLno: ln o rides in the column term, so exp64(power64) is alpha itself
      const double hadxx = kLno ? fma(d1.x, dx * dx, d2.y) : d1.x * (dx * dx), nbdx = d1.y * dx;
#if PUV_FWD_BRANCHFREE
      // both pixels' bodies run under selects (no divergent branches): the contract on a safe
      // argument (power 0) where the pixel did not hit, every state update gated by its flags
#pragma unroll
      for (int k = 0; k < kFwdPPT; ++k) {
        const float ao = mul(B.z, exp_c_core(hit[k] ? power[k] : 0.0f));
        const bool capped = !(ao < 0.99f);
        const float alpha = capped ? 0.99f : ao;
        const float Tn = mul(T[k], sub(1.0f, alpha));
        const bool term = hit[k] && Tn < 1e-4f;
        comp[k] = hit[k] && !term;
        exam[k] = term ? e + 1 : exam[k];
        done[k] = done[k] || term;
        T[k] = comp[k] ? Tn : T[k];
        last[k] = comp[k] ? e + 1 : last[k];
        n_comp += comp[k] ? 1u : 0u;
        const double pw = power64(d2.x, hadxx, nbdx, d0.y - dj[k]);
        const double a64 = capped ? 0.99 : (kLno ? 1.0 : d2.y) * exp64(fmax(pw, -700.0), sExp);
        const double w = comp[k] ? a64 * T64[k] : 0.0;
        C[k][0] = fma(d3.x, w, C[k][0]);
        C[k][1] = fma(d3.y, w, C[k][1]);
        C[k][2] = fma(d4x, w, C[k][2]);
        T64[k] -= w;   // T64 * (1 - a64)
      }
#else
#pragma unroll
      for (int k = 0; k < kFwdPPT; ++k) {
        if (!hit[k]) continue;
        const float ao = mul(B.z, exp_c_core(power[k]));   // power in [t_g, 0] here
        const bool capped = !(ao < 0.99f);
        const float alpha = capped ? 0.99f : ao;
        const float Tn = mul(T[k], sub(1.0f, alpha));
        if (Tn < 1e-4f) {
          done[k] = true;
          exam[k] = e + 1;
          continue;
        }
        T[k] = Tn;
        last[k] = e + 1;
        comp[k] = true;
#if !PUV_FWD_POPCNT
        ++n_comp;
#endif
        // fp64 value of the composited pair
        const double pw = power64(d2.x, hadxx, nbdx, d0.y - dj[k]);
        const double a64 = capped ? 0.99 : (kLno ? exp64(pw, sExp) : d2.y * exp64(pw, sExp));
        const double w = a64 * T64[k];
        C[k][0] = fma(d3.x, w, C[k][0]);
        C[k][1] = fma(d3.y, w, C[k][1]);
        C[k][2] = fma(d4x, w, C[k][2]);
        T64[k] -= w;   // T64 * (1 - a64)
      }
#endif
      if (kMaskCap > 0) {
        uint32_t m[kFwdPPT];
#pragma unroll
        for (int k = 0; k < kFwdPPT; ++k) m[k] = __ballot_sync(0xffffffffu, comp[k]);
#if PUV_FWD_POPCNT && !PUV_FWD_BRANCHFREE
#pragma unroll
        for (int k = 0; k < kFwdPPT; ++k)
          if (lane == 0) n_comp += __popc(m[k]);   // the warp's composited pairs of this entry
#endif
        if (lane == 0 && e < (uint32_t)kMaskCap) {
          MaskW mw;
#pragma unroll
          for (int k = 0; k < kFwdPPT; ++k) reinterpret_cast<uint32_t*>(&mw)[k] = m[k];
          dmask[(size_t)e * kMaskStride] = mw;
        }
      }
      if (__all_sync(0xffffffffu, all_of(done))) {
#if PUV_FWD_CULL
        stop = true;
#endif
        break;
      }
    }
#if PUV_DIRECT
    ebase += (uint32_t)nb;
    feed.pop(nb);
#endif
  }
  if constexpr (kMaskFill) {
    // zero words for the entries after this warp stopped, up to the tile's largest n_contrib (the
    // range K6 walks), so K6 never reads a stale word.  A warp with a live pixel walked (and wrote)
    // every fed entry; one whose pixels all terminated stopped right after the last termination,
    // i.e. it wrote entries [0, max exam) (exam = terminating entry + 1; 0 for off-image pixels)
    const bool wdone = __all_sync(0xffffffffu, all_of(done));
    uint32_t mx = 0;
#pragma unroll
    for (int k = 0; k < kFwdPPT; ++k) mx = max(mx, done[k] ? exam[k] : 0u);
    const uint32_t wfill = __reduce_max_sync(0xffffffffu, mx);   // used only when wdone
    __shared__ uint32_t sLmax[kRasterThreads / 32];
    uint32_t lm = 0;
#pragma unroll
    for (int k = 0; k < kFwdPPT; ++k) lm = max(lm, last[k]);
    lm = __reduce_max_sync(0xffffffffu, lm);
    if (lane == 0) sLmax[warp] = lm;
    __syncthreads();
    uint32_t Lmax = 0;
#pragma unroll
    for (int w = 0; w < kRasterThreads / 32; ++w) Lmax = max(Lmax, sLmax[w]);
    const uint32_t fe = min(Lmax, (uint32_t)kMaskCap);
    if (wdone)
      for (uint32_t e = wfill + lane; e < fe; e += 32) dmask[(size_t)e * kMaskStride] = MaskW{};
  }
#if PUV_DIRECT
  const uint32_t list_len = ebase;   // the whole list was fed unless every pixel terminated first
#else
  const uint32_t list_len = end - start;
#endif
  uint32_t n_exam = 0;
#pragma unroll
  for (int k = 0; k < kFwdPPT; ++k) n_exam += done[k] ? exam[k] : (px < W && py0 + 4 * k < H ? list_len : 0u);
  {  // pair statistics (one atomic per warp)
    const uint32_t we = __reduce_add_sync(0xffffffffu, n_exam), wc = __reduce_add_sync(0xffffffffu, n_comp);
    if (lane == 0 && (we | wc)) {
      atomicAdd((unsigned long long*)&v.hdr[view].examined, (unsigned long long)we);
      atomicAdd((unsigned long long*)&v.hdr[view].composited, (unsigned long long)wc);
    }
  }
  const size_t HW = (size_t)W * H;
#pragma unroll
  for (int k = 0; k < kFwdPPT; ++k) {
    const int py = py0 + 4 * k;
    if (px < W && py < H) {
      const size_t p = (size_t)py * W + px;
      const double c0 = fma(T64[k], (double)bg0, C[k][0]);
      const double c1 = fma(T64[k], (double)bg1, C[k][1]);
      const double c2 = fma(T64[k], (double)bg2, C[k][2]);
      image[p] = (float)c0;
      image[HW + p] = (float)c1;
      image[2 * HW + p] = (float)c2;
      double* cf = v.cfull + 3 * ((size_t)view * HW + p);
      cf[0] = c0;
      cf[1] = c1;
      cf[2] = c2;
      v.tfinal[(size_t)view * HW + p] = T[k];
      v.ncontrib[(size_t)view * HW + p] = last[k];
    }
  }
}

void launch_raster_fwd(const Plan& p, const Views& v, const uint32_t* arena, float* images, int view0, int n_views,
                       const float bg[3], cudaStream_t s) {
  if (n_views <= 0 || p.ntiles <= 0) return;
  const dim3 grid(p.ntiles, n_views);
#if PUV_RASTER_CARVEOUT >= 0
  // shared-memory carveout preference (percent): lets the driver pick a larger carveout so the
  // register-limited residency is not capped by the shared-memory configuration
  static const bool carve_once =
      cudaFuncSetAttribute(k_raster_fwd, cudaFuncAttributePreferredSharedMemoryCarveout, PUV_RASTER_CARVEOUT) == cudaSuccess;
  (void)carve_once;
#endif
  k_raster_fwd<<<grid, kRasterThreads, 0, s>>>(arena, v, view0, p.N, p.W, p.H, p.gx, p.ntiles, bg[0], bg[1], bg[2],
                                               images);
  count_launches(1);
}

}  // namespace puv
