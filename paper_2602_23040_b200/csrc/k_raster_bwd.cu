// K6 k_raster_bwd — per-tile gradient of the front-to-back composite (row a7).
//
// One 64-thread block (2 warps) per (16x16 tile, view) — all views of a call in one launch;
// warp w owns the 8-column half 8w of the tile; lane l owns column l & 7 and rows (l >> 3) + 4k,
// k < PPT = 4 (PPT = 2 with 4 warps of 8x8 quadrants is the -DPUV_BWD_PPT=2 build).  Four pixels
// per thread halve the per-pixel share of the per-entry warp reduction, which bounds the
// shared-memory pipe at two pixels per thread (ncu: 87% -> 57% of its wavefronts).  Every decision (skip test R1, alpha cap, composited set R14) is
// replayed with the fp32 contract exactly as K5 took it; every VALUE is fp64.
// Single pass in front-to-back order, using the pixel's full colour C from K5.  With dC = dL/dC
// (3 channels) only the scalar projections of the colours are needed:
//   cd_k = dC . c_k,   Sd_k = dC . (C - P_k) = dC . C - sum_{i<=k} cd_i a_i T_i
//   dL/dc_k = a_k T_k dC,   dL/da_k = cd_k T_k - Sd_k / (1 - a_k)
//   uncapped: dL/do = G dL/da, dL/dpower = o G dL/da
// and, with power = ha dx^2 + nb dx dy + hc dy^2 ((dx, dy) = mean - pixel), the mean and conic
// gradients are o-scaled moments of GdL = G dL/da over the pixels:
//   dL/dmx = o (2 ha Mx + nb My), dL/dmy = o (nb Mx + 2 hc My), dL/d(ha, nb, hc) = o (Mxx, Mxy, Myy)
//   Mx = sum GdL dx, My = sum GdL dy, Mxx = sum GdL dx^2, Mxy = sum GdL dx dy, Myy = sum GdL dy^2.
// K6 accumulates the raw moments (Mx, My, Mxx, Mxy, Myy, sum GdL, dL/dc) per (view, Gaussian);
// K7 applies the (linear) o-scaling and the conic mixing once per (view, Gaussian).  With kLno
// (default) the record holds ln o, exp64 returns alpha = o G directly and the moments are taken of
// o GdL (the o-scaling is already in; sum o GdL = o dL/do), so K7 only mixes.
// The per-pixel body is branch-free (inactive pixels get a = 0 and masked terms), so the
// pixels' fp64 chains interleave.  A thread sums the 9 moments of an entry over its pixels; the
// warp sums them with a transposing shuffle butterfly and 9 lanes issue one fp64 atomic
// each into the (view, Gaussian) slot.
#include <type_traits>

#include "contract.cuh"
#include "feed.cuh"
#include "internal.cuh"

namespace puv {

#ifndef PUV_BWD_PPT
#define PUV_BWD_PPT 4
#endif
#ifndef PUV_BWD_MINB
#define PUV_BWD_MINB 10
#endif
#if PUV_BWD_MINB > 0
#define PUV_BWD_BOUNDS __launch_bounds__(kTile * kTile / PUV_BWD_PPT, PUV_BWD_MINB)
#else
#define PUV_BWD_BOUNDS __launch_bounds__(kTile * kTile / PUV_BWD_PPT)
#endif
constexpr int kBwdPPT = PUV_BWD_PPT;                       // pixels per thread (one column, rows r + 4k)
constexpr int kBwdThreads = kTile * kTile / kBwdPPT;        // 128 (PPT 2) or 64 (PPT 4)
constexpr int kRedRow = 34;   // row stride (doubles) of the transpose buffer: 4-bank skew per row
#ifndef PUV_BWD_EXPSEL
#define PUV_BWD_EXPSEL 1
#endif
#ifndef PUV_BWD_CULL
#define PUV_BWD_CULL 1
#endif
#ifndef PUV_BWD_CAPSPLIT
#define PUV_BWD_CAPSPLIT 1
#endif
#ifndef PUV_BWD_BATCH
#define PUV_BWD_BATCH 64
#endif
#ifndef PUV_BWD_KSKIP
#define PUV_BWD_KSKIP 0
#endif
constexpr int kBwdBatch = PUV_BWD_BATCH;                   // entries staged per batch

// Alternative reduction (-DPUV_BWD_SMEM_RED).  Sum the 9 per-lane values x[0..8] over the warp
// through shared memory: lane l stores x[k] at
// buf[34 k + l] (conflict-free), then lanes 3v, 3v+1, 3v+2 (v < 9) sum value v over lanes
// [0, 12), [12, 24), [24, 32) with 16-byte loads, and two shuffles fold the thirds into lane 3v.
// The row stride of 34 doubles skews row v by 4v banks, so the 27 reading lanes spread over the
// 8 four-bank groups ((v + 6 part) mod 8): 4 wavefronts per 16-byte load, the minimum.  About
// 35 instructions per entry.  `buf` is the warp's 9 x 34 slice (16-byte aligned).
__device__ __forceinline__ double warp_sum9(const double (&x)[9], double* buf, int lane) {
#pragma unroll
  for (int k = 0; k < 9; ++k) buf[kRedRow * k + lane] = x[k];
  __syncwarp();
  const int v = lane / 3, part = lane - 3 * v;
  double s0 = 0.0, s1 = 0.0;
  if (lane < 27) {
    const double2* col = reinterpret_cast<const double2*>(buf + kRedRow * v + 12 * part);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 q = col[i];
      s0 += q.x;
      s1 += q.y;
    }
    if (part < 2) {
#pragma unroll
      for (int i = 4; i < 6; ++i) {
        const double2 q = col[i];
        s0 += q.x;
        s1 += q.y;
      }
    }
  }
  __syncwarp();
  double s = s0 + s1;
  const double p1 = __shfl_down_sync(0xffffffffu, s, 1);
  const double p2 = __shfl_down_sync(0xffffffffu, s, 2);
  return s + p1 + p2;   // valid in lanes 3v, v < 9
}

// Default reduction: transposing shuffle butterfly (8 values in 9 double shuffles, v8 in 5);
// lane l ends with the total of value (l >> 2) & 7, v8 in all lanes.  A/B on one B200 (C3, 64
// views, tools/ab_raster.py): 54.4 ms against 55.6 ms for the shared-memory transpose below
// (-DPUV_BWD_SMEM_RED), which moves more bytes through the MIO pipe per entry.
__device__ __forceinline__ double warp_reduce9_shfl(double (&x)[9]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int level = 0; level < 3; ++level) {
    const int half = 4 >> level;
    const int off = 16 >> level;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? x[i] : x[i + half];
      const double keep = upper ? x[i + half] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  double s = x[0] + __shfl_xor_sync(0xffffffffu, x[0], 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x[8] += __shfl_xor_sync(0xffffffffu, x[8], off);
  return s;
}

__global__ void PUV_BWD_BOUNDS k_raster_bwd(const uint32_t* __restrict__ arena, Views v, int N,
                                                           int W, int H, int gx, int ntiles, int view0,
                                                           const float* __restrict__ dL_dimages) {
  __shared__ float4 sA[kBwdBatch], sB[kBwdBatch];
  __shared__ double2 sD[5][kBwdBatch];
  __shared__ uint32_t sG[kBwdBatch];
  __shared__ uint4 sM[kBwdBatch][2];   // K5's composited-pixel words of the staged entries (K6 order)
  __shared__ uint32_t smax[kBwdThreads / 32];
#ifdef PUV_BWD_SMEM_RED
  __shared__ __align__(16) double sRed[kBwdThreads / 32][kRedRow * 9];
#endif
  __shared__ double sExp[kExpTab];
  exp64_table_fill(sExp);
  const int tile = blockIdx.x, view = view0 + blockIdx.y;   // dL_dimages starts at view0
  const int tx = tile % gx, ty = tile / gx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const ViewHdr& hdr = v.hdr[view];
  if (hdr.overflow) return;
#if PUV_DIRECT
  // the tile's entries: its super-tile's level-1 rank range, filtered by rect (feed.cuh)
  __shared__ uint32_t sGid[2 * kBwdBatch], sFeedCnt[kBwdThreads / 32 + 1];
  TileFeed<kBwdThreads, kBwdBatch> feed;
  {
    const ViewHdr& l1 = v.l1[view];
    const int st = (ty / kSup) * v.sgx + (tx / kSup);
    const uint32_t c0 = l1.overflow ? 0u : v.sst[(size_t)view * (v.nst + 1) + st];
    const uint32_t c1 = l1.overflow ? 0u : v.sen[(size_t)view * (v.nst + 1) + st];
    feed.init(sGid, sFeedCnt, c0, c1);
  }
  const uint32_t* list1 = arena + v.l1[view].list_base;
  const uint32_t* sorted_v = v.sorted + (size_t)view * N;
  const uint2* rect_v = v.rect + (size_t)view * N;
#else
  const uint32_t start = v.tstart[(size_t)view * ntiles + tile];
  const uint32_t* list = arena + hdr.list_base + start;
#endif
  const float4* rec = v.rec + (size_t)view * N * 2;
  const double2* rec64 = v.rec64 + (size_t)view * N * 5;
  double* g2 = v.grad2d + (size_t)view * N * 9;
  const size_t HW = (size_t)W * H;
  const float* dL_dimage = dL_dimages + (size_t)blockIdx.y * 3 * HW;
  float fi[kBwdPPT], fj[kBwdPPT];
  double di = 0.0, dj[kBwdPPT];
  uint32_t last[kBwdPPT];
  double dC[kBwdPPT][3], Sd[kBwdPPT], T[kBwdPPT];
  uint32_t tlast = 0;
#pragma unroll
  for (int k = 0; k < kBwdPPT; ++k) {
    // warp w owns columns 8(w&1).. of rows 4 PPT (w>>1)..; lane l column l&7, rows (l>>3)+4k
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTile + (warp >> 1) * 4 * kBwdPPT + (lane >> 3) + 4 * k;
    fi[k] = (float)px;
    fj[k] = (float)py;
    di = px;   // the same column for every k
    dj[k] = py;
    last[k] = 0;
    T[k] = 1.0;
    Sd[k] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) dC[k][c] = 0.0;
    if (px < W && py < H) {
      const size_t p = (size_t)py * W + px;
      last[k] = v.ncontrib[(size_t)view * HW + p];
      const double* cf = v.cfull + 3 * ((size_t)view * HW + p);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dC[k][c] = dL_dimage[c * HW + p];
        Sd[k] = fma(dC[k][c], cf[c], Sd[k]);   // Sd starts at dC . C (the full colour)
      }
    }
    tlast = max(tlast, last[k]);
  }
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, tlast);
  if (lane == 0) smax[warp] = wlast;
  __syncthreads();
  uint32_t bmax = 0;
#pragma unroll
  for (int w = 0; w < kBwdThreads / 32; ++w) bmax = max(bmax, smax[w]);

#if PUV_DIRECT
  for (uint32_t lo = 0; lo < bmax;) {
    const int nb = feed.next(list1, sorted_v, rect_v, tx, ty);
    if (nb == 0) break;
    const int n = (int)min((uint32_t)nb, bmax - lo);
    for (int i = threadIdx.x; i < n; i += kBwdThreads) {
      const uint32_t g = sGid[i];
      PUV_CHECK(g < (uint32_t)N);
      sG[i] = g;
#else
  for (uint32_t lo = 0; lo < bmax; lo += kBwdBatch) {
    const int n = (int)min((uint32_t)kBwdBatch, bmax - lo);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kBwdThreads) {
      const uint32_t g = list[lo + i];
      PUV_CHECK(g < (uint32_t)N && start + lo + i < hdr.K);
      sG[i] = g;
#endif
      sA[i] = rec[2 * (size_t)g + 0];
      sB[i] = rec[2 * (size_t)g + 1];
#pragma unroll
      for (int k = 0; k < 5; ++k) sD[k][i] = rec64[5 * (size_t)g + k];
      if (lo + i < (uint32_t)kMaskCap) {
        const uint4* m = reinterpret_cast<const uint4*>(v.dmask + (((size_t)view * ntiles + tile) * kMaskCap + lo + i) * 8);
        sM[i][0] = m[0];
        sM[i][1] = m[1];
      }
    }
    __syncthreads();
#if PUV_BWD_CULL
    // per-warp entry filter: an entry is walked only if some pixel of this warp may composite it --
    // K5's composited-pixel words of the warp are nonzero (first kMaskCap entries; stale words past
    // a pixel's end only keep an entry, never drop one), or, beyond the mask, the conservative
    // ellipse-vs-block test of K5 for the warp's 8 x 16 pixels
    uint32_t mwords[kBwdBatch / 32];
#pragma unroll
    for (int q = 0; q < kBwdBatch / 32; ++q) {
      const int j = 32 * q + lane;
      bool may = false;
      if (j < n && lo + j < wlast) {
        if (lo + j < (uint32_t)kMaskCap) {
          const uint4 w = sM[j][warp];
          may = (w.x | w.y | w.z | w.w) != 0u;
        } else {
          const float4 A = sA[j];
          const float4 B = sB[j];
          may = block_may_hit(A.x, A.y, A.z, A.w, B.x, B.y, (float)(tx * kTile + (warp & 1) * 8),
                              (float)(ty * kTile + (warp >> 1) * 4 * kBwdPPT), 7.f, (float)(4 * kBwdPPT - 1));
        }
      }
      mwords[q] = __ballot_sync(0xffffffffu, may);
    }
    static_assert(kBwdBatch == 64, "the walk keeps the batch's entry bits in one 64-bit word");
    for (uint64_t bits = ((uint64_t)mwords[1] << 32) | mwords[0]; bits; bits &= bits - 1) {
      const int j = __ffsll((long long)bits) - 1;
      const uint32_t e = lo + j;
#else
    for (int j = 0; j < n; ++j) {
      const uint32_t e = lo + j;
      if (e >= wlast) break;  // warp-uniform: no pixel of this warp reaches entry e
#endif
      const float4 B = sB[j];
      // decisions (fp32 contract), per pixel: the first kMaskCap entries from K5's composited
      // bits (bit = composited at this entry; guarded by e < last since K5 writes a warp's words
      // only until all its pixels terminated), later entries by replaying the skip test.  The cap
      // needs o (x) exp_c(power) >= 0.99 with power <= 0, where exp_c <= 1 (its last Horner step is
      // 1 + p r with r <= 0, or 2^k <= 1/2), so an entry with o < 0.99 is never capped: the
      // exp_c replay runs only for the (rare) entries with o >= 0.99 (warp-uniform branch).
      const bool may_cap = !(B.z < 0.99f);
      bool act[kBwdPPT], cap[kBwdPPT];
      bool any = false;
      // kact[k] (warp-uniform): some lane's pixel k (the warp's 8x4 sub-block k) may composite the
      // entry; a sub-block with none skips its body (PUV_BWD_KSKIP)
      bool kact[kBwdPPT];
      if (e < (uint32_t)kMaskCap) {
        static_assert(kBwdPPT == 4, "the K5 mask layout assumes 4 pixels per K6 thread");
        const uint4 mw = sM[j][warp];
        const uint32_t words[4] = {mw.x, mw.y, mw.z, mw.w};
#pragma unroll
        for (int k = 0; k < kBwdPPT; ++k) {
          // kMaskFill: every word up to the tile's largest n_contrib was written by K5 (zero past a
          // pixel's end), so the bit alone decides; else stale words past a K5 warp's stop need e < last
          act[k] = (kMaskFill || e < last[k]) && ((words[k] >> lane) & 1u);
          kact[k] = words[k] != 0u;   // a superset of the lanes' act (stale bits past last only add)
          any |= act[k];
        }
      } else {
        const float4 A = sA[j];
#pragma unroll
        for (int k = 0; k < kBwdPPT; ++k) {
          const float power = pair_power(A.x, A.y, A.z, A.w, B.x, fi[k], fj[k]);
          act[k] = e < last[k] && !(power > 0.0f || power < B.y);
          kact[k] = __any_sync(0xffffffffu, act[k]);
          any |= act[k];
        }
      }
#pragma unroll
      for (int k = 0; k < kBwdPPT; ++k) cap[k] = false;
      if (may_cap) {
        const float4 A = sA[j];
#pragma unroll
        for (int k = 0; k < kBwdPPT; ++k) {
          const float power = pair_power(A.x, A.y, A.z, A.w, B.x, fi[k], fj[k]);
          cap[k] = act[k] && !(mul(B.z, exp_c(fminf(power, 0.0f))) < 0.99f);
        }
      }
      if (!__any_sync(0xffffffffu, any)) continue;
      const double2 d0 = sD[0][j], d1 = sD[1][j], d2 = sD[2][j], d3 = sD[3][j];
      const double cb = sD[4][j].x;
      const double o = d2.y;
      // the thread's pixels share the column px: dx and its terms are computed once, and the
      // dx-only moments follow from the thread's sum of GdL (Mx = dx S, Mxx = dx^2 S)
      const double dx = d0.x - di, dxx = dx * dx;
      // kLno: ln o rides in the column term: exp64(power64) = alpha = o G, and GdL below is o G dL/da
      const double hadxx = kLno ? fma(d1.x, dxx, d2.y) : d1.x * dxx, nbdx = d1.y * dx;
      double gv[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};   // Mx, My, Mxx, Mxy, Myy, sum GdL, colour r, g, b
      double sdy = 0.0;                              // sum GdL dy (-> Mxy = dx sdy)
      // The pixel bodies, compiled twice: the alpha-cap selects exist only in the (warp-uniform,
      // rare: o >= 0.99) capped variant, so the common path carries no cap logic at all.
      auto bodies = [&](auto cap_tag) {
        constexpr bool kCap = decltype(cap_tag)::value;
#pragma unroll
        for (int k = 0; k < kBwdPPT; ++k) {
#if PUV_BWD_KSKIP
          if (!kact[k]) continue;   // warp-uniform: no pixel of sub-block k composites this entry
#endif
          const double dy = d0.y - dj[k];
#if PUV_BWD_EXPSEL
          // an inactive pixel gets G = e^-700 (~1e-304): its alpha, moments and colour terms vanish
          // below any nonzero fp64 sum, so the two result selects become one argument select
          const double pw = power64(d2.x, hadxx, nbdx, dy);
          const double G = exp64(act[k] ? pw : -700.0, sExp);
          double a = kLno ? G : o * G;
#else
          const double G = exp64(power64(d2.x, hadxx, nbdx, dy), sExp);
          double a = act[k] ? (kLno ? G : o * G) : 0.0;
#endif
          if (kCap) a = cap[k] ? 0.99 : a;
          const double aT = a * T[k];
          const double cd = fma(dC[k][0], d3.x, fma(dC[k][1], d3.y, dC[k][2] * cb));
          Sd[k] = fma(-cd, aT, Sd[k]);
          const double dLda = fma(cd, T[k], -Sd[k] * rcp64(1.0 - a));
          gv[6] = fma(aT, dC[k][0], gv[6]);
          gv[7] = fma(aT, dC[k][1], gv[7]);
          gv[8] = fma(aT, dC[k][2], gv[8]);
#if PUV_BWD_EXPSEL
          double GdL = G * dLda;
#else
          double GdL = act[k] ? G * dLda : 0.0;
#endif
          if (kCap) GdL = cap[k] ? 0.0 : GdL;   // capped: no gradient through alpha
          gv[5] += GdL;
          sdy = fma(GdL, dy, sdy);
          gv[4] = fma(GdL * dy, dy, gv[4]);
          T[k] -= aT;                             // T_{k+1} = T_k (1 - a_k)
        }
      };
#if PUV_BWD_CAPSPLIT
      if (__builtin_expect(may_cap, 0)) bodies(std::true_type{});
      else bodies(std::false_type{});
#else
      bodies(std::true_type{});   // (A/B reference: one body with the cap selects; cap[] is all-false unless may_cap)
#endif
      gv[0] = dx * gv[5];
      gv[1] = sdy;
      gv[2] = dxx * gv[5];
      gv[3] = dx * sdy;
      // raw moments into the (view, Gaussian) slot; K7 turns them into dL/d(mx, my, ha, nb, hc)
#ifndef PUV_BWD_SMEM_RED
      const double s = warp_reduce9_shfl(gv);
      double* dst = g2 + 9 * (size_t)sG[j];
      if ((lane & 3) == 0) atomicAdd(dst + (lane >> 2), s);
      if (lane == 1) atomicAdd(dst + 8, gv[8]);
#else
      const double s = warp_sum9(gv, sRed[warp], lane);
      if (lane < 27 && lane % 3 == 0) atomicAdd(g2 + 9 * (size_t)sG[j] + lane / 3, s);
#endif
    }
#if PUV_DIRECT
    lo += (uint32_t)nb;
    feed.pop(nb);
#endif
  }
}

void launch_raster_bwd(const Plan& p, const Views& v, const uint32_t* arena, const float* dL_dimages, int view0,
                       int n_views, cudaStream_t s) {
  if (n_views <= 0 || p.ntiles <= 0) return;
  const dim3 grid(p.ntiles, n_views);
#if PUV_RASTER_CARVEOUT >= 0
  // shared-memory carveout preference (percent): lets the driver pick a larger carveout so the
  // register-limited residency is not capped by the shared-memory configuration
  static const bool carve_once =
      cudaFuncSetAttribute(k_raster_bwd, cudaFuncAttributePreferredSharedMemoryCarveout, PUV_RASTER_CARVEOUT) == cudaSuccess;
  (void)carve_once;
#endif
  k_raster_bwd<<<grid, kBwdThreads, 0, s>>>(arena, v, p.N, p.W, p.H, p.gx, p.ntiles, view0, dL_dimages);
  count_launches(1);
}

}  // namespace puv
