// K6 k_raster_bwd — per-tile gradient of the front-to-back composite (row a7).
//
// One 128-thread block (4 warps) per 16x16 tile; warp w owns the 8x8 pixel
// quadrant (8(w&1), 8(w>>1)); lane l owns column l & 7 and rows (l >> 3) + 4k,
// k < PPT = 2.  Every decision (skip test R1, alpha cap, composited set R14) is
// replayed with the fp32 contract exactly as K5 took it; every VALUE is fp64
// (DESIGN.md §5).  Single pass in front-to-back order, using the pixel's full
// colour C from K5:
//   T_k = prod_{i<k} (1 - a_i),   P_k = sum_{i<=k} c_i a_i T_i,   S_k = C - P_k
//   dL/dc_k = a_k T_k dL/dC
//   dL/da_k = sum_ch dL/dC (T_k c_k - S_k / (1 - a_k))
//   uncapped: dL/do = G dL/da, dL/dpower = o G dL/da -> (mx, my, ha, nb, hc)
// The per-pixel body is branch-free (inactive pixels get a = 0 and masked
// terms), so the pixels' fp64 chains interleave (ncu: the branchy version was
// bound by fixed-latency "wait" stalls).  A thread sums the 9 values of an
// entry over its pixels; the warp sums them with a transposing butterfly
// (8 values in 9 double shuffles, the 9th in 5) and 9 lanes issue one fp64
// atomic each into the (view, Gaussian) gradient slot.
#include "contract.cuh"
#include "internal.cuh"

namespace puv {

constexpr int kBwdPPT = 2;                                 // pixels per thread
constexpr int kBwdThreads = kTile * kTile / kBwdPPT;        // 128
constexpr int kBwdBatch = 128;                             // entries staged per batch

// Sum v[0..7] across the warp (lane l ends with the total of value (l >> 2) & 7) and v8 (all lanes).
__device__ __forceinline__ double warp_reduce9(double (&x)[8], double& v8) {
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
  for (int off = 16; off > 0; off >>= 1) v8 += __shfl_xor_sync(0xffffffffu, v8, off);
  return s;
}

// 1/y for y in [0.01, 1]: fp32 reciprocal estimate + two Newton steps in fp64 (~1 ulp)
__device__ __forceinline__ double rcp64(double y) {
  double r = (double)__frcp_rn((float)y);
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

__global__ void __launch_bounds__(kBwdThreads) k_raster_bwd(const uint32_t* __restrict__ arena, Views v, int view,
                                                           int N, int W, int H, int gx, int ntiles,
                                                           const float* __restrict__ dL_dimage) {
  __shared__ float4 sA[kBwdBatch], sB[kBwdBatch];
  __shared__ double2 sD[5][kBwdBatch];
  __shared__ uint32_t sG[kBwdBatch];
  __shared__ uint32_t smax[kBwdThreads / 32];
  __shared__ double sExp[64];
  exp64_table_fill(sExp);
  const int tile = blockIdx.x;
  const int tx = tile % gx, ty = tile / gx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const ViewHdr& hdr = v.hdr[view];
  if (hdr.overflow) return;
  const uint32_t start = v.tstart[(size_t)view * ntiles + tile];
  const uint32_t* list = arena + hdr.list_base + start;
  const float4* rec = v.rec + (size_t)view * N * 3;
  const double2* rec64 = v.rec64 + (size_t)view * N * 5;
  double* g2 = v.grad2d + (size_t)view * N * 9;
  const size_t HW = (size_t)W * H;
  float fi[kBwdPPT], fj[kBwdPPT];
  uint32_t last[kBwdPPT];
  float dC[kBwdPPT][3];
  double S[kBwdPPT][3], T[kBwdPPT];
  uint32_t tlast = 0;
#pragma unroll
  for (int k = 0; k < kBwdPPT; ++k) {
    // compact 8x8 warp footprint: warp w owns quadrant (8(w&1), 8(w>>1)), lane l column l&7, rows (l>>3)+4k
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTile + (warp >> 1) * 8 + (lane >> 3) + 4 * k;
    fi[k] = (float)px;
    fj[k] = (float)py;
    last[k] = 0;
    T[k] = 1.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) { dC[k][c] = 0.f; S[k][c] = 0.0; }
    if (px < W && py < H) {
      const size_t p = (size_t)py * W + px;
      last[k] = v.ncontrib[(size_t)view * HW + p];
      const double* cf = v.cfull + 3 * ((size_t)view * HW + p);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dC[k][c] = dL_dimage[c * HW + p];
        S[k][c] = cf[c];           // S starts at the full colour C; S_k = C - P_k
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

  for (uint32_t lo = 0; lo < bmax; lo += kBwdBatch) {
    const int n = (int)min((uint32_t)kBwdBatch, bmax - lo);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kBwdThreads) {
      const uint32_t g = list[lo + i];
      sG[i] = g;
      sA[i] = rec[3 * (size_t)g + 0];
      sB[i] = rec[3 * (size_t)g + 1];
#pragma unroll
      for (int k = 0; k < 5; ++k) sD[k][i] = rec64[5 * (size_t)g + k];
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const uint32_t e = lo + j;
      if (e >= wlast) break;  // warp-uniform: no pixel of this warp reaches entry e
      const float4 A = sA[j], B = sB[j];
      // decisions (fp32 contract), per pixel
      bool act[kBwdPPT], cap[kBwdPPT];
      bool any = false;
#pragma unroll
      for (int k = 0; k < kBwdPPT; ++k) {
        const float power = pair_power(A.x, A.y, A.z, A.w, B.x, fi[k], fj[k]);
        act[k] = e < last[k] && !(power > 0.0f || power < B.y);
        cap[k] = act[k] && !(mul(B.z, exp_c(fminf(power, 0.0f))) < 0.99f);
        any |= act[k];
      }
      if (!__any_sync(0xffffffffu, any)) continue;
      const double2 d0 = sD[0][j], d1 = sD[1][j], d2 = sD[2][j], d3 = sD[3][j];
      const double d4x = sD[4][j].x;
      double gv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      double gb = 0.0;
#pragma unroll
      for (int k = 0; k < kBwdPPT; ++k) {
        const double dx = d0.x - (double)fi[k], dy = d0.y - (double)fj[k];
        const double pw = fmax(fma(d1.x * dx, dx, fma(d1.y * dx, dy, d2.x * dy * dy)), -700.0);
        const double G = exp64(fmin(pw, 0.0), sExp);
        const double a = act[k] ? (cap[k] ? 0.99 : d2.y * G) : 0.0;
        const double aT = a * T[k];
        S[k][0] = fma(-d3.x, aT, S[k][0]);
        S[k][1] = fma(-d3.y, aT, S[k][1]);
        S[k][2] = fma(-d4x, aT, S[k][2]);
        const double iom = rcp64(1.0 - a);
        const double c0 = dC[k][0], c1 = dC[k][1], c2 = dC[k][2];
        const double dLda = c0 * (T[k] * d3.x - S[k][0] * iom) + c1 * (T[k] * d3.y - S[k][1] * iom) +
                            c2 * (T[k] * d4x - S[k][2] * iom);
        gv[6] = fma(aT, c0, gv[6]);
        gv[7] = fma(aT, c1, gv[7]);
        gb = fma(aT, c2, gb);
        const double GdL = (act[k] && !cap[k]) ? G * dLda : 0.0;
        const double dP = d2.y * GdL;                        // d alpha / d power = o G
        gv[5] += GdL;                                        // d alpha / d o = G
        gv[2] = fma(dx * dx, dP, gv[2]);
        gv[3] = fma(dx * dy, dP, gv[3]);
        gv[4] = fma(dy * dy, dP, gv[4]);
        gv[0] = fma(2.0 * d1.x * dx + d1.y * dy, dP, gv[0]);
        gv[1] = fma(d1.y * dx + 2.0 * d2.x * dy, dP, gv[1]);
        T[k] -= aT;                                          // T_{k+1} = T_k (1 - a_k)
      }
      const double s = warp_reduce9(gv, gb);
      double* dst = g2 + 9 * (size_t)sG[j];
      if ((lane & 3) == 0) atomicAdd(dst + (lane >> 2), s);
      if (lane == 1) atomicAdd(dst + 8, gb);
    }
  }
}

void launch_raster_bwd(const Plan& p, const Views& v, const uint32_t* arena, const float* dL_dimage, int view,
                       const float bg[3], cudaStream_t s) {
  (void)bg;  // the background enters through the forward's full colour C
  k_raster_bwd<<<p.ntiles, kBwdThreads, 0, s>>>(arena, v, view, p.N, p.W, p.H, p.gx, p.ntiles, dL_dimage);
  count_launches(1);
}

}  // namespace puv
