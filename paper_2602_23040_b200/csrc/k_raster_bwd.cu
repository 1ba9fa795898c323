// K6 k_raster_bwd — per-tile gradient of the front-to-back composite (row a7).
//
// One 256-thread block per 16x16 tile, one pixel per thread.  Every decision
// (skip test R1, alpha cap and composited set R14) is replayed with the fp32
// contract exactly as K5 took it; every VALUE is fp64 from the 80-byte value
// record (fp32 values cannot hold 1e-3 relative per component
// on cancellation-heavy gradient components).
//   pass A (front to back): T_final = prod (1 - alpha_k) over the composited entries
//   pass B (back to front): T_k = T_{k+1} / (1 - alpha_k);
//     dL/dc_k = alpha_k T_k dL/dC
//     dL/dalpha_k = sum_c dL/dC_c (T_k c_k,c - S_k,c / (1 - alpha_k)),  S_k = sum_{i>k} c_i alpha_i T_i + T_final bg
//     uncapped: dL/do = G dL/dalpha, dL/dpower = o G dL/dalpha -> (mx, my, ha, nb, hc)
// The 9 values of an entry are summed across the warp with a transposing
// butterfly (16 double shuffles instead of 45), then 9 lanes issue one fp64
// atomic each into the (view, Gaussian) gradient slot.
#include "contract.cuh"
#include "internal.cuh"

namespace puv {

constexpr int kBwdThreads = kTile * kTile;

// Sum 16 values across the warp; afterwards lane l holds the total of value (l >> 1).
__device__ __forceinline__ double butterfly16(double (&x)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int level = 0; level < 4; ++level) {
    const int half = 8 >> level;
    const int off = 16 >> level;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? x[i] : x[i + half];
      const double keep = upper ? x[i + half] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return x[0] + __shfl_xor_sync(0xffffffffu, x[0], 1);
}

struct PairEval {
  bool act;
  bool capped;
  double a, G, dx, dy;
};

// Decision (fp32 contract) + value (fp64) of one (pixel, entry) pair.
__device__ __forceinline__ PairEval eval_pair(const float4& A, const float4& B, const double2& d0, const double2& d1,
                                              const double2& d2, float fi, float fj) {
  PairEval e;
  const float power = pair_power(A.x, A.y, A.z, A.w, B.x, fi, fj);
  e.act = !(power > 0.0f || power < B.y);
  if (!e.act) return e;
  const float ao = mul(B.z, exp_c(power));
  e.capped = !(ao < 0.99f);
  e.dx = d0.x - (double)fi;
  e.dy = d0.y - (double)fj;
  const double pw = d1.x * e.dx * e.dx + d1.y * e.dx * e.dy + d2.x * e.dy * e.dy;
  e.G = exp(pw);
  e.a = e.capped ? 0.99 : d2.y * e.G;
  return e;
}

__global__ void __launch_bounds__(kBwdThreads) k_raster_bwd(const uint32_t* __restrict__ arena, Views v, int view,
                                                           int N, int W, int H, int gx, int ntiles, float bg0,
                                                           float bg1, float bg2, const float* __restrict__ dL_dimage) {
  __shared__ float4 sA[kBwdThreads], sB[kBwdThreads];
  __shared__ double2 sD[5][kBwdThreads];
  __shared__ uint32_t sG[kBwdThreads];
  __shared__ uint32_t smax[kBwdThreads / 32];
  const int tile = blockIdx.x;
  const int tx = tile % gx, ty = tile / gx;
  const int px = tx * kTile + (threadIdx.x & (kTile - 1));
  const int py = ty * kTile + (threadIdx.x / kTile);
  const bool inside = px < W && py < H;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const ViewHdr& hdr = v.hdr[view];
  if (hdr.overflow) return;
  const uint32_t start = v.tstart[(size_t)view * ntiles + tile];
  const uint32_t* list = arena + hdr.list_base + start;
  const float4* rec = v.rec + (size_t)view * N * 3;
  const double2* rec64 = v.rec64 + (size_t)view * N * 5;
  double* g2 = v.grad2d + (size_t)view * N * 9;
  const size_t HW = (size_t)W * H, p = (size_t)py * W + px;
  double d0 = 0.0, d1 = 0.0, d2 = 0.0;
  uint32_t last = 0;
  if (inside) {
    last = v.ncontrib[(size_t)view * HW + p];
    d0 = dL_dimage[p];
    d1 = dL_dimage[HW + p];
    d2 = dL_dimage[2 * HW + p];
  }
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, last);
  if (lane == 0) smax[warp] = wlast;
  __syncthreads();
  uint32_t bmax = 0;
#pragma unroll
  for (int w = 0; w < kBwdThreads / 32; ++w) bmax = max(bmax, smax[w]);
  const float fi = (float)px, fj = (float)py;

  auto load = [&](uint32_t lo, int n) {
    if ((int)threadIdx.x < n) {
      const uint32_t g = list[lo + threadIdx.x];
      sG[threadIdx.x] = g;
      sA[threadIdx.x] = rec[3 * (size_t)g + 0];
      sB[threadIdx.x] = rec[3 * (size_t)g + 1];
#pragma unroll
      for (int k = 0; k < 5; ++k) sD[k][threadIdx.x] = rec64[5 * (size_t)g + k];
    }
  };

  // pass A: fp64 transmittance after the last composited entry
  double T = 1.0;
  for (uint32_t lo = 0; lo < bmax; lo += kBwdThreads) {
    const int n = (int)min((uint32_t)kBwdThreads, bmax - lo);
    __syncthreads();
    load(lo, n);
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const uint32_t e = lo + j;
      if (e >= wlast) break;  // warp-uniform
      if (e < last) {
        const PairEval pe = eval_pair(sA[j], sB[j], sD[0][j], sD[1][j], sD[2][j], fi, fj);
        if (pe.act) T *= 1.0 - pe.a;
      }
    }
  }
  double S0 = T * bg0, S1 = T * bg1, S2 = T * bg2;

  // pass B: reverse replay
  for (int64_t hi = (int64_t)bmax; hi > 0; hi -= kBwdThreads) {
    const int64_t lo = hi - kBwdThreads > 0 ? hi - kBwdThreads : 0;
    const int n = (int)(hi - lo);
    __syncthreads();
    load((uint32_t)lo, n);
    __syncthreads();
    for (int j = n - 1; j >= 0; --j) {
      const uint32_t e = (uint32_t)(lo + j);
      if (e >= wlast) continue;  // warp-uniform: no pixel of this warp reached entry e
      double gv[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) gv[k] = 0.0;
      bool act = false;
      if (e < last) {
        const PairEval pe = eval_pair(sA[j], sB[j], sD[0][j], sD[1][j], sD[2][j], fi, fj);
        act = pe.act;
        if (act) {
          const double2 c01 = sD[3][j], c2x = sD[4][j];
          const double om = 1.0 - pe.a;
          const double iom = 1.0 / om;
          T *= iom;                                    // T_k (before compositing entry k)
          const double aT = pe.a * T;
          gv[6] = aT * d0;
          gv[7] = aT * d1;
          gv[8] = aT * d2;
          const double dLda = d0 * (T * c01.x - S0 * iom) + d1 * (T * c01.y - S1 * iom) + d2 * (T * c2x.x - S2 * iom);
          S0 = fma(c01.x, aT, S0);
          S1 = fma(c01.y, aT, S1);
          S2 = fma(c2x.x, aT, S2);
          if (!pe.capped) {
            const double2 m = sD[0][j], hn = sD[1][j], ho = sD[2][j];
            const double dP = ho.y * pe.G * dLda;       // d alpha / d power = o G
            gv[5] = pe.G * dLda;                          // d alpha / d o = G
            gv[2] = pe.dx * pe.dx * dP;
            gv[3] = pe.dx * pe.dy * dP;
            gv[4] = pe.dy * pe.dy * dP;
            gv[0] = (2.0 * hn.x * pe.dx + hn.y * pe.dy) * dP;
            gv[1] = (hn.y * pe.dx + 2.0 * ho.x * pe.dy) * dP;
            (void)m;
          }
        }
      }
      if (__any_sync(0xffffffffu, act)) {
        const double s = butterfly16(gv);
        const int vi = lane >> 1;
        if ((lane & 1) == 0 && vi < 9) atomicAdd(g2 + 9 * (size_t)sG[j] + vi, s);
      }
    }
  }
}

void launch_raster_bwd(const Plan& p, const Views& v, const uint32_t* arena, const float* dL_dimage, int view,
                       const float bg[3], cudaStream_t s) {
  k_raster_bwd<<<p.ntiles, kBwdThreads, 0, s>>>(arena, v, view, p.N, p.W, p.H, p.gx, p.ntiles, bg[0], bg[1], bg[2],
                                                dL_dimage);
  count_launches(1);
}

}  // namespace puv
