// K1 k_project — fused atlas unpack + EWA projection + SH colour + tile rect (rows a1, a2).
//
// One thread per texel; the texel's planes are read ONCE (coalesced SoA loads)
// and the thread loops over up to kCamBatch views.  Per visible (view, Gaussian)
// it writes: the depth key and tile rect (fp32 contract, R13 -> binning), the
// 32-byte fp32 record (contract conic/mean/t_g/o -> every compositing decision, and
// the SH clamp bits for K7) and the 80-byte fp64 value record (mean, conic, o and
// colour in double -> the composited values of K5 and K6): 124 B.  The (view, Gaussian) 2D-gradient slots
// K6 accumulates into are zeroed by the backward call itself (re-entrant backward).
#include "project.cuh"

namespace puv {

template <int DEG, bool LPO>
#ifndef PUV_PROJ_SH_SMEM
#define PUV_PROJ_SH_SMEM 1
#endif
#ifndef PUV_PROJ_MINB
#define PUV_PROJ_MINB 4
#endif
__global__ void __launch_bounds__(128, PUV_PROJ_MINB) k_project(PlaneTab P, PosMode pm, const uint8_t* __restrict__ occ, int N,
                                                 const __grid_constant__ CamBatch cb, Views v, int gx, int gy,
                                                 int g0, int g1) {
  const int g = g0 + blockIdx.x * blockDim.x + threadIdx.x;   // texels [g0, g1) of the N
  if (g >= g1) return;
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const bool occupied = occ == nullptr || occ[g] != 0;
  float mux = 0.f, muy = 0.f, muz = 0.f;
  if (occupied) texel_mu<LPO>(P, pm, g, mux, muy, muz);
  const float ls0 = plane_value<LPO>(P, 3, g), ls1 = plane_value<LPO>(P, 4, g), ls2 = plane_value<LPO>(P, 5, g);
  const float qw = plane_value<LPO>(P, 6, g), qx = plane_value<LPO>(P, 7, g), qy = plane_value<LPO>(P, 8, g),
              qz = plane_value<LPO>(P, 9, g);
  const float logit = plane_value<LPO>(P, 10, g);
  const Unpacked u = unpack_contract(ls0, ls1, ls2, qw, qx, qy, qz, logit);
  bool any = false;
  Unpacked64 u64;
  double lno = 0.0;   // ln o = -log1p(e^-logit), once per texel (kLno)
#if PUV_PROJ_SH_SMEM
  // the texel's SH coefficients widened to fp64 once (not per view): [3 NK][128] doubles
  __shared__ double sSH[3 * NK][128];
  const int tid = threadIdx.x;
#define PUV_SH(k) sSH[k][tid]
#else
  float sh[3 * NK];
#define PUV_SH(k) ((double)sh[k])
#endif

  for (int i = 0; i < cb.n; ++i) {
    const CamDev& c = cb.c[i];
    const size_t o = (size_t)(cb.v0 + i) * (size_t)N + (size_t)g;
    Proj pr;
    pr.vis = false;
    CamPoint cp;
    if (occupied && u.ok) {
      cp = cam_point(c, mux, muy, muz);
      pr = project_contract(c, cp, u, gx, gy);
    }
    if (!pr.vis) {
      v.depth[o] = kInvisible;
      continue;
    }
    if (!any) {  // first visible view of this texel: fp64 unpack + SH coefficients
      any = true;
      u64 = unpack64(ls0, ls1, ls2, qw, qx, qy, qz, logit);
      if (kLno) lno = -log1p(exp(-(double)logit));
#pragma unroll
#if PUV_PROJ_SH_SMEM
      for (int k = 0; k < 3 * NK; ++k) sSH[k][tid] = plane_value<LPO>(P, 11 + k, g);
#else
      for (int k = 0; k < 3 * NK; ++k) sh[k] = plane_value<LPO>(P, 11 + k, g);
#endif
    }
    const Proj64 p64 = project64(c, mux, muy, muz, u64, cp.clx, cp.cly);
    // SH colour (R3) in fp64; the clamp decision is recorded for K7
    double dx = (double)mux - c.campos64[0], dy = (double)muy - c.campos64[1], dz = (double)muz - c.campos64[2];
    const double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    dx *= inv; dy *= inv; dz *= inv;
    double Y[NK];
    sh_basis<DEG, double>(dx, dy, dz, Y);
    double rgb[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double acc = 0.5;
#pragma unroll
      for (int k = 0; k < NK; ++k) acc = fma(Y[k], PUV_SH(3 * k + ch), acc);
      rgb[ch] = acc;
    }
    uint32_t flags = 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      if (rgb[ch] < 0.0) { rgb[ch] = 0.0; flags |= 1u << ch; }
    v.depth[o] = pr.depth_bits;
    v.rect[o] = make_uint2((uint32_t)pr.x0 | ((uint32_t)pr.x1 << 16), (uint32_t)pr.y0 | ((uint32_t)pr.y1 << 16));
    float4* rec = v.rec + 2 * o;
    rec[0] = make_float4(pr.mx, pr.my, pr.ha, pr.nb);
    rec[1] = make_float4(pr.hc, u.t_g, u.o, __uint_as_float(flags));
    double2* r64 = v.rec64 + 5 * o;
    r64[0] = make_double2(p64.mx, p64.my);
    r64[1] = make_double2(p64.ha, p64.nb);
    r64[2] = make_double2(p64.hc, kLno ? lno : u64.o);
    r64[3] = make_double2(rgb[0], rgb[1]);
    r64[4] = make_double2(rgb[2], 0.0);
  }
}

void launch_project(const Plan& p, const Views& v, const PlaneTab& P, const uint8_t* occ, const CamBatch& cb,
                    cudaStream_t s, int g0, int g1) {
  if (g1 < 0) g1 = p.N;
  if (g1 <= g0) return;
  const int threads = 128;
  const int blocks = (g1 - g0 + threads - 1) / threads;
#define PUV_K1(D, L) k_project<D, L><<<blocks, threads, 0, s>>>(P, p.pm, occ, p.N, cb, v, p.gx, p.gy, g0, g1)
  const bool lpo = P.qspec != nullptr;
  switch (p.deg) {
    case 0: if (lpo) PUV_K1(0, true); else PUV_K1(0, false); break;
    case 1: if (lpo) PUV_K1(1, true); else PUV_K1(1, false); break;
    case 2: if (lpo) PUV_K1(2, true); else PUV_K1(2, false); break;
    default: if (lpo) PUV_K1(3, true); else PUV_K1(3, false); break;
  }
#undef PUV_K1
  count_launches(1);
}

}  // namespace puv
