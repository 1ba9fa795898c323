// K7 k_project_bwd — projection backward + unpack backward + scatter to texels (rows a8, a9).
//
// One thread per texel.  For each view of the batch it reads the 9 per-(view,
// Gaussian) 2D gradients accumulated by K6 (mean2D 2, conic 3, opacity 1,
// rgb 3; fp64) and applies the chain rule of DESIGN.md §1 in fp64 (§5):
// conic <- Sigma2D (+0.3), Sigma2D <- (T = J V, Sigma), J <- camera-space mean
// (a J-clamped coordinate has zero derivative, R5 — the clamp decision is the
// fp32 contract one), mean2D <- mean, colour <- (view direction, SH
// coefficients) with clamped channels zeroed (R3).  Covariance gradients are
// summed over the views first (Sigma does not depend on the view) and pushed
// through Sigma = R diag(s^2) R^T, q_hat = q/|q|, s = exp(ls), o = sigmoid(l)
// once.  The texel's gradient is multiplied by its dynamic label D_i
// and ACCUMULATED into the caller's fp32 gradient planes.
#include "project.cuh"

namespace puv {

#ifndef PUV_PBWD_PREFETCH
#define PUV_PBWD_PREFETCH 1
#endif

// cp.async (global -> shared, asynchronous, per thread): the next view's depth key and 9 moments
// are in flight while the current view's chain rule runs, without registers to hold them.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
#ifndef PUV_PBWD_STAGES
#define PUV_PBWD_STAGES 4
#endif
constexpr int kPbwdStages = PUV_PBWD_STAGES;   // staging buffers: views in flight = stages - 1

#ifndef PUV_PBWD_SH_SMEM
#define PUV_PBWD_SH_SMEM 1
#endif
template <int DEG, bool LPO>
#ifndef PUV_PBWD_MINB
#define PUV_PBWD_MINB 1
#endif
__global__ void __launch_bounds__(128, PUV_PBWD_MINB) k_project_bwd(PlaneTab P, PosMode pm, const uint8_t* __restrict__ occ,
                                                    const uint8_t* __restrict__ mask, int N,
                                                    const __grid_constant__ CamBatch cb, Views v, GradTab Gt,
                                                    int g0, int g1, int overwrite) {
  const int g = g0 + blockIdx.x * blockDim.x + threadIdx.x;   // texels [g0, g1) of the N
  if (g >= g1) return;
  constexpr int NK = (DEG + 1) * (DEG + 1);
  // overwrite: the first K7 of a train step WRITES the texel's gradient (zeros where it has none),
  // so the step needs neither a memset of the planes nor a read-modify-write
  auto put = [&](int d, float x) {
    if (overwrite) Gt.p[d][g] = x;
    else Gt.p[d][g] += x;
  };
  auto zero_all = [&]() {
    if (!overwrite) return;
#pragma unroll
    for (int d = 0; d < 11 + 3 * NK; ++d)
      if (Gt.p[d]) Gt.p[d][g] = 0.0f;
  };
  if (occ != nullptr && occ[g] == 0) { zero_all(); return; }
  if (mask != nullptr && mask[g] == 0) { zero_all(); return; }   // gradient freezing: D_i = 0 (no work)
  bool any = false;
  for (int i = 0; i < cb.n; ++i) any |= v.depth[(size_t)(cb.v0 + i) * N + g] != kInvisible;
  if (!any) { zero_all(); return; }

  float fmx, fmy, fmz;
  texel_mu<LPO>(P, pm, g, fmx, fmy, fmz);   // the fp32 position the render saw (xyz or c (+) rho (x) ray)
  const double mux = fmx, muy = fmy, muz = fmz;
  const float ls0 = plane_value<LPO>(P, 3, g), ls1 = plane_value<LPO>(P, 4, g), ls2 = plane_value<LPO>(P, 5, g);
  const float qw = plane_value<LPO>(P, 6, g), qx = plane_value<LPO>(P, 7, g), qy = plane_value<LPO>(P, 8, g),
              qz = plane_value<LPO>(P, 9, g);
  const float logit = plane_value<LPO>(P, 10, g);
  const Unpacked64 u = unpack64(ls0, ls1, ls2, qw, qx, qy, qz, logit);

  double dmu0 = 0, dmu1 = 0, dmu2 = 0, dop = 0;
  double G00 = 0, G01 = 0, G02 = 0, G11 = 0, G12 = 0, G22 = 0;  // G = dSigma + dSigma^T
#if PUV_PBWD_SH_SMEM
  // the texel's SH coefficients k >= 1 widened to fp64 once (dynamic smem [3 (NK - 1)][128]), not
  // re-read and converted per view
  extern __shared__ double sSHd[];
  for (int k = 3; k < 3 * NK; ++k) sSHd[(k - 3) * 128 + threadIdx.x] = plane_value<LPO>(P, 11 + k, g);
#define PUV_SHW(i) sSHd[((i) - 3) * 128 + threadIdx.x]
#else
#define PUV_SHW(i) ((double)plane_value<LPO>(P, 11 + (i), g))
#endif
  double dsh[3 * NK];
#pragma unroll
  for (int k = 0; k < 3 * NK; ++k) dsh[k] = 0.0;

#if PUV_PBWD_PREFETCH
  // double-buffered per-thread staging of (depth key, 9 moments) of view i + 1 while view i runs
  __shared__ double sG2[kPbwdStages][9][128];
  __shared__ uint32_t sDep[kPbwdStages][128];
  const int tid = threadIdx.x;
  auto prefetch = [&](int i, int buf) {
    if (i < cb.n) {
      const size_t o = (size_t)(cb.v0 + i) * N + g;
      cp_async4(&sDep[buf][tid], v.depth + o);
      const double* src = v.grad2d + 9 * o;
#pragma unroll
      for (int k = 0; k < 9; ++k) cp_async8(&sG2[buf][k][tid], src + k);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int j = 0; j < kPbwdStages - 1; ++j) prefetch(j, j);
#endif
  for (int i = 0; i < cb.n; ++i) {
    const size_t o = (size_t)(cb.v0 + i) * N + g;
#if PUV_PBWD_PREFETCH
    prefetch(i + kPbwdStages - 1, (i + kPbwdStages - 1) % kPbwdStages);
    cp_async_wait<kPbwdStages - 1>();   // view i's group has landed (only the next views' may be pending)
    const int buf = i % kPbwdStages;
    if (sDep[buf][tid] == kInvisible) continue;
    // K6's raw moments (Mx, My, Mxx, Mxy, Myy, dL/do, dL/drgb): see k_raster_bwd.cu
    const double Mx = sG2[buf][0][tid], My = sG2[buf][1][tid], Mxx = sG2[buf][2][tid], Mxy = sG2[buf][3][tid],
                 Myy = sG2[buf][4][tid], dO = sG2[buf][5][tid];
    const double dr = sG2[buf][6][tid], dg = sG2[buf][7][tid], db_ = sG2[buf][8][tid];
#else
    if (v.depth[o] == kInvisible) continue;
    // K6's raw moments (Mx, My, Mxx, Mxy, Myy, dL/do, dL/drgb): see k_raster_bwd.cu
    const double* g2 = v.grad2d + 9 * o;
    const double Mx = g2[0], My = g2[1], Mxx = g2[2], Mxy = g2[3], Myy = g2[4], dO = g2[5];
    const double dr = g2[6], dg = g2[7], db_ = g2[8];
#endif
    if (Mx == 0 && My == 0 && Mxx == 0 && Mxy == 0 && Myy == 0 && dO == 0 && dr == 0 && dg == 0 && db_ == 0)
      continue;
    const CamDev& c = cb.c[i];
    const CamPoint cp = cam_point(c, fmx, fmy, fmz);  // fp32 contract: the same J-clamp decisions as K1
    const Proj64 p = project64(c, mux, muy, muz, u, cp.clx, cp.cly);
    const double a = p.a, b = p.b, cc = p.c, id2 = 1.0 / (p.det * p.det);
    // power = ha dx^2 + nb dx dy + hc dy^2 with (ha, nb, hc) = (-c/2, b, -a/2) / det, alpha = o e^power
    const double idet = 1.0 / p.det, ha = -0.5 * cc * idet, nb = b * idet, hc = -0.5 * a * idet;
    // kLno: K6's moments are already o-scaled (sums of alpha dL/dalpha = o G dL/dalpha)
    const double os = kLno ? 1.0 : u.o;
    const double dmx = os * (2.0 * ha * Mx + nb * My), dmy = os * (nb * Mx + 2.0 * hc * My);
    const double dha = os * Mxx, dnb = os * Mxy, dhc = os * Myy;
    // conic (ha, nb, hc) = (-c/2, b, -a/2) / det
    const double da = (dha * 0.5 * cc * cc - dnb * b * cc + dhc * 0.5 * b * b) * id2;
    const double db = (-dha * b * cc + dnb * (a * cc + b * b) - dhc * a * b) * id2;
    const double dc = (dha * 0.5 * b * b - dnb * a * b + dhc * 0.5 * a * a) * id2;
    const double* T0 = p.T0;
    const double* T1 = p.T1;
    // G += dS + dS^T,  dS_ij = da t0i t0j + db t0i t1j + dc t1i t1j
    G00 += 2 * (da * T0[0] * T0[0] + db * T0[0] * T1[0] + dc * T1[0] * T1[0]);
    G11 += 2 * (da * T0[1] * T0[1] + db * T0[1] * T1[1] + dc * T1[1] * T1[1]);
    G22 += 2 * (da * T0[2] * T0[2] + db * T0[2] * T1[2] + dc * T1[2] * T1[2]);
    G01 += 2 * da * T0[0] * T0[1] + db * (T0[0] * T1[1] + T1[0] * T0[1]) + 2 * dc * T1[0] * T1[1];
    G02 += 2 * da * T0[0] * T0[2] + db * (T0[0] * T1[2] + T1[0] * T0[2]) + 2 * dc * T1[0] * T1[2];
    G12 += 2 * da * T0[1] * T0[2] + db * (T0[1] * T1[2] + T1[1] * T0[2]) + 2 * dc * T1[1] * T1[2];
    // dT = (2 da S t0 + db S t1, 2 dc S t1 + db S t0)
    const double St0[3] = {u.S00 * T0[0] + u.S01 * T0[1] + u.S02 * T0[2], u.S01 * T0[0] + u.S11 * T0[1] + u.S12 * T0[2],
                           u.S02 * T0[0] + u.S12 * T0[1] + u.S22 * T0[2]};
    const double St1[3] = {u.S00 * T1[0] + u.S01 * T1[1] + u.S02 * T1[2], u.S01 * T1[0] + u.S11 * T1[1] + u.S12 * T1[2],
                           u.S02 * T1[0] + u.S12 * T1[1] + u.S22 * T1[2]};
    double dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double dT0 = 2 * da * St0[k] + db * St1[k];
      const double dT1 = 2 * dc * St1[k] + db * St0[k];
      dJ00 += dT0 * c.V64[k];
      dJ02 += dT0 * c.V64[8 + k];
      dJ11 += dT1 * c.V64[4 + k];
      dJ12 += dT1 * c.V64[8 + k];
    }
    const double fx = c.fx64, fy = c.fy64, iz = 1.0 / p.z, iz2 = iz * iz;
    double dpx = 0, dpy = 0, dpz = -(dJ00 * fx + dJ11 * fy) * iz2;
    if (cp.clx == 0) { dpx -= dJ02 * fx * iz2; dpz += 2 * dJ02 * fx * p.x * iz2 * iz; }
    else dpz += dJ02 * fx * p.cxp * iz2;
    if (cp.cly == 0) { dpy -= dJ12 * fy * iz2; dpz += 2 * dJ12 * fy * p.y * iz2 * iz; }
    else dpz += dJ12 * fy * p.cyp * iz2;
    // mean2D: mx = fx x/z + cx
    dpx += dmx * fx * iz;
    dpy += dmy * fy * iz;
    dpz -= (dmx * fx * p.x + dmy * fy * p.y) * iz2;
    dmu0 += c.V64[0] * dpx + c.V64[4] * dpy + c.V64[8] * dpz;
    dmu1 += c.V64[1] * dpx + c.V64[5] * dpy + c.V64[9] * dpz;
    dmu2 += c.V64[2] * dpx + c.V64[6] * dpy + c.V64[10] * dpz;
    dop += dO;
    // colour
    const uint32_t flags = __float_as_uint(v.rec[2 * o + 1].w);
    const double drgb[3] = {(flags & 1u) ? 0.0 : dr, (flags & 2u) ? 0.0 : dg, (flags & 4u) ? 0.0 : db_};
    double ex = mux - c.campos64[0], ey = muy - c.campos64[1], ez = muz - c.campos64[2];
    const double dist = sqrt(ex * ex + ey * ey + ez * ez), idist = 1.0 / dist;
    ex *= idist; ey *= idist; ez *= idist;
    double Y[NK];
    sh_basis<DEG, double>(ex, ey, ez, Y);
#pragma unroll
    for (int k = 0; k < NK; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) dsh[3 * k + ch] = fma(Y[k], drgb[ch], dsh[3 * k + ch]);
    if (DEG > 0) {
      double dY[NK][3];
      sh_basis_grad<DEG, double>(ex, ey, ez, dY);
      double dd0 = 0, dd1 = 0, dd2 = 0;
#pragma unroll
      for (int k = 1; k < NK; ++k) {
        const double w = PUV_SHW(3 * k) * drgb[0] + PUV_SHW(3 * k + 1) * drgb[1] + PUV_SHW(3 * k + 2) * drgb[2];
        dd0 = fma(w, dY[k][0], dd0);
        dd1 = fma(w, dY[k][1], dd1);
        dd2 = fma(w, dY[k][2], dd2);
      }
      const double dot = ex * dd0 + ey * dd1 + ez * dd2;
      dmu0 += (dd0 - ex * dot) * idist;
      dmu1 += (dd1 - ey * dot) * idist;
      dmu2 += (dd2 - ez * dot) * idist;
    }
  }

  // Sigma = R diag(t) R^T  ->  t, R  ->  (ls, q)
  const double s0 = exp((double)ls0), s1 = exp((double)ls1), s2 = exp((double)ls2);
  const double t0 = s0 * s0, t1 = s1 * s1, t2 = s2 * s2;
  const double qn = sqrt((double)qw * qw + (double)qx * qx + (double)qy * qy + (double)qz * qz), iq = 1.0 / qn;
  const double w = qw * iq, x = qx * iq, y = qy * iq, z = qz * iq;
  const double R00 = 1 - 2 * (y * y + z * z), R01 = 2 * (x * y - w * z), R02 = 2 * (x * z + w * y);
  const double R10 = 2 * (x * y + w * z), R11 = 1 - 2 * (x * x + z * z), R12 = 2 * (y * z - w * x);
  const double R20 = 2 * (x * z - w * y), R21 = 2 * (y * z + w * x), R22 = 1 - 2 * (x * x + y * y);
  const double GR00 = G00 * R00 + G01 * R10 + G02 * R20, GR01 = G00 * R01 + G01 * R11 + G02 * R21,
               GR02 = G00 * R02 + G01 * R12 + G02 * R22;
  const double GR10 = G01 * R00 + G11 * R10 + G12 * R20, GR11 = G01 * R01 + G11 * R11 + G12 * R21,
               GR12 = G01 * R02 + G11 * R12 + G12 * R22;
  const double GR20 = G02 * R00 + G12 * R10 + G22 * R20, GR21 = G02 * R01 + G12 * R11 + G22 * R21,
               GR22 = G02 * R02 + G12 * R12 + G22 * R22;
  // dt_k = 1/2 (R^T G R)_kk ; dR_ab = t_b (G R)_ab
  const double dt0 = 0.5 * (R00 * GR00 + R10 * GR10 + R20 * GR20);
  const double dt1 = 0.5 * (R01 * GR01 + R11 * GR11 + R21 * GR21);
  const double dt2 = 0.5 * (R02 * GR02 + R12 * GR12 + R22 * GR22);
  const double dR00 = t0 * GR00, dR01 = t1 * GR01, dR02 = t2 * GR02;
  const double dR10 = t0 * GR10, dR11 = t1 * GR11, dR12 = t2 * GR12;
  const double dR20 = t0 * GR20, dR21 = t1 * GR21, dR22 = t2 * GR22;
  const double dqw = 2 * (-z * dR01 + y * dR02 + z * dR10 - x * dR12 - y * dR20 + x * dR21);
  const double dqx = 2 * (y * dR01 + z * dR02 + y * dR10 - 2 * x * dR11 - w * dR12 + z * dR20 + w * dR21 - 2 * x * dR22);
  const double dqy = 2 * (-2 * y * dR00 + x * dR01 + w * dR02 + x * dR10 + z * dR12 - w * dR20 + z * dR21 - 2 * y * dR22);
  const double dqz = 2 * (-2 * z * dR00 - w * dR01 + x * dR02 + w * dR10 - 2 * z * dR11 + y * dR12 + x * dR20 + y * dR21);
  const double qd = w * dqw + x * dqx + y * dqy + z * dqz;
  if (pm.rho) {   // d rho = ray . d mu, in fp64 before the one rounding (planes 1, 2 untouched)
    put(0, (float)((double)__ldg(P.p[pm.D] + g) * dmu0 + (double)__ldg(P.p[pm.D + 1] + g) * dmu1 +
                          (double)__ldg(P.p[pm.D + 2] + g) * dmu2));
  } else {
    put(0, (float)dmu0);
    put(1, (float)dmu1);
    put(2, (float)dmu2);
  }
  put(3, (float)(2 * t0 * dt0));
  put(4, (float)(2 * t1 * dt1));
  put(5, (float)(2 * t2 * dt2));
  put(6, (float)((dqw - w * qd) * iq));
  put(7, (float)((dqx - x * qd) * iq));
  put(8, (float)((dqy - y * qd) * iq));
  put(9, (float)((dqz - z * qd) * iq));
  // dL/dlogit = dL/do o (1 - o); with kLno dop already sums o dL/do
  put(10, (float)(dop * (kLno ? 1.0 : u.o) * (1.0 - u.o)));
#pragma unroll
  for (int k = 0; k < 3 * NK; ++k) put(11 + k, (float)dsh[k]);
}

void launch_project_bwd(const Plan& p, const Views& v, const PlaneTab& P, const uint8_t* occ, const uint8_t* mask,
                        const CamBatch& cb, const GradTab& G, cudaStream_t s, int g0, int g1, bool overwrite) {
  if (g1 < 0) g1 = p.N;
  if (g1 <= g0) return;
  const int threads = 128;
  const int blocks = (g1 - g0 + threads - 1) / threads;
#if PUV_PBWD_SH_SMEM
#define PUV_K7(D, L)                                                                                      \
  do {                                                                                                    \
    constexpr int smem = 3 * ((D + 1) * (D + 1) - 1) * 128 * 8;                                           \
    static const bool attr =                                                                              \
        cudaFuncSetAttribute(k_project_bwd<D, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) ==   \
        cudaSuccess;                                                                                      \
    (void)attr;                                                                                           \
    k_project_bwd<D, L><<<blocks, threads, smem, s>>>(P, p.pm, occ, mask, p.N, cb, v, G, g0, g1,          \
                                                      overwrite ? 1 : 0);                                 \
  } while (0)
#else
#define PUV_K7(D, L) k_project_bwd<D, L><<<blocks, threads, 0, s>>>(P, p.pm, occ, mask, p.N, cb, v, G, g0, g1, overwrite ? 1 : 0)
#endif
  const bool lpo = P.qspec != nullptr;
  switch (p.deg) {
    case 0: if (lpo) PUV_K7(0, true); else PUV_K7(0, false); break;
    case 1: if (lpo) PUV_K7(1, true); else PUV_K7(1, false); break;
    case 2: if (lpo) PUV_K7(2, true); else PUV_K7(2, false); break;
    default: if (lpo) PUV_K7(3, true); else PUV_K7(3, false); break;
  }
#undef PUV_K7
  count_launches(1);
}

}  // namespace puv
