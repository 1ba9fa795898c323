// project.cuh — atlas unpack (U1-U5), EWA projection (P1-P12) and SH colour.
//
// PAPER.md:383-390 and Alg. 1: Sigma = R diag(s^2) R^T,
// Sigma2D = J T Sigma T^T J^T + 0.3 I, det <= 1e-7 / z <= near rejection,
// r = ceil(3 sqrt(lambda_max)).  Texel contents and activations: PAPER.md:297-303
// with DESIGN.md R1-R8.  Every operation that decides an integer follows the
// fp32 contract of DESIGN.md R13 (explicit _rn intrinsics).
#pragma once
#include "contract.cuh"
#include "internal.cuh"

namespace puv {

// Texel position (a1): explicit xyz planes, or mu = c (+) rho (x) ray in the fp32 contract (PUV_POS_RHO).
template <bool LPO = false>
PUV_DEV void texel_mu(const PlaneTab& P, const PosMode& pm, int g, float& x, float& y, float& z) {
  if (pm.rho) {
    const float r = plane_value<LPO>(P, 0, g);
    x = add(pm.c[0], mul(r, __ldg(P.p[pm.D] + g)));
    y = add(pm.c[1], mul(r, __ldg(P.p[pm.D + 1] + g)));
    z = add(pm.c[2], mul(r, __ldg(P.p[pm.D + 2] + g)));
  } else {
    x = plane_value<LPO>(P, 0, g);
    y = plane_value<LPO>(P, 1, g);
    z = plane_value<LPO>(P, 2, g);
  }
}

struct Unpacked {
  float S00, S01, S02, S11, S12, S22;  // world covariance (U4)
  float o, t_g;                        // opacity (U5) and log-threshold
  bool ok;                             // false: zero quaternion (R16)
};

// U1-U5 (view independent).
PUV_DEV Unpacked unpack_contract(float ls0, float ls1, float ls2, float qw, float qx, float qy, float qz,
                                 float logit) {
  Unpacked u;
  const float s0 = exp_c(ls0), s1 = exp_c(ls1), s2 = exp_c(ls2);
  const float t0 = mul(s0, s0), t1 = mul(s1, s1), t2 = mul(s2, s2);
  const float n2 = add(add(add(mul(qw, qw), mul(qx, qx)), mul(qy, qy)), mul(qz, qz));
  u.ok = n2 != 0.0f;
  const float n = sqrt_(n2);
  const float w = dvd(qw, n), x = dvd(qx, n), y = dvd(qy, n), z = dvd(qz, n);
  const float xx = mul(x, x), yy = mul(y, y), zz = mul(z, z);
  const float xy = mul(x, y), xz = mul(x, z), yz = mul(y, z);
  const float wx = mul(w, x), wy = mul(w, y), wz = mul(w, z);
  const float R00 = sub(1.0f, mul(2.0f, add(yy, zz))), R01 = mul(2.0f, sub(xy, wz)), R02 = mul(2.0f, add(xz, wy));
  const float R10 = mul(2.0f, add(xy, wz)), R11 = sub(1.0f, mul(2.0f, add(xx, zz))), R12 = mul(2.0f, sub(yz, wx));
  const float R20 = mul(2.0f, sub(xz, wy)), R21 = mul(2.0f, add(yz, wx)), R22 = sub(1.0f, mul(2.0f, add(xx, yy)));
  // U4: ((R_a0 t0) R_b0 + (R_a1 t1) R_b1) + (R_a2 t2) R_b2
#define PUV_SIG(a0, a1, a2, b0, b1, b2) \
  add(add(mul(mul(a0, t0), b0), mul(mul(a1, t1), b1)), mul(mul(a2, t2), b2))
  u.S00 = PUV_SIG(R00, R01, R02, R00, R01, R02);
  u.S01 = PUV_SIG(R00, R01, R02, R10, R11, R12);
  u.S02 = PUV_SIG(R00, R01, R02, R20, R21, R22);
  u.S11 = PUV_SIG(R10, R11, R12, R10, R11, R12);
  u.S12 = PUV_SIG(R10, R11, R12, R20, R21, R22);
  u.S22 = PUV_SIG(R20, R21, R22, R20, R21, R22);
#undef PUV_SIG
  u.o = dvd(1.0f, add(1.0f, exp_c(-logit)));
  u.t_g = -log_c(mul(255.0f, u.o));
  return u;
}

struct CamPoint {
  float x, y, z;   // camera-space mean (P1)
  float ux, uy;    // x/z, y/z (P3)
  float cxp, cyp;  // clamped (R5)
  int clx, cly;    // clamp flags: 0, +1, -1
};

// P1, P3 (P2 is the caller's z test).
PUV_DEV CamPoint cam_point(const CamDev& c, float mx, float my, float mz) {
  CamPoint p;
  p.x = add(add(add(mul(c.V[0], mx), mul(c.V[1], my)), mul(c.V[2], mz)), c.V[3]);
  p.y = add(add(add(mul(c.V[4], mx), mul(c.V[5], my)), mul(c.V[6], mz)), c.V[7]);
  p.z = add(add(add(mul(c.V[8], mx), mul(c.V[9], my)), mul(c.V[10], mz)), c.V[11]);
  p.ux = dvd(p.x, p.z);
  p.uy = dvd(p.y, p.z);
  p.cxp = fminf(c.limx, fmaxf(-c.limx, p.ux));
  p.cyp = fminf(c.limy, fmaxf(-c.limy, p.uy));
  p.clx = p.ux > c.limx ? 1 : (p.ux < -c.limx ? -1 : 0);
  p.cly = p.uy > c.limy ? 1 : (p.uy < -c.limy ? -1 : 0);
  return p;
}

struct Proj {
  bool vis;
  float mx, my, ha, nb, hc;
  uint32_t depth_bits;
  int x0, x1, y0, y1;
};

// P2, P4-P12 given U and the camera point.
PUV_DEV Proj project_contract(const CamDev& c, const CamPoint& p, const Unpacked& u, int gx, int gy) {
  Proj r;
  r.vis = false;
  if (!(p.z > c.near_plane)) return r;
  const float J00 = dvd(c.fx, p.z), J02 = -dvd(mul(c.fx, p.cxp), p.z);
  const float J11 = dvd(c.fy, p.z), J12 = -dvd(mul(c.fy, p.cyp), p.z);
  // P4: T0k = J00 V0k + J02 V2k ; T1k = J11 V1k + J12 V2k
  const float T00 = add(mul(J00, c.V[0]), mul(J02, c.V[8]));
  const float T01 = add(mul(J00, c.V[1]), mul(J02, c.V[9]));
  const float T02 = add(mul(J00, c.V[2]), mul(J02, c.V[10]));
  const float T10 = add(mul(J11, c.V[4]), mul(J12, c.V[8]));
  const float T11 = add(mul(J11, c.V[5]), mul(J12, c.V[9]));
  const float T12 = add(mul(J11, c.V[6]), mul(J12, c.V[10]));
  // P5: W_a,i = (S_i0 T_a0 + S_i1 T_a1) + S_i2 T_a2
  const float W00 = add(add(mul(u.S00, T00), mul(u.S01, T01)), mul(u.S02, T02));
  const float W01 = add(add(mul(u.S01, T00), mul(u.S11, T01)), mul(u.S12, T02));
  const float W02 = add(add(mul(u.S02, T00), mul(u.S12, T01)), mul(u.S22, T02));
  const float W10 = add(add(mul(u.S00, T10), mul(u.S01, T11)), mul(u.S02, T12));
  const float W11 = add(add(mul(u.S01, T10), mul(u.S11, T11)), mul(u.S12, T12));
  const float W12 = add(add(mul(u.S02, T10), mul(u.S12, T11)), mul(u.S22, T12));
  float a = add(add(mul(T00, W00), mul(T01, W01)), mul(T02, W02));
  const float b = add(add(mul(T10, W00), mul(T11, W01)), mul(T12, W02));
  float cc = add(add(mul(T10, W10), mul(T11, W11)), mul(T12, W12));
  // P6
  a = add(a, 0.3f);
  cc = add(cc, 0.3f);
  // P7
  const float det = sub(mul(a, cc), mul(b, b));
  if (!(det > 1e-7f)) return r;
  // P8
  r.ha = mul(-0.5f, dvd(cc, det));
  r.nb = dvd(b, det);
  r.hc = mul(-0.5f, dvd(a, det));
  // P9
  const float tr = add(a, cc);
  const float disc = sub(mul(tr, tr), mul(4.0f, det));
  const float lam = mul(0.5f, add(tr, sqrt_(fmaxf(0.0f, disc))));
  const float rf = ceilf(mul(3.0f, sqrt_(lam)));
  // P10
  r.mx = add(mul(c.fx, p.ux), c.cx);
  r.my = add(mul(c.fy, p.uy), c.cy);
  // P11 conservative rect
  const float fgx = (float)gx, fgy = (float)gy;
  const float fx0 = fminf(fmaxf(floorf(mul(sub(r.mx, rf), 0.0625f)), 0.0f), fgx);
  const float fx1 = fminf(fmaxf(add(floorf(mul(add(r.mx, rf), 0.0625f)), 1.0f), 0.0f), fgx);
  const float fy0 = fminf(fmaxf(floorf(mul(sub(r.my, rf), 0.0625f)), 0.0f), fgy);
  const float fy1 = fminf(fmaxf(add(floorf(mul(add(r.my, rf), 0.0625f)), 1.0f), 0.0f), fgy);
  r.x0 = (int)fx0; r.x1 = (int)fx1; r.y0 = (int)fy0; r.y1 = (int)fy1;
  if (r.x0 >= r.x1 || r.y0 >= r.y1) return r;
  r.depth_bits = __float_as_uint(p.z);  // P12
  r.vis = true;
  return r;
}

// ---- spherical harmonics (R3): real basis, 3DGS constants/signs; free fp32 arithmetic ----
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_0 = 1.0925484305920792, kC2_1 = -1.0925484305920792, kC2_2 = 0.31539156525252005,
                 kC2_3 = -1.0925484305920792, kC2_4 = 0.5462742152960396;
constexpr double kC3_0 = -0.5900435899266435, kC3_1 = 2.890611442640554, kC3_2 = -0.4570457994644658,
                 kC3_3 = 0.3731763325901154, kC3_4 = -0.4570457994644658, kC3_5 = 1.445305721320277,
                 kC3_6 = -0.5900435899266435;

template <int DEG, typename T>
PUV_DEV void sh_basis(T x, T y, T z, T* Y) {
  Y[0] = T(kC0);
  if (DEG >= 1) { Y[1] = -T(kC1) * y; Y[2] = T(kC1) * z; Y[3] = -T(kC1) * x; }
  if (DEG >= 2) {
    const T xx = x * x, yy = y * y, zz = z * z;
    Y[4] = T(kC2_0) * x * y; Y[5] = T(kC2_1) * y * z; Y[6] = T(kC2_2) * (T(2) * zz - xx - yy);
    Y[7] = T(kC2_3) * x * z; Y[8] = T(kC2_4) * (xx - yy);
    if (DEG >= 3) {
      Y[9] = T(kC3_0) * y * (T(3) * xx - yy);
      Y[10] = T(kC3_1) * x * y * z;
      Y[11] = T(kC3_2) * y * (T(4) * zz - xx - yy);
      Y[12] = T(kC3_3) * z * (T(2) * zz - T(3) * xx - T(3) * yy);
      Y[13] = T(kC3_4) * x * (T(4) * zz - xx - yy);
      Y[14] = T(kC3_5) * z * (xx - yy);
      Y[15] = T(kC3_6) * x * (xx - T(3) * yy);
    }
  }
}

// dY_k / d(x,y,z) of the basis polynomials (not projected on the sphere).
template <int DEG, typename T>
PUV_DEV void sh_basis_grad(T x, T y, T z, T (*dY)[3]) {
#pragma unroll
  for (int k = 0; k < (DEG + 1) * (DEG + 1); ++k) dY[k][0] = dY[k][1] = dY[k][2] = T(0);
  if (DEG >= 1) { dY[1][1] = -T(kC1); dY[2][2] = T(kC1); dY[3][0] = -T(kC1); }
  if (DEG >= 2) {
    dY[4][0] = T(kC2_0) * y; dY[4][1] = T(kC2_0) * x;
    dY[5][1] = T(kC2_1) * z; dY[5][2] = T(kC2_1) * y;
    dY[6][0] = T(-2) * T(kC2_2) * x; dY[6][1] = T(-2) * T(kC2_2) * y; dY[6][2] = T(4) * T(kC2_2) * z;
    dY[7][0] = T(kC2_3) * z; dY[7][2] = T(kC2_3) * x;
    dY[8][0] = T(2) * T(kC2_4) * x; dY[8][1] = T(-2) * T(kC2_4) * y;
    if (DEG >= 3) {
      const T xx = x * x, yy = y * y, zz = z * z;
      dY[9][0] = T(kC3_0) * T(6) * x * y; dY[9][1] = T(kC3_0) * (T(3) * xx - T(3) * yy);
      dY[10][0] = T(kC3_1) * y * z; dY[10][1] = T(kC3_1) * x * z; dY[10][2] = T(kC3_1) * x * y;
      dY[11][0] = T(-2) * T(kC3_2) * x * y; dY[11][1] = T(kC3_2) * (T(4) * zz - xx - T(3) * yy);
      dY[11][2] = T(8) * T(kC3_2) * y * z;
      dY[12][0] = T(-6) * T(kC3_3) * x * z; dY[12][1] = T(-6) * T(kC3_3) * y * z;
      dY[12][2] = T(kC3_3) * (T(6) * zz - T(3) * xx - T(3) * yy);
      dY[13][0] = T(kC3_4) * (T(4) * zz - T(3) * xx - yy); dY[13][1] = T(-2) * T(kC3_4) * x * y;
      dY[13][2] = T(8) * T(kC3_4) * x * z;
      dY[14][0] = T(2) * T(kC3_5) * x * z; dY[14][1] = T(-2) * T(kC3_5) * y * z; dY[14][2] = T(kC3_5) * (xx - yy);
      dY[15][0] = T(kC3_6) * (T(3) * xx - T(3) * yy); dY[15][1] = T(-6) * T(kC3_6) * x * y;
    }
  }
}

// ---- fp64 value path: the same Sigma / EWA / conic / mean, in double, with the
// J-clamp decisions taken from the fp32 contract (cam_point) ----

struct Unpacked64 {
  double S00, S01, S02, S11, S12, S22, o;
};

PUV_DEV Unpacked64 unpack64(float ls0, float ls1, float ls2, float qw, float qx, float qy, float qz, float logit) {
  Unpacked64 u;
  const double s0 = exp((double)ls0), s1 = exp((double)ls1), s2 = exp((double)ls2);
  const double t0 = s0 * s0, t1 = s1 * s1, t2 = s2 * s2;
  const double n = sqrt((double)qw * qw + (double)qx * qx + (double)qy * qy + (double)qz * qz);
  const double w = qw / n, x = qx / n, y = qy / n, z = qz / n;
  const double R00 = 1 - 2 * (y * y + z * z), R01 = 2 * (x * y - w * z), R02 = 2 * (x * z + w * y);
  const double R10 = 2 * (x * y + w * z), R11 = 1 - 2 * (x * x + z * z), R12 = 2 * (y * z - w * x);
  const double R20 = 2 * (x * z - w * y), R21 = 2 * (y * z + w * x), R22 = 1 - 2 * (x * x + y * y);
  u.S00 = R00 * t0 * R00 + R01 * t1 * R01 + R02 * t2 * R02;
  u.S01 = R00 * t0 * R10 + R01 * t1 * R11 + R02 * t2 * R12;
  u.S02 = R00 * t0 * R20 + R01 * t1 * R21 + R02 * t2 * R22;
  u.S11 = R10 * t0 * R10 + R11 * t1 * R11 + R12 * t2 * R12;
  u.S12 = R10 * t0 * R20 + R11 * t1 * R21 + R12 * t2 * R22;
  u.S22 = R20 * t0 * R20 + R21 * t1 * R21 + R22 * t2 * R22;
  u.o = 1.0 / (1.0 + exp(-(double)logit));
  return u;
}

struct Proj64 {
  double x, y, z, ux, uy, cxp, cyp;  // camera-space mean, x/z, y/z, J-clamped coordinates
  double T0[3], T1[3];               // T = J V (rows)
  double a, b, c, det;               // Sigma2D (+0.3 on a, c)
  double mx, my, ha, nb, hc;
};

PUV_DEV Proj64 project64(const CamDev& cam, double mx_, double my_, double mz_, const Unpacked64& u, int clx,
                         int cly) {
  Proj64 p;
  const double* V = cam.V64;
  p.x = V[0] * mx_ + V[1] * my_ + V[2] * mz_ + V[3];
  p.y = V[4] * mx_ + V[5] * my_ + V[6] * mz_ + V[7];
  p.z = V[8] * mx_ + V[9] * my_ + V[10] * mz_ + V[11];
  p.ux = p.x / p.z;
  p.uy = p.y / p.z;
  p.cxp = clx ? clx * cam.limx64 : p.ux;
  p.cyp = cly ? cly * cam.limy64 : p.uy;
  const double fx = cam.fx64, fy = cam.fy64;
  const double J00 = fx / p.z, J02 = -fx * p.cxp / p.z, J11 = fy / p.z, J12 = -fy * p.cyp / p.z;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    p.T0[k] = J00 * V[k] + J02 * V[8 + k];
    p.T1[k] = J11 * V[4 + k] + J12 * V[8 + k];
  }
  const double St0[3] = {u.S00 * p.T0[0] + u.S01 * p.T0[1] + u.S02 * p.T0[2],
                         u.S01 * p.T0[0] + u.S11 * p.T0[1] + u.S12 * p.T0[2],
                         u.S02 * p.T0[0] + u.S12 * p.T0[1] + u.S22 * p.T0[2]};
  const double St1[3] = {u.S00 * p.T1[0] + u.S01 * p.T1[1] + u.S02 * p.T1[2],
                         u.S01 * p.T1[0] + u.S11 * p.T1[1] + u.S12 * p.T1[2],
                         u.S02 * p.T1[0] + u.S12 * p.T1[1] + u.S22 * p.T1[2]};
  p.a = p.T0[0] * St0[0] + p.T0[1] * St0[1] + p.T0[2] * St0[2] + 0.3;
  p.b = p.T1[0] * St0[0] + p.T1[1] * St0[1] + p.T1[2] * St0[2];
  p.c = p.T1[0] * St1[0] + p.T1[1] * St1[1] + p.T1[2] * St1[2] + 0.3;
  p.det = p.a * p.c - p.b * p.b;
  p.ha = -0.5 * p.c / p.det;
  p.nb = p.b / p.det;
  p.hc = -0.5 * p.a / p.det;
  p.mx = fx * p.ux + cam.cx64;
  p.my = fy * p.uy + cam.cy64;
  return p;
}

}  // namespace puv
