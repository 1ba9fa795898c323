// contract.cuh — fp32 arithmetic contract for every decision on the render path.
//
// DESIGN.md §2 R13/R14: visibility, tile rect, depth key, J clamp, the pair
// skip test, the alpha cap and the transmittance termination are computed with
// explicit IEEE round-to-nearest intrinsics (never contracted into FMAs), so the
// decisions are bit-identical to the CPU oracle's.  Written from DESIGN.md, not
// from the oracle's source (they share no code).
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#include "exp2_table.h"
#include "internal.cuh"

namespace puv {

#define PUV_DEV __device__ __forceinline__

PUV_DEV float add(float a, float b) { return __fadd_rn(a, b); }
PUV_DEV float sub(float a, float b) { return __fsub_rn(a, b); }
PUV_DEV float mul(float a, float b) { return __fmul_rn(a, b); }
PUV_DEV float dvd(float a, float b) { return __fdiv_rn(a, b); }
PUV_DEV float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
PUV_DEV float sqrt_(float a) { return __fsqrt_rn(a); }

constexpr float kLn2Hi = 0.693145751953125f;
constexpr float kLn2Lo = 1.42860677e-6f;
constexpr float kLog2e = 1.44269504f;

// exp_c (R13): Cody-Waite reduction by ln2 (hi/lo) + degree-7 Taylor, Horner with fma.
// exp_c_core is exp_c without the range clamps, for callers whose argument is known to lie in (-87, 88) (the
// compositing range: power in [t_g, 0] with t_g = -log_c(255 o) >= -5.55): bit-identical there.
#ifndef PUV_EXPC_MAGIC
#define PUV_EXPC_MAGIC 1
#endif
PUV_DEV float exp_c_core(float x) {
#if PUV_EXPC_MAGIC
  // rint by the 1.5 * 2^23 shifter: for |v| < 2^22 the RN addition rounds v to the nearest integer
  // (ties to even), exactly rintf(v), and the sum's low mantissa bits are that integer -- one FADD
  // pair instead of FRND + F2I (conversion-pipe ops); bit-identical to the rintf form
  constexpr float kShifter = 12582912.0f;   // 1.5 * 2^23
  const float t = add(mul(x, kLog2e), kShifter);
  const float k = sub(t, kShifter);
  const int ki = __float_as_int(t) - 0x4b400000;
#else
  const float k = rintf(mul(x, kLog2e));
  const int ki = (int)k;
#endif
  float r = fma_(-k, kLn2Hi, x);
  r = fma_(-k, kLn2Lo, r);
  float p = (float)(1.0 / 5040.0);
  p = fma_(p, r, (float)(1.0 / 720.0));
  p = fma_(p, r, (float)(1.0 / 120.0));
  p = fma_(p, r, (float)(1.0 / 24.0));
  p = fma_(p, r, (float)(1.0 / 6.0));
  p = fma_(p, r, 0.5f);
  p = fma_(p, r, 1.0f);
  p = fma_(p, r, 1.0f);
  const float two_k = __int_as_float((ki + 127) << 23);
  return mul(p, two_k);
}

PUV_DEV float exp_c(float x) {
  if (x >= 88.0f) return __int_as_float(0x7f800000);
  if (x <= -87.0f) return 0.0f;
  return exp_c_core(x);
}

// log_c (R13): m in [sqrt(1/2), sqrt(2)], atanh series in s = f/(2+f).
PUV_DEV float log_c(float y) {
  const uint32_t b = __float_as_uint(y);
  if (y != y || y < 0.0f) return __int_as_float(0x7fc00000);
  if (b == 0x7f800000u) return y;
  if ((b & 0x7f800000u) == 0u) return __int_as_float(0xff800000);
  int e = (int)((b >> 23) & 0xffu) - 127;
  float m = __uint_as_float((b & 0x007fffffu) | 0x3f800000u);
  if (m > 1.41421356f) { m = mul(m, 0.5f); e += 1; }
  const float f = sub(m, 1.0f);
  const float s = dvd(f, add(2.0f, f));
  const float z = mul(s, s);
  float P = fma_(z, (float)(2.0 / 9.0), (float)(2.0 / 7.0));
  P = fma_(z, P, (float)(2.0 / 5.0));
  P = fma_(z, P, (float)(2.0 / 3.0));
  P = fma_(z, P, 2.0f);
  const float fe = (float)e;
  return fma_(fe, kLn2Hi, fma_(fe, kLn2Lo, mul(s, P)));
}

// Pair skip test R1 and alpha/termination R14.  Returns power; sets skip.
PUV_DEV float pair_power(float mx, float my, float ha, float nb, float hc, float fi, float fj) {
  const float dx = sub(mx, fi), dy = sub(my, fj);
  const float u = fma_(nb, dy, mul(ha, dx));
  return fma_(dx, u, mul(mul(hc, dy), dy));
}

// LPO fake quantiser (NEXT-2, DESIGN.md §13 Q1-Q8), fp32 contract: code and proxy of one value.
PUV_DEV void quant1(float x, float mn, float mx, int bits, uint32_t& code, float& prox) {
  if (bits < 0) {   // reading Q8: IEEE binary16 (round to nearest even); code = its bit pattern
    const __half h = __float2half_rn(x);
    code = __half_as_ushort(h);
    prox = __half2float(h);
    return;
  }
  code = 0;
  if (mx == mn) { prox = mn; return; }
  const float L = (float)((1u << bits) - 1u);
  float t = mul(dvd(sub(x, mn), sub(mx, mn)), L);
  if (!(t > 0.f)) t = 0.f;
  if (t > L) t = L;
  code = (uint32_t)roundf(t);
  prox = add(mn, mul(dvd((float)code, L), sub(mx, mn)));
}

// A texel plane value as the render reads it: the master value, or with LPO its proxy.
// LPO = true only in the PUV_RENDER_LPO instantiations of K1 / K7 (the plain kernels stay free of the
// quantiser code: compiled in, it cost the plain K1 +1.4 ms per C3 step in an A/B).
template <bool LPO>
PUV_DEV float plane_value(const PlaneTab& P, int d, int g) {
  const float x = __ldg(P.p[d] + g);
  if (!LPO || P.qbits[d] == 0) return x;
  uint32_t code;
  float prox;
  quant1(x, __ldg(P.qspec + 2 * d), __ldg(P.qspec + 2 * d + 1), P.qbits[d], code, prox);
  return prox;
}

// ---- fp64 value path helpers (not part of the contract) ---------------------------------------
// exp(x) = 2^m * 2^(j/256) * e^r,  k = rint(256 x / ln2) = 256 m + j,  r = x - k ln2/256 (one fma:
// the rounding of ln2/256 costs |k| * 3e-19 < 1e-13 over the valid range), |r| <= ln2/512,
// e^r by its degree-3 Taylor polynomial (truncation < 1.5e-13).  Max relative error vs libm over
// [-700, 0] below 3e-13 (tools/exp64_check.py) -- far below what the gradient tolerance needs
// (DESIGN.md §5).  `tab` = 2^(j/256), j < 256, staged in shared memory (exp64_table_fill).
// Valid for x in [-700, 1]; for far-out x (inactive pixels of the branch-free backward) the
// result is garbage but finite-or-inf, and the callers select it away.
constexpr int kExpTab = 256;
PUV_DEV void exp64_table_fill(double* tab) {
  for (int j = threadIdx.x; j < kExpTab; j += blockDim.x) tab[j] = kExp2Tab256[j];   // exp2_table.h
}

PUV_DEV double exp64(double x, const double* tab) {
  constexpr double kInvL = 369.3299304675746;            // 256 / ln 2
  constexpr double kL = 0.0027076061740622863;           // ln 2 / 256
  constexpr double kShift = 6755399441055744.0;          // 1.5 * 2^52: rint by addition
  const double t = fma(x, kInvL, kShift);
  const int k = (int)__double2loint(t);                  // low word = rint(256 x / ln2) (two's complement)
  const double r = fma(-(t - kShift), kL, x);
  double p = fma(r, 1.0 / 6.0, 0.5);
  p = fma(r, p, 1.0);
  p = fma(r, p, 1.0);
  const double v = tab[k & (kExpTab - 1)] * p;
  return __hiloint2double(__double2hiint(v) + ((k >> 8) << 20), __double2loint(v));
}

// Gaussian exponent in fp64, power = ha dx^2 + dy (nb dx + hc dy) with (dx, dy) = mean - pixel,
// from the column terms hadxx = ha dx^2 and nbdx = nb dx (shared by the pixels of a thread, which
// sit in one pixel column).  K5 and K6 evaluate it identically.
PUV_DEV double power64(double hc, double hadxx, double nbdx, double dy) { return fma(dy, fma(hc, dy, nbdx), hadxx); }

// 1/y for y in [0.01, 1]: MUFU fp64 reciprocal estimate (~2^-23 relative) + one Newton step
// (error squared: ~2^-46 = 1.4e-14 relative, far below what the gradients need)
PUV_DEV double rcp64(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  const double e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

// Conservative per-warp entry filter of K5/K6 (not part of the contract and not a decision: every
// composited pair is still decided by the per-pixel skip test R1).  Can any pixel centre (i, j) of
// the block i in [x0, x0 + ex], j in [y0, y0 + ey] reach power = ha dx^2 + nb dx dy + hc dy^2 >= t_g ((dx, dy) = mean - pixel)?
// The quadratic is concave (the conic of Sigma2D + 0.3 I), so its maximum over the box is 0 if the
// mean lies inside, else the largest of the four edge maxima (each a clamped 1-D vertex).  Kept
// when that maximum is >= t_g - margin, the margin (1e-3 of the terms' magnitude bound over the
// box + 1e-4) dwarfing the fp32 rounding of both this test and the contract's power: an entry
// whose pairs could pass R1 somewhere in the block is never dropped.
__device__ __forceinline__ bool block_may_hit(float mx, float my, float ha, float nb, float hc, float tg, float x0,
                                              float y0, float ex, float ey) {
  const float dxl = mx - (x0 + ex), dxh = mx - x0, dyl = my - (y0 + ey), dyh = my - y0;
  if (dxl <= 0.f && dxh >= 0.f && dyl <= 0.f && dyh >= 0.f) return tg <= 0.f;
  const float dxm = fmaxf(fabsf(dxl), fabsf(dxh)), dym = fmaxf(fabsf(dyl), fabsf(dyh));
  const float margin = 1e-3f * (fabsf(ha) * dxm * dxm + fabsf(nb) * dxm * dym + fabsf(hc) * dym * dym) + 1e-4f;
  // vertex of q along y (resp. x): d* = -nb e / (2 hc); a fast reciprocal is enough: a vertex off by
  // delta ~ 1e-7 |d*| only lowers that edge's value by |hc| delta^2 < 1e-9, far inside the margin
  const float ihc = __fdividef(-0.5f, hc), iha = __fdividef(-0.5f, ha);
  float best = -INFINITY;
  {
    const float dy = fminf(fmaxf(nb * dxl * ihc, dyl), dyh);
    best = fmaxf(best, dxl * (ha * dxl + nb * dy) + hc * dy * dy);
  }
  {
    const float dy = fminf(fmaxf(nb * dxh * ihc, dyl), dyh);
    best = fmaxf(best, dxh * (ha * dxh + nb * dy) + hc * dy * dy);
  }
  {
    const float dx = fminf(fmaxf(nb * dyl * iha, dxl), dxh);
    best = fmaxf(best, dx * (ha * dx + nb * dyl) + hc * dyl * dyl);
  }
  {
    const float dx = fminf(fmaxf(nb * dyh * iha, dxl), dxh);
    best = fmaxf(best, dx * (ha * dx + nb * dyh) + hc * dyh * dyh);
  }
  return best >= tg - margin;
}

}  // namespace puv
