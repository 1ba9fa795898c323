// contract.cuh — fp32 arithmetic contract for every decision on the render path.
//
// DESIGN.md §2 R13/R14: visibility, tile rect, depth key, J clamp, the pair
// skip test, the alpha cap and the transmittance termination are computed with
// explicit IEEE round-to-nearest intrinsics (never contracted into FMAs), so the
// decisions are bit-identical to the CPU oracle's.  Written from DESIGN.md, not
// from the oracle's source (they share no code).
#pragma once
#include <cstdint>

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
PUV_DEV float exp_c(float x) {
  if (x >= 88.0f) return __int_as_float(0x7f800000);
  if (x <= -87.0f) return 0.0f;
  const float k = rintf(mul(x, kLog2e));
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
  const float two_k = __int_as_float(((int)k + 127) << 23);
  return mul(p, two_k);
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

}  // namespace puv
