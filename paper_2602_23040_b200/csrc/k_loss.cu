// K12 / K13: the paper's training objective (NEXT-4).
//
// K12 photometric loss  L = sum_views (1 - lam) mean|I^ - I| + lam (1 - mean SSIM(I^, I))  and dL/dI^.
//   SSIM: 11 x 11 Gaussian window (sigma 1.5, separable), C1 = 0.01^2, C2 = 0.03^2, zero-padded
//   'same' windows, per channel; every statistic in fp64.
//   k_ssim_fwd  one CTA per 32 x 32 output tile of one (view, channel): stage the (32+10) x (32+10)
//               halo of I^, I in shared memory, horizontal 11-tap pass of x, y, x^2, y^2, xy, vertical
//               pass, then per pixel SSIM and the three window-sum sensitivities
//                 A = dS/dmu_x - 2 mu_x dS/dvar_x - mu_y dS/dcov,  B = dS/dvar_x,  Cc = dS/dcov
//               (fp64, rounded once to fp32 in the workspace) and a per-CTA partial (sum S, sum |d|).
//   k_ssim_bwd  same tiling over A, B, Cc: their window sums (gather; the window is symmetric) give
//               dS/dx(q) = W*A + 2 x W*B + y W*Cc; dL = (1-lam)/n sign(d) - lam/n dS/dx, one fp32 rounding.
//   k_photo_fin one CTA: per view the partials in a fixed order -> loss (deterministic).
// K13 regularisers  lam_s E_i[max(0, max s_i - s_max)]^2 + lam_o E_i alpha_i (1 - alpha_i) over the
//   occupied (and dynamic, if a mask is given) texels, gradients ACCUMULATED onto planes 3..5, 10.
#include "internal.cuh"

namespace puv {

namespace {

constexpr int kTX = 32, kTY = 32, kR = 5, kWin = 11;
constexpr int kHX = kTX + 2 * kR, kHY = kTY + 2 * kR;   // 42 x 42 halo
constexpr int kXS = 45;                                  // fp32 halo row stride: 45 = 13 mod 32, conflict-free strips
constexpr int kSX = 4, kSY = 4;                          // register strips: 4 columns (horizontal), 4 rows (vertical)
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;
constexpr int kHS = kTX + 1;                             // fp64 horizontal-sum row stride (conflict-free strips)
constexpr int kAS = 45;                                  // fp32 A/B/C halo row stride (13 mod 32 banks)
constexpr int kFwdSmem = 2 * kHY * kXS * (int)sizeof(float) + 5 * kHY * kHS * (int)sizeof(double);
constexpr int kBwdSmem = 3 * kHY * kAS * (int)sizeof(float) + 3 * kHY * kHS * (int)sizeof(double);

struct Win { double g[kWin]; };

__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
  // fixed-order reduction: warp butterfly then warp 0 over the 8 warp sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
  return s;
}

// One CTA per 32 x 32 output tile of one (view, channel).  Horizontal pass: a thread owns a strip of
// 4 adjacent columns of one halo row (14 loads -> 4 x 5 window sums); vertical pass: a thread owns 4
// adjacent rows of one column (14 loads per statistic -> 4 outputs).
__global__ void __launch_bounds__(256, 3) k_ssim_fwd(const float* __restrict__ img, const float* __restrict__ tgt,
                                                     int W, int H, Win win, float* __restrict__ abc,
                                                     double2* __restrict__ part) {
  extern __shared__ double smem[];
  double (*hs)[kHY][kHS] = reinterpret_cast<double (*)[kHY][kHS]>(smem);
  float* xs = reinterpret_cast<float*>(smem + 5 * kHY * kHS);
  float* ys = xs + kHY * kXS;
  __shared__ double red[8];
  const int plane = blockIdx.z;                       // view * 3 + channel within the chunk
  const size_t HW = (size_t)W * H;
  const float* X = img + plane * HW;
  const float* Y = tgt + plane * HW;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  for (int i = threadIdx.x; i < kHY * kHX; i += blockDim.x) {
    const int r = i / kHX, c = i % kHX;
    const int gy = y0 - kR + r, gx = x0 - kR + c;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    xs[r * kXS + c] = in ? __ldg(X + (size_t)gy * W + gx) : 0.f;
    ys[r * kXS + c] = in ? __ldg(Y + (size_t)gy * W + gx) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHY * (kTX / kSX); i += blockDim.x) {
    const int r = i / (kTX / kSX), c0 = (i % (kTX / kSX)) * kSX;
    double a[kSX], b[kSX], aa[kSX], bb[kSX], ab[kSX];
#pragma unroll
    for (int j = 0; j < kSX; ++j) a[j] = b[j] = aa[j] = bb[j] = ab[j] = 0.0;
#pragma unroll
    for (int t = 0; t < kWin + kSX - 1; ++t) {
      const double x = (double)xs[r * kXS + c0 + t], y = (double)ys[r * kXS + c0 + t];
      const double xx = x * x, yy = y * y, xy = x * y;
#pragma unroll
      for (int j = 0; j < kSX; ++j) {
        const int k = t - j;
        if (k < 0 || k >= kWin) continue;
        const double g = win.g[k];
        a[j] = fma(g, x, a[j]);
        b[j] = fma(g, y, b[j]);
        aa[j] = fma(g, xx, aa[j]);
        bb[j] = fma(g, yy, bb[j]);
        ab[j] = fma(g, xy, ab[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kSX; ++j) {
      hs[0][r][c0 + j] = a[j]; hs[1][r][c0 + j] = b[j]; hs[2][r][c0 + j] = aa[j];
      hs[3][r][c0 + j] = bb[j]; hs[4][r][c0 + j] = ab[j];
    }
  }
  __syncthreads();
  double sS = 0.0, sA = 0.0;
  {
    const int c = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * kSY;   // 8 warps x 4 rows = 32 rows
    double m[5][kSY];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
#pragma unroll
      for (int j = 0; j < kSY; ++j) m[q][j] = 0.0;
#pragma unroll
      for (int t = 0; t < kWin + kSY - 1; ++t) {
        const double h = hs[q][r0 + t][c];
#pragma unroll
        for (int j = 0; j < kSY; ++j) {
          const int k = t - j;
          if (k < 0 || k >= kWin) continue;
          m[q][j] = fma(win.g[k], h, m[q][j]);
        }
      }
    }
    const int gx = x0 + c;
#pragma unroll
    for (int j = 0; j < kSY; ++j) {
      const int gy = y0 + r0 + j;
      if (gx >= W || gy >= H) continue;
      const double mx = m[0][j], my = m[1][j];
      const double vx = m[2][j] - mx * mx, vy = m[3][j] - my * my, cov = m[4][j] - mx * my;
      const double n1 = 2.0 * mx * my + kC1, n2 = 2.0 * cov + kC2;
      const double d1 = mx * mx + my * my + kC1, d2 = vx + vy + kC2;
      const double rdd = 1.0 / (d1 * d2);
      const double S = n1 * n2 * rdd;
      const double dS_dmx = 2.0 * my * n2 * rdd - 2.0 * mx * S / d1;
      const double dS_dvx = -S / d2;
      const double dS_dcov = 2.0 * n1 * rdd;
      const size_t o = (size_t)gy * W + gx;
      float* P = abc + (size_t)plane * 3 * HW;     // one fp32 rounding each (DESIGN.md §12 L8)
      P[o] = (float)(dS_dmx - 2.0 * mx * dS_dvx - my * dS_dcov);
      P[HW + o] = (float)dS_dvx;
      P[2 * HW + o] = (float)dS_dcov;
      sS += S;
      sA += fabs((double)xs[(r0 + j + kR) * kXS + c + kR] - (double)ys[(r0 + j + kR) * kXS + c + kR]);
    }
  }
  const double tS = block_sum_fixed(sS, red);
  const double tA = block_sum_fixed(sA, red);
  if (threadIdx.x == 0)
    part[((size_t)plane * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(tS, tA);
}

__global__ void __launch_bounds__(256, 3) k_ssim_bwd(const float* __restrict__ img, const float* __restrict__ tgt,
                                                     int W, int H, Win win, const float* __restrict__ abc,
                                                     double cl1, double cs, float* __restrict__ dl) {
  extern __shared__ double smem[];
  double (*hs)[kHY][kHS] = reinterpret_cast<double (*)[kHY][kHS]>(smem);
  float (*as)[kHY][kAS] = reinterpret_cast<float (*)[kHY][kAS]>(smem + 3 * kHY * kHS);
  const int plane = blockIdx.z;
  const size_t HW = (size_t)W * H;
  const float* P = abc + (size_t)plane * 3 * HW;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  for (int i = threadIdx.x; i < kHY * kHX; i += blockDim.x) {
    const int r = i / kHX, c = i % kHX;
    const int gy = y0 - kR + r, gx = x0 - kR + c;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const size_t o = (size_t)gy * W + gx;
    as[0][r][c] = in ? __ldcs(P + o) : 0.f;
    as[1][r][c] = in ? __ldcs(P + HW + o) : 0.f;
    as[2][r][c] = in ? __ldcs(P + 2 * HW + o) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHY * (kTX / kSX); i += blockDim.x) {
    const int r = i / (kTX / kSX), c0 = (i % (kTX / kSX)) * kSX;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double acc[kSX];
#pragma unroll
      for (int j = 0; j < kSX; ++j) acc[j] = 0.0;
#pragma unroll
      for (int t = 0; t < kWin + kSX - 1; ++t) {
        const double v = (double)as[q][r][c0 + t];
#pragma unroll
        for (int j = 0; j < kSX; ++j) {
          const int k = t - j;
          if (k < 0 || k >= kWin) continue;
          acc[j] = fma(win.g[k], v, acc[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < kSX; ++j) hs[q][r][c0 + j] = acc[j];
    }
  }
  __syncthreads();
  const int c = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * kSY;
  double m[3][kSY];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
#pragma unroll
    for (int j = 0; j < kSY; ++j) m[q][j] = 0.0;
#pragma unroll
    for (int t = 0; t < kWin + kSY - 1; ++t) {
      const double h = hs[q][r0 + t][c];
#pragma unroll
      for (int j = 0; j < kSY; ++j) {
        const int k = t - j;
        if (k < 0 || k >= kWin) continue;
        m[q][j] = fma(win.g[k], h, m[q][j]);
      }
    }
  }
  const int gx = x0 + c;
#pragma unroll
  for (int j = 0; j < kSY; ++j) {
    const int gy = y0 + r0 + j;
    if (gx >= W || gy >= H) continue;
    const size_t o = plane * HW + (size_t)gy * W + gx;
    const double x = (double)img[o], y = (double)tgt[o];
    const double dS = m[0][j] + 2.0 * x * m[1][j] + y * m[2][j];
    const double sg = x > y ? 1.0 : (x < y ? -1.0 : 0.0);
    dl[o] = (float)(cl1 * sg - cs * dS);
  }
}

__global__ void __launch_bounds__(256) k_photo_fin(const double2* __restrict__ part, int nviews, int blocks_per_plane,
                                                   double inv_n, double lam, double* __restrict__ loss, bool first) {
  __shared__ double red[8];
  double acc = first ? 0.0 : *loss;
  for (int v = 0; v < nviews; ++v) {
    const double2* p = part + (size_t)v * 3 * blocks_per_plane;
    double s = 0.0, a = 0.0;
    for (int i = threadIdx.x; i < 3 * blocks_per_plane; i += blockDim.x) { s += p[i].x; a += p[i].y; }
    const double tS = block_sum_fixed(s, red);
    const double tA = block_sum_fixed(a, red);
    if (threadIdx.x == 0) acc += (1.0 - lam) * tA * inv_n + lam * (1.0 - tS * inv_n);
  }
  if (threadIdx.x == 0) *loss = acc;
}

// ---- K13 regularisers -------------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_reg_partial(PlaneTab P, const uint8_t* __restrict__ occ,
                                                     const uint8_t* __restrict__ mask, int64_t N, double s_max,
                                                     double* __restrict__ part) {
  __shared__ double red[8];
  double cnt = 0.0, hs = 0.0, op = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if ((occ && !occ[i]) || (mask && !mask[i])) continue;
    const float l0 = P.p[3][i], l1 = P.p[4][i], l2 = P.p[5][i];
    const float lm = l1 > l0 ? (l2 > l1 ? l2 : l1) : (l2 > l0 ? l2 : l0);
    const double h = fmax(0.0, exp((double)lm) - s_max);
    const double a = 1.0 / (1.0 + exp(-(double)P.p[10][i]));
    cnt += 1.0;
    hs += h * h;
    op += a * (1.0 - a);
  }
  const double c = block_sum_fixed(cnt, red);
  const double t = block_sum_fixed(hs, red);
  const double u = block_sum_fixed(op, red);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = c;
    part[3 * blockIdx.x + 1] = t;
    part[3 * blockIdx.x + 2] = u;
  }
}

__global__ void __launch_bounds__(256) k_reg_fin(const double* __restrict__ part, int nb, double lam_s, double lam_o,
                                                 double* __restrict__ loss, double* __restrict__ hdr) {
  __shared__ double red[8];
  double c = 0, t = 0, u = 0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) { c += part[3 * i]; t += part[3 * i + 1]; u += part[3 * i + 2]; }
  c = block_sum_fixed(c, red);
  t = block_sum_fixed(t, red);
  u = block_sum_fixed(u, red);
  if (threadIdx.x == 0) {
    *loss = c > 0 ? (lam_s * t + lam_o * u) / c : 0.0;
    hdr[0] = c > 0 ? 1.0 / c : 0.0;
  }
}

__global__ void __launch_bounds__(256) k_reg_grad(PlaneTab P, const uint8_t* __restrict__ occ,
                                                  const uint8_t* __restrict__ mask, int64_t N, double s_max,
                                                  double lam_s, double lam_o, const double* __restrict__ hdr,
                                                  GradTab G) {
  const double inv_n = *hdr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if ((occ && !occ[i]) || (mask && !mask[i])) continue;
    const float l0 = P.p[3][i], l1 = P.p[4][i], l2 = P.p[5][i];
    int am = 0;
    float lm = l0;
    if (l1 > lm) { lm = l1; am = 1; }
    if (l2 > lm) { lm = l2; am = 2; }
    const double s = exp((double)lm);
    const double h = fmax(0.0, s - s_max);
    if (h > 0.0) {
      float* g = G.p[3 + am] + i;
      *g = (float)((double)*g + lam_s * 2.0 * h * s * inv_n);
    }
    const double a = 1.0 / (1.0 + exp(-(double)P.p[10][i]));
    float* go = G.p[10] + i;
    *go = (float)((double)*go + lam_o * (1.0 - 2.0 * a) * a * (1.0 - a) * inv_n);
  }
}

Win make_window() {
  // g_i = exp(-(i - 5)^2 / (2 sigma^2)) / sum, sigma = 1.5, in fp64 on the host
  Win w;
  double s = 0.0;
  for (int i = 0; i < kWin; ++i) { w.g[i] = std::exp(-(double)((i - kR) * (i - kR)) / (2.0 * 1.5 * 1.5)); s += w.g[i]; }
  for (int i = 0; i < kWin; ++i) w.g[i] /= s;
  return w;
}

}  // namespace

size_t photo_view_bytes(int W, int H) {
  const size_t bx = (W + kTX - 1) / kTX, by = (H + kTY - 1) / kTY;
  return (size_t)3 * 3 * W * H * sizeof(float) + 3 * bx * by * sizeof(double2) + 256;   // + alignment slack
}

void launch_photo_loss(int nviews, int W, int H, const float* img, const float* tgt, double lam, float* dl,
                       double* loss, void* ws, int chunk, cudaStream_t s) {
  static const bool attr = [] {
    cudaFuncSetAttribute(k_ssim_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    cudaFuncSetAttribute(k_ssim_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    cudaFuncSetAttribute(k_ssim_fwd, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_ssim_bwd, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return true;
  }();
  (void)attr;
  const Win win = make_window();
  const int bx = (W + kTX - 1) / kTX, by = (H + kTY - 1) / kTY;
  const size_t HW = (size_t)W * H;
  const double inv_n = 1.0 / (3.0 * (double)HW);
  for (int v0 = 0; v0 < nviews; v0 += chunk) {
    const int nv = nviews - v0 < chunk ? nviews - v0 : chunk;
    float* abc = (float*)ws;
    double2* part = (double2*)((char*)ws + (((size_t)chunk * 9 * HW * sizeof(float) + 255) & ~(size_t)255));
    const size_t off = (size_t)v0 * 3 * HW;
    const dim3 grid(bx, by, 3 * nv);
    k_ssim_fwd<<<grid, 256, kFwdSmem, s>>>(img + off, tgt + off, W, H, win, abc, part);
    k_ssim_bwd<<<grid, 256, kBwdSmem, s>>>(img + off, tgt + off, W, H, win, abc, (1.0 - lam) * inv_n, lam * inv_n, dl + off);
    k_photo_fin<<<1, 256, 0, s>>>(part, nv, bx * by, inv_n, lam, loss, v0 == 0);
    count_launches(3);
  }
}

size_t reg_workspace_bytes() { return (size_t)(3 * 4 * 148 + 8) * sizeof(double); }

void launch_reg_loss(const PlaneTab& P, const uint8_t* occ, const uint8_t* mask, int64_t N, double lam_s,
                     double lam_o, double s_max, const GradTab& G, double* loss, void* ws, cudaStream_t s) {
  const int nb = 4 * 148;
  double* part = (double*)ws;
  double* hdr = part + 3 * nb;
  k_reg_partial<<<nb, 256, 0, s>>>(P, occ, mask, N, s_max, part);
  k_reg_fin<<<1, 256, 0, s>>>(part, nb, lam_s, lam_o, loss, hdr);
  k_reg_grad<<<nb, 256, 0, s>>>(P, occ, mask, N, s_max, lam_s, lam_o, hdr, G);
  count_launches(3);
}

}  // namespace puv
