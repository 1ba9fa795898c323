// K11 — covariance-aware flow masking, supp. Algorithm 1.
//
// Per camera: a summed-area table of the motion mask (two scan kernels), then
// one thread per texel: Sigma3D (contract U1-U4), camera-space mean, UNclamped
// EWA Jacobian, Sigma2D + 0.3, validity (z <= 0 or det <= 1e-7 -> static), radius
// r = min(r_max, ceil(3 sqrt(lambda_max))), window = integer pixels with
// |p - m|_inf <= r inside the image; dynamic iff some window pixel has mask = 1
// and d^2 <= 9 (contract R1 power >= -4.5).  The SAT answers "does the window /
// this window row contain any mask pixel" in O(1), so empty windows and rows are
// skipped without changing any decision.  D_i = OR over cameras, accumulated in
// the thread's own label byte across the per-camera launches (no atomics).
// Every decision uses the fp32 contract, so labels are bit-identical to the
// oracle's plain window scan.
#include "contract.cuh"
#include "internal.cuh"
#include "project.cuh"

namespace puv {

// S[(y+1)*(W+1) + (x+1)] = sum of mask[0..y][0..x]; row 0 / column 0 are zero.
__global__ void __launch_bounds__(1024) k_sat_rows(const uint8_t* __restrict__ mask, int W, int H,
                                                   uint32_t* __restrict__ S) {
  __shared__ uint32_t part[1024];
  const int y = blockIdx.x;            // one block per image row (y < H), block H writes row 0 of S
  if (y == H) {
    for (int x = threadIdx.x; x <= W; x += blockDim.x) S[x] = 0;
    return;
  }
  const uint8_t* row = mask + (size_t)y * W;
  uint32_t* out = S + (size_t)(y + 1) * (W + 1);
  if (threadIdx.x == 0) out[0] = 0;
  const int per = (W + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(W, lo + per);
  uint32_t s = 0;
  for (int x = lo; x < hi; ++x) s += row[x] != 0;
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t t = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;
  for (int x = lo; x < hi; ++x) {
    run += row[x] != 0;
    out[x + 1] = run;
  }
}

// Column prefix over rows 1..H: block = 32 columns x 32 warps, warp w owns a chunk of rows.
__global__ void __launch_bounds__(1024) k_sat_cols(int W, int H, uint32_t* __restrict__ S) {
  __shared__ uint32_t part[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = blockIdx.x * 32 + lane;
  const int per = (H + 31) / 32;
  const int r0 = 1 + warp * per, r1 = min(H + 1, r0 + per);
  uint32_t s = 0;
  if (x <= W)
    for (int y = r0; y < r1; ++y) s += S[(size_t)y * (W + 1) + x];
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    uint32_t run = 0;
    for (int w = 0; w < 32; ++w) { const uint32_t t = part[w][lane]; part[w][lane] = run; run += t; }
  }
  __syncthreads();
  if (x <= W) {
    uint32_t run = part[warp][lane];
    for (int y = r0; y < r1; ++y) {
      uint32_t* p = S + (size_t)y * (W + 1) + x;
      run += *p;
      *p = run;
    }
  }
}

__device__ __forceinline__ uint32_t sat_count(const uint32_t* S, int W1, int x0, int x1, int y0, int y1) {
  // mask pixels in [x0, x1] x [y0, y1] (inclusive)
  return S[(size_t)(y1 + 1) * W1 + (x1 + 1)] - S[(size_t)y0 * W1 + (x1 + 1)] - S[(size_t)(y1 + 1) * W1 + x0] +
         S[(size_t)y0 * W1 + x0];
}

__device__ bool project_window(const PlaneTab& P, const PosMode& pm, int g, const CamDev& cam, int r_max, const uint32_t* S, float& mx,
                               float& my, float& ha, float& nb, float& hc, int& x0, int& x1, int& y0, int& y1);

__global__ void __launch_bounds__(128) k_label(PlaneTab P, PosMode pm, const uint8_t* __restrict__ occ, int N,
                                               const __grid_constant__ CamDev cam, const uint8_t* __restrict__ mask,
                                               const uint32_t* __restrict__ S, int r_max, int first,
                                               uint8_t* __restrict__ labels) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  // phase 1 (per lane): projection, validity, window and the O(1) "window holds a mask pixel" test
  bool cand = false;
  float mx = 0.f, my = 0.f, ha = 0.f, nb = 0.f, hc = 0.f;
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
  if (g < N) {
    if (first) labels[g] = 0;
    cand = (first || !labels[g]) && (occ == nullptr || occ[g] != 0);   // OR over cameras: skip if dynamic
  }
  if (cand) cand = project_window(P, pm, g, cam, r_max, S, mx, my, ha, nb, hc, x0, x1, y0, y1);
  // phase 2 (warp-cooperative): scan the candidate windows one at a time, 32 pixels per step
  uint32_t todo = __ballot_sync(0xffffffffu, cand);
  const int W1 = cam.W + 1;
  while (todo) {
    const int leader = __ffs(todo) - 1;
    todo &= todo - 1;
    const float lmx = __shfl_sync(0xffffffffu, mx, leader), lmy = __shfl_sync(0xffffffffu, my, leader);
    const float lha = __shfl_sync(0xffffffffu, ha, leader), lnb = __shfl_sync(0xffffffffu, nb, leader);
    const float lhc = __shfl_sync(0xffffffffu, hc, leader);
    const int lx0 = __shfl_sync(0xffffffffu, x0, leader), lx1 = __shfl_sync(0xffffffffu, x1, leader);
    const int ly0 = __shfl_sync(0xffffffffu, y0, leader), ly1 = __shfl_sync(0xffffffffu, y1, leader);
    bool hit = false;
    for (int j = ly0; j <= ly1 && !hit; ++j) {
      if (sat_count(S, W1, lx0, lx1, j, j) == 0) continue;      // no mask pixel in this window row
      const uint8_t* row = mask + (size_t)j * cam.W;
      const float fj = (float)j;
      for (int i0 = lx0; i0 <= lx1 && !hit; i0 += 32) {
        const int i = i0 + lane;
        const bool h = i <= lx1 && row[i] && pair_power(lmx, lmy, lha, lnb, lhc, (float)i, fj) >= -4.5f;
        hit = __any_sync(0xffffffffu, h);
      }
    }
    if (hit && lane == leader) labels[g] = 1;
  }
}

// Alg. 1 steps 1-4 for texel g and camera `cam`; returns false when the camera cannot mark the
// texel (invalid projection, empty window, or no mask pixel inside the window).
__device__ bool project_window(const PlaneTab& P, const PosMode& pm, int g, const CamDev& cam, int r_max, const uint32_t* S, float& mx,
                               float& my, float& ha, float& nb, float& hc, int& x0, int& x1, int& y0, int& y1) {
  const Unpacked u = unpack_contract(__ldg(P.p[3] + g), __ldg(P.p[4] + g), __ldg(P.p[5] + g), __ldg(P.p[6] + g),
                                     __ldg(P.p[7] + g), __ldg(P.p[8] + g), __ldg(P.p[9] + g), __ldg(P.p[10] + g));
  if (!u.ok) return false;
  float mux, muy, muz;
  texel_mu(P, pm, g, mux, muy, muz);
  const CamPoint cp = cam_point(cam, mux, muy, muz);
  if (!(cp.z > 0.0f)) return false;                             // Alg. 1: z <= 0 -> static
  // Alg. 1's Jacobian has no clamp: J02 = -fx x / z^2 with the unclamped x/z
  const float J00 = dvd(cam.fx, cp.z), J02 = -dvd(mul(cam.fx, cp.ux), cp.z);
  const float J11 = dvd(cam.fy, cp.z), J12 = -dvd(mul(cam.fy, cp.uy), cp.z);
  const float* V = cam.V;
  const float T00 = add(mul(J00, V[0]), mul(J02, V[8])), T01 = add(mul(J00, V[1]), mul(J02, V[9]));
  const float T02 = add(mul(J00, V[2]), mul(J02, V[10]));
  const float T10 = add(mul(J11, V[4]), mul(J12, V[8])), T11 = add(mul(J11, V[5]), mul(J12, V[9]));
  const float T12 = add(mul(J11, V[6]), mul(J12, V[10]));
  const float W00 = add(add(mul(u.S00, T00), mul(u.S01, T01)), mul(u.S02, T02));
  const float W01 = add(add(mul(u.S01, T00), mul(u.S11, T01)), mul(u.S12, T02));
  const float W02 = add(add(mul(u.S02, T00), mul(u.S12, T01)), mul(u.S22, T02));
  const float W10 = add(add(mul(u.S00, T10), mul(u.S01, T11)), mul(u.S02, T12));
  const float W11 = add(add(mul(u.S01, T10), mul(u.S11, T11)), mul(u.S12, T12));
  const float W12 = add(add(mul(u.S02, T10), mul(u.S12, T11)), mul(u.S22, T12));
  const float a = add(add(add(mul(T00, W00), mul(T01, W01)), mul(T02, W02)), 0.3f);
  const float b = add(add(mul(T10, W00), mul(T11, W01)), mul(T12, W02));
  const float c = add(add(add(mul(T10, W10), mul(T11, W11)), mul(T12, W12)), 0.3f);
  const float det = sub(mul(a, c), mul(b, b));
  if (!(det > 1e-7f)) return false;
  ha = mul(-0.5f, dvd(c, det));
  nb = dvd(b, det);
  hc = mul(-0.5f, dvd(a, det));
  const float tr = add(a, c);
  const float lam = mul(0.5f, add(tr, sqrt_(fmaxf(0.0f, sub(mul(tr, tr), mul(4.0f, det))))));
  const float rf = fminf((float)r_max, ceilf(mul(3.0f, sqrt_(lam))));
  mx = add(mul(cam.fx, cp.ux), cam.cx);
  my = add(mul(cam.fy, cp.uy), cam.cy);
  const float fx0 = fmaxf(ceilf(sub(mx, rf)), 0.0f), fx1 = fminf(floorf(add(mx, rf)), (float)(cam.W - 1));
  const float fy0 = fmaxf(ceilf(sub(my, rf)), 0.0f), fy1 = fminf(floorf(add(my, rf)), (float)(cam.H - 1));
  if (fx0 > fx1 || fy0 > fy1) return false;
  x0 = (int)fx0; x1 = (int)fx1; y0 = (int)fy0; y1 = (int)fy1;
  return sat_count(S, cam.W + 1, x0, x1, y0, y1) != 0;          // any mask pixel in the window?
}

void launch_label(const Plan& p, const PlaneTab& P, const uint8_t* occ, const CamDev& cam, const uint8_t* mask,
                  uint32_t* sat, int r_max, int first, uint8_t* labels, cudaStream_t s) {
  k_sat_rows<<<cam.H + 1, 1024, 0, s>>>(mask, cam.W, cam.H, sat);
  k_sat_cols<<<(cam.W + 1 + 31) / 32, 1024, 0, s>>>(cam.W, cam.H, sat);
  k_label<<<(p.N + 127) / 128, 128, 0, s>>>(P, p.pm, occ, p.N, cam, mask, sat, r_max, first, labels);
  count_launches(3);
}

}  // namespace puv
