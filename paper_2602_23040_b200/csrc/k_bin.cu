// K2/K4 — key generation and the stable tile pass of the (tile, depth) radix sort (rows a3, a4).
//
// After K3 the visible Gaussians of a view are in (depth_bits, gid) order
// ("rank" order).  Expanding each rank into the tiles of its rect, row-major,
// gives the key sequence in depth order; a STABLE counting sort of that
// sequence by tile id (the high digit, one pass with ntiles buckets) yields
// every tile's list sorted by (depth_bits, gid) — the same order as a full
// LSD radix sort of (tile << 32 | depth_bits) keys emitted in gid order (R8).
//
//   k_koff_*        exclusive scan of tiles-touched over ranks -> key offset per rank, K
//   k_view_finalize carve this view's lists from the arena (device-side bump), overflow flag
//   k_tile_count    per key block b: count[b][tile]                      (smem histogram)
//   k_col_scan      count[b][t] <- sum_{b'<b} count[b'][t]; total[t]
//   k_tile_ranges   tile_start = exclusive scan of total; tile_end
//   k_tile_scatter  per key block: stable placement.  Keys are processed in
//                   groups of 32 consecutive ranks; a per-tile 32-bit mask in
//                   shared memory records which group members hit the tile,
//                   so member m's slot is cursor[t] + popc(mask[t] & (2^m - 1)).
#include "internal.cuh"

namespace puv {

constexpr int kBinThreads = 512;

__device__ __forceinline__ uint32_t rect_tiles(uint2 r) {
  const uint32_t x0 = r.x & 0xffffu, x1 = r.x >> 16, y0 = r.y & 0xffffu, y1 = r.y >> 16;
  return (x1 - x0) * (y1 - y0);
}

// ---- key offsets per rank ----------------------------------------------------------------------

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* sh, uint32_t& total) {
  // 256-thread block exclusive scan (warp shuffles + smem)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (kScanThreads / 32) ? sh[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < (kScanThreads / 32)) sh[lane] = w;
  }
  __syncthreads();
  total = sh[kScanThreads / 32 - 1];
  const uint32_t before = warp > 0 ? sh[warp - 1] : 0u;
  __syncthreads();
  return before + v - x;
}

__global__ void __launch_bounds__(kScanThreads) k_koff_reduce(const uint32_t* __restrict__ sorted,
                                                             const uint2* __restrict__ rect, const ViewHdr* hdr,
                                                             uint32_t* __restrict__ bsum) {
  __shared__ uint32_t sh[32];
  const uint32_t n = hdr->n_vis;
  const uint32_t base = blockIdx.x * kScanTile;
  uint32_t s = 0;
  if (base < n) {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const uint32_t r = base + threadIdx.x * kScanItems + i;
      if (r < n) s += rect_tiles(rect[sorted[r]]);
    }
  }
  uint32_t tot;
  block_excl_scan(s, sh, tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_bsum(uint32_t* data, int m, uint64_t* total_out) {
  __shared__ unsigned long long part[1024];
  const int per = (m + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(m, lo + per);
  unsigned long long s = 0;
  for (int i = lo; i < hi; ++i) s += data[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const unsigned long long t = threadIdx.x >= off ? part[threadIdx.x - off] : 0ull;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  unsigned long long run = part[threadIdx.x] - s;
  for (int i = lo; i < hi; ++i) {
    const uint32_t x = data[i];
    data[i] = (uint32_t)run;   // per-view K < 2^32 is checked in k_view_finalize
    run += x;
  }
  if (threadIdx.x == 1023) *total_out = part[1023];
}

__global__ void __launch_bounds__(kScanThreads) k_koff_write(const uint32_t* __restrict__ sorted,
                                                            const uint2* __restrict__ rect, const ViewHdr* hdr,
                                                            const uint32_t* __restrict__ bsum,
                                                            uint32_t* __restrict__ koff) {
  __shared__ uint32_t sh[32];
  const uint32_t n = hdr->n_vis;
  const uint32_t base = blockIdx.x * kScanTile;
  if (base > n) return;
  uint32_t t[kScanItems], s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint32_t r = base + threadIdx.x * kScanItems + i;
    t[i] = r < n ? rect_tiles(rect[sorted[r]]) : 0u;
    s += t[i];
  }
  uint32_t tot;
  uint32_t run = bsum[blockIdx.x] + block_excl_scan(s, sh, tot);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint32_t r = base + threadIdx.x * kScanItems + i;
    if (r <= n) koff[r] = run;   // koff[n] = K
    run += t[i];
  }
}

__global__ void k_view_finalize(ViewHdr* hdr, CallHdr* call, const uint64_t* ktotal) {
  const uint64_t K = *ktotal;
  hdr->K = K;
  call->arena_need += K;
  const bool fits = K < 0xffffffffull && call->arena_used + K <= call->arena_cap;
  if (fits) {
    hdr->list_base = call->arena_used;
    call->arena_used += K;
    hdr->overflow = 0;
    uint64_t kb = (K + kNbMax - 1) / kNbMax;
    if (kb < 65536) kb = 65536;
    hdr->kb = (uint32_t)kb;
    hdr->nb = (uint32_t)((K + kb - 1) / kb);
  } else {
    hdr->list_base = 0;
    hdr->overflow = 1;
    call->overflow_any = 1;
    hdr->kb = 65536;
    hdr->nb = 0;
  }
}

// ---- key-block enumeration shared by count and scatter ----------------------------------------

struct GroupSmem {
  uint32_t ioff[257];   // item offsets of members (exclusive prefix), [G] = items
  uint32_t j0[256];     // first local key of the member inside this key block
  uint32_t x0[256], y0[256], w[256];
  uint32_t gid[256];
};

// Loads the group of G ranks starting at r into smem; returns items in the group within [klo, khi).
template <int G>
__device__ uint32_t load_group(GroupSmem& gs, uint32_t r, uint32_t n_vis, uint64_t klo, uint64_t khi,
                               const uint32_t* __restrict__ koff, const uint32_t* __restrict__ sorted,
                               const uint2* __restrict__ rect, uint32_t* scan_sh) {
  uint32_t cnt = 0;
  if (threadIdx.x < G) {
    const uint32_t rr = r + threadIdx.x;
    if (rr < n_vis) {
      const uint64_t ks = koff[rr], ke = koff[rr + 1];
      const uint64_t s = ks > klo ? ks : klo, e = ke < khi ? ke : khi;
      cnt = e > s ? (uint32_t)(e - s) : 0u;
      const uint32_t gid = sorted[rr];
      const uint2 rc = rect[gid];
      gs.j0[threadIdx.x] = (uint32_t)(s - ks);
      gs.x0[threadIdx.x] = rc.x & 0xffffu;
      gs.y0[threadIdx.x] = rc.y & 0xffffu;
      gs.w[threadIdx.x] = (rc.x >> 16) - (rc.x & 0xffffu);
      gs.gid[threadIdx.x] = gid;
    }
  }
  // exclusive scan of cnt over the first G threads (G <= 256)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = threadIdx.x < G ? cnt : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (G > 32) {
    if (lane == 31 && warp < G / 32) scan_sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (int w2 = 0; w2 < G / 32; ++w2) { const uint32_t t = scan_sh[w2]; scan_sh[w2] = run; run += t; }
      scan_sh[G / 32] = run;
    }
    __syncthreads();
    if (threadIdx.x < G) gs.ioff[threadIdx.x] = scan_sh[warp] + v - cnt;
    if (threadIdx.x == 0) gs.ioff[G] = scan_sh[G / 32];
  } else {
    if (threadIdx.x < G) gs.ioff[threadIdx.x] = v - cnt;
    if (threadIdx.x == G - 1) gs.ioff[G] = v;
  }
  __syncthreads();
  return gs.ioff[G];
}

// item -> (member, tile)
template <int G>
__device__ __forceinline__ uint32_t item_tile(const GroupSmem& gs, uint32_t it, int gx, uint32_t& m) {
  uint32_t lo = 0, hi = G;  // largest m with ioff[m] <= it
#pragma unroll
  for (int s = G / 2; s >= 1; s >>= 1) {
    const uint32_t mid = lo + s;
    if (mid < hi && gs.ioff[mid] <= it) lo = mid;
  }
  m = lo;
  const uint32_t j = gs.j0[lo] + (it - gs.ioff[lo]);
  const uint32_t w = gs.w[lo];
  const uint32_t q = j / w;
  return (gs.y0[lo] + q) * (uint32_t)gx + gs.x0[lo] + (j - q * w);
}

__device__ __forceinline__ uint32_t first_rank(const uint32_t* __restrict__ koff, uint32_t n_vis, uint64_t klo) {
  // largest r < n_vis with koff[r] <= klo  (koff strictly increasing: every rank has >= 1 key)
  uint32_t lo = 0, hi = n_vis;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)koff[mid] <= klo) lo = mid; else hi = mid;
  }
  return lo;
}

template <int G>
__global__ void __launch_bounds__(kBinThreads) k_tile_count(const ViewHdr* hdr, const uint32_t* __restrict__ koff,
                                                           const uint32_t* __restrict__ sorted,
                                                           const uint2* __restrict__ rect, int gx, int ntiles,
                                                           uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t scnt[];
  __shared__ GroupSmem gs;
  __shared__ uint32_t scan_sh[16];
  const ViewHdr h = *hdr;
  if (h.overflow) return;
  for (uint32_t b = blockIdx.x; b < h.nb; b += gridDim.x) {
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) scnt[t] = 0;
    const uint64_t klo = (uint64_t)b * h.kb;
    const uint64_t khi = klo + h.kb < h.K ? klo + h.kb : h.K;
    uint32_t r = first_rank(koff, h.n_vis, klo);
    __syncthreads();
    while (r < h.n_vis && (uint64_t)koff[r] < khi) {
      const uint32_t items = load_group<G>(gs, r, h.n_vis, klo, khi, koff, sorted, rect, scan_sh);
      for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        uint32_t m;
        atomicAdd(&scnt[item_tile<G>(gs, it, gx, m)], 1u);
      }
      r += G;
      __syncthreads();
    }
    uint32_t* row = cnt + (size_t)b * ntiles;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) row[t] = scnt[t];
    __syncthreads();
  }
}

// Column exclusive scan: block = 32 tiles x 32 warps; warp w owns a chunk of rows.
__global__ void __launch_bounds__(1024) k_col_scan(const ViewHdr* hdr, uint32_t* __restrict__ cnt, int ntiles,
                                                   uint32_t* __restrict__ total) {
  __shared__ uint32_t part[32][33];
  const uint32_t nb = hdr->overflow ? 0u : hdr->nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const uint32_t per = (nb + 31) / 32;
  const uint32_t b0 = warp * per, b1 = min(nb, b0 + per);
  uint32_t s = 0;
  if (t < ntiles)
    for (uint32_t b = b0; b < b1; ++b) s += cnt[(size_t)b * ntiles + t];
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    uint32_t run = 0;
    for (int w = 0; w < 32; ++w) { const uint32_t x = part[w][lane]; part[w][lane] = run; run += x; }
    if (t < ntiles) total[t] = run;
  }
  __syncthreads();
  if (t < ntiles) {
    uint32_t run = part[warp][lane];
    for (uint32_t b = b0; b < b1; ++b) {
      const size_t i = (size_t)b * ntiles + t;
      const uint32_t x = cnt[i];
      cnt[i] = run;
      run += x;
    }
  }
}

// `total` may alias `tend` (each thread reads its own totals before writing them back)
__global__ void __launch_bounds__(1024) k_tile_ranges(const uint32_t* total, int ntiles, uint32_t* tstart,
                                                      uint32_t* tend) {
  __shared__ uint32_t part[1024];
  const int per = (ntiles + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(ntiles, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += total[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t x = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += x;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;
  for (int i = lo; i < hi; ++i) {
    tstart[i] = run;
    run += total[i];
    tend[i] = run;
  }
}

template <bool SMEM_CURSOR>
__global__ void __launch_bounds__(kBinThreads) k_tile_scatter(const ViewHdr* hdr, const uint32_t* __restrict__ koff,
                                                             const uint32_t* __restrict__ sorted,
                                                             const uint2* __restrict__ rect, int gx, int ntiles,
                                                             uint32_t* __restrict__ cnt,
                                                             const uint32_t* __restrict__ tstart,
                                                             uint32_t* __restrict__ arena) {
  constexpr int G = 32;
  extern __shared__ uint32_t dyn[];
  uint32_t* smask = dyn;
  __shared__ GroupSmem gs;
  __shared__ uint32_t scan_sh[16];
  const ViewHdr h = *hdr;
  if (h.overflow) return;
  uint32_t* list = arena + h.list_base;
  for (uint32_t b = blockIdx.x; b < h.nb; b += gridDim.x) {
    uint32_t* row = cnt + (size_t)b * ntiles;
    uint32_t* cursor = SMEM_CURSOR ? dyn + ntiles : row;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
      smask[t] = 0;
      if (SMEM_CURSOR) cursor[t] = tstart[t] + row[t];
      else row[t] += tstart[t];
    }
    const uint64_t klo = (uint64_t)b * h.kb;
    const uint64_t khi = klo + h.kb < h.K ? klo + h.kb : h.K;
    uint32_t r = first_rank(koff, h.n_vis, klo);
    __syncthreads();
    while (r < h.n_vis && (uint64_t)koff[r] < khi) {
      const uint32_t items = load_group<G>(gs, r, h.n_vis, klo, khi, koff, sorted, rect, scan_sh);
      // phase A: mark members per tile
      for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        uint32_t m;
        const uint32_t t = item_tile<G>(gs, it, gx, m);
        atomicOr(&smask[t], 1u << m);
      }
      __syncthreads();
      // phase B: place
      for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        uint32_t m;
        const uint32_t t = item_tile<G>(gs, it, gx, m);
        const uint32_t mk = smask[t];
        list[cursor[t] + __popc(mk & ((1u << m) - 1u))] = gs.gid[m];
      }
      __syncthreads();
      // phase C: the highest member of each touched tile advances its cursor and clears the mask
      for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        uint32_t m;
        const uint32_t t = item_tile<G>(gs, it, gx, m);
        const uint32_t mk = smask[t];
        if (mk != 0u && (31u - __clz(mk)) == m) {
          cursor[t] += __popc(mk);
          smask[t] = 0;
        }
      }
      r += G;
      __syncthreads();
    }
  }
}

void launch_bin(const Plan& p, const Views& v, void* state, uint32_t* arena, int view, cudaStream_t s) {
  char* st = (char*)state;
  const uint32_t* sorted = v.sorted + (size_t)view * p.N;
  const uint2* rect = v.rect + (size_t)view * p.N;
  ViewHdr* hdr = v.hdr + view;
  uint32_t* bsum = (uint32_t*)(st + p.bsum);
  uint32_t* koff = (uint32_t*)(st + p.koff);
  uint32_t* cnt = (uint32_t*)(st + p.cnt);
  uint64_t* ktot = &hdr->ktotal;  // scratch: K of this view before finalize
  uint32_t* tstart = v.tstart + (size_t)view * p.ntiles;
  uint32_t* tend = v.tend + (size_t)view * p.ntiles;
  const int nsb = p.N / kScanTile + 1;   // one extra block so koff[n_vis] (= K) is always written
  k_koff_reduce<<<nsb, kScanThreads, 0, s>>>(sorted, rect, hdr, bsum);
  k_scan_bsum<<<1, 1024, 0, s>>>(bsum, nsb, ktot);
  k_koff_write<<<nsb, kScanThreads, 0, s>>>(sorted, rect, hdr, bsum, koff);
  k_view_finalize<<<1, 1, 0, s>>>(hdr, v.call, ktot);

  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t cnt_smem = (size_t)p.ntiles * 4;
  cudaFuncSetAttribute(k_tile_count<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cnt_smem);
  k_tile_count<256><<<2 * nsm, kBinThreads, cnt_smem, s>>>(hdr, koff, sorted, rect, p.gx, p.ntiles, cnt);
  k_col_scan<<<(p.ntiles + 31) / 32, 1024, 0, s>>>(hdr, cnt, p.ntiles, tend /* totals */);
  k_tile_ranges<<<1, 1024, 0, s>>>(tend, p.ntiles, tstart, tend);
  const bool smem_cursor = (size_t)p.ntiles * 8 <= 160 * 1024;
  const size_t sc_smem = (size_t)p.ntiles * (smem_cursor ? 8 : 4);
  if (smem_cursor) {
    cudaFuncSetAttribute(k_tile_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc_smem);
    k_tile_scatter<true><<<2 * nsm, kBinThreads, sc_smem, s>>>(hdr, koff, sorted, rect, p.gx, p.ntiles, cnt, tstart,
                                                               arena);
  } else {
    cudaFuncSetAttribute(k_tile_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc_smem);
    k_tile_scatter<false><<<2 * nsm, kBinThreads, sc_smem, s>>>(hdr, koff, sorted, rect, p.gx, p.ntiles, cnt, tstart,
                                                                arena);
  }
  count_launches(8);
}

}  // namespace puv
