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
//   k_block_starts  first rank of every key block (one binary search per block)
//   k_tile_count    per (key block b, tile band): count[b][tile]           (smem histogram)
//   k_col_scan      count[b][t] <- sum_{b'<b} count[b'][t]; total[t]
//   k_tile_ranges   tile_start = exclusive scan of total; tile_end
//   k_tile_scatter  per (key block, tile band): stable placement.  Ranks are
//                   staged 256 at a time ("super-group"); keys are placed in
//                   sub-groups of 32 consecutive ranks; a per-tile 32-bit mask
//                   in shared memory records which sub-group members hit the
//                   tile, so member m's slot is cursor[t] + popc(mask[t] & (2^m-1)).
//                   Masks are double-buffered so "advance cursors" of one
//                   sub-group and "mark" of the next share a barrier interval.
// A tile band is a run of whole tile rows (<= kBandTiles tiles); every key of a
// block falls in exactly one band, so bands split the work without changing the
// order, and a CTA only holds its band's masks and cursors in shared memory.
#include "internal.cuh"

namespace puv {

constexpr int kBinThreads = 512;
constexpr int kSG = 256;          // ranks staged per super-group
constexpr int kSub = 32;          // ranks per placement sub-group (mask width)
constexpr int kItemCache = 2048;  // items of a sub-group whose (tile, member) are cached in smem
constexpr int kBandTiles = 2048;  // max tiles per band

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

// Views are binned concurrently on several streams: the arena is carved with atomics (a view's
// list_base depends on the completion order; its contents do not).
__global__ void k_view_finalize(ViewHdr* hdr, CallHdr* call, const uint64_t* ktotal) {
  const uint64_t K = *ktotal;
  hdr->K = K;
  atomicAdd((unsigned long long*)&call->arena_need, (unsigned long long)K);
  const uint64_t base = K < 0xffffffffull ? atomicAdd((unsigned long long*)&call->arena_used, (unsigned long long)K)
                                          : ~0ull;
  const bool fits = base != ~0ull && base + K <= call->arena_cap;
  if (fits) {
    hdr->list_base = base;
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

// bstart[b] = largest rank r < n_vis with koff[r] <= b*kb  (koff strictly increasing: every rank has >= 1 key)
__global__ void k_block_starts(const ViewHdr* hdr, const uint32_t* __restrict__ koff, uint32_t* __restrict__ bstart) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  const ViewHdr h = *hdr;
  if (h.overflow || b >= h.nb) return;
  const uint64_t klo = (uint64_t)b * h.kb;
  uint32_t lo = 0, hi = h.n_vis;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)koff[mid] <= klo) lo = mid; else hi = mid;
  }
  bstart[b] = lo;
}

// ---- key-block x band enumeration shared by count and scatter ---------------------------------

struct Band {
  uint32_t y0, y1;     // tile rows [y0, y1)
  uint32_t t0, nt;     // first tile id, tiles in the band
};

__device__ __forceinline__ Band band_of(uint32_t band, int band_rows, int gx, int gy) {
  Band b;
  b.y0 = band * band_rows;
  b.y1 = min((uint32_t)gy, b.y0 + band_rows);
  b.t0 = b.y0 * gx;
  b.nt = (b.y1 - b.y0) * gx;
  return b;
}

struct SuperGroup {
  uint32_t ioff[kSG + 1];   // item offsets of members (exclusive prefix), [kSG] = items
  uint32_t j0[kSG];         // first local key (row-major index in the rect) of the member
  uint32_t x0[kSG], y0[kSG], w[kSG];
  float iw[kSG];            // 1 / w
  uint32_t gid[kSG];
  uint32_t scan[kBinThreads / 32 + 1];
};

// Stage ranks [r, r + kSG) clipped to the key block [klo, khi) and to the band rows; returns items.
__device__ uint32_t load_super(SuperGroup& sg, uint32_t r, uint32_t n_vis, uint64_t klo, uint64_t khi,
                               const Band& bd, const uint32_t* __restrict__ koff,
                               const uint32_t* __restrict__ sorted, const uint2* __restrict__ rect) {
  uint32_t cnt = 0;
  if (threadIdx.x < kSG) {
    const uint32_t rr = r + threadIdx.x;
    if (rr < n_vis) {
      const uint64_t ks = koff[rr], ke = koff[rr + 1];
      const uint64_t s = ks > klo ? ks : klo, e = ke < khi ? ke : khi;
      if (e > s) {
        const uint32_t gid = sorted[rr];
        const uint2 rc = rect[gid];
        const uint32_t x0 = rc.x & 0xffffu, w = (rc.x >> 16) - x0;
        const uint32_t y0 = rc.y & 0xffffu, y1 = rc.y >> 16;
        const uint32_t ry0 = max(y0, bd.y0), ry1 = min(y1, bd.y1);
        uint32_t js = (uint32_t)(s - ks), je = (uint32_t)(e - ks);
        if (ry1 > ry0) {
          js = max(js, (ry0 - y0) * w);
          je = min(je, (ry1 - y0) * w);
          cnt = je > js ? je - js : 0u;
        }
        if (cnt) {
          sg.j0[threadIdx.x] = js;
          sg.x0[threadIdx.x] = x0;
          sg.y0[threadIdx.x] = y0;
          sg.w[threadIdx.x] = w;
          sg.iw[threadIdx.x] = 1.0f / (float)w;
          sg.gid[threadIdx.x] = gid;
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = threadIdx.x < kSG ? cnt : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31 && warp < kSG / 32) sg.scan[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int w2 = 0; w2 < kSG / 32; ++w2) { const uint32_t t = sg.scan[w2]; sg.scan[w2] = run; run += t; }
    sg.scan[kSG / 32] = run;
  }
  __syncthreads();
  if (threadIdx.x < kSG) sg.ioff[threadIdx.x] = sg.scan[warp] + v - cnt;
  if (threadIdx.x == 0) sg.ioff[kSG] = sg.scan[kSG / 32];
  __syncthreads();
  return sg.ioff[kSG];
}

// item `it` of members [mlo, mlo + SPAN) -> (member, band-local tile)
template <int SPAN>
__device__ __forceinline__ uint32_t item_tile(const SuperGroup& sg, uint32_t mlo, uint32_t it, int gx, uint32_t by0,
                                              uint32_t& m) {
  uint32_t lo = mlo;  // largest m in [mlo, mlo + SPAN) with ioff[m] <= it
#pragma unroll
  for (int s = SPAN / 2; s >= 1; s >>= 1)
    if (sg.ioff[lo + s] <= it) lo += s;
  m = lo;
  const uint32_t j = sg.j0[lo] + (it - sg.ioff[lo]);
  const uint32_t w = sg.w[lo];
  uint32_t q = (uint32_t)((float)j * sg.iw[lo]);
  int32_t rem = (int32_t)(j - q * w);
  if (rem < 0) { --q; rem += (int32_t)w; }
  if (rem >= (int32_t)w) { ++q; rem -= (int32_t)w; }
  return (sg.y0[lo] + q - by0) * (uint32_t)gx + sg.x0[lo] + (uint32_t)rem;
}

__global__ void __launch_bounds__(kBinThreads) k_tile_count(const ViewHdr* hdr, const uint32_t* __restrict__ koff,
                                                           const uint32_t* __restrict__ sorted,
                                                           const uint2* __restrict__ rect,
                                                           const uint32_t* __restrict__ bstart, int gx, int gy,
                                                           int band_rows, int nbands, int ntiles,
                                                           uint32_t* __restrict__ cnt) {
  __shared__ uint32_t scnt[kBandTiles];
  __shared__ SuperGroup sg;
  const ViewHdr h = *hdr;
  if (h.overflow) return;
  for (uint32_t wi = blockIdx.x; wi < h.nb * (uint32_t)nbands; wi += gridDim.x) {
    const uint32_t b = wi / nbands;
    const Band bd = band_of(wi % nbands, band_rows, gx, gy);
    for (uint32_t t = threadIdx.x; t < bd.nt; t += blockDim.x) scnt[t] = 0;
    const uint64_t klo = (uint64_t)b * h.kb;
    const uint64_t khi = klo + h.kb < h.K ? klo + h.kb : h.K;
    uint32_t r = bstart[b];
    __syncthreads();
    while (r < h.n_vis && (uint64_t)koff[r] < khi) {
      const uint32_t items = load_super(sg, r, h.n_vis, klo, khi, bd, koff, sorted, rect);
      for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        uint32_t m;
        atomicAdd(&scnt[item_tile<kSG>(sg, 0, it, gx, bd.y0, m)], 1u);
      }
      r += kSG;
      __syncthreads();
    }
    uint32_t* row = cnt + (size_t)b * ntiles + bd.t0;
    for (uint32_t t = threadIdx.x; t < bd.nt; t += blockDim.x) row[t] = scnt[t];
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

// advance cursors of a finished sub-group from its cached items and clear its mask
__device__ __forceinline__ void advance_cached(const uint32_t* icache, uint32_t items, uint32_t* mask,
                                               uint32_t* cursor) {
  for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
    const uint32_t c = icache[it];
    const uint32_t t = c & 0x7ffffffu, m = c >> 27;
    const uint32_t mk = mask[t];
    if (mk != 0u && (31u - __clz(mk)) == m) {
      cursor[t] += __popc(mk);
      mask[t] = 0;
    }
  }
}

__global__ void __launch_bounds__(kBinThreads) k_tile_scatter(const ViewHdr* hdr, const uint32_t* __restrict__ koff,
                                                             const uint32_t* __restrict__ sorted,
                                                             const uint2* __restrict__ rect,
                                                             const uint32_t* __restrict__ bstart, int gx, int gy,
                                                             int band_rows, int nbands, int ntiles,
                                                             const uint32_t* __restrict__ cnt,
                                                             const uint32_t* __restrict__ tstart,
                                                             uint32_t* __restrict__ arena) {
  __shared__ uint32_t smask[2][kBandTiles];
  __shared__ uint32_t cursor[kBandTiles];
  __shared__ SuperGroup sg;
  __shared__ uint32_t icache[2][kItemCache];   // tile | member << 27 of the current / previous sub-group
  const ViewHdr h = *hdr;
  if (h.overflow) return;
  uint32_t* list = arena + h.list_base;
  for (uint32_t wi = blockIdx.x; wi < h.nb * (uint32_t)nbands; wi += gridDim.x) {
    const uint32_t b = wi / nbands;
    const Band bd = band_of(wi % nbands, band_rows, gx, gy);
    const uint32_t* row = cnt + (size_t)b * ntiles + bd.t0;
    for (uint32_t t = threadIdx.x; t < bd.nt; t += blockDim.x) {
      smask[0][t] = 0;
      smask[1][t] = 0;
      cursor[t] = tstart[bd.t0 + t] + row[t];
    }
    const uint64_t klo = (uint64_t)b * h.kb;
    const uint64_t khi = klo + h.kb < h.K ? klo + h.kb : h.K;
    uint32_t r = bstart[b];
    __syncthreads();
    uint32_t par = 0;
    uint32_t prev_items = 0;   // items of the previous (cached) sub-group whose cursors still advance
    while (r < h.n_vis && (uint64_t)koff[r] < khi) {
      load_super(sg, r, h.n_vis, klo, khi, bd, koff, sorted, rect);
      for (int s = 0; s < kSG / kSub; ++s) {
        const uint32_t mlo = s * kSub;
        const uint32_t i0 = sg.ioff[mlo], i1 = sg.ioff[mlo + kSub];
        const uint32_t items = i1 - i0;
        if (items == 0) continue;   // uniform
        uint32_t* mk_cur = smask[par];
        // phase A: mark members per tile; advance the previous sub-group (other buffers)
        for (uint32_t k = threadIdx.x; k < items; k += blockDim.x) {
          uint32_t m;
          const uint32_t t = item_tile<kSub>(sg, mlo, i0 + k, gx, bd.y0, m);
          const uint32_t ml = m - mlo;
          if (k < kItemCache) icache[par][k] = t | (ml << 27);
          atomicOr(&mk_cur[t], 1u << ml);
        }
        if (prev_items) {
          advance_cached(icache[par ^ 1], prev_items, smask[par ^ 1], cursor);
          prev_items = 0;
        }
        __syncthreads();
        // phase B: place
        for (uint32_t k = threadIdx.x; k < items; k += blockDim.x) {
          uint32_t t, ml;
          if (k < kItemCache) {
            const uint32_t c = icache[par][k];
            t = c & 0x7ffffffu;
            ml = c >> 27;
          } else {
            uint32_t m;
            t = item_tile<kSub>(sg, mlo, i0 + k, gx, bd.y0, m);
            ml = m - mlo;
          }
          const uint32_t mk = mk_cur[t];
          list[cursor[t] + __popc(mk & ((1u << ml) - 1u))] = sg.gid[mlo + ml];
        }
        __syncthreads();
        if (items > kItemCache) {
          // rare oversized sub-group: advance now (uncached items need sg), one extra barrier
          for (uint32_t k = threadIdx.x; k < items; k += blockDim.x) {
            uint32_t t, ml;
            if (k < kItemCache) {
              const uint32_t c = icache[par][k];
              t = c & 0x7ffffffu;
              ml = c >> 27;
            } else {
              uint32_t m;
              t = item_tile<kSub>(sg, mlo, i0 + k, gx, bd.y0, m);
              ml = m - mlo;
            }
            const uint32_t mk = mk_cur[t];
            if (mk != 0u && (31u - __clz(mk)) == ml) {
              cursor[t] += __popc(mk);
              mk_cur[t] = 0;
            }
          }
          __syncthreads();
        } else {
          prev_items = items;   // advanced together with the next sub-group's phase A
          par ^= 1;
        }
      }
      r += kSG;
    }
    // (the last cached sub-group's advance is not needed: masks and cursors are re-initialised)
    __syncthreads();
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
  uint32_t* bstart = (uint32_t*)(st + p.bstart);
  uint64_t* ktot = &hdr->ktotal;  // scratch: K of this view before finalize
  uint32_t* tstart = v.tstart + (size_t)view * p.ntiles;
  uint32_t* tend = v.tend + (size_t)view * p.ntiles;
  const int nsb = p.N / kScanTile + 1;   // one extra block so koff[n_vis] (= K) is always written
  k_koff_reduce<<<nsb, kScanThreads, 0, s>>>(sorted, rect, hdr, bsum);
  k_scan_bsum<<<1, 1024, 0, s>>>(bsum, nsb, ktot);
  k_koff_write<<<nsb, kScanThreads, 0, s>>>(sorted, rect, hdr, bsum, koff);
  k_view_finalize<<<1, 1, 0, s>>>(hdr, v.call, ktot);
  k_block_starts<<<(kNbMax + 255) / 256, 256, 0, s>>>(hdr, koff, bstart);

  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int band_rows = p.gx >= kBandTiles ? 1 : (kBandTiles / p.gx < p.gy ? kBandTiles / p.gx : p.gy);
  const int nbands = (p.gy + band_rows - 1) / band_rows;
  k_tile_count<<<4 * nsm, kBinThreads, 0, s>>>(hdr, koff, sorted, rect, bstart, p.gx, p.gy, band_rows, nbands,
                                              p.ntiles, cnt);
  k_col_scan<<<(p.ntiles + 31) / 32, 1024, 0, s>>>(hdr, cnt, p.ntiles, tend /* totals */);
  k_tile_ranges<<<1, 1024, 0, s>>>(tend, p.ntiles, tstart, tend);
  k_tile_scatter<<<4 * nsm, kBinThreads, 0, s>>>(hdr, koff, sorted, rect, bstart, p.gx, p.gy, band_rows, nbands,
                                                p.ntiles, cnt, tstart, arena);
  count_launches(9);
}

}  // namespace puv
