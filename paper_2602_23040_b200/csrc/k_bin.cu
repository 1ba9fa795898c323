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

#ifndef PUV_BIN_THREADS
#define PUV_BIN_THREADS 256
#endif
#ifndef PUV_BIN_CTAS_PER_SM
#define PUV_BIN_CTAS_PER_SM 8
#endif
constexpr int kBinThreads = PUV_BIN_THREADS;
constexpr int kSG = kBinThreads < 256 ? kBinThreads : 256;   // ranks staged per super-group
constexpr int kSub = 32;          // ranks per placement sub-group (mask width)
#ifndef PUV_BIN_ITEM_CACHE
#define PUV_BIN_ITEM_CACHE 1024
#endif
#ifndef PUV_BIN_BAND_TILES
#define PUV_BIN_BAND_TILES 512
#endif
constexpr int kItemCache = PUV_BIN_ITEM_CACHE;  // items of a sub-group whose (tile, member) are cached in smem
constexpr int kBandTiles = PUV_BIN_BAND_TILES;  // max tiles per band

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
      if (r < n) s += rect_tiles(rect[sorted ? sorted[r] : r]);
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
    t[i] = r < n ? rect_tiles(rect[sorted ? sorted[r] : r]) : 0u;
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
// list_base depends on the completion order; its contents do not) -- see k_view_finalize2.

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
        const uint32_t gid = sorted ? sorted[rr] : rr;
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
          PUV_CHECK(cursor[t] + __popc(mk & ((1u << ml) - 1u)) < h.K);
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

// ---- two-level tile pass ---------------------------------------------------------------------
//
// Level 1 bins the RANKS into super-tiles of kSup x kSup tiles with the stable counting sort
// above (k_tile_count / k_col_scan / k_tile_ranges / k_tile_scatter over super-tile rects: ~K/10
// keys at C3).  Level 2 splits every super-tile's rank list into segments of `seglen` ranks; one
// warp per segment walks 32 ranks at a time and, for each of the kSup^2 tiles of its super-tile,
// takes a ballot of the lanes whose rect covers the tile: popc(ballot) counts (pass 1), and
// popc(ballot & lanes-below) is a lane's stable slot inside the tile's run (pass 2), so every
// tile list comes out in rank = (depth_bits, gid) order with one coalesced run of writes per
// (32 ranks, tile).

#ifndef PUV_SEG_MIN
#define PUV_SEG_MIN 512
#endif
constexpr int kSegMin = PUV_SEG_MIN;       // ranks per level-2 segment (at least)
constexpr int kSegTarget = 32768;          // seglen >= K1 / kSegTarget, so segments <= kSegTarget + nst

__host__ __device__ inline size_t max_segments(int ntiles) { return (size_t)kSegTarget + (size_t)ntiles; }

struct L2Info { uint32_t seglen, nseg, pad0, pad1; };

// Per rank: the tile rect + gid (for level 2) and the super-tile rect (level 1); K = sum of tiles.
__global__ void __launch_bounds__(256) k_bin_prep(const ViewHdr* hdr, const uint32_t* __restrict__ sorted,
                                                  const uint2* __restrict__ rect, uint4* __restrict__ rk,
                                                  uint2* __restrict__ srect, unsigned long long* __restrict__ ktotal) {
  __shared__ unsigned long long part[8];
  const uint32_t n = hdr->n_vis;
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t t = 0;
  if (r < n) {
    const uint32_t gid = sorted[r];
    const uint2 rc = rect[gid];
    rk[r] = make_uint4(rc.x, rc.y, gid, 0u);
    const uint32_t x0 = rc.x & 0xffffu, x1 = rc.x >> 16, y0 = rc.y & 0xffffu, y1 = rc.y >> 16;
    t = (x1 - x0) * (y1 - y0);
    const uint32_t sx0 = x0 / kSup, sx1 = (x1 + kSup - 1) / kSup, sy0 = y0 / kSup, sy1 = (y1 + kSup - 1) / kSup;
    srect[r] = make_uint2(sx0 | (sx1 << 16), sy0 | (sy1 << 16));
  }
  unsigned long long w = __reduce_add_sync(0xffffffffu, t);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (int k = 0; k < 8; ++k) b += part[k];
    if (b) atomicAdd(ktotal, b);
  }
}

// Carve this view's final lists (K keys) and its level-1 rank lists (K1) from the arena.
__global__ void k_view_finalize2(ViewHdr* hdr, CallHdr* call, const unsigned long long* ktotal,
                                 const uint64_t* k1total, ViewHdr* l1) {
  const uint64_t K = *ktotal, K1 = *k1total, need = K + K1;
  hdr->K = K;
  atomicAdd((unsigned long long*)&call->arena_need, (unsigned long long)need);
  const uint64_t base = K < 0xffffffffull ? atomicAdd((unsigned long long*)&call->arena_used, (unsigned long long)need)
                                          : ~0ull;
  const bool fits = base != ~0ull && base + need <= call->arena_cap;
  l1->n_vis = hdr->n_vis;
  l1->K = K1;
  if (fits) {
    hdr->list_base = base;
    hdr->overflow = 0;
    l1->list_base = base + K;
    l1->overflow = 0;
    uint64_t kb = (K1 + kNbMax - 1) / kNbMax;
    if (kb < 2048) kb = 2048;
    l1->kb = (uint32_t)kb;
    l1->nb = (uint32_t)((K1 + kb - 1) / kb);
  } else {
    hdr->list_base = 0;
    hdr->overflow = 1;
    call->overflow_any = 1;
    l1->list_base = 0;
    l1->overflow = 1;
    l1->kb = 2048;
    l1->nb = 0;
  }
}

// Level-2 segment plan (one block): seglen, segments per super-tile (prefix in segbase), seg -> st.
__global__ void __launch_bounds__(1024) k_seg_plan(const ViewHdr* l1, const uint32_t* __restrict__ sst,
                                                   const uint32_t* __restrict__ sen, int nst,
                                                   uint32_t* __restrict__ segbase, uint32_t* __restrict__ segst,
                                                   L2Info* info) {
  __shared__ uint32_t part[1024];
  __shared__ uint32_t s_len;
  if (threadIdx.x == 0) {
    const uint64_t K1 = l1->overflow ? 0 : l1->K;
    uint64_t len = (K1 + kSegTarget - 1) / kSegTarget;
    if (len < kSegMin) len = kSegMin;
    s_len = (uint32_t)len;
  }
  __syncthreads();
  const uint32_t seglen = s_len;
  const bool ov = l1->overflow != 0;
  const int per = (nst + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(nst, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += ov ? 0u : (sen[i] - sst[i] + seglen - 1) / seglen;
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
    const uint32_t c = ov ? 0u : (sen[i] - sst[i] + seglen - 1) / seglen;
    segbase[i] = run;
    for (uint32_t k = 0; k < c; ++k) segst[run + k] = (uint32_t)i;
    run += c;
  }
  if (threadIdx.x == 1023) {
    segbase[nst] = part[1023];
    info->seglen = seglen;
    info->nseg = part[1023];
  }
}

// 16-bit mask of the tiles of super-tile (sx, sy) covered by tile rect q (bit = ly * kSup + lx).
__device__ __forceinline__ uint32_t cover_mask(const uint4& q, uint32_t sx, uint32_t sy) {
  const uint32_t x0 = q.x & 0xffffu, x1 = q.x >> 16, y0 = q.y & 0xffffu, y1 = q.y >> 16;
  const uint32_t bx = sx * kSup, by = sy * kSup;
  const uint32_t lx0 = x0 > bx ? x0 - bx : 0u, lx1 = min(x1 - bx, (uint32_t)kSup);
  const uint32_t ly0 = y0 > by ? y0 - by : 0u, ly1 = min(y1 - by, (uint32_t)kSup);
  const uint32_t row = ((1u << lx1) - 1u) & ~((1u << lx0) - 1u);
  const uint32_t rows = ((1u << ly1) - 1u) & ~((1u << ly0) - 1u);   // bit per local row
  uint32_t m = 0;
#pragma unroll
  for (int ly = 0; ly < kSup; ++ly) m |= ((rows >> ly) & 1u) ? row << (kSup * ly) : 0u;
  return m;
}

// Walk segment `seg` 32 ranks at a time; PASS 1 counts per tile, PASS 2 places.
template <int PASS>
__global__ void __launch_bounds__(256) k_seg_walk(const ViewHdr* hdr, const ViewHdr* l1, const L2Info* info,
                                                  const uint32_t* __restrict__ segbase,
                                                  const uint32_t* __restrict__ segst,
                                                  const uint32_t* __restrict__ sst, const uint32_t* __restrict__ sen,
                                                  const uint32_t* __restrict__ arena, const uint4* __restrict__ rk,
                                                  int sgx, int gx, int gy, uint32_t* __restrict__ cnt2,
                                                  const uint32_t* __restrict__ tstart, uint32_t* __restrict__ out) {
  if (l1->overflow) return;
  const uint32_t nseg = info->nseg, seglen = info->seglen;
  const int lane = threadIdx.x & 31;
  const uint32_t* list1 = arena + l1->list_base;
  PUV_CHECK(nseg <= max_segments(gx * gy));
  uint32_t* list = out + hdr->list_base;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; seg < nseg; seg += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t st = segst[seg];
    const uint32_t sx = st % sgx, sy = st / sgx;
    const uint32_t i0 = sst[st] + (seg - segbase[st]) * seglen;
    const uint32_t i1 = min(sen[st], i0 + seglen);
    uint32_t base[kSupT];
#pragma unroll
    for (int b = 0; b < kSupT; ++b) {
      base[b] = 0;
      if (PASS == 2) {
        const uint32_t tx = sx * kSup + (b % kSup), ty = sy * kSup + (b / kSup);
        if (tx < (uint32_t)gx && ty < (uint32_t)gy) base[b] = tstart[ty * gx + tx] + cnt2[(size_t)seg * kSupT + b];
      }
    }
    // software pipeline: the next batch's rank and rect are loaded before this batch is placed
    uint32_t i = i0 + lane;
    uint4 q = make_uint4(0, 0, 0, 0);
    if (i < i1) q = rk[list1[i]];
    for (uint32_t b0 = i0; b0 < i1; b0 += 32) {
      const bool valid = b0 + lane < i1;
      const uint4 cur = q;
      const uint32_t inx = b0 + 32 + lane;
      if (inx < i1) q = rk[list1[inx]];
      const uint32_t m = valid ? cover_mask(cur, sx, sy) : 0u;
#pragma unroll
      for (int b = 0; b < kSupT; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (m >> b) & 1u);
        if (PASS == 2 && ((m >> b) & 1u)) {
          PUV_CHECK(base[b] + __popc(bal & lt) < hdr->K);
          list[base[b] + __popc(bal & lt)] = cur.z;
        }
        base[b] += __popc(bal);
      }
    }
    if (PASS == 1 && lane < kSupT) {
      uint32_t c = 0;
#pragma unroll
      for (int b = 0; b < kSupT; ++b) c = lane == b ? base[b] : c;
      cnt2[(size_t)seg * kSupT + lane] = c;
    }
  }
}

// Per tile: exclusive offsets of its super-tile's segments (in place in cnt2) and the tile total.
// One warp per super-tile, lane b < kSupT walks column b of the super-tile's segment rows (16
// consecutive words per row: coalesced, and the loads run ahead of the running sum).
__global__ void __launch_bounds__(256) k_seg_offsets(const ViewHdr* l1, const uint32_t* __restrict__ segbase,
                                                     int sgx, int nst, int gx, int gy, uint32_t* __restrict__ cnt2,
                                                     uint32_t* __restrict__ total) {
  const int st = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, b = threadIdx.x & 31;
  if (st >= nst || b >= kSupT) return;
  const int tx = (st % sgx) * kSup + b % kSup, ty = (st / sgx) * kSup + b / kSup;
  uint32_t run = 0;
  if (!l1->overflow) {
    const uint32_t s0 = segbase[st], s1 = segbase[st + 1];
    uint32_t* c = cnt2 + (size_t)s0 * kSupT + b;
#pragma unroll 8
    for (uint32_t k = 0; k < s1 - s0; ++k) {
      const uint32_t x = c[(size_t)k * kSupT];
      c[(size_t)k * kSupT] = run;
      run += x;
    }
  }
  if (tx < gx && ty < gy) total[ty * gx + tx] = run;
}

size_t bin_scratch_bytes(size_t N, int ntiles) {
  const size_t ms = max_segments(ntiles);
  return align_up(16 * N) + align_up(8 * N) + align_up(sizeof(ViewHdr)) + align_up(16) + align_up(sizeof(L2Info)) +
         3 * align_up(4 * ((size_t)ntiles + 1)) + align_up(4 * ms) + align_up(4 * ms * kSupT);
}

// Level-2 scratch carved from a binning scratch block (at p.bin2).
struct Bin2 {
  uint4* rk;
  uint2* srect;
  unsigned long long* ktot;
  L2Info* info;
  uint32_t *segbase, *segst, *cnt2;
};

static Bin2 bin2_of(const Plan& p, void* state) {
  char* b2 = (char*)state + p.bin2;
  size_t o = 0;
  auto take = [&](size_t bytes) { char* q = b2 + o; o += align_up(bytes); return q; };
  Bin2 b;
  b.rk = (uint4*)take(16 * (size_t)p.N);
  b.srect = (uint2*)take(8 * (size_t)p.N);
  b.ktot = (unsigned long long*)take(16);
  b.info = (L2Info*)take(sizeof(L2Info));
  b.segbase = (uint32_t*)take(4 * ((size_t)p.ntiles + 1));
  b.segst = (uint32_t*)take(4 * max_segments(p.ntiles));
  b.cnt2 = (uint32_t*)take(4 * max_segments(p.ntiles) * kSupT);
  return b;
}

// Level 2 (per-tile lists from the super-tile rank lists): on the render path when !kDirect, else on
// demand for the debug / parity view of one view (the level-1 lists, super-tile ranges and header
// persist per view; rk is rebuilt here since a later view may have reused the scratch block).
static void level2(const Plan& p, const Views& v, const Bin2& b, uint32_t* arena, int view, cudaStream_t s) {
  ViewHdr* hdr = v.hdr + view;
  const ViewHdr* l1 = v.l1 + view;
  const uint32_t* sst = v.sst + (size_t)view * (p.nst + 1);
  const uint32_t* sen = v.sen + (size_t)view * (p.nst + 1);
  uint32_t* tstart = v.tstart + (size_t)view * p.ntiles;
  uint32_t* tend = v.tend + (size_t)view * p.ntiles;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  k_seg_plan<<<1, 1024, 0, s>>>(l1, sst, sen, p.nst, b.segbase, b.segst, b.info);
#ifndef PUV_WALK_CTAS_PER_SM
#define PUV_WALK_CTAS_PER_SM 8
#endif
  const int wblocks = PUV_WALK_CTAS_PER_SM * nsm;   // 8 warps per block, grid-stride over segments
  k_seg_walk<1><<<wblocks, 256, 0, s>>>(hdr, l1, b.info, b.segbase, b.segst, sst, sen, arena, b.rk, p.sgx, p.gx,
                                        p.gy, b.cnt2, nullptr, nullptr);
  k_seg_offsets<<<(p.nst + 7) / 8, 256, 0, s>>>(l1, b.segbase, p.sgx, p.nst, p.gx, p.gy, b.cnt2, tend /* totals */);
  k_tile_ranges<<<1, 1024, 0, s>>>(tend, p.ntiles, tstart, tend);
  k_seg_walk<2><<<wblocks, 256, 0, s>>>(hdr, l1, b.info, b.segbase, b.segst, sst, sen, arena, b.rk, p.sgx, p.gx,
                                        p.gy, b.cnt2, tstart, arena);
  count_launches(5);
}

void launch_bin(const Plan& p, const Views& v, void* state, uint32_t* arena, int view, cudaStream_t s, bool with_level2) {
  char* st = (char*)state;
  const uint32_t* sorted = v.sorted + (size_t)view * p.N;
  const uint2* rect = v.rect + (size_t)view * p.N;
  ViewHdr* hdr = v.hdr + view;
  uint32_t* bsum = (uint32_t*)(st + p.bsum);
  uint32_t* koff1 = (uint32_t*)(st + p.koff);
  uint32_t* cnt = (uint32_t*)(st + p.cnt);
  uint32_t* bstart = (uint32_t*)(st + p.bstart);
  const Bin2 b = bin2_of(p, state);
  ViewHdr* l1 = v.l1 + view;
  uint32_t* sst = v.sst + (size_t)view * (p.nst + 1);
  uint32_t* sen = v.sen + (size_t)view * (p.nst + 1);
  const int sgx = p.sgx, sgy = (p.gy + kSup - 1) / kSup, nst = p.nst;
  uint64_t* k1tot = &l1->ktotal;

  cudaMemsetAsync(b.ktot, 0, 16, s);
  k_bin_prep<<<(p.N + 255) / 256, 256, 0, s>>>(hdr, sorted, rect, b.rk, b.srect, b.ktot);
  // level-1 key offsets per rank (super-tile keys), K1
  const int nsb = p.N / kScanTile + 1;   // one extra block so koff1[n_vis] (= K1) is always written
  k_koff_reduce<<<nsb, kScanThreads, 0, s>>>(nullptr, b.srect, hdr, bsum);
  k_scan_bsum<<<1, 1024, 0, s>>>(bsum, nsb, k1tot);
  k_koff_write<<<nsb, kScanThreads, 0, s>>>(nullptr, b.srect, hdr, bsum, koff1);
  k_view_finalize2<<<1, 1, 0, s>>>(hdr, v.call, b.ktot, k1tot, l1);
  k_block_starts<<<(kNbMax + 255) / 256, 256, 0, s>>>(l1, koff1, bstart);

  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // level 1: stable counting sort of super-tile keys (ranks) by super-tile
  const int band_rows = sgx >= kBandTiles ? 1 : (kBandTiles / sgx < sgy ? kBandTiles / sgx : sgy);
  const int nbands = (sgy + band_rows - 1) / band_rows;
  k_tile_count<<<PUV_BIN_CTAS_PER_SM * nsm, kBinThreads, 0, s>>>(l1, koff1, nullptr, b.srect, bstart, sgx, sgy,
                                                                 band_rows, nbands, nst, cnt);
  k_col_scan<<<(nst + 31) / 32, 1024, 0, s>>>(l1, cnt, nst, sen /* totals */);
  k_tile_ranges<<<1, 1024, 0, s>>>(sen, nst, sst, sen);
  k_tile_scatter<<<PUV_BIN_CTAS_PER_SM * nsm, kBinThreads, 0, s>>>(l1, koff1, nullptr, b.srect, bstart, sgx, sgy,
                                                                   band_rows, nbands, nst, cnt, sst, arena + 0);
  count_launches(11);
  if (with_level2) level2(p, v, b, arena, view, s);
}

void launch_bin_level2(const Plan& p, const Views& v, void* state, uint32_t* arena, int view, cudaStream_t s) {
  const Bin2 b = bin2_of(p, state);
  // rk (rect + gid per rank) of this view, again
  cudaMemsetAsync(b.ktot, 0, 16, s);
  k_bin_prep<<<(p.N + 255) / 256, 256, 0, s>>>(v.hdr + view, v.sorted + (size_t)view * p.N,
                                               v.rect + (size_t)view * p.N, b.rk, b.srect, b.ktot);
  count_launches(1);
  level2(p, v, b, arena, view, s);
}

}  // namespace puv
