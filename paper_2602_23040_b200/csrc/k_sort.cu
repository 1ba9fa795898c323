// K3 — stable LSD radix sort of the visible Gaussians of one view by depth key
// (the low "digit" of the (tile, depth) key, row a4), with the culling
// compaction folded into the first pass.
//
// Four 8-bit passes over the 32-bit depth bits.  Each pass: upsweep (per-block
// digit histogram) -> one-block exclusive scan of the digit-major histogram
// -> downsweep (stable block-local rank by warp match_any + per-warp digit
// counters, then scatter).  Input of pass 0 is gid order, so ties in depth
// keep ascending gid (R8) without carrying the gid in the key.
#include "internal.cuh"

namespace puv {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 8;                              // per thread
constexpr int kSortTile = kSortThreads * kSortItems;       // 2048 items per block

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// digit of an item, 256 = "no item" (outside n, or culled in pass 0)
template <bool FIRST>
__device__ __forceinline__ uint32_t item_digit(const uint32_t* keys, uint32_t idx, uint32_t n, int shift,
                                               uint32_t& key) {
  if (idx >= n) return 256u;
  key = keys[idx];
  if (FIRST && key == kInvisible) return 256u;
  return (key >> shift) & 0xffu;
}

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads) k_radix_upsweep(const uint32_t* __restrict__ keys,
                                                                 const uint32_t* n_ptr, uint32_t n_fixed, int shift,
                                                                 uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[256];
  const uint32_t n = FIRST ? n_fixed : *n_ptr;
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * kSortTile;
  if (base < n) {
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      uint32_t key;
      const uint32_t d = item_digit<FIRST>(keys, base + i * kSortThreads + threadIdx.x, n, shift, key);
      if (d < 256u) atomicAdd(&h[d], 1u);
    }
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of `m` u32 in one block of 1024 threads.  If total_out, writes the total.
__global__ void __launch_bounds__(1024) k_scan_one_block(uint32_t* data, int m, uint32_t* total_out) {
  __shared__ uint32_t part[1024];
  const int per = (m + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(m, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += data[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t t = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;  // exclusive
  for (int i = lo; i < hi; ++i) {
    const uint32_t x = data[i];
    data[i] = run;
    run += x;
  }
  if (total_out && threadIdx.x == 1023) *total_out = part[1023];
}

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads) k_radix_downsweep(const uint32_t* __restrict__ keys_in,
                                                                   const uint32_t* __restrict__ vals_in,
                                                                   uint32_t* __restrict__ keys_out,
                                                                   uint32_t* __restrict__ vals_out,
                                                                   const uint32_t* n_ptr, uint32_t n_fixed, int shift,
                                                                   const uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t wh[kSortWarps][256];
  __shared__ uint32_t goff[256];
  const uint32_t n = FIRST ? n_fixed : *n_ptr;
  const uint32_t base = blockIdx.x * kSortTile;
  if (base >= n) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&wh[0][0])[i] = 0;
  goff[threadIdx.x] = hist[(size_t)threadIdx.x * nblocks + blockIdx.x];
  __syncthreads();
  uint32_t key[kSortItems], dig[kSortItems], loc[kSortItems], val[kSortItems];
  const uint32_t wbase = base + warp * (32 * kSortItems);
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const uint32_t idx = wbase + r * 32 + lane;
    key[r] = 0;
    dig[r] = item_digit<FIRST>(keys_in, idx, n, shift, key[r]);
    val[r] = (dig[r] < 256u) ? (FIRST ? idx : vals_in[idx]) : 0u;
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[r]);
    const uint32_t rank = __popc(peers & lanemask_lt());
    const uint32_t cur = dig[r] < 256u ? wh[warp][dig[r]] : 0u;
    __syncwarp();
    if (dig[r] < 256u && rank == 0) wh[warp][dig[r]] = cur + __popc(peers);
    __syncwarp();
    loc[r] = cur + rank;
  }
  __syncthreads();
  {  // per digit: exclusive prefix over warps
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t t = wh[w][threadIdx.x];
      wh[w][threadIdx.x] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    if (dig[r] < 256u) {
      const uint32_t pos = goff[dig[r]] + wh[warp][dig[r]] + loc[r];
      keys_out[pos] = key[r];
      vals_out[pos] = val[r];
    }
  }
}

void launch_depth_sort(const Plan& p, const Views& v, void* state, int view, cudaStream_t s) {
  char* st = (char*)state;
  uint32_t* sk0 = (uint32_t*)(st + p.sk0);
  uint32_t* sv0 = (uint32_t*)(st + p.sv0);
  uint32_t* sk1 = (uint32_t*)(st + p.sk1);
  uint32_t* sv1 = (uint32_t*)(st + p.sv1);
  uint32_t* hist = (uint32_t*)(st + p.hist);
  const int nb = (int)p.sort_blocks;
  const uint32_t* depth = v.depth + (size_t)view * p.N;
  uint32_t* nvis = &v.hdr[view].n_vis;
  uint32_t* sorted = v.sorted + (size_t)view * p.N;
  const int m = 256 * nb;
  // pass 0: depth[] (gid order) -> (sk0, sv0), dropping culled Gaussians; writes n_vis
  k_radix_upsweep<true><<<nb, kSortThreads, 0, s>>>(depth, nullptr, (uint32_t)p.N, 0, hist, nb);
  k_scan_one_block<<<1, 1024, 0, s>>>(hist, m, nvis);
  k_radix_downsweep<true><<<nb, kSortThreads, 0, s>>>(depth, nullptr, sk0, sv0, nullptr, (uint32_t)p.N, 0, hist, nb);
  const uint32_t* ki[3] = {sk0, sk1, sk0};
  const uint32_t* vi[3] = {sv0, sv1, sv0};
  uint32_t* ko[3] = {sk1, sk0, sk1};
  uint32_t* vo[3] = {sv1, sv0, sorted};
  for (int pass = 1; pass < 4; ++pass) {
    const int sh = 8 * pass;
    k_radix_upsweep<false><<<nb, kSortThreads, 0, s>>>(ki[pass - 1], nvis, 0, sh, hist, nb);
    k_scan_one_block<<<1, 1024, 0, s>>>(hist, m, nullptr);
    k_radix_downsweep<false><<<nb, kSortThreads, 0, s>>>(ki[pass - 1], vi[pass - 1], ko[pass - 1], vo[pass - 1], nvis,
                                                          0, sh, hist, nb);
  }
  count_launches(12);
}

}  // namespace puv
