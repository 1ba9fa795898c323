// K3 — onesweep LSD radix sort of the visible Gaussians of one view by depth key
// (the low "digit" of the (tile, depth) key, row a4), with the culling
// compaction folded into the first pass.
//
//   k_os_hist   one read of every depth key: the four 8-bit digit histograms of
//               the visible keys (smem histograms, one global atomic per bin and CTA)
//   k_os_scan   exclusive scan of each histogram -> global digit offsets; n_vis
//   k_os_pass   x4: each CTA takes a 4096-item tile by atomic ticket, ranks its
//               items stably per digit (warp match_any + per-warp counters),
//               publishes its per-digit count, resolves its exclusive prefix by
//               decoupled look-back over the preceding tiles' status words, and
//               scatters.  One read and one write of (key, value) per pass.
// Pass 0 reads the depth keys in gid order and drops culled texels, so ties in
// depth keep ascending gid (R8) without carrying the gid in the key.
#include "internal.cuh"

namespace puv {

constexpr int kOsThreads = 256;
constexpr int kOsWarps = kOsThreads / 32;
#ifndef PUV_OS_ITEMS
#define PUV_OS_ITEMS 16
#endif
constexpr int kOsItems = PUV_OS_ITEMS;               // per thread
constexpr int kOsTile = kOsThreads * kOsItems;       // 4096 items per CTA
constexpr uint32_t kFlagAgg = 1u << 30, kFlagPre = 2u << 30, kCountMask = (1u << 30) - 1u;
#ifndef PUV_OS_WINDOW
#define PUV_OS_WINDOW 8
#endif
constexpr int kOsWindow = PUV_OS_WINDOW;   // predecessor status words read per look-back round (1 = serial walk)
#ifndef PUV_OS_STAGE
#define PUV_OS_STAGE 1
#endif
// 1: the scatter goes through shared memory in tile-local digit order, so consecutive threads write
// consecutive addresses of a digit's run (coalesced) instead of each item straight to its slot
constexpr bool kOsStage = PUV_OS_STAGE != 0;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kOsThreads) k_os_hist(const uint32_t* __restrict__ keys, uint32_t n,
                                                       uint32_t* __restrict__ ghist, size_t vstride) {
  // grid.y: the views of a sort group (keys of view y at keys + y n, its scratch at + y vstride)
  keys += (size_t)blockIdx.y * n;
  ghist += (size_t)blockIdx.y * vstride;
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += kOsThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * kOsThreads * 4;
  for (uint32_t i = (blockIdx.x * kOsThreads + threadIdx.x) * 4; i < n; i += stride) {
    uint32_t k4[4];
    if (i + 3 < n && (((uintptr_t)(keys + i)) & 15) == 0) {
      const uint4 q = *reinterpret_cast<const uint4*>(keys + i);
      k4[0] = q.x; k4[1] = q.y; k4[2] = q.z; k4[3] = q.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) k4[j] = i + j < n ? keys[i + j] : kInvisible;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t k = k4[j];
      if (k == kInvisible) continue;
      atomicAdd(&h[0][k & 0xffu], 1u);
      atomicAdd(&h[1][(k >> 8) & 0xffu], 1u);
      atomicAdd(&h[2][(k >> 16) & 0xffu], 1u);
      atomicAdd(&h[3][k >> 24], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 256; i += kOsThreads) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(ghist + i, c);
  }
}

// ghist[4][256] counts -> exclusive offsets in place; n_vis; reset the pass tickets.
__global__ void __launch_bounds__(256) k_os_scan(uint32_t* ghist, uint32_t* tickets, uint32_t* n_vis,
                                                 size_t vstride, size_t nvstride) {
  // block x: view x of the sort group
  ghist += (size_t)blockIdx.x * vstride;
  tickets += (size_t)blockIdx.x * vstride;
  n_vis += (size_t)blockIdx.x * nvstride;
  __shared__ uint32_t s[256];
  for (int p = 0; p < 4; ++p) {
    const uint32_t c = ghist[p * 256 + threadIdx.x];
    s[threadIdx.x] = c;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
      const uint32_t t = threadIdx.x >= off ? s[threadIdx.x - off] : 0u;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    ghist[p * 256 + threadIdx.x] = s[threadIdx.x] - c;
    if (p == 0 && threadIdx.x == 255) *n_vis = s[255];
    __syncthreads();
  }
  if (threadIdx.x < 4) tickets[threadIdx.x] = 0;
}

template <bool FIRST>
__global__ void __launch_bounds__(kOsThreads) k_os_pass(const uint32_t* __restrict__ keys_in,
                                                       const uint32_t* __restrict__ vals_in,
                                                       uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                       const uint32_t* n_ptr, uint32_t n_fixed, int shift,
                                                       const uint32_t* __restrict__ goff, uint32_t* status,
                                                       uint32_t* ticket, int write_keys, uint32_t kvstride,
                                                       size_t vstride, size_t nvstride) {
  __shared__ uint32_t wh[kOsWarps][256];
  __shared__ uint32_t excl[256];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t tstart[kOsStage ? 256 : 1], wsum[kOsWarps];
  __shared__ uint32_t skey[kOsStage ? kOsTile : 1], sval[kOsStage ? kOsTile : 1];
  {  // grid.y: view y of the sort group -- its keys / values (stride kvstride), its histogram
     // offsets, look-back status words and ticket (stride vstride), its visible count (nvstride)
    const size_t y = blockIdx.y;
    keys_in += y * kvstride;
    if (!FIRST) vals_in += y * kvstride;
    keys_out += y * kvstride;
    vals_out += y * kvstride;
    goff += y * vstride;
    status += y * vstride;
    ticket += y * vstride;
    if (!FIRST) n_ptr += y * nvstride;
  }
  const uint32_t n = FIRST ? n_fixed : *n_ptr;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = threadIdx.x; i < kOsWarps * 256; i += kOsThreads) (&wh[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kOsTile;
  if (base >= n) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t key[kOsItems], dig[kOsItems], loc[kOsItems], val[kOsItems];
  const uint32_t wbase = base + warp * (32 * kOsItems);
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const uint32_t idx = wbase + r * 32 + lane;
    key[r] = kInvisible;
    dig[r] = 256u;
    val[r] = 0u;
    if (idx < n) {
      key[r] = keys_in[idx];
      if (!FIRST || key[r] != kInvisible) {
        dig[r] = (key[r] >> shift) & 0xffu;
        val[r] = FIRST ? idx : vals_in[idx];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[r]);
    const uint32_t rank = __popc(peers & lanemask_lt());
    const uint32_t cur = dig[r] < 256u ? wh[warp][dig[r]] : 0u;
    __syncwarp();
    if (dig[r] < 256u && rank == 0) wh[warp][dig[r]] = cur + __popc(peers);
    __syncwarp();
    loc[r] = cur + rank;
  }
  __syncthreads();
  // per digit (thread d): exclusive prefix over warps, publish, decoupled look-back
  {
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kOsWarps; ++w) {
      const uint32_t t = wh[w][d];
      wh[w][d] = run;
      run += t;
    }
    uint32_t* st = status + (size_t)tile * 256 + d;
    if (tile == 0) {
      st_release(st, kFlagPre | run);
      excl[d] = 0;
    } else {
      st_release(st, kFlagAgg | run);
      // decoupled look-back, kOsWindow predecessors per round (independent loads in flight): sum
      // aggregates from the nearest tile back until an inclusive prefix; an unpublished tile
      // restarts the round at that tile (spin)
      uint32_t acc = 0;
      for (int64_t t = (int64_t)tile - 1; t >= 0;) {
        uint32_t sw[kOsWindow];
#pragma unroll
        for (int w = 0; w < kOsWindow; ++w)
          sw[w] = t - w >= 0 ? ld_volatile(status + (size_t)(t - w) * 256 + d) : kFlagPre;
        bool found = false;
        int w = 0;
        for (; w < kOsWindow; ++w) {
          const uint32_t flag = sw[w] & ~kCountMask;
          if (flag == 0u) break;               // not published yet: re-read from tile t - w
          acc += sw[w] & kCountMask;
          if (flag == kFlagPre) { found = true; break; }
        }
        if (found) break;
        t -= w;
      }
      st_release(st, kFlagPre | (acc + run));
      excl[d] = acc;
    }
    if (kOsStage) {
      // tile-local start of digit d's run: exclusive scan of the tile's digit counts
      uint32_t x = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      tstart[d] = x - run;   // warp-local exclusive; the warp offsets are added below
    }
  }
  __syncthreads();
  if (kOsStage) {
    uint32_t wo = 0;
    for (int w = 0; w < warp; ++w) wo += wsum[w];
    tstart[threadIdx.x] += wo;
    uint32_t cnt = 0;
    for (int w = 0; w < kOsWarps; ++w) cnt += wsum[w];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
      if (dig[r] < 256u) {
        const uint32_t li = tstart[dig[r]] + wh[warp][dig[r]] + loc[r];
        skey[li] = key[r];
        sval[li] = val[r];
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += kOsThreads) {
      const uint32_t k = skey[i];
      const uint32_t dd = (k >> shift) & 0xffu;
      const uint32_t pos = goff[dd] + excl[dd] + (i - tstart[dd]);
      if (write_keys) keys_out[pos] = k;
      vals_out[pos] = sval[i];
    }
  } else {
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
      if (dig[r] < 256u) {
        const uint32_t pos = goff[dig[r]] + excl[dig[r]] + wh[warp][dig[r]] + loc[r];
        if (write_keys) keys_out[pos] = key[r];
        vals_out[pos] = val[r];
      }
    }
  }
}

size_t depth_sort_scratch_bytes(size_t N) {
  const size_t tiles = (N + kOsTile - 1) / kOsTile;
  return 4 * (4 * 256 * tiles + 4 * 256 + 8);
}

void launch_depth_sort(const Plan& p, const Views& v, void* state, int view, int nv, cudaStream_t s) {
  // views [view, view + nv) in one set of launches (grid.y = view of the group, nv <= kSortGroup):
  // the per-view sorts are independent (own histograms, tickets, look-back chains), batched only
  // for parallelism -- one view's ~836k visible keys fill ~1.4 onesweep CTAs per SM
  char* st = (char*)state;
  const size_t N = p.N;
  uint32_t* sk0 = (uint32_t*)(st + p.sk0);   // [kSortGroup][N] each
  uint32_t* sv0 = (uint32_t*)(st + p.sv0);
  uint32_t* sk1 = (uint32_t*)(st + p.sk1);
  uint32_t* sv1 = (uint32_t*)(st + p.sv1);
  const size_t tiles = (N + kOsTile - 1) / kOsTile;
  // per view: status [4][tiles][256], ghist [4][256], tickets [4] (+ pad): depth_sort_scratch_bytes
  const size_t vstride = depth_sort_scratch_bytes(N) / 4;
  uint32_t* status = (uint32_t*)(st + p.hist);
  uint32_t* ghist = status + 4 * 256 * tiles;
  uint32_t* tickets = ghist + 4 * 256;
  const uint32_t* depth = v.depth + (size_t)view * N;
  uint32_t* nvis = &v.hdr[view].n_vis;
  const size_t nvstride = sizeof(ViewHdr) / sizeof(uint32_t);
  static_assert(sizeof(ViewHdr) % sizeof(uint32_t) == 0, "ViewHdr stride in words");
  uint32_t* sorted = v.sorted + (size_t)view * N;
  cudaMemsetAsync(status, 0, 4 * vstride * nv, s);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t hwant = (N + 4 * kOsThreads - 1) / (4 * kOsThreads);
  const size_t hcap = (size_t)4 * nsm / nv > 0 ? (size_t)4 * nsm / nv : 1;
  const int hb = (int)(hwant < hcap ? (hwant > 0 ? hwant : 1) : hcap);
  k_os_hist<<<dim3(hb, nv), kOsThreads, 0, s>>>(depth, (uint32_t)N, ghist, vstride);
  k_os_scan<<<nv, 256, 0, s>>>(ghist, tickets, nvis, vstride, nvstride);
  const uint32_t* ki[4] = {depth, sk0, sk1, sk0};
  const uint32_t* vi[4] = {nullptr, sv0, sv1, sv0};
  uint32_t* ko[4] = {sk0, sk1, sk0, sk1};
  uint32_t* vo[4] = {sv0, sv1, sv0, sorted};
  const dim3 grid((unsigned)tiles, nv);
  k_os_pass<true><<<grid, kOsThreads, 0, s>>>(ki[0], vi[0], ko[0], vo[0], nullptr, (uint32_t)N, 0, ghist, status,
                                              tickets, 1, (uint32_t)N, vstride, nvstride);
  for (int pass = 1; pass < 4; ++pass)   // the last pass writes only the depth order (its keys are not read)
    k_os_pass<false><<<grid, kOsThreads, 0, s>>>(ki[pass], vi[pass], ko[pass], vo[pass], nvis, 0, 8 * pass,
                                                 ghist + 256 * pass, status + (size_t)pass * 256 * tiles,
                                                 tickets + pass, pass < 3 ? 1 : 0, (uint32_t)N, vstride, nvstride);
  count_launches(6);
}

}  // namespace puv
