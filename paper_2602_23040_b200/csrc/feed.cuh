// feed.cuh — the tile's entry stream of K5/K6 straight from the level-1 super-tile rank list
// (internal.cuh kDirect).
//
// The level-1 pass leaves, per super-tile of 4 x 4 tiles, the ranks of every visible Gaussian whose
// rect touches it, in rank = (depth_bits, gid) order.  A tile's list (R8) is the subsequence whose
// rect contains the tile -- exactly what level 2 would have written, in the same order.  The block
// walks its super-tile's ranks NT at a time (gid = depth order[rank], rect[gid], 4 compares), keeps
// the passing gids in order with a block-wide stable compaction (warp ballots + warp offsets), and
// hands out batches of NB of them; a round's overflow past NB stays queued for the next batch.
#pragma once
#include "internal.cuh"

namespace puv {

template <int NT, int NB>
struct TileFeed {
  static_assert(NT <= NB, "one round adds at most NT entries, so the queue never exceeds 2 NB");
  uint32_t* q;          // smem, 2 NB: queued gids (passing, in list order)
  uint32_t* cnt;        // smem, NT / 32 + 1: per-warp pass counts; cnt[NT / 32] = queue length
  uint32_t c, cend;     // next candidate / end in the super-tile's rank range (block-uniform)

  __device__ __forceinline__ void init(uint32_t* q_, uint32_t* cnt_, uint32_t c0, uint32_t c1) {
    q = q_;
    cnt = cnt_;
    c = c0;
    cend = c1;
    if (threadIdx.x == 0) cnt[NT / 32] = 0;
  }

  // Fill the queue to >= NB entries (or to the end of the candidates); returns the batch size
  // min(queued, NB), block-uniform; q[0, n) are the batch's gids.  Contains barriers: call with the
  // whole block.
  __device__ __forceinline__ int next(const uint32_t* __restrict__ list1, const uint32_t* __restrict__ sorted,
                                      const uint2* __restrict__ rect, uint32_t tx, uint32_t ty) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    uint32_t queued = cnt[NT / 32];
    while (queued < (uint32_t)NB && c < cend) {
      const uint32_t i = c + threadIdx.x;
      bool pass = false;
      uint32_t gid = 0;
      if (i < cend) {
        gid = sorted[list1[i]];
        const uint2 rc = rect[gid];
        pass = tx >= (rc.x & 0xffffu) && tx < (rc.x >> 16) && ty >= (rc.y & 0xffffu) && ty < (rc.y >> 16);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, pass);
      if (lane == 0) cnt[warp] = __popc(bal);
      __syncthreads();
      uint32_t before = queued, total = 0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) {
        const uint32_t x = cnt[w];
        before += w < warp ? x : 0u;
        total += x;
      }
      if (pass) q[before + __popc(bal & ((1u << lane) - 1u))] = gid;
      queued += total;
      c += NT;
      __syncthreads();
    }
    if (threadIdx.x == 0) cnt[NT / 32] = queued;
    return (int)min(queued, (uint32_t)NB);
  }

  // After the batch of n entries is consumed: move the queued remainder to the front.
  __device__ __forceinline__ void pop(int n) {
    __syncthreads();
    const uint32_t queued = cnt[NT / 32], rem = queued - (uint32_t)n;   // rem < NT <= n when rem > 0
    const uint32_t x = threadIdx.x < rem ? q[n + threadIdx.x] : 0u;
    __syncthreads();
    if (threadIdx.x < rem) q[threadIdx.x] = x;
    if (threadIdx.x == 0) cnt[NT / 32] = rem;
  }
};

}  // namespace puv
