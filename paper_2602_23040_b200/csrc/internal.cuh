// internal.cuh — device-side types, state layout and launchers of libpuv.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#include "../../include/puv.h"

// PUV_LNO: the fp64 value record carries ln(o) instead of o, folded into the Gaussian exponent
// (alpha = exp(power + ln o): one DMUL less per composited pixel in K5 and K6); K6's moments are
// then o-scaled (sums of alpha dL/dalpha) and K7 drops its o factors
#ifndef PUV_LNO
#define PUV_LNO 1
#endif
constexpr bool kLno = PUV_LNO != 0;

#ifndef PUV_K1_HEAD
#define PUV_K1_HEAD 0
#endif
constexpr int kK1Head = PUV_K1_HEAD;   // views projected ahead of the rest (0: one K1 for all views)

#ifndef PUV_STEP_OVERLAP
#define PUV_STEP_OVERLAP 0
#endif
constexpr bool kStepOverlap = PUV_STEP_OVERLAP != 0;   // train step: per-view K6 beside later K5s

#ifndef PUV_RASTER_CARVEOUT
#define PUV_RASTER_CARVEOUT -1   // -1: driver default
#endif

namespace puv {

constexpr int kMaxPlanes = 11 + 3 * 16 + 3;   // SH degree 3 + the 3 ray planes of PUV_POS_RHO
constexpr int kCamBatch = 64;             // views per K1/K7 launch (cameras passed by value, 6 KB of params)
constexpr int kTile = PUV_TILE;
constexpr int kNbMax = 1024;              // max key blocks of the stable tile pass per view
#ifndef PUV_BIN_STREAMS
#define PUV_BIN_STREAMS 4
#endif
constexpr int kBinStreams = PUV_BIN_STREAMS;  // views binned concurrently (one scratch block each)
#ifndef PUV_SORT_GROUP
#define PUV_SORT_GROUP 1
#endif
// views depth-sorted by one set of onesweep launches (grid.y); their tile passes stay per view
constexpr int kSortGroup = PUV_SORT_GROUP;
#ifndef PUV_BIN_PRIORITY
#define PUV_BIN_PRIORITY 0
#endif
constexpr int kBinPriority = PUV_BIN_PRIORITY;  // 1: binning streams at the highest priority (A/B: +2 ms/step, off)
#ifndef PUV_DMASK
#define PUV_DMASK 1
#endif
#ifndef PUV_DMASK_CAP
#define PUV_DMASK_CAP 384
#endif
// K5 records, for the first kMaskCap entries of every tile list, which of the tile's 256 pixels
// composited the entry (8 words in K6's pixel order); K6 reads the bits instead of replaying the
// fp32 skip test (entries beyond the cap: replay).  DESIGN.md §6.
constexpr int kMaskCap = PUV_DMASK ? PUV_DMASK_CAP : 0;
#ifndef PUV_FWD_GROUP
#define PUV_FWD_GROUP 4
#endif
constexpr int kFwdGroup = PUV_FWD_GROUP;  // consecutive views per forward-composite launch (4: K5 47.3 -> 42.8 ms/step)
constexpr int kSup = 4;                   // tiles per super-tile side (level 1 of the tile pass)
constexpr int kSupT = kSup * kSup;        // tiles per super-tile
#ifndef PUV_DIRECT
#define PUV_DIRECT 1
#endif
// 1: K5/K6 consume each tile's entries straight from its super-tile's rank list (level 1 of the
// tile pass, in (depth, gid) order) with the rect test of level 2 applied as they stage a batch,
// so level 2 (materialising the per-tile lists) runs only for the parity / debug view.
constexpr bool kDirect = PUV_DIRECT != 0;
#ifndef PUV_MASK_FILL
#define PUV_MASK_FILL 0
#endif
// K5 writes zero mask words for a warp's entries after it stopped (all its pixels terminated) up to
// the tile's largest n_contrib, so every word K6 reads is valid and a set bit alone means
// "composited" (K6 drops its per-pixel e < n_contrib guard)
constexpr bool kMaskFill = PUV_MASK_FILL != 0 && kDirect && kMaskCap > 0;
constexpr uint32_t kInvisible = 0xFFFFFFFFu;

// Plane table of a render call; with LPO (PUV_RENDER_LPO) every atlas plane value is read through its
// proxy (qspec = D x (min, max), qbits[d] = bits, -1 = binary16, 0 = read as is; the ray planes of
// PUV_POS_RHO are never quantised).
struct PlaneTab {
  const float* p[kMaxPlanes];
  const float* qspec;
  int8_t qbits[kMaxPlanes];
};
struct GradTab { float* p[kMaxPlanes]; };

// Per-view camera constants (viewmat rows 0..2, intrinsics, lim = fp32(1.3*W/(2 fx)) (R5)).
struct CamDev {
  float V[12];
  float fx, fy, cx, cy;
  int W, H;
  float near_plane;
  float campos[3];
  float limx, limy;
  // the same values widened on the host (exact): the fp64 value path reads these instead of
  // converting the fp32 fields per (view, texel) (F2F is a quarter-rate conversion op)
  double V64[12];
  double fx64, fy64, cx64, cy64, limx64, limy64, campos64[3];
};
struct CamBatch { CamDev c[kCamBatch]; int n; int v0; };

// Position storage (puv_layout.position_mode): rho mode reads mu = c (+) rho (x) ray with the ray in
// planes [D, D+3) of the plane table.
struct PosMode { int rho; int D; float c[3]; };

// Device header of one view (written by kernels; read by later kernels and by the host once per step).
struct ViewHdr {
  uint32_t n_vis;
  uint32_t overflow;      // 1 if this view's keys did not fit in the arena
  uint64_t K;             // keys of this view
  uint64_t list_base;     // offset (in keys) of this view's lists inside the arena
  uint32_t kb;            // keys per block of the stable tile pass
  uint32_t nb;            // blocks of the stable tile pass
  uint64_t ktotal;        // scratch: K before the arena is carved
  uint64_t examined;      // (pixel, entry) pairs that ran the skip test in K5
  uint64_t composited;    // pairs composited in K5
  uint64_t pad;
};
struct CallHdr {
  uint64_t arena_used;    // keys handed out so far (running sum over views)
  uint64_t arena_need;    // keys requested (>= arena_used when overflowing)
  uint32_t overflow_any;
  uint32_t n_views;       // views of the call (puv_view_counts checks against it)
  uint64_t arena_cap;     // capacity in keys (copied at launch)
  uint64_t pad[4];
};

// Offsets (bytes) of every array inside the caller's state buffer.
struct Plan {
  int n_views, N, W, H, HW, gx, gy, ntiles, D, deg;
  PosMode pm;
  size_t call_hdr, view_hdr;
  // per view arrays, each [n_views][...]
  size_t depth, rect, rec, rec64, grad2d, sorted, tstart, tend, tfinal, ncontrib, cfull, dmask;
  size_t sst, sen, l1hdr;  // per view: super-tile ranges into the level-1 rank list, its header
  int sgx, nst;            // super-tiles per row, super-tiles
  // scratch shared by all views (reused in stream order)
  // (offsets relative to one scratch block; block i starts at scratch0 + i * scratch_stride)
  size_t sk0, sv0, sk1, sv1, hist, koff, bsum, cnt, bstart, bin2;
  size_t scratch0, scratch_stride;
  int nscratch;            // binning streams / scratch blocks of this call
  size_t sort_blocks;      // blocks of one radix pass over N items
  size_t total;
};

// Records of a visible (view, Gaussian):
//  rec   (fp32 contract, 32 B): A=(mx,my,ha,nb) B=(hc,t_g,o,flags)  -> every decision; flags = SH clamp bits (K7)
//  rec64 (fp64 values,   80 B): (mx,my) (ha,nb) (hc,ln o) (r,g) (b,-)   (o itself when !kLno)               -> backward values
struct Views {
  uint32_t* depth;   // [V][N]
  uint2* rect;       // [V][N]  (x0 | x1<<16, y0 | y1<<16)
  float4* rec;       // [V][N][2]
  double2* rec64;    // [V][N][5]
  double* grad2d;    // [V][N][9]  d/d(mx,my,ha,nb,hc,o,r,g,b), fp64
  uint32_t* sorted;  // [V][N]  gids in (depth, gid) order, first n_vis valid
  uint32_t* tstart;  // [V][ntiles]
  uint32_t* tend;    // [V][ntiles]
  float* tfinal;     // [V][HW]
  uint32_t* ncontrib;// [V][HW]
  double* cfull;     // [V][HW][3]  fp64 full colour sum c a T + T_final bg (forward -> backward)
  uint32_t* dmask;   // [V][ntiles][kMaskCap][8]  composited-pixel bitmask per (tile, entry) (K5 -> K6)
  uint32_t* sst;     // [V][nst + 1]  super-tile range start in the view's level-1 rank list
  uint32_t* sen;     // [V][nst + 1]  ... end
  ViewHdr* l1;       // [V]  level-1 header (list_base of the rank lists, K1, overflow)
  int sgx, nst;      // super-tiles per row, super-tiles
  ViewHdr* hdr;      // [V]
  CallHdr* call;
};

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Device-side bounds checks of the data-dependent indexing (arena writes and reads, gids), on in
// the -DPUV_DEBUG_CHECKS build only (compute-sanitizer is not available on the GPU pool): a
// violated check traps the kernel, and the call surfaces PUV_E_CUDA.
#ifdef PUV_DEBUG_CHECKS
#define PUV_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define PUV_CHECK(cond) do { } while (0)
#endif

Plan make_plan(const puv_layout& L, int n_views, int W, int H);
Views views_of(const Plan& p, void* state);

// ---- launch accounting (every kernel launch of the library is counted; see puv_profile_read) ----
void count_launches(int n);
size_t depth_sort_scratch_bytes(size_t N);
size_t bin_scratch_bytes(size_t N, int ntiles);

// ---- launchers (all asynchronous on `s`) ----
void launch_project(const Plan& p, const Views& v, const PlaneTab& P, const uint8_t* occ, const CamBatch& cb,
                    cudaStream_t s, int g0 = 0, int g1 = -1);
void launch_depth_sort(const Plan& p, const Views& v, void* state, int view, int nv, cudaStream_t s);
void launch_bin(const Plan& p, const Views& v, void* state, uint32_t* arena, int view, cudaStream_t s, bool level2);
void launch_bin_level2(const Plan& p, const Views& v, void* state, uint32_t* arena, int view, cudaStream_t s);
void launch_raster_fwd(const Plan& p, const Views& v, const uint32_t* arena, float* images, int view0, int n_views,
                       const float bg[3], cudaStream_t s);
void launch_raster_bwd(const Plan& p, const Views& v, const uint32_t* arena, const float* dL_dimages, int view0,
                       int n_views, cudaStream_t s);
void launch_project_bwd(const Plan& p, const Views& v, const PlaneTab& P, const uint8_t* occ, const uint8_t* mask,
                        const CamBatch& cb, const GradTab& G, cudaStream_t s, int g0 = 0, int g1 = -1,
                        bool overwrite = false);
void launch_l2_loss(int64_t n, const float* img, const float* tgt, float* dl, double* loss, cudaStream_t s,
                    bool accumulate);
void launch_pack(const puv_layout& L, const float* const* level_planes, const uint8_t* const* level_occ,
                 float* const* atlas_planes, uint8_t* atlas_occ, cudaStream_t s);
void launch_unpack(const puv_layout& L, const float* const* atlas_planes, float* const* level_planes, cudaStream_t s);
void launch_contract(int op, const float* in, float* out, int64_t n, cudaStream_t s);
void launch_label(const Plan& p, const PlaneTab& P, const uint8_t* occ, const CamDev& cam, const uint8_t* mask,
                  uint32_t* sat, int r_max, int first, uint8_t* labels, cudaStream_t s);
size_t photo_view_bytes(int W, int H);
void launch_photo_loss(int nviews, int W, int H, const float* img, const float* tgt, double lam, float* dl,
                       double* loss, void* ws, int chunk, cudaStream_t s);
size_t reg_workspace_bytes();
void launch_reg_loss(const PlaneTab& P, const uint8_t* occ, const uint8_t* mask, int64_t N, double lam_s,
                     double lam_o, double s_max, const GradTab& G, double* loss, void* ws, cudaStream_t s);
void launch_quant_fit(const PlaneTab& P, int D, const uint8_t* occ, int64_t N, float* spec, cudaStream_t s);
void launch_quantize(const float* const* x, float* const* proxy, void* const* code, const int8_t* bits, int D,
                     const float* spec, const uint8_t* occ, int64_t N, cudaStream_t s);
void launch_begin_call(const Plan& p, const Views& v, uint64_t arena_cap, cudaStream_t s);
void launch_overflow_acc(const void* state, uint32_t* flag, uint64_t* need, cudaStream_t s);

}  // namespace puv
