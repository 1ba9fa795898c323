/*
 * puv.h — C ABI of libpuv: the differentiable splat render of UV-atlas Gaussians
 * (PackUV-GS, arXiv 2602.23040) for NVIDIA B200 (sm_100a).
 *
 * The paper's problem statement: fit Gaussians stored in UV maps
 * U[u,v,k] = {rho, r, s, o, c} to multi-view images by
 * rendering them "as 2D splats ... combined with alpha-blending using a
 * tile-based rasterizer" and back-propagating the image loss
 * onto the texels, with gradient freezing of static Gaussians.
 * Levels are packed into one atlas.  Every reading of a
 * point the paper leaves open is listed in DESIGN.md §2 (R1..R16).
 *
 * Conventions (all entry points):
 *  - extern "C", never throw; return puv_status (0 = PUV_OK, < 0 = error).
 *  - The caller owns every buffer.  The library never allocates device memory.
 *    "device pointer" = a pointer valid on the current CUDA device;
 *    "host pointer" = ordinary process memory.  Arrays of device pointers
 *    (plane tables) are themselves HOST arrays.
 *  - Calls that take `stream` (a cudaStream_t, NULL = legacy default stream)
 *    are asynchronous: argument errors are returned synchronously before any
 *    work is enqueued; CUDA launch errors surface as PUV_E_CUDA.
 *  - After an error, puv_last_error() returns a thread-local message.
 *  - Thread safety: calls may come from several host threads, also on one
 *    device (the library's internal binning streams are shared per device and
 *    their enqueue is serialised by a lock); two calls must not share a state
 *    or arena buffer concurrently.
 *  - Texel planes are fp32, SoA: plane d of an atlas is H_A*W_A floats, row
 *    major; texel id (gid) = y*W_A + x.  Plane order (R2):
 *      [x, y, z, ls0, ls1, ls2, qw, qx, qy, qz, logit_o, sh(k,c) at 11+3k+c]
 *    D = 11 + 3*(sh_degree+1)^2.
 *  - Images are fp32 planar (3, H, W) per view, views concatenated.
 */
#ifndef PUV_H_
#define PUV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t puv_status;
enum {
  PUV_OK = 0,
  PUV_E_INVALID_ARGUMENT = -1,    /* null pointer, bad count, bad size */
  PUV_E_INVALID_CONFIG = -2,      /* bad level list / sh_degree */
  PUV_E_LAYOUT_OVERFLOW = -3,     /* placement outside the atlas */
  PUV_E_DIMENSION_MISMATCH = -4,  /* plane count / image size mismatch */
  PUV_E_INVALID_CAMERA = -5,      /* fx,fy <= 0, empty image, rotation not orthonormal within 1e-5 */
  PUV_E_WORKSPACE_TOO_SMALL = -6, /* state buffer smaller than puv_query_sizes() */
  PUV_E_STATE_MISMATCH = -7,      /* state was written by a different call signature */
  PUV_E_CUDA = -8,                /* a CUDA runtime error (message in puv_last_error) */
  PUV_E_UNSUPPORTED = -9          /* outside the built envelope (e.g. > 16 levels) */
};

#define PUV_MAX_LEVELS 16
#define PUV_MAX_SH_DEGREE 3
#define PUV_TILE 16

/* One UV level placed in the atlas.  rows x cols = M_k x N_k.
 * Unrotated: cell (r, c) -> atlas (y + r, x + c).  rot90ccw: the placement is
 * cols tall and rows wide; cell (r, c) -> atlas (y + cols - 1 - c, x + r) (R15). */
typedef struct {
  int32_t rows, cols;
  int32_t x, y;
  int32_t rot90ccw;
} puv_placement;

typedef struct {
  int32_t num_levels;   /* K, 1..16 */
  int32_t sh_degree;    /* 0..3 */
  int32_t planes;       /* D = 11 + 3*(sh_degree+1)^2 */
  int32_t atlas_w, atlas_h;
  puv_placement level[PUV_MAX_LEVELS];
  /* Position storage:
   *  PUV_POS_XYZ: planes 0..2 hold the world position (default).
   *  PUV_POS_RHO: plane 0 holds rho, the distance from `center` along the texel's UV ray; planes 1..2
   *    are unused (their table entries may be NULL and their gradients are left untouched) and the
   *    plane table passed to render/backward has D + 3 entries: [D..D+2] = the ray-direction planes
   *    written by puv_ray_planes.  The texel position is mu = center (+) rho (x) ray in the fp32
   *    contract; d rho = ray . d mu. */
  int32_t position_mode;
  float center[3];
} puv_layout;

enum { PUV_POS_XYZ = 0, PUV_POS_RHO = 1 };

/* Pinhole camera, OpenCV axes (x right, y down, z forward) (R4).  Pixel (i, j)
 * is sampled at integer coordinates. */
typedef struct {
  float viewmat[16];    /* row-major world -> camera rigid transform */
  float fx, fy, cx, cy; /* pixels */
  int32_t width, height;
  float near_plane;     /* cull z <= near (0.2 in every config) */
  float campos[3];      /* camera centre in world space (SH view direction, R3) */
} puv_camera;

typedef struct {
  float bg[3];          /* background colour, composited with T_final (R9) */
  uint32_t flags;       /* 0, or PUV_RENDER_LPO */
  /* PUV_RENDER_LPO (NEXT-2 fused into the render): every texel plane value the
   * render and its backward read is replaced, as it is read, by its LPO proxy -- exactly the value
   * puv_quantize would write (Q1-Q8): the per-plane range lpo_spec (device, D x 2 floats, from
   * puv_quant_fit), lpo_pos_bits for the position planes (1..16 or PUV_QUANT_FP16), lpo_attr_bits
   * (1..16) for the others.  The backward then returns the straight-through (STE) gradient of the
   * fp32 master planes without a proxy atlas in memory. */
  const float* lpo_spec;
  int32_t lpo_pos_bits, lpo_attr_bits;
} puv_render_opts;
#define PUV_RENDER_LPO 1u

/* Column layout (R15): L0 at (0,0); levels 1.. stacked top-down at x = cols[0],
 * unrotated; W_A = cols0 + max_{k>=1} cols_k, H_A = max(rows0, sum_{k>=1} rows_k).
 * rows/cols: host arrays of K.  out: host. */
puv_status puv_layout_for_levels(int32_t K, const int32_t* rows, const int32_t* cols, int32_t sh_degree,
                                 puv_layout* out);

/* The paper's pyramid schedule and recursive atlas layout: level 0
 * is M0 x N0 and levels alternate halving N and M (odd k: N/2, even k: M/2).  A level is an image of
 * M_k columns (u, azimuth) by N_k rows (v, polar).  Placement (x, y of the top-left corner): L0 at
 * (S/2, 0); L1 rotated 90 deg CCW at (0, 0); L2 at (0, S); L3 (rotated) right of L2, L4 right of L3,
 * L5 (rotated) below L4, L6 right of L5, L7 (rotated) below L6 — odd levels rotated, even levels not.
 * M0 = N0 = S (a power of two >= 16), 1 <= K <= 8.  For S = 1024, K = 8: atlas 1536 x 1536 with
 * 2,088,960 used texels (0.8854, "88.5% efficiency").  position_mode = PUV_POS_XYZ. */
puv_status puv_layout_paper(int32_t S, int32_t K, int32_t sh_degree, puv_layout* out);

/* Ray-direction planes of an atlas (for PUV_POS_RHO): for level k cell (v = row, u = column),
 * theta = (u + 0.5)/M_k 2 pi - pi, phi = (v + 0.5)/N_k pi, ray = (sin phi cos theta, sin phi sin theta,
 * cos phi) (the inverse of PAPER.md eq. uvgs2 at pixel centres), evaluated in fp64 on
 * the host and rounded to fp32, written at the texel's atlas position; unplaced texels get 0.
 * ray_planes: host array of 3 device pointers (H_A*W_A floats each).  Synchronous. */
puv_status puv_ray_planes(const puv_layout* layout, float* const* ray_planes, void* stream);

/* Pack K levels into the atlas.  level_planes: host array of
 * K*D device pointers, k-major (level k plane d at [k*D + d]), each rows_k*cols_k
 * floats.  level_occ: host array of K device pointers to rows_k*cols_k bytes
 * (occupancy), or NULL (all occupied).  atlas_planes: host array of D device
 * pointers (H_A*W_A floats); atlas_occ: device, H_A*W_A bytes.  Pixels outside
 * every placement are written 0 / unoccupied.  Errors: INVALID_ARGUMENT,
 * LAYOUT_OVERFLOW (a placement leaves the atlas or two overlap). */
puv_status puv_pack_atlas(const puv_layout* layout, const float* const* level_planes,
                          const uint8_t* const* level_occ, float* const* atlas_planes, uint8_t* atlas_occ,
                          void* stream);

/* Inverse of pack for D planes (used for gradients): atlas -> levels. */
puv_status puv_unpack_levels(const puv_layout* layout, const float* const* atlas_planes, float* const* level_planes,
                             void* stream);

/* Sizes for a render/backward call over n_views cameras (host array).
 * state_bytes: the fixed-size per-call state (per-view records, depth order,
 *   per-pixel transmittance, tile ranges, 2D gradients, scratch).
 * arena_hint: a first guess for the key arena (tile lists); the exact need is
 *   data dependent and reported by puv_check_overflow after a render. */
puv_status puv_query_sizes(const puv_layout* layout, int32_t n_views, const puv_camera* cams,
                           const puv_render_opts* opts, size_t* state_bytes, size_t* arena_hint);

/* Forward render of n_views views (steps a1-a5 of DESIGN.md §1).
 * atlas_planes: host array of D device pointers; atlas_occ: device H_A*W_A bytes
 * or NULL (all occupied).  cams: host array of n_views.  images: device,
 * n_views*3*H*W floats (all views must share W, H).  state: device, >= state_bytes.
 * arena: device, arena_bytes.  Per view it holds the K tile-list keys (4 bytes
 * each) followed by the K1 keys of the level-1 super-tile pass of the binning
 * (4x4-tile super-tiles, K1 = sum over visible Gaussians of the super-tile
 * rect areas, ~K/10 at C3).  If a view does not fit, the
 * overflow flag is set on device, the affected views render nothing, and
 * puv_check_overflow reports the size needed (4 (K + K1) bytes summed over views). */
puv_status puv_render_views(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                            int32_t n_views, const puv_camera* cams, const puv_render_opts* opts, float* images,
                            void* state, size_t state_bytes, void* arena, size_t arena_bytes, void* stream);

/* L = 1/2 sum (images - targets)^2 (R11) over n floats; dL_dimages = images -
 * targets.  loss: device double, OVERWRITTEN with L.  All device pointers. */
puv_status puv_l2_loss_grad(int64_t n, const float* images, const float* targets, float* dL_dimages, double* loss,
                            void* stream);

/* The paper's photometric objective (NEXT-4; readings L1-L4 of DESIGN.md §12):
 *   loss = sum_views (1 - lambda_ssim) mean|I^ - I| + lambda_ssim (1 - mean SSIM(I^, I)),
 * means over the view's 3 H W entries; SSIM of Wang et al. with an 11 x 11 Gaussian window
 * (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero-padded windows, per channel; statistics in fp64.
 * dL_dimages = d loss / d images (sign(0) = 0 for the L1 term), OVERWRITTEN; loss: device double,
 * OVERWRITTEN.  images/targets/dL_dimages: device, n_views*3*H*W floats (CHW per view).
 * workspace: device, >= puv_photo_workspace_bytes(W, H, 1) bytes; views are processed in chunks of
 * as many as the workspace holds (puv_photo_workspace_bytes(W, H, v) for v views per chunk).
 * lambda_ssim in [0, 1] (0.2 when the caller has no value: L1). */
size_t puv_photo_workspace_bytes(int32_t width, int32_t height, int32_t views_per_chunk);
puv_status puv_photo_loss_grad(int32_t n_views, int32_t width, int32_t height, const float* images,
                               const float* targets, double lambda_ssim, float* dL_dimages, double* loss,
                               void* workspace, size_t workspace_bytes, void* stream);

/* The paper's regularisers (readings L5-L7 of DESIGN.md §12):
 *   loss = lambda_scale E_i[max(0, max_a exp(ls_ia) - s_max)]^2 + lambda_opacity E_i alpha_i (1 - alpha_i),
 * alpha = sigmoid(opacity logit), E_i the mean over occupied texels (atlas_occ != 0, or all if NULL)
 * that are dynamic (dynamic_mask != 0; all if NULL).  loss: device double, OVERWRITTEN (0 when no
 * texel is selected).  Gradients are ACCUMULATED (+=) onto atlas_grad planes 3, 4, 5 (the argmax
 * axis; ties -> lowest) and 10; only those four entries of atlas_planes / atlas_grad are read.
 * workspace: device, >= puv_reg_workspace_bytes() bytes.  (lambdas 1e-4.) */
size_t puv_reg_workspace_bytes(void);
puv_status puv_reg_loss_grad(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                             const uint8_t* dynamic_mask, double lambda_scale, double lambda_opacity, double s_max,
                             float* const* atlas_grad, double* loss, void* workspace, size_t workspace_bytes,
                             void* stream);

/* Low-precision optimisation (LPO, NEXT-2; readings Q1-Q7 of
 * DESIGN.md §13).  Training renders a uniformly quantised proxy of the fp32 master planes and
 * passes gradients straight through (STE): call puv_quantize for the proxy, render / backward the
 * proxy with the usual calls, and accumulate the backward into the MASTER gradient planes.
 *
 * puv_quant_fit: per-plane (min, max) over occupied texels -> spec, a device array
 * of D x 2 floats (OVERWRITTEN; (0, 0) for a plane with no occupied texel and for the unused planes
 * 1, 2 of PUV_POS_RHO).  Exact (order independent).
 * puv_quantize: per texel and plane, in the fp32 contract,
 *   L = 2^bits - 1, t = clamp(((x - min) / (max - min)) * L, 0, L), code = round half away (t),
 *   proxy = min + (code / L) * (max - min);  max == min -> code 0, proxy = min;
 * bits = pos_bits for the position planes (0..2, or plane 0 = rho), attr_bits for the others
 * (16 and 8; each 1..16).  Unoccupied texels: code 0, proxy 0.  codes: NULL, or a
 * host table of D device pointers to uint8 planes (bits <= 8) / uint16 planes (bits > 8; the two
 * bytes are the hi/lo 8-bit planes of SPEC.md:313); proxy: NULL or a host table of D device fp32
 * planes.  Entries for rho mode's planes 1, 2 are ignored (may be NULL).
 * pos_bits = PUV_QUANT_FP16 (reading Q8, "we retain them in FP16"): the position
 * planes are instead stored as IEEE binary16 (round to nearest even; the range is not used):
 * code = the 16-bit pattern (uint16 plane; its two bytes are the 8-bit storage split of
 * PAPER.md:1303), proxy = the half's value. */
#define PUV_QUANT_FP16 256
puv_status puv_quant_fit(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                         float* spec, void* stream);
puv_status puv_quantize(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                        const float* spec, int32_t pos_bits, int32_t attr_bits, void* const* codes,
                        float* const* proxy, void* stream);

/* Backward of the last puv_render_views with the same layout/cams/opts/state/arena
 * (steps a7-a9).  dL_dimages: device, like images.  dynamic_mask: device
 * H_A*W_A bytes (D_i of PAPER.md:410-414) or NULL.  atlas_grad: host array of D
 * device pointers; gradients w.r.t. the texel planes are ACCUMULATED (+=).
 * Re-entrant: the per-(view, Gaussian) moment slots in `state` are reset by every call, so k
 * calls after one render add k times the gradient (e.g. two loss terms on one forward). */
puv_status puv_render_backward(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                               int32_t n_views, const puv_camera* cams, const puv_render_opts* opts,
                               const float* dL_dimages, const uint8_t* dynamic_mask, void* state, size_t state_bytes,
                               void* arena, size_t arena_bytes, float* const* atlas_grad, void* stream);

/* Covariance-aware flow masking, supp. Algorithm 1: the dynamic label
 *   D_i = OR_c [ exists integer pixel p inside the image with |p - m_ic|_inf <= r_ic,
 *                mask_c(p) != 0 and (p - m_ic)^T (Sigma2D_ic)^-1 (p - m_ic) <= 9 ],
 *   r_ic = min(r_max, ceil(3 sqrt(lambda_max))), Sigma2D with the UNclamped EWA Jacobian + 0.3,
 *   camera c skipped for texel i when z <= 0 or det <= 1e-7 (readings M1-M6).
 * The labels feed render_backward's dynamic_mask (gradient freezing).
 * masks: device, n_cams*H*W bytes (all cameras share W, H).  labels: device, H_A*W_A bytes,
 * OVERWRITTEN (1 dynamic / 0 static; unoccupied texels 0).  workspace: device, at least
 * puv_label_workspace_bytes(W, H) bytes.  r_max >= 0 (SPEC.md:472 default 64). */
size_t puv_label_workspace_bytes(int32_t width, int32_t height);
puv_status puv_label_dynamic(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                             int32_t n_cams, const puv_camera* cams, const uint8_t* masks, int32_t r_max,
                             uint8_t* labels, void* workspace, size_t workspace_bytes, void* stream);

/* One fused training step of the L2 harness (steps a1-a9): puv_render_views, then per view
 * puv_l2_loss_grad and the composite backward, then the projection backward of all views —
 * the same results as the three calls in sequence (images, T_final, n_contrib and tile lists
 * bit-identical; loss and gradients up to the order of fp64 atomic additions), but each view's
 * loss gradient and composite backward run on a second internal stream as soon as the view is
 * composited, overlapping the compositing and binning of later views.  targets, dL_dimages:
 * device, like images.  loss: device double, OVERWRITTEN with 1/2 sum (images - targets)^2.
 * atlas_grad: ACCUMULATED (+=) like puv_render_backward.  On arena overflow the affected views
 * render nothing and their gradients are not computed (puv_check_overflow, then re-run).
 * targets_ready: a cudaEvent_t or NULL; the loss gradients wait for it (not the render), so a
 * host->device copy of the targets recorded on another stream overlaps the render. */
puv_status puv_render_l2_step(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                              int32_t n_views, const puv_camera* cams, const puv_render_opts* opts, float* images,
                              const float* targets, float* dL_dimages, double* loss, const uint8_t* dynamic_mask,
                              void* state, size_t state_bytes, void* arena, size_t arena_bytes,
                              float* const* atlas_grad, void* targets_ready, void* stream);

/* Device buffers of a training step (puv_train_step / puv_train_step_host).  images and
 * dL_dimages hold views_per_call views (n*3*H*W floats); loss: double, OVERWRITTEN with
 * L = 1/2 sum over all views (R11); overflow (uint32) / arena_need (uint64): OVERWRITTEN with
 * "some view chunk overflowed the key arena" and the largest arena bytes a chunk needed (the
 * step's result is then incomplete: grow the arena to arena_need and re-run the step);
 * state / arena as for puv_render_views with n_views = views_per_call. */
typedef struct {
  float* images;
  float* dL_dimages;
  double* loss;
  uint32_t* overflow;
  uint64_t* arena_need;
  void* state;
  size_t state_bytes;
  void* arena;
  size_t arena_bytes;
} puv_step_buffers;

/* One training step of the L2 harness over n_views views (rows a1-a9), in chunks of
 * views_per_call views (<= 0: all in one chunk; the state is sized for one chunk, so a large
 * rig fits HBM): per chunk puv_render_views, the L2 loss gradient against `targets` (device,
 * n_views*3*H*W floats), the composite and projection backward.  atlas_grad (host table of D
 * device planes) is OVERWRITTEN with dL/d(texel planes) summed over all views, x D_i when
 * dynamic_mask is given.  Results equal the separate calls. */
puv_status puv_train_step(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                          int32_t n_views, const puv_camera* cams, const puv_render_opts* opts, const float* targets,
                          const uint8_t* dynamic_mask, int32_t views_per_call, const puv_step_buffers* buffers,
                          float* const* atlas_grad, void* stream);

/* One host<->device copy: src / dst are a HOST and a DEVICE pointer (direction given by the call). */
typedef struct {
  const void* src;
  void* dst;
  size_t bytes;
} puv_copy;

/* puv_train_step from HOST inputs, end to end: enqueues on `stream` the `uploads`
 * (host -> device, e.g. the atlas planes), copies targets_host (host, n_views*3*H*W floats) into
 * `targets` (device) on an internal copy stream that overlaps the render (the first loss waits
 * for it), runs the step, then the `downloads` (device -> host, e.g. the gradient planes and the
 * loss).  Asynchronous like every call: synchronise `stream` before reading the downloads.
 * Pinned host memory makes the copies asynchronous (pageable memory works, synchronously). */
puv_status puv_train_step_host(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                               int32_t n_views, const puv_camera* cams, const puv_render_opts* opts,
                               const puv_copy* uploads, int32_t n_uploads, const float* targets_host, float* targets,
                               const uint8_t* dynamic_mask, int32_t views_per_call, const puv_step_buffers* buffers,
                               float* const* atlas_grad, const puv_copy* downloads, int32_t n_downloads,
                               void* stream);

/* puv_train_step from HOST buffers with the host link overlapped (the e2e path of a training loop):
 * atlas_host (host, D x H_A*W_A floats, plane-major) is uploaded into the device planes atlas_planes
 * (a host table; rho mode's unused planes 1, 2 may be NULL and the ray planes stay resident) in 4
 * texel chunks on an internal copy stream, K1 projecting each chunk as soon as it has landed; the
 * targets follow on that stream (the first loss waits for them); the gradient (OVERWRITTEN in
 * atlas_grad) goes back into grad_host (host, D x H_A*W_A) in 4 texel chunks on a second copy
 * stream as K7 finishes each, then the loss into *loss_host.  Same results as puv_train_step.
 * Asynchronous: synchronise `stream` before reading grad_host / loss_host (pinned memory makes the
 * copies asynchronous).  Every argument is checked before anything is enqueued. */
puv_status puv_train_step_host_atlas(const puv_layout* layout, float* const* atlas_planes, const float* atlas_host,
                                     const uint8_t* atlas_occ, int32_t n_views, const puv_camera* cams,
                                     const puv_render_opts* opts, const float* targets_host, float* targets,
                                     const uint8_t* dynamic_mask, int32_t views_per_call,
                                     const puv_step_buffers* buffers, float* const* atlas_grad, float* grad_host,
                                     double* loss_host, void* stream);

/* The one host synchronisation per step: waits for `stream`, then reports
 * whether any view of the last render overflowed the arena and the arena
 * bytes the call needs.  Host outputs. */
puv_status puv_check_overflow(const void* state, int32_t n_views, void* stream, int32_t* overflowed,
                              uint64_t* needed_arena_bytes);

/* The asynchronous form of puv_check_overflow for callers that chain several render calls
 * (e.g. view chunks of one step) without a host sync: enqueues on `stream`
 *   *flag |= (the last render call on `state` overflowed);
 *   *needed_arena_bytes = max(*needed_arena_bytes, the arena bytes that call needed).
 * flag, needed_arena_bytes: DEVICE pointers (uint32, uint64), caller-initialised. */
puv_status puv_overflow_accumulate(const void* state, uint32_t* flag, uint64_t* needed_arena_bytes, void* stream);

/* Counters of one view of the last render on `state` (synchronises `stream`), without the tile-list
 * materialisation of puv_debug_view: counts[0..4] = visible Gaussians, K (keys = sum of tiles
 * touched), (pixel, entry) pairs examined and composited by the forward, overflow flag.  Host out.
 * `view` must be < the n_views of that render (PUV_E_INVALID_ARGUMENT otherwise). */
puv_status puv_view_counts(const void* state, int32_t view, void* stream, uint64_t* counts);

/* Per-view debug/parity view of the state (synchronises `stream`).  Host out.
 * Device pointers inside point into state/arena and stay valid until the next call.  The render
 * consumes each tile's entries straight from the level-1 super-tile lists (the rect test applied
 * while K5/K6 stage them), so this call first materialises the view's per-tile lists (level 2 of
 * the tile pass, into the arena space the render reserved for them): state and arena are written. */
typedef struct {
  uint32_t n_visible;            /* Gaussians surviving culling in this view */
  uint32_t ntiles, tiles_x, tiles_y;
  uint64_t n_keys;               /* K = sum of tiles touched */
  const uint32_t* tile_start;    /* device, ntiles: range start into `keys_gid` */
  const uint32_t* tile_end;      /* device, ntiles: range end (exclusive) */
  const uint32_t* keys_gid;      /* device, n_keys gids, sorted by (tile, depth_bits, gid) */
  const uint32_t* depth_key;     /* device, H_A*W_A: depth bits of z, 0xFFFFFFFF if culled */
  const float* t_final;          /* device, H*W: fp32 contract transmittance after the last entry */
  const uint32_t* n_contrib;     /* device, H*W: list position after the last composited entry */
  const double* grad2d;          /* device, H_A*W_A*9 fp64, per Gaussian, of the last backward: pixel moments
                                    (Mx,My,Mxx,Mxy,Myy) of alpha dL/dalpha (= o G dL/dalpha), o dL/do, dL/d(r,g,b);
                                    dL/d(mx,my,ha,nb,hc) = (2ha Mx + nb My, nb Mx + 2hc My, Mxx, Mxy, Myy)
                                    (k_raster_bwd.cu; a -DPUV_LNO=0 build stores the moments of G dL/dalpha) */
  const uint32_t* depth_order;   /* device, n_visible gids sorted by (depth_bits, gid) */
  uint64_t n_examined;           /* (pixel, entry) pairs that ran the skip test in the forward */
  uint64_t n_composited;         /* pairs composited in the forward */
} puv_view_debug;

puv_status puv_debug_view(const puv_layout* layout, int32_t n_views, const puv_camera* cams, void* state,
                          size_t state_bytes, void* arena, int32_t view, void* stream, puv_view_debug* out);

/* Stage profiling.  When enabled, every library call records a CUDA event pair
 * around each stage on the call's stream (asynchronous, no host sync).
 * puv_profile_read synchronises those events and returns, per stage, the summed
 * device milliseconds, the kernels launched and the number of timed stage
 * instances; kernel_launches counts every kernel the library launched since it
 * was loaded (profiling on or off).  Stages: */
#define PUV_NUM_STAGES 11
enum {
  PUV_STAGE_PROJECT = 0,      /* K1 unpack + EWA projection + SH colour + rect (rows a1, a2) */
  PUV_STAGE_DEPTH_SORT = 1,   /* K3 depth radix sort with culling compaction (row a4, low digit) */
  PUV_STAGE_BIN = 2,          /* K2/K4 key generation + stable tile pass + tile ranges (rows a3, a4) */
  PUV_STAGE_RASTER_FWD = 3,   /* K5 composite (row a5) */
  PUV_STAGE_LOSS = 4,         /* K10 L2 loss gradient (row a6) */
  PUV_STAGE_RASTER_BWD = 5,   /* K6 composite backward (row a7) */
  PUV_STAGE_PROJECT_BWD = 6,  /* K7 projection + unpack backward, scatter to texels (rows a8, a9) */
  PUV_STAGE_PACK = 7,         /* K9 pack / unpack */
  PUV_STAGE_LABEL = 8,        /* K11 flow masking (supp. Alg. 1) */
  PUV_STAGE_OBJECTIVE = 9,    /* K12/K13 L1+SSIM photometric loss, regularisers (NEXT-4) */
  PUV_STAGE_QUANT = 10        /* K14 LPO range fit + fake quantiser (NEXT-2) */
};
typedef struct {
  double ms[PUV_NUM_STAGES];
  uint64_t launches[PUV_NUM_STAGES];
  uint64_t calls[PUV_NUM_STAGES];
  uint64_t kernel_launches;
} puv_profile;
/* Measurement aid: with on != 0, later render calls run the depth sort and binning of each view
 * on the caller's stream instead of the internal binning streams, so every stage runs alone and
 * its per-stage event time (puv_profile_read) is its serialised cost.  Results are identical. */
puv_status puv_profile_serial(int32_t on);
/* The recorded stage instances since the last reset, in enqueue order (synchronises): per instance
 * out[3i] = stage id, out[3i+1] / out[3i+2] = start / end in ms relative to the first instance's
 * start (a timeline of the overlapped stages).  Host outputs; at most max_events instances. */
puv_status puv_profile_timeline(double* out, int32_t max_events, int32_t* n_events);
puv_status puv_profile_enable(int32_t on);
puv_status puv_profile_read(puv_profile* out, int32_t reset);

/* Evaluate a contract function of DESIGN.md R13 elementwise on device arrays (for the
 * exhaustive GPU-vs-oracle bit-equality test).  op: 0 = exp_c, 1 = log_c.  in/out: device, n floats. */
puv_status puv_debug_contract(int32_t op, const float* in, float* out, int64_t n, void* stream);

/* Thread-local message of the last error; returns its length (writes up to len-1 chars + NUL). */
size_t puv_last_error(char* buf, size_t len);

/* Library build id, e.g. "libpuv sm_100a <git describe>". */
const char* puv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PUV_H_ */
