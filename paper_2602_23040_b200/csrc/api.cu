// api.cu — the C ABI of include/puv.h: validation, state carving, stream sequencing.
//
// Host runtime only: every step of the path runs in the kernels of this
// directory.  Argument errors are returned before anything is enqueued.
#include <nvtx3/nvToolsExt.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <atomic>
#include <mutex>
#include <vector>

#include "internal.cuh"

#ifndef PUV_VERSION
#define PUV_VERSION "dev"
#endif

namespace puv {

static thread_local std::string g_err;

// ---- launch accounting and stage profiling ------------------------------------------------------
static std::atomic<uint64_t> g_launches{0};
void count_launches(int n) { g_launches += (uint64_t)n; }

struct ProfEvent { int stage; cudaEvent_t a, b; uint64_t launches; };
static std::mutex g_prof_mu;
static std::atomic<bool> g_prof_on{false};
static std::atomic<bool> g_serial{false};   // puv_profile_serial: binning on the caller's stream
static std::vector<ProfEvent> g_prof_events;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t take_event() {
  if (!g_event_pool.empty()) { cudaEvent_t e = g_event_pool.back(); g_event_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

static const char* const kStageName[] = {"puv:project", "puv:depth_sort", "puv:bin", "puv:raster_fwd",
                                         "puv:loss", "puv:raster_bwd", "puv:project_bwd", "puv:pack",
                                         "puv:label", "puv:objective", "puv:quant"};

// RAII: an NVTX range around the host-side enqueue of one stage (for ncu --nvtx filtering and
// timeline tools; a no-op without a tool attached), and an event pair around the stage on `s`
// when profiling is on.
struct StageScope {
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  uint64_t l0 = 0;
  StageScope(int st, cudaStream_t stream) : stage(st), s(stream) {
    nvtxRangePushA(kStageName[st]);
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    a = take_event();
    cudaEventRecord(a, s);
    l0 = g_launches;
  }
  ~StageScope() {
    nvtxRangePop();
    if (!a) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = take_event();
    cudaEventRecord(b, s);
    g_prof_events.push_back({stage, a, b, g_launches - l0});
  }
};

// ---- internal streams for the binning pipeline (one set per device, created on first use) ----
// One set per device, shared by every call on that device: `mu` serialises the enqueue of a
// render pipeline (the growable event pools and the fork/join events are not thread-safe), so
// host threads may call the library concurrently on one device.
struct StreamSet {
  std::mutex mu;
  cudaStream_t s[kBinStreams] = {};
  cudaStream_t s2 = nullptr;     // per-view loss + composite backward of the fused L2 step
  cudaStream_t cp = nullptr;     // host->device uploads of the host-buffer steps
  cudaStream_t cp2 = nullptr;    // device->host downloads of puv_train_step_host_atlas
  cudaStream_t k1 = nullptr;     // K1 of the views after the head (kK1Head), beside their binning
  cudaEvent_t fork = nullptr, join = nullptr, k1fork = nullptr, k1tail = nullptr;
  std::vector<cudaEvent_t> ev, fev, sev;
  static cudaEvent_t pooled(std::vector<cudaEvent_t>& pool, int v) {
    while ((int)pool.size() <= v) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      pool.push_back(e);
    }
    return pool[v];
  }
  cudaEvent_t view_event(int v) { return pooled(ev, v); }
  cudaEvent_t fwd_event(int v) { return pooled(fev, v); }
  cudaEvent_t sort_event(int g) { return pooled(sev, g); }
};

static StreamSet& stream_set(int /*n*/) {
  static std::mutex mu;
  static std::vector<StreamSet*> sets;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if ((int)sets.size() <= dev) sets.resize(dev + 1, nullptr);
  if (!sets[dev]) {
    StreamSet* ss = new StreamSet();
    // Binning streams at the highest stream priority only with -DPUV_BIN_PRIORITY=1: the step is
    // SM-time bound, and prioritised binning slows the compositing by more than it removes from the
    // composite waits (A/B on one B200: +2 ms per C3 step).
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    for (int i = 0; i < kBinStreams; ++i)
      cudaStreamCreateWithPriority(&ss->s[i], cudaStreamNonBlocking, kBinPriority ? prio_hi : prio_lo);
    cudaEventCreateWithFlags(&ss->fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss->join, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&ss->s2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ss->cp, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ss->cp2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ss->k1, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ss->k1fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss->k1tail, cudaEventDisableTiming);
    sets[dev] = ss;
  }
  return *sets[dev];
}

static puv_status fail(puv_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static puv_status cuda_check(const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PUV_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return PUV_OK;
}

static puv_status check_layout(const puv_layout* L) {
  if (!L) return fail(PUV_E_INVALID_ARGUMENT, "layout is NULL");
  if (L->num_levels < 1 || L->num_levels > PUV_MAX_LEVELS)
    return fail(PUV_E_INVALID_CONFIG, "num_levels %d outside 1..%d", L->num_levels, PUV_MAX_LEVELS);
  if (L->sh_degree < 0 || L->sh_degree > PUV_MAX_SH_DEGREE)
    return fail(PUV_E_INVALID_CONFIG, "sh_degree %d outside 0..3", L->sh_degree);
  const int D = 11 + 3 * (L->sh_degree + 1) * (L->sh_degree + 1);
  if (L->planes != D) return fail(PUV_E_DIMENSION_MISMATCH, "planes %d != 11 + 3 (deg+1)^2 = %d", L->planes, D);
  if (L->atlas_w < 1 || L->atlas_h < 1 || (int64_t)L->atlas_w * L->atlas_h >= (int64_t)1 << 31)
    return fail(PUV_E_INVALID_CONFIG, "atlas %d x %d", L->atlas_w, L->atlas_h);
  if (L->position_mode != PUV_POS_XYZ && L->position_mode != PUV_POS_RHO)
    return fail(PUV_E_INVALID_CONFIG, "position_mode %d", L->position_mode);
  for (int k = 0; k < L->num_levels; ++k) {
    const puv_placement& a = L->level[k];
    if (a.rows < 1 || a.cols < 1) return fail(PUV_E_INVALID_CONFIG, "level %d is empty", k);
    const int w = a.rot90ccw ? a.rows : a.cols, h = a.rot90ccw ? a.cols : a.rows;
    if (a.x < 0 || a.y < 0 || a.x + w > L->atlas_w || a.y + h > L->atlas_h)
      return fail(PUV_E_LAYOUT_OVERFLOW, "level %d (%dx%d at %d,%d) leaves the %dx%d atlas", k, h, w, a.x, a.y,
                  L->atlas_w, L->atlas_h);
    for (int j = 0; j < k; ++j) {
      const puv_placement& b = L->level[j];
      const int wb = b.rot90ccw ? b.rows : b.cols, hb = b.rot90ccw ? b.cols : b.rows;
      if (a.x < b.x + wb && b.x < a.x + w && a.y < b.y + hb && b.y < a.y + h)
        return fail(PUV_E_LAYOUT_OVERFLOW, "levels %d and %d overlap", j, k);
    }
  }
  return PUV_OK;
}

static puv_status check_cameras(int n, const puv_camera* cams, int& W, int& H) {
  if (n < 1) return fail(PUV_E_INVALID_ARGUMENT, "n_views %d < 1", n);
  if (!cams) return fail(PUV_E_INVALID_ARGUMENT, "cams is NULL");
  W = cams[0].width;
  H = cams[0].height;
  for (int i = 0; i < n; ++i) {
    const puv_camera& c = cams[i];
    if (!(c.fx > 0.f) || !(c.fy > 0.f) || c.width < 1 || c.height < 1 || !(c.near_plane > 0.f))
      return fail(PUV_E_INVALID_CAMERA, "camera %d: fx, fy, near must be > 0 and the image non-empty", i);
    if (c.width != W || c.height != H)
      return fail(PUV_E_DIMENSION_MISMATCH, "camera %d: %dx%d differs from camera 0 (%dx%d)", i, c.width, c.height, W, H);
    if ((int64_t)W * H >= (int64_t)1 << 30 || (W + kTile - 1) / kTile > 2048 || (H + kTile - 1) / kTile > 65535)
      return fail(PUV_E_UNSUPPORTED, "camera %d: image %dx%d too large", i, W, H);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double dot = 0;
        for (int k = 0; k < 3; ++k) dot += (double)c.viewmat[4 * a + k] * c.viewmat[4 * b + k];
        if (std::fabs(dot - (a == b ? 1.0 : 0.0)) > 1e-5)
          return fail(PUV_E_INVALID_CAMERA, "camera %d: rotation not orthonormal within 1e-5", i);
      }
    if (c.viewmat[12] != 0.f || c.viewmat[13] != 0.f || c.viewmat[14] != 0.f || c.viewmat[15] != 1.f)
      return fail(PUV_E_INVALID_CAMERA, "camera %d: last row of viewmat must be (0,0,0,1)", i);
  }
  return PUV_OK;
}

static CamDev cam_dev(const puv_camera& c) {
  CamDev d;
  for (int k = 0; k < 12; ++k) d.V[k] = c.viewmat[k];
  d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy;
  d.W = c.width; d.H = c.height;
  d.near_plane = c.near_plane;
  for (int k = 0; k < 3; ++k) d.campos[k] = c.campos[k];
  // R5: lim = 1.3 * tan(fov/2) = 1.3 * 0.5 * W / fx in fp64, rounded to fp32
  d.limx = (float)(1.3 * 0.5 * (double)c.width / (double)c.fx);
  d.limy = (float)(1.3 * 0.5 * (double)c.height / (double)c.fy);
  for (int k = 0; k < 12; ++k) d.V64[k] = d.V[k];
  d.fx64 = d.fx; d.fy64 = d.fy; d.cx64 = d.cx; d.cy64 = d.cy;
  d.limx64 = d.limx; d.limy64 = d.limy;
  for (int k = 0; k < 3; ++k) d.campos64[k] = d.campos[k];
  return d;
}

Plan make_plan(const puv_layout& L, int n_views, int W, int H) {
  Plan p{};
  p.n_views = n_views;
  p.N = L.atlas_w * L.atlas_h;
  p.W = W; p.H = H; p.HW = W * H;
  p.gx = (W + kTile - 1) / kTile;
  p.gy = (H + kTile - 1) / kTile;
  p.ntiles = p.gx * p.gy;
  p.D = L.planes;
  p.deg = L.sh_degree;
  p.pm.rho = L.position_mode == PUV_POS_RHO;
  p.pm.D = L.planes;
  for (int k = 0; k < 3; ++k) p.pm.c[k] = L.center[k];
  const size_t V = n_views, N = p.N;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += align_up(bytes); return o; };
  p.call_hdr = take(sizeof(CallHdr));
  p.view_hdr = take(sizeof(ViewHdr) * V);
  p.depth = take(4 * V * N);
  p.rect = take(8 * V * N);
  p.rec = take(32 * V * N);
  p.rec64 = take(80 * V * N);
  p.grad2d = take(72 * V * N);
  p.sorted = take(4 * V * N);
  p.tstart = take(4 * V * p.ntiles);
  p.tend = take(4 * V * p.ntiles);
  p.tfinal = take(4 * V * p.HW);
  p.ncontrib = take(4 * V * p.HW);
  p.cfull = take(24 * V * p.HW);
  p.dmask = take(32 * V * (size_t)p.ntiles * (size_t)(kMaskCap > 0 ? kMaskCap : 1));
  p.sgx = (p.gx + kSup - 1) / kSup;
  p.nst = p.sgx * ((p.gy + kSup - 1) / kSup);
  p.sst = take(4 * V * (size_t)(p.nst + 1));
  p.sen = take(4 * V * (size_t)(p.nst + 1));
  p.l1hdr = take(sizeof(ViewHdr) * V);
  p.sort_blocks = (N + 2047) / 2048;
  // binning scratch: one block per binning stream; offsets below are relative to a block
  size_t soff = 0;
  auto stake = [&](size_t bytes) { const size_t o = soff; soff += align_up(bytes); return o; };
  p.sk0 = stake(4 * N * kSortGroup);   // onesweep ping-pong of a sort group of views
  p.sv0 = stake(4 * N * kSortGroup);
  p.sk1 = stake(4 * N * kSortGroup);
  p.sv1 = stake(4 * N * kSortGroup);
  p.hist = stake(depth_sort_scratch_bytes(N) * kSortGroup);
  p.koff = stake(4 * (N + 1));
  p.bsum = stake(4 * (N / 2048 + 2));
  p.cnt = stake(4 * (size_t)kNbMax * p.ntiles);
  p.bstart = stake(4 * (size_t)(kNbMax + 1));
  p.bin2 = stake(bin_scratch_bytes(N, p.ntiles));
  p.nscratch = n_views < kBinStreams ? n_views : kBinStreams;
  p.scratch_stride = soff;
  p.scratch0 = take(soff * p.nscratch);
  p.total = off;
  return p;
}

Views views_of(const Plan& p, void* state) {
  char* s = (char*)state;
  Views v;
  v.depth = (uint32_t*)(s + p.depth);
  v.rect = (uint2*)(s + p.rect);
  v.rec = (float4*)(s + p.rec);
  v.rec64 = (double2*)(s + p.rec64);
  v.grad2d = (double*)(s + p.grad2d);
  v.sorted = (uint32_t*)(s + p.sorted);
  v.tstart = (uint32_t*)(s + p.tstart);
  v.tend = (uint32_t*)(s + p.tend);
  v.tfinal = (float*)(s + p.tfinal);
  v.ncontrib = (uint32_t*)(s + p.ncontrib);
  v.cfull = (double*)(s + p.cfull);
  v.dmask = (uint32_t*)(s + p.dmask);
  v.sst = (uint32_t*)(s + p.sst);
  v.sen = (uint32_t*)(s + p.sen);
  v.l1 = (ViewHdr*)(s + p.l1hdr);
  v.sgx = p.sgx;
  v.nst = p.nst;
  v.hdr = (ViewHdr*)(s + p.view_hdr);
  v.call = (CallHdr*)(s + p.call_hdr);
  return v;
}

struct Common {
  Plan plan;
  Views views;
  PlaneTab P;
  int W, H;
};

// Plane table of a render/backward/label call: D entries, + the 3 ray planes in PUV_POS_RHO mode
// (where entries 1 and 2 are unused and may be NULL).
static puv_status fill_planes(const puv_layout* L, const float* const* tab, PlaneTab& P) {
  if (!tab) return fail(PUV_E_INVALID_ARGUMENT, "atlas_planes is NULL");
  const bool rho = L->position_mode == PUV_POS_RHO;
  const int n = L->planes + (rho ? 3 : 0);
  P.qspec = nullptr;
  for (int d = 0; d < kMaxPlanes; ++d) P.qbits[d] = 0;
  for (int d = 0; d < n; ++d) {
    if (rho && (d == 1 || d == 2)) { P.p[d] = nullptr; continue; }
    if (!tab[d]) return fail(PUV_E_INVALID_ARGUMENT, "atlas plane %d is NULL", d);
    P.p[d] = tab[d];
  }
  return PUV_OK;
}

static puv_status prepare(const puv_layout* L, const float* const* atlas_planes, int32_t n_views,
                          const puv_camera* cams, const puv_render_opts* opts, void* state, size_t state_bytes,
                          Common& c) {
  puv_status st = check_layout(L);
  if (st) return st;
  st = fill_planes(L, atlas_planes, c.P);
  if (st) return st;
  if (opts && opts->flags != 0) {
    if (opts->flags != PUV_RENDER_LPO) return fail(PUV_E_UNSUPPORTED, "opts.flags %u: only PUV_RENDER_LPO", opts->flags);
    const int pb = opts->lpo_pos_bits, ab = opts->lpo_attr_bits;
    if (!opts->lpo_spec) return fail(PUV_E_INVALID_ARGUMENT, "PUV_RENDER_LPO without lpo_spec");
    if ((pb != PUV_QUANT_FP16 && (pb < 1 || pb > 16)) || ab < 1 || ab > 16)
      return fail(PUV_E_INVALID_ARGUMENT, "LPO bits (%d, %d) outside 1..16 (pos: or PUV_QUANT_FP16)", pb, ab);
    c.P.qspec = opts->lpo_spec;
    const bool rho = L->position_mode == PUV_POS_RHO;
    for (int d = 0; d < L->planes; ++d) {
      if (rho && (d == 1 || d == 2)) continue;   // unused planes; the ray planes are never quantised
      c.P.qbits[d] = (int8_t)(d < 3 ? (pb == PUV_QUANT_FP16 ? -1 : pb) : ab);
    }
  }
  st = check_cameras(n_views, cams, c.W, c.H);
  if (st) return st;
  if (!state) return fail(PUV_E_INVALID_ARGUMENT, "state is NULL");
  c.plan = make_plan(*L, n_views, c.W, c.H);
  if (state_bytes < c.plan.total)
    return fail(PUV_E_WORKSPACE_TOO_SMALL, "state_bytes %zu < %zu", state_bytes, c.plan.total);
  c.views = views_of(c.plan, state);
  return PUV_OK;
}

}  // namespace puv

using namespace puv;

extern "C" {

puv_status puv_layout_for_levels(int32_t K, const int32_t* rows, const int32_t* cols, int32_t sh_degree,
                                 puv_layout* out) {
  if (!rows || !cols || !out) return fail(PUV_E_INVALID_ARGUMENT, "NULL argument");
  if (K < 1 || K > PUV_MAX_LEVELS) return fail(PUV_E_INVALID_CONFIG, "K %d outside 1..%d", K, PUV_MAX_LEVELS);
  if (sh_degree < 0 || sh_degree > PUV_MAX_SH_DEGREE) return fail(PUV_E_INVALID_CONFIG, "sh_degree %d", sh_degree);
  puv_layout L;
  std::memset(&L, 0, sizeof L);
  L.num_levels = K;
  L.sh_degree = sh_degree;
  L.planes = 11 + 3 * (sh_degree + 1) * (sh_degree + 1);
  int64_t y = 0, colw = 0;
  for (int k = 0; k < K; ++k) {
    if (rows[k] < 1 || cols[k] < 1) return fail(PUV_E_INVALID_CONFIG, "level %d is empty", k);
    L.level[k].rows = rows[k];
    L.level[k].cols = cols[k];
    L.level[k].rot90ccw = 0;
    if (k == 0) { L.level[k].x = 0; L.level[k].y = 0; continue; }
    L.level[k].x = cols[0];
    L.level[k].y = (int32_t)y;
    y += rows[k];
    if (cols[k] > colw) colw = cols[k];
  }
  const int64_t W = (int64_t)cols[0] + colw, H = rows[0] > y ? rows[0] : y;
  if (W * H >= (int64_t)1 << 31) return fail(PUV_E_LAYOUT_OVERFLOW, "atlas %lld x %lld too large", (long long)W,
                                               (long long)H);
  L.atlas_w = (int32_t)W;
  L.atlas_h = (int32_t)H;
  *out = L;
  return PUV_OK;
}

puv_status puv_layout_paper(int32_t S, int32_t K, int32_t sh_degree, puv_layout* out) {
  if (!out) return fail(PUV_E_INVALID_ARGUMENT, "NULL output");
  if (K < 1 || K > 8) return fail(PUV_E_INVALID_CONFIG, "K %d outside 1..8", K);
  if (S < 16 || (S & (S - 1))) return fail(PUV_E_INVALID_CONFIG, "S %d must be a power of two >= 16", S);
  if (sh_degree < 0 || sh_degree > PUV_MAX_SH_DEGREE) return fail(PUV_E_INVALID_CONFIG, "sh_degree %d", sh_degree);
  puv_layout L;
  std::memset(&L, 0, sizeof L);
  L.num_levels = K;
  L.sh_degree = sh_degree;
  L.planes = 11 + 3 * (sh_degree + 1) * (sh_degree + 1);
  // schedule: (M_k, N_k) = (M, N/2) for odd k, (M/2, N) for even k; level = N rows x M cols
  int M = S, Nn = S;
  int px = 0, py = 0, pw = 0, ph = 0;   // previous placement (x, y, width, height)
  for (int k = 0; k < K; ++k) {
    if (k > 0) { if (k & 1) Nn /= 2; else M /= 2; }
    puv_placement& a = L.level[k];
    a.rows = Nn;
    a.cols = M;
    a.rot90ccw = k & 1;
    const int w = a.rot90ccw ? a.rows : a.cols, h = a.rot90ccw ? a.cols : a.rows;
    if (k == 0) { a.x = K > 1 ? S / 2 : 0; a.y = 0; }
    else if (k == 1) { a.x = 0; a.y = 0; }
    else if (k == 2) { a.x = 0; a.y = S; }
    else if (k == 3 || k == 4 || k == 6) { a.x = px + pw; a.y = py; }      // right of the previous level
    else { a.x = px; a.y = py + ph; }                                      // k = 5, 7: below the previous
    px = a.x; py = a.y; pw = w; ph = h;
  }
  L.atlas_w = K > 1 ? S + S / 2 : S;
  L.atlas_h = K > 2 ? S + S / 2 : S;
  const puv_status st = check_layout(&L);
  if (st) return st;
  *out = L;
  return PUV_OK;
}

puv_status puv_ray_planes(const puv_layout* layout, float* const* ray_planes, void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!ray_planes || !ray_planes[0] || !ray_planes[1] || !ray_planes[2])
    return fail(PUV_E_INVALID_ARGUMENT, "NULL ray plane");
  const size_t NA = (size_t)layout->atlas_w * layout->atlas_h;
  std::vector<float> host(3 * NA, 0.0f);
  const double kPi = 3.14159265358979323846;
  for (int k = 0; k < layout->num_levels; ++k) {
    const puv_placement& a = layout->level[k];
    for (int r = 0; r < a.rows; ++r)
      for (int c = 0; c < a.cols; ++c) {
        // level image: u = column (azimuth, M_k = cols), v = row (polar, N_k = rows); pixel centres
        const double theta = (c + 0.5) / a.cols * 2.0 * kPi - kPi, phi = (r + 0.5) / a.rows * kPi;
        const size_t ay = a.rot90ccw ? (size_t)(a.y + a.cols - 1 - c) : (size_t)(a.y + r);
        const size_t ax = a.rot90ccw ? (size_t)(a.x + r) : (size_t)(a.x + c);
        const size_t o = ay * layout->atlas_w + ax;
        host[o] = (float)(std::sin(phi) * std::cos(theta));
        host[NA + o] = (float)(std::sin(phi) * std::sin(theta));
        host[2 * NA + o] = (float)std::cos(phi);
      }
  }
  cudaStream_t s = (cudaStream_t)stream;
  for (int d = 0; d < 3; ++d) cudaMemcpyAsync(ray_planes[d], host.data() + d * NA, NA * 4, cudaMemcpyHostToDevice, s);
  const cudaError_t e = cudaStreamSynchronize(s);   // host staging buffer must outlive the copies
  if (e != cudaSuccess) return fail(PUV_E_CUDA, "puv_ray_planes: %s", cudaGetErrorString(e));
  return PUV_OK;
}

puv_status puv_pack_atlas(const puv_layout* layout, const float* const* level_planes, const uint8_t* const* level_occ,
                          float* const* atlas_planes, uint8_t* atlas_occ, void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!level_planes || !atlas_planes || !atlas_occ) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer table");
  for (int i = 0; i < layout->num_levels * layout->planes; ++i)
    if (!level_planes[i]) return fail(PUV_E_INVALID_ARGUMENT, "level plane %d is NULL", i);
  for (int d = 0; d < layout->planes; ++d)
    if (!atlas_planes[d]) return fail(PUV_E_INVALID_ARGUMENT, "atlas plane %d is NULL", d);
  { StageScope sc(PUV_STAGE_PACK, (cudaStream_t)stream);
    launch_pack(*layout, level_planes, level_occ, atlas_planes, atlas_occ, (cudaStream_t)stream); }
  return cuda_check("puv_pack_atlas");
}

puv_status puv_unpack_levels(const puv_layout* layout, const float* const* atlas_planes, float* const* level_planes,
                             void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!level_planes || !atlas_planes) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer table");
  { StageScope sc(PUV_STAGE_PACK, (cudaStream_t)stream);
    launch_unpack(*layout, atlas_planes, level_planes, (cudaStream_t)stream); }
  return cuda_check("puv_unpack_levels");
}

puv_status puv_query_sizes(const puv_layout* layout, int32_t n_views, const puv_camera* cams,
                           const puv_render_opts* opts, size_t* state_bytes, size_t* arena_hint) {
  puv_status st = check_layout(layout);
  if (st) return st;
  int W, H;
  st = check_cameras(n_views, cams, W, H);
  if (st) return st;
  if (!state_bytes || !arena_hint) return fail(PUV_E_INVALID_ARGUMENT, "NULL output");
  const Plan p = make_plan(*layout, n_views, W, H);
  *state_bytes = p.total;
  // first guess: 48 keys per Gaussian per view (C3 measures ~37-43)
  *arena_hint = (size_t)4 * 48 * (size_t)p.N * n_views;
  return PUV_OK;
}

// Per-view work the fused L2 step (puv_render_l2_step) attaches to the render pipeline: the loss
// gradient and the composite backward of view v run on a second compute stream as soon as view
// v is composited, under the compositing of later views and the binning of the views after them.
struct L2Hook {
  const float* targets;
  float* dL;
  double* loss;
  cudaEvent_t targets_ready;   // nullable: the per-view losses wait for it (e.g. an H2D copy of targets)
  bool backward;               // also the per-view composite backward (the fused step); else losses only
  void* zero_ptr;              // nullable: zeroed on the second stream first (K6's moment slots)
  size_t zero_bytes;
};

// Project, bin and composite all views of a call (rows a1-a5); with `hook`, also rows a6-a7 per
// view.  `s` is ordered after everything enqueued here when the function returns.
// Host-link overlap of puv_train_step_host_atlas: the atlas arrives in texel chunks and K1 projects
// each chunk once it has landed (`ready`); the gradient leaves in texel chunks, each copied out
// as soon as K7 has finished it (`done`).
#ifndef PUV_TEXEL_CHUNKS
#define PUV_TEXEL_CHUNKS 4
#endif
constexpr int kTexelChunks = PUV_TEXEL_CHUNKS;
struct TexelPipe {
  int n;                              // chunks (<= kTexelChunks)
  int bound[kTexelChunks + 1];        // texel ranges [bound[i], bound[i+1])
  cudaEvent_t ready[kTexelChunks];    // K1 of chunk i waits for it (nullable)
  cudaEvent_t done[kTexelChunks];     // recorded after K7 of chunk i (nullable)
};

static void render_pipeline(const Common& c, const uint8_t* atlas_occ, int n_views, const puv_camera* cams,
                            const float bg[3], float* images, void* state, void* arena, size_t arena_bytes,
                            cudaStream_t s, const L2Hook* hook, const TexelPipe* tin = nullptr) {
  const Plan& p = c.plan;
  cudaMemsetAsync(c.views.hdr, 0, sizeof(ViewHdr) * n_views, s);
  launch_begin_call(p, c.views, arena_bytes / 4, s);
  StreamSet& ss = stream_set(p.nscratch);
  std::lock_guard<std::mutex> lock(ss.mu);
  // K1 head split: project the first kK1Head views first (one more pass over the atlas) so their
  // binning starts while K1 of the other views runs on its own stream; those views' binning waits
  // for that K1 (k1tail).  Device-resident atlas only (the texel-chunk host path keeps one K1).
  const bool head_split = kK1Head > 0 && !tin && n_views > kK1Head && n_views <= kCamBatch;
  if (head_split) {
    cudaEventRecord(ss.k1fork, s);
    CamBatch ch;
    ch.v0 = 0;
    ch.n = kK1Head;
    for (int i = 0; i < ch.n; ++i) ch.c[i] = cam_dev(cams[i]);
    { StageScope sc(PUV_STAGE_PROJECT, s); launch_project(p, c.views, c.P, atlas_occ, ch, s); }
    cudaStreamWaitEvent(ss.k1, ss.k1fork, 0);
    CamBatch ct;
    ct.v0 = kK1Head;
    ct.n = n_views - kK1Head;
    for (int i = 0; i < ct.n; ++i) ct.c[i] = cam_dev(cams[kK1Head + i]);
    { StageScope sc(PUV_STAGE_PROJECT, ss.k1); launch_project(p, c.views, c.P, atlas_occ, ct, ss.k1); }
    cudaEventRecord(ss.k1tail, ss.k1);
  }
  for (int v0 = 0; v0 < n_views && !head_split; v0 += kCamBatch) {
    CamBatch cb;
    cb.v0 = v0;
    cb.n = n_views - v0 < kCamBatch ? n_views - v0 : kCamBatch;
    for (int i = 0; i < cb.n; ++i) cb.c[i] = cam_dev(cams[v0 + i]);
    StageScope sc(PUV_STAGE_PROJECT, s);
    if (tin) {
      for (int i = 0; i < tin->n; ++i) {
        if (tin->ready[i]) cudaStreamWaitEvent(s, tin->ready[i], 0);
        launch_project(p, c.views, c.P, atlas_occ, cb, s, tin->bound[i], tin->bound[i + 1]);
      }
    } else {
      launch_project(p, c.views, c.P, atlas_occ, cb, s);
    }
  }
  // Pipeline: view v is depth-sorted and binned on binning stream v % nscratch (its own scratch
  // block) while earlier views composite on `s`; `s` waits on view v's binning event only.
  cudaEventRecord(ss.fork, s);
  for (int i = 0; i < p.nscratch; ++i) cudaStreamWaitEvent(ss.s[i], ss.fork, 0);
  if (hook) {
    cudaStreamWaitEvent(ss.s2, ss.fork, 0);
    // HBM-bound zeroing beside the compute-bound compositing instead of in front of the backward
    if (hook->zero_bytes) cudaMemsetAsync(hook->zero_ptr, 0, hook->zero_bytes, ss.s2);
    if (hook->targets_ready) cudaStreamWaitEvent(ss.s2, hook->targets_ready, 0);
  }
  // Views are composited in groups of kFwdGroup consecutive views per launch (grid.y), each
  // group once all its views are binned.
  const bool serial = g_serial;
  for (int v = 0; v < n_views; ++v) {
    const int i = v % p.nscratch;
    cudaStream_t bs = serial ? s : ss.s[i];
    if (head_split && v >= kK1Head) cudaStreamWaitEvent(bs, ss.k1tail, 0);
    void* scratch = (char*)state + p.scratch0 + (size_t)i * p.scratch_stride;
    if (kSortGroup == 1) {
      { StageScope sc(PUV_STAGE_DEPTH_SORT, bs); launch_depth_sort(p, c.views, scratch, v, 1, bs); }
#ifdef PUV_SORT_TWICE   // measurement only: the marginal step cost of the depth sort's SM time
      launch_depth_sort(p, c.views, scratch, v, 1, bs);
#endif
    } else {
      // sort group gi = views [gi G, gi G + G) depth-sorted together on binning stream gi % nscratch
      // (its scratch block holds G views of onesweep scratch); each view's tile pass then runs on
      // stream v % nscratch as before, after its group's sort
      const int gi = v / kSortGroup;
      if (v % kSortGroup == 0) {
        const int si = gi % p.nscratch;
        cudaStream_t gs = serial ? s : ss.s[si];
        void* gscratch = (char*)state + p.scratch0 + (size_t)si * p.scratch_stride;
        const int nv = n_views - v < kSortGroup ? n_views - v : kSortGroup;
        { StageScope sc(PUV_STAGE_DEPTH_SORT, gs); launch_depth_sort(p, c.views, gscratch, v, nv, gs); }
        cudaEventRecord(ss.sort_event(gi), gs);
      }
      if (!serial) cudaStreamWaitEvent(bs, ss.sort_event(gi), 0);
    }
    { StageScope sc(PUV_STAGE_BIN, bs); launch_bin(p, c.views, scratch, (uint32_t*)arena, v, bs, !kDirect); }
    cudaEvent_t done = ss.view_event(v);
    cudaEventRecord(done, bs);
    cudaStreamWaitEvent(s, done, 0);
    const int g0 = v - v % kFwdGroup;
    if (v == n_views - 1 || (v + 1) % kFwdGroup == 0) {
      {
        StageScope sc(PUV_STAGE_RASTER_FWD, s);
        launch_raster_fwd(p, c.views, (const uint32_t*)arena, images + (size_t)g0 * 3 * p.HW, g0, v + 1 - g0, bg, s);
      }
      if (hook) {
        cudaEvent_t fdone = ss.fwd_event(v);
        cudaEventRecord(fdone, s);
        cudaStreamWaitEvent(ss.s2, fdone, 0);
        const size_t off = (size_t)g0 * 3 * p.HW, n = (size_t)(v + 1 - g0) * 3 * p.HW;
        { StageScope sc(PUV_STAGE_LOSS, ss.s2);
          launch_l2_loss((int64_t)n, images + off, hook->targets + off, hook->dL + off, hook->loss, ss.s2, true); }
        if (hook->backward) {
          StageScope sc(PUV_STAGE_RASTER_BWD, ss.s2);
          launch_raster_bwd(p, c.views, (const uint32_t*)arena, hook->dL + off, g0, v + 1 - g0, ss.s2);
        }
      }
    }
  }
  if (hook) {
    cudaEventRecord(ss.join, ss.s2);
    cudaStreamWaitEvent(s, ss.join, 0);
  }
}

puv_status puv_render_views(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                            int32_t n_views, const puv_camera* cams, const puv_render_opts* opts, float* images,
                            void* state, size_t state_bytes, void* arena, size_t arena_bytes, void* stream) {
  Common c;
  puv_status st = prepare(layout, atlas_planes, n_views, cams, opts, state, state_bytes, c);
  if (st) return st;
  if (!images) return fail(PUV_E_INVALID_ARGUMENT, "images is NULL");
  if (!arena && arena_bytes) return fail(PUV_E_INVALID_ARGUMENT, "arena is NULL");
  const float bg[3] = {opts ? opts->bg[0] : 0.f, opts ? opts->bg[1] : 0.f, opts ? opts->bg[2] : 0.f};
  render_pipeline(c, atlas_occ, n_views, cams, bg, images, state, arena, arena_bytes, (cudaStream_t)stream, nullptr);
  return cuda_check("puv_render_views");
}

puv_status puv_l2_loss_grad(int64_t n, const float* images, const float* targets, float* dL_dimages, double* loss,
                            void* stream) {
  if (n < 0 || (n > 0 && (!images || !targets || !dL_dimages)) || !loss)
    return fail(PUV_E_INVALID_ARGUMENT, "bad loss arguments");
  { StageScope sc(PUV_STAGE_LOSS, (cudaStream_t)stream);
    launch_l2_loss(n, images, targets, dL_dimages, loss, (cudaStream_t)stream, false); }
  return cuda_check("puv_l2_loss_grad");
}

puv_status puv_quant_fit(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                         float* spec, void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!atlas_planes || !spec) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer");
  const bool rho = layout->position_mode == PUV_POS_RHO;
  PlaneTab P{};
  for (int d = 0; d < layout->planes; ++d) {
    if (rho && (d == 1 || d == 2)) continue;
    if (!atlas_planes[d]) return fail(PUV_E_INVALID_ARGUMENT, "atlas plane %d is NULL", d);
    P.p[d] = atlas_planes[d];
  }
  { StageScope sc(PUV_STAGE_QUANT, (cudaStream_t)stream);
    puv::launch_quant_fit(P, layout->planes, atlas_occ, (int64_t)layout->atlas_w * layout->atlas_h, spec,
                          (cudaStream_t)stream); }
  return cuda_check("puv_quant_fit");
}

puv_status puv_quantize(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                        const float* spec, int32_t pos_bits, int32_t attr_bits, void* const* codes,
                        float* const* proxy, void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!atlas_planes || !spec) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer");
  if ((pos_bits != PUV_QUANT_FP16 && (pos_bits < 1 || pos_bits > 16)) || attr_bits < 1 || attr_bits > 16)
    return fail(PUV_E_INVALID_ARGUMENT, "bits (%d, %d) outside 1..16 (pos: or PUV_QUANT_FP16)", pos_bits, attr_bits);
  if (!codes && !proxy) return fail(PUV_E_INVALID_ARGUMENT, "codes and proxy are both NULL");
  const bool rho = layout->position_mode == PUV_POS_RHO;
  const int D = layout->planes;
  const float* x[kMaxPlanes] = {};
  int8_t bits[kMaxPlanes] = {};
  for (int d = 0; d < D; ++d) {
    if (rho && (d == 1 || d == 2)) continue;
    if (!atlas_planes[d]) return fail(PUV_E_INVALID_ARGUMENT, "atlas plane %d is NULL", d);
    if (codes && !codes[d]) return fail(PUV_E_INVALID_ARGUMENT, "code plane %d is NULL", d);
    if (proxy && !proxy[d]) return fail(PUV_E_INVALID_ARGUMENT, "proxy plane %d is NULL", d);
    x[d] = atlas_planes[d];
    bits[d] = (int8_t)((d < 3) ? (pos_bits == PUV_QUANT_FP16 ? -1 : pos_bits) : attr_bits);
  }
  { StageScope sc(PUV_STAGE_QUANT, (cudaStream_t)stream);
    puv::launch_quantize(x, proxy, codes, bits, D, spec, atlas_occ, (int64_t)layout->atlas_w * layout->atlas_h,
                         (cudaStream_t)stream); }
  return cuda_check("puv_quantize");
}

size_t puv_photo_workspace_bytes(int32_t width, int32_t height, int32_t views_per_chunk) {
  if (width < 1 || height < 1 || views_per_chunk < 1) return 0;
  return (size_t)views_per_chunk * puv::photo_view_bytes(width, height);
}

puv_status puv_photo_loss_grad(int32_t n_views, int32_t width, int32_t height, const float* images,
                               const float* targets, double lambda_ssim, float* dL_dimages, double* loss,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (n_views < 1 || width < 1 || height < 1) return fail(PUV_E_INVALID_ARGUMENT, "bad sizes %d x %d x %d",
                                                          n_views, width, height);
  if ((int64_t)width * height > ((int64_t)1 << 28)) return fail(PUV_E_UNSUPPORTED, "image too large");
  if (!images || !targets || !dL_dimages || !loss || !workspace) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer");
  if (!(lambda_ssim >= 0.0 && lambda_ssim <= 1.0)) return fail(PUV_E_INVALID_ARGUMENT, "lambda_ssim outside [0, 1]");
  const size_t per = puv::photo_view_bytes(width, height);
  if (workspace_bytes < per)
    return fail(PUV_E_WORKSPACE_TOO_SMALL, "workspace_bytes %zu < %zu (one view)", workspace_bytes, per);
  const int chunk = (int)std::min<size_t>((size_t)n_views, workspace_bytes / per);
  { StageScope sc(PUV_STAGE_OBJECTIVE, (cudaStream_t)stream);
    puv::launch_photo_loss(n_views, width, height, images, targets, lambda_ssim, dL_dimages, loss, workspace, chunk,
                           (cudaStream_t)stream); }
  return cuda_check("puv_photo_loss_grad");
}

size_t puv_reg_workspace_bytes(void) { return puv::reg_workspace_bytes(); }

puv_status puv_reg_loss_grad(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                             const uint8_t* dynamic_mask, double lambda_scale, double lambda_opacity, double s_max,
                             float* const* atlas_grad, double* loss, void* workspace, size_t workspace_bytes,
                             void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!atlas_planes || !atlas_grad || !loss || !workspace) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer");
  if (workspace_bytes < puv::reg_workspace_bytes())
    return fail(PUV_E_WORKSPACE_TOO_SMALL, "workspace_bytes %zu < %zu", workspace_bytes, puv::reg_workspace_bytes());
  PlaneTab P{};
  GradTab G{};
  for (int d : {3, 4, 5, 10}) {
    if (!atlas_planes[d] || !atlas_grad[d]) return fail(PUV_E_INVALID_ARGUMENT, "plane %d is NULL", d);
    P.p[d] = atlas_planes[d];
    G.p[d] = atlas_grad[d];
  }
  const int64_t N = (int64_t)layout->atlas_w * layout->atlas_h;
  { StageScope sc(PUV_STAGE_OBJECTIVE, (cudaStream_t)stream);
    puv::launch_reg_loss(P, atlas_occ, dynamic_mask, N, lambda_scale, lambda_opacity, s_max, G, loss, workspace,
                         (cudaStream_t)stream); }
  return cuda_check("puv_reg_loss_grad");
}

static puv_status grad_table(const puv_layout* layout, float* const* atlas_grad, GradTab& G) {
  if (!atlas_grad) return fail(PUV_E_INVALID_ARGUMENT, "atlas_grad is NULL");
  for (int d = 0; d < layout->planes; ++d) {
    if (layout->position_mode == PUV_POS_RHO && (d == 1 || d == 2)) { G.p[d] = nullptr; continue; }
    if (!atlas_grad[d]) return fail(PUV_E_INVALID_ARGUMENT, "grad plane %d is NULL", d);
    G.p[d] = atlas_grad[d];
  }
  return PUV_OK;
}

// K7 over all views of the call, in camera batches (rows a8, a9)
static void project_backward(const Common& c, const uint8_t* atlas_occ, int n_views, const puv_camera* cams,
                             const uint8_t* dynamic_mask, const GradTab& G, cudaStream_t s,
                             const TexelPipe* tout = nullptr, bool overwrite = false) {
  const int nchunk = tout ? tout->n : 1;
  for (int k = 0; k < nchunk; ++k) {
    const int g0 = tout ? tout->bound[k] : 0, g1 = tout ? tout->bound[k + 1] : -1;
    for (int v0 = 0; v0 < n_views; v0 += kCamBatch) {
      CamBatch cb;
      cb.v0 = v0;
      cb.n = n_views - v0 < kCamBatch ? n_views - v0 : kCamBatch;
      for (int i = 0; i < cb.n; ++i) cb.c[i] = cam_dev(cams[v0 + i]);
      StageScope sc(PUV_STAGE_PROJECT_BWD, s);
      // with `overwrite`, the first camera batch writes every texel of the range, the later ones add
      launch_project_bwd(c.plan, c.views, c.P, atlas_occ, dynamic_mask, cb, G, s, g0, g1, overwrite && v0 == 0);
    }
    if (tout && tout->done[k]) cudaEventRecord(tout->done[k], s);
  }
}

puv_status puv_render_backward(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                               int32_t n_views, const puv_camera* cams, const puv_render_opts* opts,
                               const float* dL_dimages, const uint8_t* dynamic_mask, void* state, size_t state_bytes,
                               void* arena, size_t arena_bytes, float* const* atlas_grad, void* stream) {
  Common c;
  puv_status st = prepare(layout, atlas_planes, n_views, cams, opts, state, state_bytes, c);
  if (st) return st;
  if (!dL_dimages) return fail(PUV_E_INVALID_ARGUMENT, "dL_dimages is NULL");
  GradTab G;
  if ((st = grad_table(layout, atlas_grad, G))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  // the (view, Gaussian) moment slots K6 accumulates into start at zero on every backward call,
  // so backward can be called repeatedly on one forward state (each call adds its gradient once)
  cudaMemsetAsync(c.views.grad2d, 0, (size_t)72 * n_views * c.plan.N, s);
  // all views in one launch (grid = tiles x views): no per-view tail; the background enters
  // through the forward's full colour C
  { StageScope sc(PUV_STAGE_RASTER_BWD, s);
    launch_raster_bwd(c.plan, c.views, (const uint32_t*)arena, dL_dimages, 0, n_views, s); }
  project_backward(c, atlas_occ, n_views, cams, dynamic_mask, G, s);
  return cuda_check("puv_render_backward");
}

puv_status puv_render_l2_step(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                              int32_t n_views, const puv_camera* cams, const puv_render_opts* opts, float* images,
                              const float* targets, float* dL_dimages, double* loss, const uint8_t* dynamic_mask,
                              void* state, size_t state_bytes, void* arena, size_t arena_bytes,
                              float* const* atlas_grad, void* targets_ready, void* stream) {
  Common c;
  puv_status st = prepare(layout, atlas_planes, n_views, cams, opts, state, state_bytes, c);
  if (st) return st;
  if (!images || !targets || !dL_dimages || !loss)
    return fail(PUV_E_INVALID_ARGUMENT, "NULL images / targets / dL_dimages / loss");
  if (!arena && arena_bytes) return fail(PUV_E_INVALID_ARGUMENT, "arena is NULL");
  GradTab G;
  if ((st = grad_table(layout, atlas_grad, G))) return st;
  const float bg[3] = {opts ? opts->bg[0] : 0.f, opts ? opts->bg[1] : 0.f, opts ? opts->bg[2] : 0.f};
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(loss, 0, sizeof(double), s);
  cudaMemsetAsync(c.views.grad2d, 0, (size_t)72 * n_views * c.plan.N, s);   // K6's moment slots
  const L2Hook hook{targets, dL_dimages, loss, (cudaEvent_t)targets_ready, true, nullptr, 0};
  render_pipeline(c, atlas_occ, n_views, cams, bg, images, state, arena, arena_bytes, s, &hook);
  project_backward(c, atlas_occ, n_views, cams, dynamic_mask, G, s);
  return cuda_check("puv_render_l2_step");
}

// One training step in chunks of views (rows a1-a9): per chunk render, L2 loss gradient (the
// loss accumulates over chunks), composite backward and projection backward into atlas_grad.
static puv_status train_step_enqueue(const puv_layout* layout, const float* const* atlas_planes,
                                     const uint8_t* atlas_occ, int32_t n_views, const puv_camera* cams,
                                     const puv_render_opts* opts, const float* targets, const uint8_t* dynamic_mask,
                                     int32_t views_per_call, const puv_step_buffers* b, float* const* atlas_grad,
                                     cudaEvent_t targets_ready, cudaStream_t s, bool validate_only = false,
                                     const TexelPipe* tin = nullptr, const TexelPipe* tout = nullptr) {
  if (!b) return fail(PUV_E_INVALID_ARGUMENT, "buffers is NULL");
  if (!targets || !b->images || !b->dL_dimages || !b->loss || !b->overflow || !b->arena_need)
    return fail(PUV_E_INVALID_ARGUMENT, "NULL targets / images / dL_dimages / loss / overflow / arena_need");
  if (!b->arena && b->arena_bytes) return fail(PUV_E_INVALID_ARGUMENT, "arena is NULL");
  const int chunk = (views_per_call <= 0 || views_per_call > n_views) ? n_views : views_per_call;
  Common c;
  puv_status st = prepare(layout, atlas_planes, chunk, cams, opts, b->state, b->state_bytes, c);
  if (st) return st;
  st = check_cameras(n_views, cams, c.W, c.H);   // every camera, not only the first chunk's
  if (st) return st;
  GradTab G;
  if ((st = grad_table(layout, atlas_grad, G))) return st;
  if (validate_only) return PUV_OK;
  const float bg[3] = {opts ? opts->bg[0] : 0.f, opts ? opts->bg[1] : 0.f, opts ? opts->bg[2] : 0.f};
  const size_t NA = (size_t)layout->atlas_w * layout->atlas_h, HW3 = (size_t)3 * c.W * c.H;
  (void)NA;   // OVERWRITTEN: the first chunk's K7 writes every texel (zeros where no gradient), the rest add
  cudaMemsetAsync(b->loss, 0, sizeof(double), s);
  cudaMemsetAsync(b->overflow, 0, sizeof(uint32_t), s);
  cudaMemsetAsync(b->arena_need, 0, sizeof(uint64_t), s);
  for (int v0 = 0; v0 < n_views; v0 += chunk) {
    const int n = n_views - v0 < chunk ? n_views - v0 : chunk;
    Common cc = c;
    cc.plan = make_plan(*layout, n, c.W, c.H);   // offsets of an n-view call (fits: n <= chunk)
    cc.views = views_of(cc.plan, b->state);
    // each view's loss gradient on the second stream as soon as it is composited, and the zeroing
    // of K6's moment slots there too: both overlap the compositing of later views
    // kStepOverlap: each view's composite backward also runs on the second stream right after its
    // loss gradient (beside the compositing of later views); else one K6 launch for the chunk
    const L2Hook hook{targets + (size_t)v0 * HW3, b->dL_dimages, b->loss, v0 == 0 ? targets_ready : nullptr,
                      kStepOverlap, cc.views.grad2d, (size_t)72 * n * cc.plan.N};
    render_pipeline(cc, atlas_occ, n, cams + v0, bg, b->images, b->state, b->arena, b->arena_bytes, s, &hook,
                    v0 == 0 ? tin : nullptr);
    launch_overflow_acc(b->state, b->overflow, b->arena_need, s);
    if (!kStepOverlap) {
      StageScope sc(PUV_STAGE_RASTER_BWD, s);
      launch_raster_bwd(cc.plan, cc.views, (const uint32_t*)b->arena, b->dL_dimages, 0, n, s);
    }
    project_backward(cc, atlas_occ, n, cams + v0, dynamic_mask, G, s, v0 + n >= n_views ? tout : nullptr, v0 == 0);
  }
  return PUV_OK;
}

puv_status puv_train_step(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                          int32_t n_views, const puv_camera* cams, const puv_render_opts* opts, const float* targets,
                          const uint8_t* dynamic_mask, int32_t views_per_call, const puv_step_buffers* buffers,
                          float* const* atlas_grad, void* stream) {
  const puv_status st = train_step_enqueue(layout, atlas_planes, atlas_occ, n_views, cams, opts, targets, dynamic_mask,
                                           views_per_call, buffers, atlas_grad, nullptr, (cudaStream_t)stream);
  if (st) return st;
  return cuda_check("puv_train_step");
}

puv_status puv_train_step_host(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                               int32_t n_views, const puv_camera* cams, const puv_render_opts* opts,
                               const puv_copy* uploads, int32_t n_uploads, const float* targets_host, float* targets,
                               const uint8_t* dynamic_mask, int32_t views_per_call, const puv_step_buffers* buffers,
                               float* const* atlas_grad, const puv_copy* downloads, int32_t n_downloads,
                               void* stream) {
  if (n_uploads < 0 || n_downloads < 0 || (n_uploads && !uploads) || (n_downloads && !downloads))
    return fail(PUV_E_INVALID_ARGUMENT, "bad upload / download lists");
  for (int i = 0; i < n_uploads; ++i)
    if (uploads[i].bytes && (!uploads[i].src || !uploads[i].dst)) return fail(PUV_E_INVALID_ARGUMENT, "upload %d", i);
  for (int i = 0; i < n_downloads; ++i)
    if (downloads[i].bytes && (!downloads[i].src || !downloads[i].dst))
      return fail(PUV_E_INVALID_ARGUMENT, "download %d", i);
  if (!targets || !targets_host) return fail(PUV_E_INVALID_ARGUMENT, "NULL targets");
  int W, H;
  puv_status st = check_cameras(n_views, cams, W, H);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  // every argument is checked before anything (the uploads included) is enqueued
  st = train_step_enqueue(layout, atlas_planes, atlas_occ, n_views, cams, opts, targets, dynamic_mask, views_per_call,
                          buffers, atlas_grad, nullptr, s, true);
  if (st) return st;
  StreamSet& ss = stream_set(1);
  // this call's own events (recorded once, destroyed after use: resources are released when
  // the recorded work completes), so concurrent calls never share them
  cudaEvent_t fork = nullptr, done = nullptr;
  cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  // the uploads first, alone on the host link (K1 needs all of them); then the targets on the copy
  // stream, overlapping K1 and the render (the first loss waits for them)
  for (int i = 0; i < n_uploads; ++i)
    if (uploads[i].bytes) cudaMemcpyAsync(uploads[i].dst, uploads[i].src, uploads[i].bytes, cudaMemcpyHostToDevice, s);
  {
    std::lock_guard<std::mutex> lock(ss.mu);   // the copy stream is shared per device
    cudaEventRecord(fork, s);                  // also orders the target buffer after earlier work on `s`
    cudaStreamWaitEvent(ss.cp, fork, 0);
    cudaMemcpyAsync(targets, targets_host, (size_t)n_views * 3 * W * H * sizeof(float), cudaMemcpyHostToDevice,
                    ss.cp);
    cudaEventRecord(done, ss.cp);
  }
  st = train_step_enqueue(layout, atlas_planes, atlas_occ, n_views, cams, opts, targets, dynamic_mask, views_per_call,
                          buffers, atlas_grad, done, s);
  cudaEventDestroy(fork);
  cudaEventDestroy(done);
  if (st) return st;
  for (int i = 0; i < n_downloads; ++i)
    if (downloads[i].bytes)
      cudaMemcpyAsync(downloads[i].dst, downloads[i].src, downloads[i].bytes, cudaMemcpyDeviceToHost, s);
  return cuda_check("puv_train_step_host");
}

puv_status puv_train_step_host_atlas(const puv_layout* layout, float* const* atlas_planes, const float* atlas_host,
                                     const uint8_t* atlas_occ, int32_t n_views, const puv_camera* cams,
                                     const puv_render_opts* opts, const float* targets_host, float* targets,
                                     const uint8_t* dynamic_mask, int32_t views_per_call,
                                     const puv_step_buffers* buffers, float* const* atlas_grad, float* grad_host,
                                     double* loss_host, void* stream) {
  if (!atlas_host || !grad_host || !loss_host || !targets_host || !targets || !atlas_planes)
    return fail(PUV_E_INVALID_ARGUMENT, "NULL host / device buffer");
  int W, H;
  puv_status st = check_cameras(n_views, cams, W, H);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  st = train_step_enqueue(layout, (const float* const*)atlas_planes, atlas_occ, n_views, cams, opts, targets,
                          dynamic_mask, views_per_call, buffers, atlas_grad, nullptr, s, true);
  if (st) return st;
  const size_t N = (size_t)layout->atlas_w * layout->atlas_h;
  const int D = layout->planes;
  StreamSet& ss = stream_set(1);
  TexelPipe tin{}, tout{};
  tin.n = tout.n = kTexelChunks;
  for (int i = 0; i <= kTexelChunks; ++i) tin.bound[i] = tout.bound[i] = (int)((N * (size_t)i) / kTexelChunks);
  cudaEvent_t fork = nullptr, tdone = nullptr, gdone = nullptr;
  cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&tdone, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&gdone, cudaEventDisableTiming);
  for (int i = 0; i < kTexelChunks; ++i) {
    cudaEventCreateWithFlags(&tin.ready[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&tout.done[i], cudaEventDisableTiming);
  }
  {
    std::lock_guard<std::mutex> lock(ss.mu);   // the copy streams are shared per device
    cudaEventRecord(fork, s);                  // after earlier work on `s` (the buffers are free)
    cudaStreamWaitEvent(ss.cp, fork, 0);
    // the atlas planes in texel chunks (K1 projects a chunk as soon as it has landed), then the targets
    for (int i = 0; i < kTexelChunks; ++i) {
      const size_t g0 = tin.bound[i], n = tin.bound[i + 1] - g0;
      for (int d = 0; d < D; ++d)
        if (atlas_planes[d])
          cudaMemcpyAsync(atlas_planes[d] + g0, atlas_host + (size_t)d * N + g0, n * sizeof(float),
                          cudaMemcpyHostToDevice, ss.cp);
      cudaEventRecord(tin.ready[i], ss.cp);
    }
    cudaMemcpyAsync(targets, targets_host, (size_t)n_views * 3 * W * H * sizeof(float), cudaMemcpyHostToDevice,
                    ss.cp);
    cudaEventRecord(tdone, ss.cp);
  }
  st = train_step_enqueue(layout, (const float* const*)atlas_planes, atlas_occ, n_views, cams, opts, targets,
                          dynamic_mask, views_per_call, buffers, atlas_grad, tdone, s, false, &tin, &tout);
  if (!st) {
    std::lock_guard<std::mutex> lock(ss.mu);
    // the gradient in texel chunks as K7 finishes each, then the loss; `s` waits for all of it
    for (int i = 0; i < kTexelChunks; ++i) {
      cudaStreamWaitEvent(ss.cp2, tout.done[i], 0);
      const size_t g0 = tout.bound[i], n = tout.bound[i + 1] - g0;
      for (int d = 0; d < D; ++d)
        if (atlas_grad[d])
          cudaMemcpyAsync(grad_host + (size_t)d * N + g0, atlas_grad[d] + g0, n * sizeof(float),
                          cudaMemcpyDeviceToHost, ss.cp2);
    }
    cudaMemcpyAsync(loss_host, buffers->loss, sizeof(double), cudaMemcpyDeviceToHost, ss.cp2);
    cudaEventRecord(gdone, ss.cp2);
    cudaStreamWaitEvent(s, gdone, 0);
  }
  cudaEventDestroy(fork);
  cudaEventDestroy(tdone);
  cudaEventDestroy(gdone);
  for (int i = 0; i < kTexelChunks; ++i) {
    cudaEventDestroy(tin.ready[i]);
    cudaEventDestroy(tout.done[i]);
  }
  if (st) return st;
  return cuda_check("puv_train_step_host_atlas");
}

puv_status puv_check_overflow(const void* state, int32_t n_views, void* stream, int32_t* overflowed,
                              uint64_t* needed_arena_bytes) {
  if (!state || !overflowed || !needed_arena_bytes) return fail(PUV_E_INVALID_ARGUMENT, "NULL argument");
  CallHdr h;
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemcpyAsync(&h, state, sizeof h, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(PUV_E_CUDA, "puv_check_overflow: %s", cudaGetErrorString(e));
  *overflowed = (int32_t)h.overflow_any;
  *needed_arena_bytes = 4 * h.arena_need;
  return PUV_OK;
}

puv_status puv_overflow_accumulate(const void* state, uint32_t* flag, uint64_t* needed_arena_bytes, void* stream) {
  if (!state || !flag || !needed_arena_bytes) return fail(PUV_E_INVALID_ARGUMENT, "NULL argument");
  launch_overflow_acc(state, flag, needed_arena_bytes, (cudaStream_t)stream);
  return cuda_check("puv_overflow_accumulate");
}

puv_status puv_debug_view(const puv_layout* layout, int32_t n_views, const puv_camera* cams, void* state,
                          size_t state_bytes, void* arena, int32_t view, void* stream, puv_view_debug* out) {
  puv_status st = check_layout(layout);
  if (st) return st;
  int W, H;
  st = check_cameras(n_views, cams, W, H);
  if (st) return st;
  if (!state || !out || view < 0 || view >= n_views) return fail(PUV_E_INVALID_ARGUMENT, "bad debug arguments");
  const Plan p = make_plan(*layout, n_views, W, H);
  if (state_bytes < p.total) return fail(PUV_E_WORKSPACE_TOO_SMALL, "state too small");
  const Views v = views_of(p, state);
  ViewHdr h;
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemcpyAsync(&h, v.hdr + view, sizeof h, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(PUV_E_CUDA, "puv_debug_view: %s", cudaGetErrorString(e));
  if (kDirect && !h.overflow) {
    // the render consumed the level-1 super-tile lists directly; materialise this view's per-tile
    // lists (level 2 of the tile pass, with binning scratch block 0) for the parity / debug view
    launch_bin_level2(p, v, (char*)state + p.scratch0, (uint32_t*)arena, view, s);
    const cudaError_t e2 = cudaStreamSynchronize(s);
    if (e2 != cudaSuccess) return fail(PUV_E_CUDA, "puv_debug_view: %s", cudaGetErrorString(e2));
  }
  out->n_visible = h.n_vis;
  out->ntiles = p.ntiles;
  out->tiles_x = p.gx;
  out->tiles_y = p.gy;
  out->n_keys = h.overflow ? 0 : h.K;
  out->tile_start = v.tstart + (size_t)view * p.ntiles;
  out->tile_end = v.tend + (size_t)view * p.ntiles;
  out->keys_gid = (const uint32_t*)arena + h.list_base;
  out->depth_key = v.depth + (size_t)view * p.N;
  out->t_final = v.tfinal + (size_t)view * p.HW;
  out->n_contrib = v.ncontrib + (size_t)view * p.HW;
  out->grad2d = v.grad2d + (size_t)view * p.N * 9;
  out->depth_order = v.sorted + (size_t)view * p.N;
  out->n_examined = h.examined;
  out->n_composited = h.composited;
  return PUV_OK;
}

puv_status puv_view_counts(const void* state, int32_t view, void* stream, uint64_t* counts) {
  if (!state || !counts || view < 0) return fail(PUV_E_INVALID_ARGUMENT, "bad view_counts arguments");
  // the view headers follow the call header at the start of the state (make_plan)
  cudaStream_t s = (cudaStream_t)stream;
  CallHdr ch;
  cudaMemcpyAsync(&ch, state, sizeof ch, cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(PUV_E_CUDA, "puv_view_counts: %s", cudaGetErrorString(e));
  if ((uint32_t)view >= ch.n_views)
    return fail(PUV_E_INVALID_ARGUMENT, "view %d outside the last render's %u views", view, ch.n_views);
  const ViewHdr* vh = (const ViewHdr*)((const char*)state + align_up(sizeof(CallHdr))) + view;
  ViewHdr h;
  cudaMemcpyAsync(&h, vh, sizeof h, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(PUV_E_CUDA, "puv_view_counts: %s", cudaGetErrorString(e));
  counts[0] = h.n_vis;
  counts[1] = h.overflow ? 0 : h.K;
  counts[2] = h.examined;
  counts[3] = h.composited;
  counts[4] = h.overflow;
  return PUV_OK;
}

puv_status puv_debug_contract(int32_t op, const float* in, float* out, int64_t n, void* stream) {
  if ((op != 0 && op != 1) || n < 0 || (n > 0 && (!in || !out))) return fail(PUV_E_INVALID_ARGUMENT, "bad contract args");
  if (n) launch_contract(op, in, out, n, (cudaStream_t)stream);
  return cuda_check("puv_debug_contract");
}

size_t puv_label_workspace_bytes(int32_t width, int32_t height) {
  if (width < 1 || height < 1) return 0;
  return (size_t)4 * ((size_t)width + 1) * ((size_t)height + 1);
}

puv_status puv_label_dynamic(const puv_layout* layout, const float* const* atlas_planes, const uint8_t* atlas_occ,
                             int32_t n_cams, const puv_camera* cams, const uint8_t* masks, int32_t r_max,
                             uint8_t* labels, void* workspace, size_t workspace_bytes, void* stream) {
  puv_status st = check_layout(layout);
  if (st) return st;
  if (!masks || !labels || !workspace) return fail(PUV_E_INVALID_ARGUMENT, "NULL pointer");
  PlaneTab P;
  st = fill_planes(layout, atlas_planes, P);
  if (st) return st;
  if (r_max < 0) return fail(PUV_E_INVALID_ARGUMENT, "r_max %d < 0", r_max);
  int W, H;
  st = check_cameras(n_cams, cams, W, H);
  if (st) return st;
  if (workspace_bytes < puv_label_workspace_bytes(W, H))
    return fail(PUV_E_WORKSPACE_TOO_SMALL, "workspace_bytes %zu < %zu", workspace_bytes,
                puv_label_workspace_bytes(W, H));
  Plan p{};
  p.N = layout->atlas_w * layout->atlas_h;
  p.pm.rho = layout->position_mode == PUV_POS_RHO;
  p.pm.D = layout->planes;
  for (int k = 0; k < 3; ++k) p.pm.c[k] = layout->center[k];
  cudaStream_t s = (cudaStream_t)stream;
  StageScope sc(PUV_STAGE_LABEL, s);
  for (int c = 0; c < n_cams; ++c)
    launch_label(p, P, atlas_occ, cam_dev(cams[c]), masks + (size_t)c * W * H, (uint32_t*)workspace, r_max, c == 0,
                 labels, s);
  return cuda_check("puv_label_dynamic");
}

puv_status puv_profile_serial(int32_t on) {
  g_serial = on != 0;
  return PUV_OK;
}

puv_status puv_profile_enable(int32_t on) {
  g_prof_on = on != 0;
  return PUV_OK;
}

puv_status puv_profile_timeline(double* out, int32_t max_events, int32_t* n_events) {
  if (!out || !n_events || max_events < 0) return fail(PUV_E_INVALID_ARGUMENT, "bad timeline arguments");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int n = (int)g_prof_events.size() < max_events ? (int)g_prof_events.size() : max_events;
  for (int i = 0; i < n; ++i) {
    const ProfEvent& e = g_prof_events[i];
    const cudaError_t err = cudaEventSynchronize(e.b);
    if (err != cudaSuccess) return fail(PUV_E_CUDA, "puv_profile_timeline: %s", cudaGetErrorString(err));
    float t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t0, g_prof_events[0].a, e.a);
    cudaEventElapsedTime(&t1, g_prof_events[0].a, e.b);
    out[3 * i] = e.stage;
    out[3 * i + 1] = t0;
    out[3 * i + 2] = t1;
  }
  *n_events = n;
  return PUV_OK;
}

puv_status puv_profile_read(puv_profile* out, int32_t reset) {
  if (!out) return fail(PUV_E_INVALID_ARGUMENT, "NULL profile");
  std::memset(out, 0, sizeof *out);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (const ProfEvent& e : g_prof_events) {
    const cudaError_t err = cudaEventSynchronize(e.b);
    if (err != cudaSuccess) return fail(PUV_E_CUDA, "puv_profile_read: %s", cudaGetErrorString(err));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    out->ms[e.stage] += ms;
    out->launches[e.stage] += e.launches;
    out->calls[e.stage] += 1;
  }
  if (reset) {
    for (const ProfEvent& e : g_prof_events) { g_event_pool.push_back(e.a); g_event_pool.push_back(e.b); }
    g_prof_events.clear();
  }
  out->kernel_launches = g_launches;
  return PUV_OK;
}

size_t puv_last_error(char* buf, size_t len) {
  if (buf && len) {
    const size_t n = g_err.size() < len - 1 ? g_err.size() : len - 1;
    std::memcpy(buf, g_err.data(), n);
    buf[n] = 0;
  }
  return g_err.size();
}

const char* puv_version(void) { return "libpuv sm_100a " PUV_VERSION; }

}  // extern "C"
