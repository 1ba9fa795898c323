/*
 * puv_oracle.c — CPU ORACLE for the PackUV-GS splat render (TEST INFRASTRUCTURE).
 *
 * This file is test infrastructure, not product code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * arms may load it.  It shares no code, header, table or constant generator
 * with the CUDA path in paper_2602_23040_b200/; it is written from the
 * paper and the readings listed in DESIGN.md §2.
 *
 * What it computes (the "plain definition"):
 *   for each view, each pixel p: the front-to-back alpha composite of
 *   L_p = { visible g : tile(p) in rect(g) } ordered by (depth_bits(g), gid),
 *   and the exact derivative of that piecewise-smooth function w.r.t. the
 *   atlas texel planes with every decision held constant.
 *
 * Two arithmetic paths (DESIGN.md §2 R13):
 *   (A) decisions in fp32 under the arithmetic contract of DESIGN.md §2
 *       (visibility, rect, depth bits, J clamp, alpha-skip, alpha cap,
 *       transmittance termination) — the bit-exact target;
 *   (B) values in fp64 (projection, colour, composite, analytic backward),
 *       using (A)'s decisions.  (B) can be re-evaluated at perturbed fp64
 *       parameters with (A)'s decisions frozen, for finite differences.
 *
 * Passages followed (PAPER.md line numbers):
 *   3DGS primitive + alpha-blended tile rasterizer      189-195
 *   UV texel attributes U[u,v,k] = {rho, r, s, o, c}      297-303
 *   Sigma = R diag(s^2) R^T                               383-384, 1197
 *   EWA: Sigma2D = J T Sigma T^T J^T, J = [[fx/z,0,-fx x/z^2],[0,fy/z,-fy y/z^2]]
 *                                                          386-390, 1198-1204
 *   +0.3 low-pass on the diagonal                          1205-1206
 *   det <= 1e-7 / z <= 0 rejection                         1211-1215
 *   lambda_max and r = ceil(3 sqrt(lambda_max))            1219-1221
 *   gradient freezing grad <- D_i grad                     410-414
 *   atlas layout / pack                                    261-272
 * Everything the paper leaves open follows DESIGN.md §2's readings R1..R16.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared
 *        (x86-64 SSE arithmetic; FLT_EVAL_METHOD == 0).
 *
 * Threads (OpenMP, SURVEY.md §8(d) "OpenMP over (view, tile rows)"): projection
 * and the per-tile sorts run one Gaussian / one tile per iteration; forward and
 * backward run pixel ROWS round-robin over the threads (schedule(static, 1)).
 * Every pixel is still computed exactly as written; the only effect is the
 * order of the backward's per-Gaussian sums: each thread accumulates its rows
 * into its own buffer and the buffers are added in thread order, so for a given
 * thread count the result is deterministic.  orc_set_threads(1) gives the plain
 * single-thread program.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int orc_nthreads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static int orc_thread(void)
{
#ifdef _OPENMP
    return omp_get_thread_num();
#else
    return 0;
#endif
}

/* number of threads of the following calls (n < 1: all host cores); returns the count in use */
int orc_set_threads(int n)
{
#ifdef _OPENMP
    omp_set_num_threads(n >= 1 ? n : omp_get_num_procs());
#else
    (void)n;
#endif
    return orc_nthreads();
}

#if defined(__FLT_EVAL_METHOD__) && __FLT_EVAL_METHOD__ != 0
#error "oracle needs FLT_EVAL_METHOD == 0 (SSE float arithmetic)"
#endif

/* ------------------------------------------------------------------------- */
/* types (marshalled from Python with ctypes; layout stated in oracle/orc.py) */

typedef struct {
    float viewmat[16];            /* row-major world -> camera, OpenCV axes */
    float fx, fy, cx, cy;
    int32_t width, height;
    float near_plane;
    float campos[3];
} orc_camera;

typedef struct {                  /* path (A) outputs per (Gaussian, view) */
    int32_t visible;
    uint32_t depth_bits;
    int32_t x0, x1, y0, y1;       /* tile rect [x0,x1) x [y0,y1) */
    uint32_t tiles;
    float mx, my, ha, nb, hc, o, t_g;
    int32_t clamp_x, clamp_y;     /* J clamp: 0 none, +1 at +lim, -1 at -lim */
} orc_proj;

#define ORC_TILE 16

/* ------------------------------------------------------------------------- */
/* arithmetic contract: exp_c / log_c (DESIGN.md §2 R13)                      */

static float f_from_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t bits_from_f(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

static const float LN2_HI = 0.693145751953125f;
static const float LN2_LO = 1.42860677e-6f;

float orc_exp_c(float x)
{
    if (x >= 88.0f) return INFINITY;
    if (x <= -87.0f) return 0.0f;
    float k = rintf(x * 1.44269504f);
    float r = fmaf(-k, LN2_HI, x);
    r = fmaf(-k, LN2_LO, r);
    float p = (float)(1.0 / 5040.0);
    p = fmaf(p, r, (float)(1.0 / 720.0));
    p = fmaf(p, r, (float)(1.0 / 120.0));
    p = fmaf(p, r, (float)(1.0 / 24.0));
    p = fmaf(p, r, (float)(1.0 / 6.0));
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    int ki = (int)k;
    float two_k = f_from_bits((uint32_t)(ki + 127) << 23);
    return p * two_k;
}

float orc_log_c(float y)
{
    uint32_t b = bits_from_f(y);
    if (y != y || y < 0.0f) return NAN;
    if (y == INFINITY) return INFINITY;
    if ((b & 0x7f800000u) == 0) return -INFINITY;     /* 0 and subnormals */
    int e = (int)((b >> 23) & 0xff) - 127;
    float m = f_from_bits((b & 0x007fffffu) | 0x3f800000u);
    if (m > 1.41421356f) { m = m * 0.5f; e = e + 1; }
    float f = m - 1.0f;
    float s = f / (2.0f + f);
    float z = s * s;
    float P = fmaf(z, (float)(2.0 / 9.0), (float)(2.0 / 7.0));
    P = fmaf(z, P, (float)(2.0 / 5.0));
    P = fmaf(z, P, (float)(2.0 / 3.0));
    P = fmaf(z, P, 2.0f);
    float fe = (float)e;
    return fmaf(fe, LN2_HI, fmaf(fe, LN2_LO, s * P));
}

void orc_exp_c_array(const float* x, float* y, int64_t n)
{
    #pragma omp parallel for schedule(static, 65536)
    for (int64_t i = 0; i < n; ++i) y[i] = orc_exp_c(x[i]);
}
void orc_log_c_array(const float* x, float* y, int64_t n)
{
    #pragma omp parallel for schedule(static, 65536)
    for (int64_t i = 0; i < n; ++i) y[i] = orc_log_c(x[i]);
}

/* ------------------------------------------------------------------------- */
/* spherical harmonics (real basis, 3DGS sign convention; R3)       */

static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Y[k] for k < (deg+1)^2 at unit direction d; dY[k][3] = gradient of the
 * basis polynomial w.r.t. (x, y, z) (not projected on the sphere). */
static void sh_basis(int deg, const double d[3], double* Y, double (*dY)[3])
{
    double x = d[0], y = d[1], z = d[2];
    double xx = x * x, yy = y * y, zz = z * z;
    int nk = (deg + 1) * (deg + 1);
    for (int k = 0; k < nk; ++k) { Y[k] = 0; if (dY) { dY[k][0] = dY[k][1] = dY[k][2] = 0; } }
    Y[0] = SH_C0;
    if (deg >= 1) {
        Y[1] = -SH_C1 * y; Y[2] = SH_C1 * z; Y[3] = -SH_C1 * x;
        if (dY) { dY[1][1] = -SH_C1; dY[2][2] = SH_C1; dY[3][0] = -SH_C1; }
    }
    if (deg >= 2) {
        Y[4] = SH_C2[0] * x * y;
        Y[5] = SH_C2[1] * y * z;
        Y[6] = SH_C2[2] * (2.0 * zz - xx - yy);
        Y[7] = SH_C2[3] * x * z;
        Y[8] = SH_C2[4] * (xx - yy);
        if (dY) {
            dY[4][0] = SH_C2[0] * y; dY[4][1] = SH_C2[0] * x;
            dY[5][1] = SH_C2[1] * z; dY[5][2] = SH_C2[1] * y;
            dY[6][0] = -2.0 * SH_C2[2] * x; dY[6][1] = -2.0 * SH_C2[2] * y; dY[6][2] = 4.0 * SH_C2[2] * z;
            dY[7][0] = SH_C2[3] * z; dY[7][2] = SH_C2[3] * x;
            dY[8][0] = 2.0 * SH_C2[4] * x; dY[8][1] = -2.0 * SH_C2[4] * y;
        }
    }
    if (deg >= 3) {
        Y[9] = SH_C3[0] * y * (3.0 * xx - yy);
        Y[10] = SH_C3[1] * x * y * z;
        Y[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
        Y[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        Y[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
        Y[14] = SH_C3[5] * z * (xx - yy);
        Y[15] = SH_C3[6] * x * (xx - 3.0 * yy);
        if (dY) {
            dY[9][0] = SH_C3[0] * 6.0 * x * y; dY[9][1] = SH_C3[0] * (3.0 * xx - 3.0 * yy);
            dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
            dY[11][0] = SH_C3[2] * (-2.0 * x * y); dY[11][1] = SH_C3[2] * (4.0 * zz - xx - 3.0 * yy);
            dY[11][2] = SH_C3[2] * 8.0 * y * z;
            dY[12][0] = SH_C3[3] * (-6.0 * x * z); dY[12][1] = SH_C3[3] * (-6.0 * y * z);
            dY[12][2] = SH_C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
            dY[13][0] = SH_C3[4] * (4.0 * zz - 3.0 * xx - yy); dY[13][1] = SH_C3[4] * (-2.0 * x * y);
            dY[13][2] = SH_C3[4] * 8.0 * x * z;
            dY[14][0] = SH_C3[5] * 2.0 * x * z; dY[14][1] = SH_C3[5] * (-2.0 * y * z);
            dY[14][2] = SH_C3[5] * (xx - yy);
            dY[15][0] = SH_C3[6] * (3.0 * xx - 3.0 * yy); dY[15][1] = SH_C3[6] * (-6.0 * x * y);
        }
    }
}

/* exported for the orthonormality pin */
void orc_sh_basis(int deg, const double* dirs, int64_t n, double* Y)
{
    int nk = (deg + 1) * (deg + 1);
    for (int64_t i = 0; i < n; ++i) sh_basis(deg, dirs + 3 * i, Y + nk * i, NULL);
}

/* ------------------------------------------------------------------------- */
/* path (A): fp32 contract projection, DESIGN.md §2 steps U1-U5, P1-P12        */

static float lim_of(int32_t extent, float f)
{   /* 1.3 * tan(fov/2) = 1.3 * 0.5 * extent / f, in fp64 then rounded (R5) */
    return (float)(1.3 * 0.5 * (double)extent / (double)f);
}

static float clampf(float v, float lo, float hi) { return v < lo ? lo : (v > hi ? hi : v); }

static void project_one_f32(const float* const* planes, int64_t g, const orc_camera* cam, orc_proj* P)
{
    memset(P, 0, sizeof(*P));
    /* U1 */
    float s0 = orc_exp_c(planes[3][g]), s1 = orc_exp_c(planes[4][g]), s2 = orc_exp_c(planes[5][g]);
    float t0 = s0 * s0, t1 = s1 * s1, t2 = s2 * s2;
    /* U2 */
    float w = planes[6][g], x = planes[7][g], y = planes[8][g], z = planes[9][g];
    float n2 = ((w * w + x * x) + y * y) + z * z;
    if (n2 == 0.0f) return;
    float n = sqrtf(n2);
    w = w / n; x = x / n; y = y / n; z = z / n;
    /* U3 */
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
    float wx = w * x, wy = w * y, wz = w * z;
    float R[3][3];
    R[0][0] = 1.0f - 2.0f * (yy + zz); R[0][1] = 2.0f * (xy - wz);        R[0][2] = 2.0f * (xz + wy);
    R[1][0] = 2.0f * (xy + wz);        R[1][1] = 1.0f - 2.0f * (xx + zz); R[1][2] = 2.0f * (yz - wx);
    R[2][0] = 2.0f * (xz - wy);        R[2][1] = 2.0f * (yz + wx);        R[2][2] = 1.0f - 2.0f * (xx + yy);
    /* U4: Sigma_ab = ((R_a0 t0) R_b0 + (R_a1 t1) R_b1) + (R_a2 t2) R_b2 */
    float S[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = a; b < 3; ++b) {
            float v = ((R[a][0] * t0) * R[b][0] + (R[a][1] * t1) * R[b][1]) + (R[a][2] * t2) * R[b][2];
            S[a][b] = v; S[b][a] = v;
        }
    /* U5 */
    float o = 1.0f / (1.0f + orc_exp_c(-planes[10][g]));
    float t_g = -orc_log_c(255.0f * o);
    /* P1 */
    const float* V = cam->viewmat;
    float mux = planes[0][g], muy = planes[1][g], muz = planes[2][g];
    float px = ((V[0] * mux + V[1] * muy) + V[2] * muz) + V[3];
    float py = ((V[4] * mux + V[5] * muy) + V[6] * muz) + V[7];
    float pz = ((V[8] * mux + V[9] * muy) + V[10] * muz) + V[11];
    /* P2 */
    if (!(pz > cam->near_plane)) return;
    /* P3 */
    float limx = lim_of(cam->width, cam->fx), limy = lim_of(cam->height, cam->fy);
    float ux = px / pz, uy = py / pz;
    float cxp = fminf(limx, fmaxf(-limx, ux));
    float cyp = fminf(limy, fmaxf(-limy, uy));
    int clx = ux > limx ? 1 : (ux < -limx ? -1 : 0);
    int cly = uy > limy ? 1 : (uy < -limy ? -1 : 0);
    float J00 = cam->fx / pz, J02 = -((cam->fx * cxp) / pz);
    float J11 = cam->fy / pz, J12 = -((cam->fy * cyp) / pz);
    /* P4 */
    float T[2][3];
    for (int k = 0; k < 3; ++k) {
        T[0][k] = J00 * V[0 * 4 + k] + J02 * V[2 * 4 + k];
        T[1][k] = J11 * V[1 * 4 + k] + J12 * V[2 * 4 + k];
    }
    /* P5 */
    float W[2][3];
    for (int a = 0; a < 2; ++a)
        for (int i = 0; i < 3; ++i)
            W[a][i] = (S[i][0] * T[a][0] + S[i][1] * T[a][1]) + S[i][2] * T[a][2];
    float ca = (T[0][0] * W[0][0] + T[0][1] * W[0][1]) + T[0][2] * W[0][2];
    float cb = (T[1][0] * W[0][0] + T[1][1] * W[0][1]) + T[1][2] * W[0][2];
    float cc = (T[1][0] * W[1][0] + T[1][1] * W[1][1]) + T[1][2] * W[1][2];
    /* P6 */
    ca = ca + 0.3f; cc = cc + 0.3f;
    /* P7 */
    float det = ca * cc - cb * cb;
    if (!(det > 1e-7f)) return;
    /* P8 */
    float ha = -0.5f * (cc / det);
    float nb = cb / det;
    float hc = -0.5f * (ca / det);
    /* P9 */
    float tr = ca + cc;
    float disc = tr * tr - 4.0f * det;
    float lam = 0.5f * (tr + sqrtf(fmaxf(0.0f, disc)));
    float rf = ceilf(3.0f * sqrtf(lam));
    /* P10 */
    float mx = cam->fx * ux + cam->cx;
    float my = cam->fy * uy + cam->cy;
    /* P11 (conservative rect) */
    int gx = (cam->width + ORC_TILE - 1) / ORC_TILE, gy = (cam->height + ORC_TILE - 1) / ORC_TILE;
    float fx0 = clampf(floorf((mx - rf) * 0.0625f), 0.0f, (float)gx);
    float fx1 = clampf(floorf((mx + rf) * 0.0625f) + 1.0f, 0.0f, (float)gx);
    float fy0 = clampf(floorf((my - rf) * 0.0625f), 0.0f, (float)gy);
    float fy1 = clampf(floorf((my + rf) * 0.0625f) + 1.0f, 0.0f, (float)gy);
    int x0 = (int)fx0, x1 = (int)fx1, y0 = (int)fy0, y1 = (int)fy1;
    if (x0 >= x1 || y0 >= y1) return;
    P->visible = 1;
    P->depth_bits = bits_from_f(pz);   /* P12 */
    P->x0 = x0; P->x1 = x1; P->y0 = y0; P->y1 = y1;
    P->tiles = (uint32_t)((x1 - x0) * (y1 - y0));
    P->mx = mx; P->my = my; P->ha = ha; P->nb = nb; P->hc = hc; P->o = o; P->t_g = t_g;
    P->clamp_x = clx; P->clamp_y = cly;
}

/* planes: D pointers to H_A*W_A floats; occ nullable */
int orc_project(const float* const* planes, int64_t n, const uint8_t* occ, const orc_camera* cam, orc_proj* out)
{
    #pragma omp parallel for schedule(static, 4096)
    for (int64_t g = 0; g < n; ++g) {
        if (occ && !occ[g]) { memset(&out[g], 0, sizeof(orc_proj)); continue; }
        project_one_f32(planes, g, cam, &out[g]);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* binning: per tile the list of visible g whose rect contains the tile,
 * ordered by (depth_bits, gid) (R8).  Plain construction: append
 * in gid order, then sort each tile's list with qsort.                       */

typedef struct { uint32_t depth; uint32_t gid; } orc_key;

static int cmp_key(const void* a, const void* b)
{
    const orc_key* p = (const orc_key*)a; const orc_key* q = (const orc_key*)b;
    if (p->depth != q->depth) return p->depth < q->depth ? -1 : 1;
    if (p->gid != q->gid) return p->gid < q->gid ? -1 : 1;
    return 0;
}

int64_t orc_bin_count(int64_t n, const orc_proj* P)
{
    int64_t K = 0;
    for (int64_t g = 0; g < n; ++g) if (P[g].visible) K += P[g].tiles;
    return K;
}

/* start/end: ntiles each (tile id = ty*gx + tx); gids: K entries */
int orc_bin(int64_t n, const orc_proj* P, int gx, int gy, uint32_t* start, uint32_t* end, uint32_t* gids)
{
    int64_t ntiles = (int64_t)gx * gy;
    int64_t* cnt = (int64_t*)calloc((size_t)ntiles, sizeof(int64_t));
    if (!cnt) return -1;
    for (int64_t g = 0; g < n; ++g) {
        if (!P[g].visible) continue;
        for (int ty = P[g].y0; ty < P[g].y1; ++ty)
            for (int tx = P[g].x0; tx < P[g].x1; ++tx) cnt[(int64_t)ty * gx + tx]++;
    }
    int64_t acc = 0;
    for (int64_t t = 0; t < ntiles; ++t) { start[t] = (uint32_t)acc; acc += cnt[t]; end[t] = (uint32_t)acc; cnt[t] = 0; }
    orc_key* keys = (orc_key*)malloc((size_t)(acc > 0 ? acc : 1) * sizeof(orc_key));
    if (!keys) { free(cnt); return -1; }
    for (int64_t g = 0; g < n; ++g) {
        if (!P[g].visible) continue;
        for (int ty = P[g].y0; ty < P[g].y1; ++ty)
            for (int tx = P[g].x0; tx < P[g].x1; ++tx) {
                int64_t t = (int64_t)ty * gx + tx;
                orc_key k = {P[g].depth_bits, (uint32_t)g};
                keys[start[t] + cnt[t]++] = k;
            }
    }
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < ntiles; ++t)
        qsort(keys + start[t], (size_t)(end[t] - start[t]), sizeof(orc_key), cmp_key);
    for (int64_t i = 0; i < acc; ++i) gids[i] = keys[i].gid;
    free(keys); free(cnt);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* path (B): fp64 per-Gaussian values with (A)'s decisions                    */

typedef struct {
    double mx, my, ha, nb, hc, o, rgb[3];
    int rgb_clamped[3];
} val_proj;

typedef struct {          /* intermediate values kept for the backward */
    double mu[3], s[3], t[3], qn, qh[4], R[3][3], Sig[3][3];
    double p[3], ux, uy, cxp, cyp, J00, J02, J11, J12, T[2][3];
    double a, b, c, det, o, dir[3], dist;
    double Y[16], dY[16][3];
} val_aux;

static void project_one_f64(const double* const* vp, int64_t g, int sh_degree, const orc_camera* cam,
                            const orc_proj* A, val_proj* out, val_aux* X)
{
    val_aux Xl; if (!X) X = &Xl;
    for (int k = 0; k < 3; ++k) { X->mu[k] = vp[k][g]; X->s[k] = exp(vp[3 + k][g]); X->t[k] = X->s[k] * X->s[k]; }
    double q[4] = {vp[6][g], vp[7][g], vp[8][g], vp[9][g]};
    X->qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) X->qh[k] = q[k] / X->qn;
    double w = X->qh[0], x = X->qh[1], y = X->qh[2], z = X->qh[3];
    double (*R)[3] = X->R;
    R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double v = 0;
            for (int k = 0; k < 3; ++k) v += R[a][k] * X->t[k] * R[b][k];
            X->Sig[a][b] = v;
        }
    const float* V = cam->viewmat;
    for (int r = 0; r < 3; ++r)
        X->p[r] = (double)V[4 * r] * X->mu[0] + (double)V[4 * r + 1] * X->mu[1] + (double)V[4 * r + 2] * X->mu[2] + (double)V[4 * r + 3];
    double pz = X->p[2];
    X->ux = X->p[0] / pz; X->uy = X->p[1] / pz;
    double limx = lim_of(cam->width, cam->fx), limy = lim_of(cam->height, cam->fy);
    X->cxp = A->clamp_x ? A->clamp_x * limx : X->ux;
    X->cyp = A->clamp_y ? A->clamp_y * limy : X->uy;
    X->J00 = cam->fx / pz; X->J02 = -cam->fx * X->cxp / pz;
    X->J11 = cam->fy / pz; X->J12 = -cam->fy * X->cyp / pz;
    for (int k = 0; k < 3; ++k) {
        X->T[0][k] = X->J00 * V[k] + X->J02 * V[8 + k];
        X->T[1][k] = X->J11 * V[4 + k] + X->J12 * V[8 + k];
    }
    double M[2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            double v = 0;
            for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) v += X->T[a][i] * X->Sig[i][j] * X->T[b][j];
            M[a][b] = v;
        }
    X->a = M[0][0] + 0.3; X->b = M[0][1]; X->c = M[1][1] + 0.3;
    X->det = X->a * X->c - X->b * X->b;
    out->ha = -0.5 * X->c / X->det;
    out->nb = X->b / X->det;
    out->hc = -0.5 * X->a / X->det;
    out->mx = cam->fx * X->ux + cam->cx;
    out->my = cam->fy * X->uy + cam->cy;
    X->o = 1.0 / (1.0 + exp(-vp[10][g]));
    out->o = X->o;
    double d[3], dn = 0;
    for (int k = 0; k < 3; ++k) { d[k] = X->mu[k] - (double)cam->campos[k]; dn += d[k] * d[k]; }
    X->dist = sqrt(dn);
    for (int k = 0; k < 3; ++k) X->dir[k] = d[k] / X->dist;
    sh_basis(sh_degree, X->dir, X->Y, X->dY);
    int nk = (sh_degree + 1) * (sh_degree + 1);
    for (int c = 0; c < 3; ++c) {
        double v = 0.5;
        for (int k = 0; k < nk; ++k) v += X->Y[k] * vp[11 + 3 * k + c][g];
        out->rgb_clamped[c] = v < 0.0;
        out->rgb[c] = v < 0.0 ? 0.0 : v;
    }
}

/* ------------------------------------------------------------------------- */
/* per-pixel composite (decisions from (A), values from (B))                  */

typedef struct {
    int64_t gid;
    double alpha, G, dx, dy, T;
    int capped;
} comp_entry;

/* Walks the tile list for pixel (i,j).  Fills `ce` with composited entries
 * (in order), returns their count; *n_contrib = list position after the
 * last composited entry; *T32 = final fp32 contract transmittance.        */
static int composite_pixel(int i, int j, const uint32_t* list, int64_t len, const orc_proj* P,
                           const val_proj* VP, comp_entry* ce, int32_t* n_contrib, float* T32)
{
    float T = 1.0f;
    double T64 = 1.0;
    int nc = 0;
    int32_t last = 0;
    float fi = (float)i, fj = (float)j;
    for (int64_t e = 0; e < len; ++e) {
        uint32_t g = list[e];
        const orc_proj* A = &P[g];
        /* R1 skip test, contract */
        float dx = A->mx - fi, dy = A->my - fj;
        float u = fmaf(A->nb, dy, A->ha * dx);
        float power = fmaf(dx, u, (A->hc * dy) * dy);
        if (power > 0.0f || power < A->t_g) continue;
        /* R14 alpha / termination, contract */
        float G = orc_exp_c(power);
        float ao = A->o * G;
        int capped = !(ao < 0.99f);
        float alpha = capped ? 0.99f : ao;
        float Tn = T * (1.0f - alpha);
        if (Tn < 1e-4f) break;
        /* values (fp64) */
        const val_proj* B = &VP[g];
        double ddx = B->mx - (double)i, ddy = B->my - (double)j;
        double pw = B->ha * ddx * ddx + B->nb * ddx * ddy + B->hc * ddy * ddy;
        double G64 = exp(pw);
        double a64 = capped ? 0.99 : B->o * G64;
        ce[nc].gid = g; ce[nc].alpha = a64; ce[nc].G = G64; ce[nc].dx = ddx; ce[nc].dy = ddy;
        ce[nc].T = T64; ce[nc].capped = capped;
        nc++;
        T64 = T64 * (1.0 - a64);
        T = Tn;
        last = (int32_t)(e + 1);
    }
    *n_contrib = last;
    *T32 = T;
    return nc;
}

/* ------------------------------------------------------------------------- */
/* view setup shared by forward and backward                                  */

typedef struct {
    int64_t n;
    int gx, gy;
    orc_proj* P;
    val_proj* VP;
    uint32_t *start, *end, *gids;
    int64_t K;
} view_ctx;

static void view_free(view_ctx* v)
{
    free(v->P); free(v->VP); free(v->start); free(v->end); free(v->gids);
    memset(v, 0, sizeof(*v));
}

static int view_setup(const float* const* dec, const double* const* val, int sh_degree, int64_t n,
                      const uint8_t* occ, const orc_camera* cam, view_ctx* v)
{
    memset(v, 0, sizeof(*v));
    v->n = n;
    v->gx = (cam->width + ORC_TILE - 1) / ORC_TILE;
    v->gy = (cam->height + ORC_TILE - 1) / ORC_TILE;
    v->P = (orc_proj*)malloc((size_t)n * sizeof(orc_proj));
    v->VP = (val_proj*)calloc((size_t)n, sizeof(val_proj));
    int64_t nt = (int64_t)v->gx * v->gy;
    v->start = (uint32_t*)malloc((size_t)nt * 4);
    v->end = (uint32_t*)malloc((size_t)nt * 4);
    if (!v->P || !v->VP || !v->start || !v->end) { view_free(v); return -1; }
    orc_project(dec, n, occ, cam, v->P);
    #pragma omp parallel for schedule(static, 4096)
    for (int64_t g = 0; g < n; ++g)
        if (v->P[g].visible) project_one_f64(val, g, sh_degree, cam, &v->P[g], &v->VP[g], NULL);
    v->K = orc_bin_count(n, v->P);
    v->gids = (uint32_t*)malloc((size_t)(v->K > 0 ? v->K : 1) * 4);
    if (!v->gids) { view_free(v); return -1; }
    orc_bin(n, v->P, v->gx, v->gy, v->start, v->end, v->gids);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* forward: image (3,H,W) fp64; T32 / n_contrib per pixel (nullable)          */

int orc_forward(const float* const* dec, const double* const* val, int sh_degree, int64_t n,
                const uint8_t* occ, const orc_camera* cam, const double* bg,
                double* image, float* T32_out, int32_t* ncontrib_out, int64_t* stats /* [N_vis, K, examined?] */)
{
    view_ctx v;
    if (view_setup(dec, val, sh_degree, n, occ, cam, &v)) return -1;
    int W = cam->width, H = cam->height;
    int64_t maxlen = 0;
    for (int64_t t = 0; t < (int64_t)v.gx * v.gy; ++t)
        if ((int64_t)(v.end[t] - v.start[t]) > maxlen) maxlen = v.end[t] - v.start[t];
    if (maxlen < 1) maxlen = 1;
    const int nthr = orc_nthreads();
    comp_entry* ce_all = (comp_entry*)malloc((size_t)nthr * (size_t)maxlen * sizeof(comp_entry));
    if (!ce_all) { view_free(&v); return -1; }
    int64_t composited = 0;
    #pragma omp parallel for schedule(static, 1) reduction(+ : composited)
    for (int j = 0; j < H; ++j) {
        comp_entry* ce = ce_all + (size_t)orc_thread() * (size_t)maxlen;
        for (int i = 0; i < W; ++i) {
            int64_t t = (int64_t)(j / ORC_TILE) * v.gx + (i / ORC_TILE);
            int32_t nctr; float T32;
            int nc = composite_pixel(i, j, v.gids + v.start[t], v.end[t] - v.start[t], v.P, v.VP, ce, &nctr, &T32);
            double C[3] = {0, 0, 0};
            double T = 1.0;
            for (int k = 0; k < nc; ++k) {
                const val_proj* B = &v.VP[ce[k].gid];
                for (int c = 0; c < 3; ++c) C[c] += B->rgb[c] * ce[k].alpha * T;
                T *= (1.0 - ce[k].alpha);
            }
            for (int c = 0; c < 3; ++c) image[(int64_t)c * H * W + (int64_t)j * W + i] = C[c] + T * bg[c];
            if (T32_out) T32_out[(int64_t)j * W + i] = T32;
            if (ncontrib_out) ncontrib_out[(int64_t)j * W + i] = nctr;
            composited += nc;
        }
    }
    if (stats) {
        int64_t nvis = 0;
        for (int64_t g = 0; g < n; ++g) nvis += v.P[g].visible;
        stats[0] = nvis; stats[1] = v.K; stats[2] = composited;
    }
    free(ce_all);
    view_free(&v);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* backward: grad planes (D x n) fp64, ACCUMULATED (+=).  mask nullable.       */

int orc_backward(const float* const* dec, const double* const* val, int sh_degree, int64_t n,
                 const uint8_t* occ, const orc_camera* cam, const double* bg,
                 const double* dL_dimage, const uint8_t* mask, double* const* grad)
{
    view_ctx v;
    if (view_setup(dec, val, sh_degree, n, occ, cam, &v)) return -1;
    int W = cam->width, H = cam->height;
    int64_t maxlen = 0;
    for (int64_t t = 0; t < (int64_t)v.gx * v.gy; ++t)
        if ((int64_t)(v.end[t] - v.start[t]) > maxlen) maxlen = v.end[t] - v.start[t];
    if (maxlen < 1) maxlen = 1;
    const int nthr = orc_nthreads();
    comp_entry* ce_all = (comp_entry*)malloc((size_t)nthr * (size_t)maxlen * sizeof(comp_entry));
    /* per-Gaussian 2D gradients: mx, my, ha, nb, hc, o, r, g, b; one buffer per thread */
    double* g2_all = (double*)calloc((size_t)nthr * (size_t)n * 9, sizeof(double));
    if (!ce_all || !g2_all) { free(ce_all); free(g2_all); view_free(&v); return -1; }

    #pragma omp parallel for schedule(static, 1)
    for (int j = 0; j < H; ++j) {
        comp_entry* ce = ce_all + (size_t)orc_thread() * (size_t)maxlen;
        double* g2 = g2_all + (size_t)orc_thread() * (size_t)n * 9;
        for (int i = 0; i < W; ++i) {
            int64_t t = (int64_t)(j / ORC_TILE) * v.gx + (i / ORC_TILE);
            int32_t nctr; float T32;
            int nc = composite_pixel(i, j, v.gids + v.start[t], v.end[t] - v.start[t], v.P, v.VP, ce, &nctr, &T32);
            double dC[3];
            for (int c = 0; c < 3; ++c) dC[c] = dL_dimage[(int64_t)c * H * W + (int64_t)j * W + i];
            double Tfin = 1.0;
            for (int k = 0; k < nc; ++k) Tfin *= (1.0 - ce[k].alpha);
            /* S = sum_{i>k} c_i alpha_i T_i + T_{n+1} bg */
            double S[3] = {Tfin * bg[0], Tfin * bg[1], Tfin * bg[2]};
            for (int k = nc - 1; k >= 0; --k) {
                int64_t g = ce[k].gid;
                const val_proj* B = &v.VP[g];
                double a = ce[k].alpha, T = ce[k].T;
                double dLda = 0;
                for (int c = 0; c < 3; ++c) {
                    g2[g * 9 + 6 + c] += a * T * dC[c];
                    dLda += dC[c] * (T * B->rgb[c] - S[c] / (1.0 - a));
                }
                for (int c = 0; c < 3; ++c) S[c] += B->rgb[c] * a * T;
                if (ce[k].capped) continue;
                double G = ce[k].G;
                g2[g * 9 + 5] += G * dLda;                 /* d alpha / d o = G */
                double dP = B->o * G * dLda;                /* d alpha / d power = o G */
                double dx = ce[k].dx, dy = ce[k].dy;
                g2[g * 9 + 2] += dx * dx * dP;
                g2[g * 9 + 3] += dx * dy * dP;
                g2[g * 9 + 4] += dy * dy * dP;
                g2[g * 9 + 0] += (2.0 * B->ha * dx + B->nb * dy) * dP;
                g2[g * 9 + 1] += (B->nb * dx + 2.0 * B->hc * dy) * dP;
            }
        }
    }
    /* thread buffers summed in thread order into buffer 0 */
    double* g2 = g2_all;
    #pragma omp parallel for schedule(static, 4096)
    for (int64_t q = 0; q < n * 9; ++q)
        for (int t = 1; t < nthr; ++t) g2[q] += g2_all[(size_t)t * (size_t)n * 9 + (size_t)q];

    /* per-Gaussian chain rule to texel planes (DESIGN.md §1 backward); each g writes only its own texel */
    int nk = (sh_degree + 1) * (sh_degree + 1);
    const float* V = cam->viewmat;
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t g = 0; g < n; ++g) {
        if (!v.P[g].visible) continue;
        const double* d2 = g2 + g * 9;
        int any = 0;
        for (int k = 0; k < 9; ++k) any |= d2[k] != 0.0;
        if (!any) continue;
        val_proj B; val_aux X;
        project_one_f64(val, g, sh_degree, cam, &v.P[g], &B, &X);
        double dmu[3] = {0, 0, 0}, dp[3] = {0, 0, 0};
        /* conic (ha, nb, hc) <- (a, b, c) */
        double a = X.a, b = X.b, c = X.c, det2 = X.det * X.det;
        double dha = d2[2], dnb = d2[3], dhc = d2[4];
        double da = dha * (0.5 * c * c / det2) + dnb * (-b * c / det2) + dhc * (0.5 * b * b / det2);
        double db = dha * (-b * c / det2) + dnb * ((a * c + b * b) / det2) + dhc * (-a * b / det2);
        double dc = dha * (0.5 * b * b / det2) + dnb * (-a * b / det2) + dhc * (0.5 * a * a / det2);
        /* Sigma2D = T Sigma T^T: a = t0 S t0, b = t0 S t1, c = t1 S t1 */
        double dS[3][3];
        for (int i2 = 0; i2 < 3; ++i2)
            for (int j2 = 0; j2 < 3; ++j2)
                dS[i2][j2] = da * X.T[0][i2] * X.T[0][j2] + db * X.T[0][i2] * X.T[1][j2] + dc * X.T[1][i2] * X.T[1][j2];
        double St0[3], St1[3];
        for (int i2 = 0; i2 < 3; ++i2) {
            St0[i2] = X.Sig[i2][0] * X.T[0][0] + X.Sig[i2][1] * X.T[0][1] + X.Sig[i2][2] * X.T[0][2];
            St1[i2] = X.Sig[i2][0] * X.T[1][0] + X.Sig[i2][1] * X.T[1][1] + X.Sig[i2][2] * X.T[1][2];
        }
        double dT[2][3];
        for (int k = 0; k < 3; ++k) {
            dT[0][k] = 2.0 * da * St0[k] + db * St1[k];
            dT[1][k] = 2.0 * dc * St1[k] + db * St0[k];
        }
        /* T0k = J00 V0k + J02 V2k ; T1k = J11 V1k + J12 V2k */
        double dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0;
        for (int k = 0; k < 3; ++k) {
            dJ00 += dT[0][k] * V[k]; dJ02 += dT[0][k] * V[8 + k];
            dJ11 += dT[1][k] * V[4 + k]; dJ12 += dT[1][k] * V[8 + k];
        }
        double pz = X.p[2], fx = cam->fx, fy = cam->fy;
        dp[2] += dJ00 * (-fx / (pz * pz)) + dJ11 * (-fy / (pz * pz));
        if (v.P[g].clamp_x == 0) { dp[0] += dJ02 * (-fx / (pz * pz)); dp[2] += dJ02 * (2.0 * fx * X.p[0] / (pz * pz * pz)); }
        else dp[2] += dJ02 * (fx * X.cxp / (pz * pz));
        if (v.P[g].clamp_y == 0) { dp[1] += dJ12 * (-fy / (pz * pz)); dp[2] += dJ12 * (2.0 * fy * X.p[1] / (pz * pz * pz)); }
        else dp[2] += dJ12 * (fy * X.cyp / (pz * pz));
        /* mean2D */
        dp[0] += d2[0] * fx / pz; dp[2] += d2[0] * (-fx * X.p[0] / (pz * pz));
        dp[1] += d2[1] * fy / pz; dp[2] += d2[1] * (-fy * X.p[1] / (pz * pz));
        for (int k = 0; k < 3; ++k) dmu[k] += V[k] * dp[0] + V[4 + k] * dp[1] + V[8 + k] * dp[2];
        /* Sigma = R diag(t) R^T */
        double dt[3], dR[3][3];
        for (int k = 0; k < 3; ++k) {
            double v2 = 0;
            for (int i2 = 0; i2 < 3; ++i2) for (int j2 = 0; j2 < 3; ++j2) v2 += dS[i2][j2] * X.R[i2][k] * X.R[j2][k];
            dt[k] = v2;
        }
        for (int a2 = 0; a2 < 3; ++a2)
            for (int b2 = 0; b2 < 3; ++b2) {
                double v2 = 0;
                for (int j2 = 0; j2 < 3; ++j2) v2 += (dS[a2][j2] + dS[j2][a2]) * X.R[j2][b2];
                dR[a2][b2] = v2 * X.t[b2];
            }
        double w = X.qh[0], x = X.qh[1], y = X.qh[2], z = X.qh[3];
        double dq[4];
        dq[0] = dR[0][1] * (-2 * z) + dR[0][2] * (2 * y) + dR[1][0] * (2 * z) + dR[1][2] * (-2 * x)
              + dR[2][0] * (-2 * y) + dR[2][1] * (2 * x);
        dq[1] = dR[0][1] * (2 * y) + dR[0][2] * (2 * z) + dR[1][0] * (2 * y) + dR[1][1] * (-4 * x)
              + dR[1][2] * (-2 * w) + dR[2][0] * (2 * z) + dR[2][1] * (2 * w) + dR[2][2] * (-4 * x);
        dq[2] = dR[0][0] * (-4 * y) + dR[0][1] * (2 * x) + dR[0][2] * (2 * w) + dR[1][0] * (2 * x)
              + dR[1][2] * (2 * z) + dR[2][0] * (-2 * w) + dR[2][1] * (2 * z) + dR[2][2] * (-4 * y);
        dq[3] = dR[0][0] * (-4 * z) + dR[0][1] * (-2 * w) + dR[0][2] * (2 * x) + dR[1][0] * (2 * w)
              + dR[1][1] * (-4 * z) + dR[1][2] * (2 * y) + dR[2][0] * (2 * x) + dR[2][1] * (2 * y);
        double qd = X.qh[0] * dq[0] + X.qh[1] * dq[1] + X.qh[2] * dq[2] + X.qh[3] * dq[3];
        double dqraw[4];
        for (int k = 0; k < 4; ++k) dqraw[k] = (dq[k] - X.qh[k] * qd) / X.qn;
        /* colour */
        double drgb[3] = {B.rgb_clamped[0] ? 0 : d2[6], B.rgb_clamped[1] ? 0 : d2[7], B.rgb_clamped[2] ? 0 : d2[8]};
        double ddir[3] = {0, 0, 0};
        double scale = (mask && !mask[g]) ? 0.0 : 1.0;
        for (int k = 0; k < nk; ++k)
            for (int c2 = 0; c2 < 3; ++c2) {
                double shv = val[11 + 3 * k + c2][g];
                grad[11 + 3 * k + c2][g] += scale * X.Y[k] * drgb[c2];
                for (int e = 0; e < 3; ++e) ddir[e] += shv * X.dY[k][e] * drgb[c2];
            }
        double dd = X.dir[0] * ddir[0] + X.dir[1] * ddir[1] + X.dir[2] * ddir[2];
        for (int k = 0; k < 3; ++k) dmu[k] += (ddir[k] - X.dir[k] * dd) / X.dist;
        for (int k = 0; k < 3; ++k) grad[k][g] += scale * dmu[k];
        for (int k = 0; k < 3; ++k) grad[3 + k][g] += scale * dt[k] * 2.0 * X.t[k];
        for (int k = 0; k < 4; ++k) grad[6 + k][g] += scale * dqraw[k];
        grad[10][g] += scale * d2[5] * X.o * (1.0 - X.o);
    }
    free(ce_all); free(g2_all);
    view_free(&v);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* covariance-aware flow masking, supp. Algorithm 1,
 * followed step by step with the readings M1-M6 of DESIGN.md §10:
 *   1. Sigma3D = R(q) diag(s^2) R(q)^T            (contract U1-U4)
 *   2. camera-space mean; J = [[fx/z,0,-fx x/z^2],[0,fy/z,-fy y/z^2]] UNclamped;
 *      Sigma2D = J (T Sigma T^T) J^T; +0.3 on the diagonal; m = pixel projection
 *   3. invalid (static for this camera) if det <= 1e-7, det < 0 or z <= 0
 *   4. r = min(r_max, ceil(3 sqrt(lambda_max)))
 *   5. scan integer pixels p with |p - m|_inf <= r inside the image; dynamic iff
 *      some p has d^2 <= 9 (contract: R1 power >= -4.5) and mask(p) = 1
 *   D_i = OR over cameras.  labels: n bytes, OVERWRITTEN.  masks: n_cams images
 *   of width*height bytes (0 / nonzero), camera order.                        */

static int label_one_f32(const float* const* planes, int64_t g, const orc_camera* cam, const uint8_t* mask,
                         int r_max)
{
    float s0 = orc_exp_c(planes[3][g]), s1 = orc_exp_c(planes[4][g]), s2 = orc_exp_c(planes[5][g]);
    float t0 = s0 * s0, t1 = s1 * s1, t2 = s2 * s2;
    float w = planes[6][g], x = planes[7][g], y = planes[8][g], z = planes[9][g];
    float n2 = ((w * w + x * x) + y * y) + z * z;
    if (n2 == 0.0f) return 0;
    float n = sqrtf(n2);
    w = w / n; x = x / n; y = y / n; z = z / n;
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
    float wx = w * x, wy = w * y, wz = w * z;
    float R[3][3];
    R[0][0] = 1.0f - 2.0f * (yy + zz); R[0][1] = 2.0f * (xy - wz);        R[0][2] = 2.0f * (xz + wy);
    R[1][0] = 2.0f * (xy + wz);        R[1][1] = 1.0f - 2.0f * (xx + zz); R[1][2] = 2.0f * (yz - wx);
    R[2][0] = 2.0f * (xz - wy);        R[2][1] = 2.0f * (yz + wx);        R[2][2] = 1.0f - 2.0f * (xx + yy);
    float S[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = a; b < 3; ++b) {
            float v = ((R[a][0] * t0) * R[b][0] + (R[a][1] * t1) * R[b][1]) + (R[a][2] * t2) * R[b][2];
            S[a][b] = v; S[b][a] = v;
        }
    const float* V = cam->viewmat;
    float mux = planes[0][g], muy = planes[1][g], muz = planes[2][g];
    float px = ((V[0] * mux + V[1] * muy) + V[2] * muz) + V[3];
    float py = ((V[4] * mux + V[5] * muy) + V[6] * muz) + V[7];
    float pz = ((V[8] * mux + V[9] * muy) + V[10] * muz) + V[11];
    if (!(pz > 0.0f)) return 0;
    float ux = px / pz, uy = py / pz;
    float J00 = cam->fx / pz, J02 = -((cam->fx * ux) / pz);
    float J11 = cam->fy / pz, J12 = -((cam->fy * uy) / pz);
    float T[2][3];
    for (int k = 0; k < 3; ++k) {
        T[0][k] = J00 * V[0 * 4 + k] + J02 * V[2 * 4 + k];
        T[1][k] = J11 * V[1 * 4 + k] + J12 * V[2 * 4 + k];
    }
    float Wm[2][3];
    for (int a = 0; a < 2; ++a)
        for (int i = 0; i < 3; ++i)
            Wm[a][i] = (S[i][0] * T[a][0] + S[i][1] * T[a][1]) + S[i][2] * T[a][2];
    float ca = (T[0][0] * Wm[0][0] + T[0][1] * Wm[0][1]) + T[0][2] * Wm[0][2];
    float cb = (T[1][0] * Wm[0][0] + T[1][1] * Wm[0][1]) + T[1][2] * Wm[0][2];
    float cc = (T[1][0] * Wm[1][0] + T[1][1] * Wm[1][1]) + T[1][2] * Wm[1][2];
    ca = ca + 0.3f; cc = cc + 0.3f;
    float det = ca * cc - cb * cb;
    if (!(det > 1e-7f)) return 0;
    float ha = -0.5f * (cc / det), nb = cb / det, hc = -0.5f * (ca / det);
    float tr = ca + cc;
    float lam = 0.5f * (tr + sqrtf(fmaxf(0.0f, tr * tr - 4.0f * det)));
    float rf = fminf((float)r_max, ceilf(3.0f * sqrtf(lam)));
    float mx = cam->fx * ux + cam->cx, my = cam->fy * uy + cam->cy;
    float fx0 = fmaxf(ceilf(mx - rf), 0.0f), fx1 = fminf(floorf(mx + rf), (float)(cam->width - 1));
    float fy0 = fmaxf(ceilf(my - rf), 0.0f), fy1 = fminf(floorf(my + rf), (float)(cam->height - 1));
    if (fx0 > fx1 || fy0 > fy1) return 0;
    for (int j = (int)fy0; j <= (int)fy1; ++j)
        for (int i = (int)fx0; i <= (int)fx1; ++i) {
            if (!mask[(int64_t)j * cam->width + i]) continue;
            float dx = mx - (float)i, dy = my - (float)j;
            float u = fmaf(nb, dy, ha * dx);
            float power = fmaf(dx, u, (hc * dy) * dy);
            if (power >= -4.5f) return 1;
        }
    return 0;
}

/* gids: nullable list of n_sel texel ids to label (others untouched); NULL = all n texels */
int orc_label_dynamic(const float* const* planes, int64_t n, const uint8_t* occ, int n_cams, const orc_camera* cams,
                      const uint8_t* masks, int r_max, const int64_t* gids, int64_t n_sel, uint8_t* labels)
{
    int64_t cnt = gids ? n_sel : n;
    for (int64_t s = 0; s < cnt; ++s) {
        int64_t g = gids ? gids[s] : s;
        uint8_t d = 0;
        if (!occ || occ[g])
            for (int c = 0; c < n_cams && !d; ++c)
                d = (uint8_t)label_one_f32(planes, g, &cams[c],
                                            masks + (int64_t)c * cams[0].width * cams[0].height, r_max);
        labels[g] = d;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* atlas layout and packing (R15)                 */

/* Column layout for arbitrary level lists: L0 at (0,0); levels 1.. stacked
 * top-down in one column at x = cols0, unrotated.  out: K x {x, y, rot}. */
int orc_layout_column(int K, const int32_t* rows, const int32_t* cols, int32_t* out, int32_t* W, int32_t* H)
{
    if (K < 1) return -1;
    out[0] = 0; out[1] = 0; out[2] = 0;
    int32_t w = cols[0], h = rows[0], y = 0, colw = 0;
    for (int k = 1; k < K; ++k) {
        out[3 * k] = cols[0]; out[3 * k + 1] = y; out[3 * k + 2] = 0;
        y += rows[k];
        if (cols[k] > colw) colw = cols[k];
    }
    if (y > h) h = y;
    *W = w + colw; *H = h;
    return 0;
}

/* The paper's K <= 8 pyramid atlas as the placement table of
 * scaled by S/1024 (levels: image of M_k = cols columns, N_k = rows rows; odd levels rotated):
 *   k  (M_k, N_k)        x, y (top-left)     rotated
 *   0  (S, S)            (S/2, 0)            no
 *   1  (S, S/2)          (0, 0)              yes
 *   2  (S/2, S/2)        (0, S)              no
 *   3  (S/2, S/4)        (S/2, S)            yes
 *   4  (S/4, S/4)        (3S/4, S)           no
 *   5  (S/4, S/8)        (3S/4, 5S/4)        yes
 *   6  (S/8, S/8)        (7S/8, 5S/4)        no
 *   7  (S/8, S/16)       (7S/8, 11S/8)       yes
 * atlas (3S/2)^2 for K >= 3, 3S/2 x S for K = 2, S x S for K = 1 (L0 then at (0,0)).
 * out: K x {x, y, rot}; rows/cols: K each. */
int orc_layout_paper(int S, int K, int32_t* rows, int32_t* cols, int32_t* out, int32_t* W, int32_t* H)
{
    static const int M8[8] = {8, 8, 4, 4, 2, 2, 1, 1};      /* in units of S/8 */
    static const int N16[8] = {16, 8, 8, 4, 4, 2, 2, 1};    /* in units of S/16 */
    static const int X8[8] = {4, 0, 0, 4, 6, 6, 7, 7};      /* x in units of S/8 */
    static const int Y8[8] = {0, 0, 8, 8, 8, 10, 10, 11};   /* y in units of S/8 */
    if (K < 1 || K > 8 || S < 16 || (S & (S - 1))) return -2;
    for (int k = 0; k < K; ++k) {
        cols[k] = M8[k] * (S / 8);
        rows[k] = N16[k] * (S / 16);
        out[3 * k] = (K == 1) ? 0 : X8[k] * (S / 8);
        out[3 * k + 1] = Y8[k] * (S / 8);
        out[3 * k + 2] = k & 1;
    }
    *W = K > 1 ? S + S / 2 : S;
    *H = K > 2 ? S + S / 2 : S;
    return 0;
}

/* Ray direction of every atlas texel (zero where unplaced): level cell (v = row, u = column),
 * theta = (u + 0.5)/M 2pi - pi, phi = (v + 0.5)/N pi (inverse of PAPER.md eq. uvgs2 at pixel
 * centres), dir = (sin phi cos theta, sin phi sin theta, cos phi) in fp64, rounded. */
int orc_ray_dirs(int K, const int32_t* rows, const int32_t* cols, const int32_t* place, int32_t W_A, int32_t H_A,
                 float* rx, float* ry, float* rz)
{
    const double pi = 3.14159265358979323846;
    int64_t NA = (int64_t)W_A * H_A;
    memset(rx, 0, (size_t)NA * 4); memset(ry, 0, (size_t)NA * 4); memset(rz, 0, (size_t)NA * 4);
    for (int k = 0; k < K; ++k)
        for (int r = 0; r < rows[k]; ++r)
            for (int c = 0; c < cols[k]; ++c) {
                double th = (c + 0.5) / cols[k] * 2.0 * pi - pi, ph = (r + 0.5) / rows[k] * pi;
                int64_t ay = place[3 * k + 2] ? place[3 * k + 1] + cols[k] - 1 - c : place[3 * k + 1] + r;
                int64_t ax = place[3 * k + 2] ? place[3 * k] + r : place[3 * k] + c;
                int64_t o = ay * W_A + ax;
                rx[o] = (float)(sin(ph) * cos(th));
                ry[o] = (float)(sin(ph) * sin(th));
                rz[o] = (float)cos(ph);
            }
    return 0;
}

/* PUV_POS_RHO positions: mu_k = c_k (+) rho (x) ray_k in fp32 (two IEEE ops). */
void orc_positions_from_rho(const float* rho, const float* rx, const float* ry, const float* rz, const float* c,
                            int64_t n, float* x, float* y, float* z)
{
    for (int64_t i = 0; i < n; ++i) {
        x[i] = c[0] + rho[i] * rx[i];
        y[i] = c[1] + rho[i] * ry[i];
        z[i] = c[2] + rho[i] * rz[i];
    }
}

/* d rho = ray . d mu (fp64) */
void orc_rho_grad(const float* rx, const float* ry, const float* rz, const double* gx, const double* gy,
                  const double* gz, int64_t n, double* grho)
{
    for (int64_t i = 0; i < n; ++i) grho[i] = (double)rx[i] * gx[i] + (double)ry[i] * gy[i] + (double)rz[i] * gz[i];
}

/* Level k (rows_k x cols_k, D planes) -> atlas (H_A x W_A).  Unrotated: cell
 * (r, c) -> (y + r, x + c).  rot90ccw: placement is cols_k tall, rows_k wide
 * and cell (r, c) -> (y + cols_k - 1 - c, x + r).  Unplaced pixels: zero and
 * unoccupied.  level_occ[k] nullable (all occupied). */
int orc_pack(int K, const int32_t* rows, const int32_t* cols, const int32_t* place, int D,
             const float* const* level_planes /* K*D pointers, k-major */, const uint8_t* const* level_occ,
             int32_t W_A, int32_t H_A, float* const* atlas_planes, uint8_t* atlas_occ)
{
    int64_t NA = (int64_t)W_A * H_A;
    for (int d = 0; d < D; ++d) memset(atlas_planes[d], 0, (size_t)NA * 4);
    memset(atlas_occ, 0, (size_t)NA);
    for (int k = 0; k < K; ++k) {
        int32_t x = place[3 * k], y = place[3 * k + 1], rot = place[3 * k + 2];
        for (int r = 0; r < rows[k]; ++r)
            for (int c = 0; c < cols[k]; ++c) {
                int64_t ay, ax;
                if (!rot) { ay = y + r; ax = x + c; }
                else { ay = y + cols[k] - 1 - c; ax = x + r; }
                if (ay < 0 || ay >= H_A || ax < 0 || ax >= W_A) return -3;
                int64_t dst = ay * W_A + ax, src = (int64_t)r * cols[k] + c;
                for (int d = 0; d < D; ++d) atlas_planes[d][dst] = level_planes[k * D + d][src];
                atlas_occ[dst] = level_occ && level_occ[k] ? level_occ[k][src] : 1;
            }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-2 low-precision optimisation (LPO): the uniform K-bit fake quantiser  */
/* of PAPER.md:468-474 / 1295-1311 with SPEC.md:298-313's formulas, in the   */
/* fp32 contract (readings Q1-Q7):                             */
/*   L = 2^bits - 1;  t = ((x (-) min) (/) (max (-) min)) (x) L, clamped to   */
/*   [0, L];  code = round-half-away-from-zero(t);             */
/*   proxy = min (+) ((code (/) L) (x) (max (-) min));  max == min -> code 0, */
/*   proxy = min.                                                            */

uint32_t orc_quant_code(float x, float mn, float mx, int bits)
{
    if (mx == mn) return 0;
    const float L = (float)((1u << bits) - 1u);
    float t = ((x - mn) / (mx - mn)) * L;
    if (!(t > 0.0f)) t = 0.0f;          /* also maps NaN to 0 */
    if (t > L) t = L;
    return (uint32_t)roundf(t);
}

float orc_dequant(uint32_t code, float mn, float mx, int bits)
{
    if (mx == mn) return mn;
    const float L = (float)((1u << bits) - 1u);
    return mn + ((float)code / L) * (mx - mn);
}

/* Reading Q8: "we retain them [positions] in FP16" -- the position
 * planes stored as IEEE 754 binary16.  fp32 -> binary16 with round-to-nearest-even, written out on
 * the bit fields: sign; exponent rebiased 127 -> 15; normal halves keep 10 mantissa bits; values
 * below 2^-14 become subnormal halves (mantissa shifted right with the implicit 1); overflow past
 * the largest half (65504) -> infinity; NaN -> the quiet NaN 0x7e00.  Returns the 16-bit pattern. */
uint32_t orc_fp16_bits(float x)
{
    const uint32_t b = bits_from_f(x);
    const uint32_t sign = (b >> 16) & 0x8000u;
    const int32_t e = (int32_t)((b >> 23) & 0xffu);
    uint32_t m = b & 0x7fffffu;
    if (e == 0xff) return sign | (m ? 0x7e00u : 0x7c00u);         /* inf / NaN */
    int32_t he = e - 127 + 15;                                     /* half exponent field */
    if (he >= 0x1f) return sign | 0x7c00u;                         /* too large: inf */
    uint32_t mant;                                                 /* 1.m as a 24-bit integer (normal) */
    int shift;                                                     /* bits dropped */
    if (he <= 0) {                                                 /* subnormal half (or zero) */
        if (e == 0) return sign;                                   /* fp32 zero / subnormal: |x| < 2^-126 */
        mant = m | 0x800000u;
        shift = 13 + 1 - he;
        if (shift > 24) return sign;                               /* below half the smallest subnormal */
        he = 0;
    } else {
        mant = m;
        shift = 13;
    }
    uint32_t q = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) q += 1u;          /* round to nearest, ties to even */
    /* a carry out of the mantissa bumps the exponent (also subnormal -> smallest normal, max -> inf) */
    return sign | ((((uint32_t)he << 10) + q) & 0xffffu);
}

/* The binary16 value of a 16-bit pattern, as fp32 (exact). */
float orc_fp16_value(uint32_t h)
{
    const uint32_t sign = (h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
    if (e == 0x1f) return f_from_bits(sign | 0x7f800000u | (m << 13));
    if (e == 0) {                                                  /* subnormal: m * 2^-24 */
        const float v = (float)m * 5.9604644775390625e-8f;
        return sign ? -v : v;
    }
    return f_from_bits(sign | ((e - 15 + 127) << 23) | (m << 13));
}

/* Position plane stored as binary16: code = the 16-bit pattern, proxy = its value; unoccupied 0. */
void orc_quantize_plane_fp16(const float* x, const uint8_t* occ, int64_t n, uint32_t* code, float* proxy)
{
    for (int64_t i = 0; i < n; ++i) {
        if (occ && !occ[i]) { code[i] = 0; proxy[i] = 0.0f; continue; }
        code[i] = orc_fp16_bits(x[i]);
        proxy[i] = orc_fp16_value(code[i]);
    }
}

/* Per-plane min/max over occupied texels; no occupied texel -> (0, 0). */
void orc_quant_fit(int D, const float* const* planes, const uint8_t* occ, int64_t n, float* spec /* D x 2 */)
{
    for (int d = 0; d < D; ++d) {
        float mn = 0.0f, mx = 0.0f;
        int any = 0;
        if (planes[d])
            for (int64_t i = 0; i < n; ++i) {
                if (occ && !occ[i]) continue;
                const float v = planes[d][i];
                if (!any || v < mn) mn = v;
                if (!any || v > mx) mx = v;
                any = 1;
            }
        spec[2 * d] = mn;
        spec[2 * d + 1] = mx;
    }
}

/* Codes (uint32) and proxy of one plane; unoccupied texels: code 0, proxy 0. */
void orc_quantize_plane(const float* x, const uint8_t* occ, int64_t n, float mn, float mx, int bits, uint32_t* code,
                        float* proxy)
{
    for (int64_t i = 0; i < n; ++i) {
        if (occ && !occ[i]) { code[i] = 0; proxy[i] = 0.0f; continue; }
        code[i] = orc_quant_code(x[i], mn, mx, bits);
        proxy[i] = orc_dequant(code[i], mn, mx, bits);
    }
}
