"""Seeded synthetic scenes shaped like the paper's multi-view captures.

This module is the ONE thing the CPU oracle (`oracle/`) and the CUDA path
(`paper_2602_23040_b200/`) share: it produces inputs only.  It holds none of
the method's arithmetic — no unpacking, projection, binning, compositing,
packing layout or gradient — just random draws, camera poses and the
"UV-coherent" ordering of samples inside each atlas level.

Workloads follow BASELINE.json `configs` (BJ.configs[i]); the recipe and the
draw order are stated in DESIGN.md §3.  The paper's datasets (PackUV-2B,
N3DV, SelfCap) are not available; these scenes stand in
for them with the shapes the paper names (55-88 cameras around a dynamic
scene, 1024^2 atlas levels).

Texel record (per atlas level, SoA planes, float32):
    [x, y, z, ls0, ls1, ls2, qw, qx, qy, qz, logit_o, sh(k, c) ...]
with SH plane index 11 + 3k + c, k < (deg+1)^2 (reading R2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_ROOT = (2602, 23040)
NEAR = 0.2
TILE = 16


def n_planes(sh_degree: int) -> int:
    return 11 + 3 * (sh_degree + 1) ** 2


@dataclass
class Camera:
    """Pinhole camera, OpenCV axes (x right, y down, z forward).

    viewmat: float32 (4, 4) row-major world -> camera.
    campos: float32 (3,) camera centre in world space.
    """
    viewmat: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float
    campos: np.ndarray


@dataclass
class Level:
    """One UV level: D planes of rows x cols texels (M_k x N_k)."""
    planes: np.ndarray          # float32 (D, rows, cols)
    occ: np.ndarray             # uint8 (rows, cols)
    labels: np.ndarray          # uint8 (rows, cols), dynamic label D_i

    @property
    def rows(self) -> int:
        return self.planes.shape[1]

    @property
    def cols(self) -> int:
        return self.planes.shape[2]


@dataclass
class Scene:
    cfg: int
    sh_degree: int
    levels: list[Level]
    cameras: list[Camera]
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def D(self) -> int:
        return n_planes(self.sh_degree)

    def target(self, view: int, frame: int | None = None) -> np.ndarray:
        """Seeded U[0,1] target image (3, H, W) float32 for `view` (BJ.configs[0]); for a frame
        sequence (C4) one image per (frame, view)."""
        cam = self.cameras[view]
        seq = [*SEED_ROOT, self.cfg, 1, view] if frame is None else [*SEED_ROOT, self.cfg, 3, frame, view]
        rng = np.random.default_rng(np.random.SeedSequence(seq))
        return rng.random((3, cam.height, cam.width), dtype=np.float32)


# ----------------------------------------------------------------------------
# cameras


def look_at(eye, target, width, height, f, up=(0.0, 0.0, 1.0)) -> Camera:
    """World->camera pose of a camera at `eye` looking at `target`, world z up."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    V = np.eye(4)
    V[:3, :3] = R
    V[:3, 3] = -R @ eye
    return Camera(viewmat=V.astype(np.float32), fx=float(f), fy=float(f),
                  cx=(width - 1) / 2.0, cy=(height - 1) / 2.0,
                  width=int(width), height=int(height), near=NEAR,
                  campos=eye.astype(np.float32))


def ring(n, radius, z, width, height, f, offset=0.0, target=(0.0, 0.0, 0.0)):
    cams = []
    for i in range(n):
        a = offset + 2.0 * math.pi * i / n
        cams.append(look_at((radius * math.cos(a), radius * math.sin(a), z), target, width, height, f))
    return cams


def dome(n, radius, el_lo_deg, el_hi_deg, width, height, f, target=(0.0, 0.0, 0.0)):
    """n cameras on a dome: elevations evenly in [lo, hi], golden-angle azimuths."""
    cams = []
    golden = math.pi * (3.0 - math.sqrt(5.0))
    tx, ty, tz = target
    for i in range(n):
        el = math.radians(el_lo_deg + (el_hi_deg - el_lo_deg) * (i + 0.5) / n)
        az = i * golden
        eye = (tx + radius * math.cos(el) * math.cos(az), ty + radius * math.cos(el) * math.sin(az),
               tz + radius * math.sin(el))
        cams.append(look_at(eye, target, width, height, f))
    return cams


# ----------------------------------------------------------------------------
# Gaussian attribute draws (shared distributions)


def _uv_coherent_order(pos: np.ndarray, rows: int, cols: int, centre) -> np.ndarray:
    """Order samples by their spherical UV cell about `centre`.

    Only used to lay samples out so that neighbouring texels are spatially
    coherent, like a fitted PackUV level; it is not part of the render.
    """
    d = pos.astype(np.float64) - np.asarray(centre, np.float64)
    rho = np.linalg.norm(d, axis=1)
    theta = np.arctan2(d[:, 1], d[:, 0])
    phi = np.arccos(np.clip(d[:, 2] / np.maximum(rho, 1e-12), -1.0, 1.0))
    u = np.clip(np.floor((math.pi + theta) / (2 * math.pi) * rows), 0, rows - 1).astype(np.int64)
    v = np.clip(np.floor(phi / math.pi * cols), 0, cols - 1).astype(np.int64)
    return np.lexsort((rho, v, u))


def _attributes(rng, n, sh_degree):
    """Draws in the documented order after positions: log-scales, quats, logits, SH DC, SH rest."""
    ls = rng.normal(-3.5, 0.3, size=(n, 3))
    q = rng.normal(0.0, 1.0, size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    lo = rng.normal(0.0, 1.0, size=(n, 1))
    dc = rng.random((n, 3))
    nrest = (sh_degree + 1) ** 2 - 1
    rest = rng.normal(0.0, 0.05, size=(n, 3 * nrest))
    return np.concatenate([ls, q, lo, dc, rest], axis=1)


def _blobs(rng, n, n_blobs, centre_lo, centre_hi, sig_lo, sig_hi):
    centres = rng.uniform(centre_lo, centre_hi, size=(n_blobs, 3))
    sig = rng.uniform(sig_lo, sig_hi, size=(n_blobs, 3))
    rots = []
    for _ in range(n_blobs):
        # random orthogonal frame (QR of a Gaussian matrix, sign-fixed)
        qm, rm = np.linalg.qr(rng.normal(size=(3, 3)))
        rots.append(qm * np.sign(np.diag(rm)))
    which = rng.integers(0, n_blobs, size=n)
    eps = rng.normal(size=(n, 3)) * sig[which]
    out = np.einsum("nij,nj->ni", np.stack(rots)[which], eps) + centres[which]
    return out


def _fill_levels(rng, pos, sh_degree, shapes, centre, occupied_fraction=None):
    """Split samples over levels (in order), UV-order each level, draw attributes, labels."""
    n = pos.shape[0]
    attrs = _attributes(rng, n, sh_degree)
    labels = (rng.random(n) < 0.25).astype(np.uint8)
    levels = []
    start = 0
    D = n_planes(sh_degree)
    for (rows, cols) in shapes:
        cnt = rows * cols
        sl = slice(start, start + cnt)
        p = pos[sl]
        order = _uv_coherent_order(p, rows, cols, centre)
        rec = np.concatenate([p, attrs[sl]], axis=1)[order]
        assert rec.shape[1] == D
        planes = np.ascontiguousarray(rec.T.reshape(D, rows, cols)).astype(np.float32)
        occ = np.ones((rows, cols), np.uint8)
        lab = labels[sl][order].reshape(rows, cols)
        levels.append(Level(planes=planes, occ=occ, labels=lab))
        start += cnt
    assert start == n
    return levels


# ----------------------------------------------------------------------------
# configs (BJ.configs)


def make_scene(cfg: int, views: int | None = None) -> Scene:
    """Build BASELINE.json configs[cfg-1] (cfg is 1-based like SURVEY.md's C1..C5)."""
    rng = np.random.default_rng(np.random.SeedSequence([*SEED_ROOT, cfg]))
    if cfg == 1:
        n = 64 * 64
        pos = rng.uniform(-1.0, 1.0, size=(n, 3))
        levels = _fill_levels(rng, pos, 0, [(64, 64)], (0, 0, 0))
        cams = [look_at((4.0, 0.0, 0.0), (0, 0, 0), 128, 128, 150.0)]
        sc = Scene(cfg, 0, levels, cams, "C1: 64x64 atlas, 1 view 128x128")
    elif cfg == 2:
        shapes = [(512, 512), (256, 256), (128, 128)]
        n = sum(r * c for r, c in shapes)
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pos = d * rng.uniform(0.8, 1.2, size=(n, 1))
        levels = _fill_levels(rng, pos, 1, shapes, (0, 0, 0))
        cams = ring(16, 3.0, 0.0, 1024, 768, 900.0)
        sc = Scene(cfg, 1, levels, cams, "C2: 512^2+256^2+128^2 levels, 16 views 1024x768")
    elif cfg == 3 or cfg == 4:
        n = 1024 * 1024
        nb = int(round(0.8 * n))
        blob = _blobs(rng, nb, 8, -1.5, 1.5, 0.1, 0.5)
        bg = rng.uniform(-2.0, 2.0, size=(n - nb, 3))
        pos = np.concatenate([blob, bg], axis=0)
        pos = pos[rng.permutation(n)]
        levels = _fill_levels(rng, pos, 3, [(1024, 1024)], (0, 0, 0))
        if cfg == 3:
            cams = ring(32, 3.5, 1.0, 1920, 1080, 1400.0) + \
                ring(32, 3.5, 2.0, 1920, 1080, 1400.0, offset=math.pi / 32)
            sc = Scene(cfg, 3, levels, cams, "C3: 1024^2 atlas SH3, 64 views 1920x1080")
        else:
            cams = dome(55, 3.5, 10.0, 60.0, 1920, 1080, 1400.0)
            sc = Scene(cfg, 3, levels, cams, "C4: 30 frames of 1024^2 SH3, 55 views 1920x1080")
            sc.meta["frames"] = 30
            sc.meta["flow"] = _flow_field(rng)
    elif cfg == 5:
        n0, n1 = 2048 * 2048, 1024 * 1024
        blob = _blobs(rng, n0, 32, np.array([-3.0, -3.0, 0.2]), np.array([3.0, 3.0, 2.5]), 0.1, 0.6)
        floor = np.concatenate([rng.uniform(-4.0, 4.0, size=(n1, 2)), np.zeros((n1, 1))], axis=1)
        pos = np.concatenate([blob, floor], axis=0)
        levels = _fill_levels(rng, pos, 3, [(2048, 2048), (1024, 1024)], (0, 0, 1.0))
        cams = dome(88, 6.0, 10.0, 60.0, 3840, 2160, 2800.0, target=(0.0, 0.0, 1.0))
        sc = Scene(cfg, 3, levels, cams, "C5: 2048^2+1024^2 levels SH3, 88 views 3840x2160")
    else:
        raise ValueError(f"unknown config {cfg}")
    if views is not None:
        sc.cameras = sc.cameras[:views]
    return sc


def rho_scene(cfg: int, shapes, sh_degree: int, cams, centre=(0.0, 0.0, 0.0)) -> Scene:
    """Seeded inputs of the paper-native atlas (NEXT-1): levels of the given
    (rows, cols) whose plane 0 holds rho (distance along the texel's UV ray about `centre`,
    PAPER.md:211-215) and planes 1, 2 are unused (zero).  rho = 1 + 0.25 sin(3 a + p) sin(2 b + q)
    + N(0, 0.03) on the level grid (a = 2 pi c / cols, b = pi r / rows): a smooth closed surface
    with per-texel jitter, like a fitted shell.  The remaining planes use the shared draws."""
    rng = np.random.default_rng(np.random.SeedSequence([*SEED_ROOT, cfg]))
    D = n_planes(sh_degree)
    levels = []
    for (rows, cols) in shapes:
        n = rows * cols
        p, q = rng.uniform(0, 2 * math.pi, size=2)
        b, a = np.meshgrid(math.pi * (np.arange(rows) + 0.5) / rows, 2 * math.pi * (np.arange(cols) + 0.5) / cols,
                           indexing="ij")
        rho = 1.0 + 0.25 * np.sin(3 * a + p) * np.sin(2 * b + q) + rng.normal(0, 0.03, size=(rows, cols))
        attrs = _attributes(rng, n, sh_degree)
        planes = np.zeros((D, rows, cols), np.float32)
        planes[0] = rho
        planes[3:] = attrs.T.reshape(D - 3, rows, cols)
        labels = (rng.random((rows, cols)) < 0.25).astype(np.uint8)
        levels.append(Level(planes=planes, occ=np.ones((rows, cols), np.uint8), labels=labels))
    sc = Scene(cfg, sh_degree, levels, list(cams), f"rho atlas {shapes[0]}.. K={len(shapes)}")
    sc.meta["centre"] = tuple(float(x) for x in centre)
    return sc


def _flow_field(rng):
    """Smooth seeded flow u_a(p) = sin(k_a . p + phi_a)/sqrt(3), |k_a| = 2 rad/m (C4)."""
    k = rng.normal(size=(3, 3))
    k = 2.0 * k / np.linalg.norm(k, axis=1, keepdims=True)
    ph = rng.uniform(0, 2 * math.pi, size=3)
    return k, ph


def frame_positions(scene: Scene, frame: int) -> np.ndarray:
    """C4: dynamic texels move mu_t = mu_0 + 0.05 (t/29) u(mu_0); static texels fixed."""
    k, ph = scene.meta["flow"]
    lv = scene.levels[0]
    mu0 = lv.planes[0:3].reshape(3, -1).T.astype(np.float64)
    u = np.sin(mu0 @ k.T + ph) / math.sqrt(3.0)
    dyn = lv.labels.reshape(-1).astype(bool)
    mu = mu0.copy()
    mu[dyn] += 0.05 * (frame / 29.0) * u[dyn]
    return np.ascontiguousarray(mu.T.reshape(3, lv.rows, lv.cols)).astype(np.float32)


def motion_masks(scene: Scene, views, n_blobs=6, rmin=0.03, rmax=0.12, tag=2) -> np.ndarray:
    """Seeded stand-in for thresholded + dilated optical-flow masks (RAFT is out of
    scope): per view, the union of n_blobs discs with radii U[rmin, rmax] x image height at uniform
    centres.  Returns (len(views), H, W) uint8 in {0, 1}."""
    cam0 = scene.cameras[views[0]]
    H, W = cam0.height, cam0.width
    out = np.zeros((len(views), H, W), np.uint8)
    jj, ii = np.mgrid[0:H, 0:W]
    for k, v in enumerate(views):
        rng = np.random.default_rng(np.random.SeedSequence([*SEED_ROOT, scene.cfg, tag, v]))
        for _ in range(n_blobs):
            cx, cy = rng.uniform(0, W), rng.uniform(0, H)
            r = rng.uniform(rmin, rmax) * H
            out[k][(ii - cx) ** 2 + (jj - cy) ** 2 <= r * r] = 1
    return out


def moving_region_masks(scene: Scene, views, centre, radius, tag=4) -> np.ndarray:
    """Seeded stand-in for thresholded + dilated optical-flow masks of a spatially coherent motion
    (PAPER.md:362-378): the moving part of the scene is the ball |x - centre| <= radius; in every
    view its mask is the image disc the ball projects to (centre projected, angular radius
    asin(radius / distance)), so only Gaussians that overlap the moving region in some camera can
    be labelled dynamic.  Returns (len(views), H, W) uint8 in {0, 1}."""
    cam0 = scene.cameras[views[0]]
    H, W = cam0.height, cam0.width
    out = np.zeros((len(views), H, W), np.uint8)
    jj, ii = np.mgrid[0:H, 0:W]
    c = np.asarray(centre, np.float64)
    for k, v in enumerate(views):
        cam = scene.cameras[v]
        V = cam.viewmat.astype(np.float64)
        p = V[:3, :3] @ c + V[:3, 3]
        if p[2] <= radius:
            out[k] = 1          # the camera is inside / behind the ball's near side: all pixels move
            continue
        u, w_ = cam.fx * p[0] / p[2] + cam.cx, cam.fy * p[1] / p[2] + cam.cy
        r_px = cam.fx * math.tan(math.asin(min(1.0, radius / float(np.linalg.norm(p)))))
        out[k][(ii - u) ** 2 + (jj - w_) ** 2 <= r_px * r_px] = 1
    return out


# ----------------------------------------------------------------------------
# tiny hand-built scenes for pins (tests)


def tiny_scene(mu, log_scale, quat, logit, sh, cam: Camera, sh_degree=0) -> Scene:
    """A one-level scene from explicit per-Gaussian arrays (n Gaussians in a 1 x n level)."""
    mu = np.atleast_2d(np.asarray(mu, np.float32))
    n = mu.shape[0]
    rec = np.concatenate([mu, np.broadcast_to(np.asarray(log_scale, np.float32), (n, 3)),
                          np.broadcast_to(np.asarray(quat, np.float32), (n, 4)),
                          np.broadcast_to(np.asarray(logit, np.float32).reshape(-1, 1), (n, 1)),
                          np.broadcast_to(np.asarray(sh, np.float32), (n, 3 * (sh_degree + 1) ** 2))], axis=1)
    planes = np.ascontiguousarray(rec.T.reshape(-1, 1, n)).astype(np.float32)
    lv = Level(planes=planes, occ=np.ones((1, n), np.uint8), labels=np.ones((1, n), np.uint8))
    return Scene(0, sh_degree, [lv], [cam], "tiny")
