"""Pins of the CPU oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it pins (PAPER.md line, SPEC.md line or DESIGN.md
reading).  None of them re-types the oracle's formula: they use closed forms,
independent numerical derivatives, brute force on tiny inputs, quadrature,
finite differences and invariants (DESIGN.md §4 lists what pins what).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import orc
from synth.scenes import Camera, look_at, tiny_scene, make_scene

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def ident_cam(W, H, f, cx, cy):
    return Camera(viewmat=np.eye(4, dtype=np.float32), fx=f, fy=f, cx=cx, cy=cy, width=W, height=H,
                  near=0.2, campos=np.zeros(3, np.float32))


def conic_to_cov(p):
    """(ha, nb, hc) -> Sigma2D: power = ha dx^2 + nb dx dy + hc dy^2 = -1/2 d^T Sigma^-1 d."""
    A, B, Cc = -2.0 * float(p["ha"]), -float(p["nb"]), -2.0 * float(p["hc"])
    inv = np.array([[A, B], [B, Cc]])
    return np.linalg.inv(inv)


def single(mu, ls, q, logit, dc, cam, deg=0):
    sh = np.zeros(3 * (deg + 1) ** 2, np.float32)
    sh[:3] = dc
    sc = tiny_scene(mu, ls, q, logit, sh, cam, deg)
    return sc


def planes_of(sc):
    planes, occ, _ = orc.pack(sc.levels)
    return planes, occ


# ---------------------------------------------------------------------------
# contract functions exp_c / log_c (R13)

def test_exp_c_accuracy_and_specials():
    x = np.linspace(-86.99, 87.99, 1_000_001, dtype=np.float32)
    y = orc.exp_c(x).astype(np.float64)
    ref = np.exp(x.astype(np.float64))
    rel = np.abs(y - ref) / ref
    assert rel.max() < 2 * 2.0 ** -24 * 1.01, rel.max()       # <= 2 ulp vs fp64 libm
    sp = orc.exp_c(np.array([0.0, 88.0, 100.0, -87.0, -100.0], np.float32))
    assert sp[0] == 1.0 and np.isinf(sp[1]) and np.isinf(sp[2]) and sp[3] == 0.0 and sp[4] == 0.0
    assert np.all(np.diff(y[::1000]) >= 0)                     # monotone on a coarse grid
    # near k ln2 (range-reduction boundaries) still within 2 ulp of exp of the fp32 input
    for k in (-20, -1, 1, 7, 30):
        xk = np.float32(k * math.log(2.0))
        v = float(orc.exp_c(np.array([xk], np.float32))[0])
        assert abs(v / math.exp(float(xk)) - 1.0) < 2 * 2.0 ** -24


def test_log_c_accuracy_and_specials():
    y = np.exp(np.linspace(math.log(1.2e-38), math.log(3e38), 1_000_001)).astype(np.float32)
    lc = orc.log_c(y).astype(np.float64)
    ref = np.log(y.astype(np.float64))
    err = np.abs(lc - ref)
    assert (err / np.maximum(np.abs(ref), 1e-30)).max() < 4 * 2.0 ** -24
    near1 = (np.float32(1.0) + np.arange(-3000, 3000, dtype=np.float32) * np.float32(2 ** -23)).astype(np.float32)
    lc = orc.log_c(near1).astype(np.float64)
    ref = np.log(near1.astype(np.float64))
    m = ref != 0
    assert (np.abs(lc - ref)[m] / np.abs(ref[m])).max() < 4 * 2.0 ** -24
    sp = orc.log_c(np.array([1.0, 0.0, 1e-40], np.float32))
    assert sp[0] == 0.0 and np.isneginf(sp[1]) and np.isneginf(sp[2])


# ---------------------------------------------------------------------------
# SH basis (R3): orthonormal on the sphere (pins every constant and
# polynomial; a wrong constant breaks normality, a wrong polynomial orthogonality)

def test_sh_basis_signs_vs_scipy_legendre():
    """Every basis function, sign included, against an independent construction (R3):
    the real SH formed from scipy's complex Y_l^m (associated Legendre functions WITH the
    Condon-Shortley phase (-1)^m) as  Y_{l,m} = sqrt2 Re Y_l^m (m > 0),  Y_l^0 (m = 0),
    sqrt2 Im Y_l^|m| (m < 0), index k = l^2 + l + m.  This is the convention of the 3DGS
    constants the paper's renderer inherits: at degree 1 it is sqrt(3/4pi) (-y, z, -x).
    Orthonormality alone would accept any sign flip; this pin does not."""
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(7)
    d = rng.normal(size=(500, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    polar = np.arccos(np.clip(d[:, 2], -1, 1))
    azim = np.arctan2(d[:, 1], d[:, 0])
    ref = np.zeros((d.shape[0], 16))
    for l in range(4):
        for m in range(-l, l + 1):
            c = sph_harm_y(l, abs(m), polar, azim)     # complex, Condon-Shortley phase included
            ref[:, l * l + l + m] = (math.sqrt(2) * c.real if m > 0 else
                                     (c.real if m == 0 else math.sqrt(2) * c.imag))
    Y = orc.sh_basis(3, d)
    assert np.abs(Y - ref).max() < 1e-12, np.abs(Y - ref).max(axis=0)
    c1 = math.sqrt(3 / (4 * math.pi))
    assert np.allclose(Y[:, 1:4], c1 * np.stack([-d[:, 1], d[:, 2], -d[:, 0]], 1), atol=1e-14)


def test_sh_basis_orthonormal():
    nt, nph = 64, 48
    xg, wg = np.polynomial.legendre.leggauss(nph)             # exact in cos(phi) for deg <= 95
    th = (np.arange(nt) + 0.5) * 2 * math.pi / nt
    ct = np.repeat(xg, nt)
    st = np.sqrt(1 - ct ** 2)
    tt = np.tile(th, nph)
    dirs = np.stack([st * np.cos(tt), st * np.sin(tt), ct], axis=1)
    w = np.repeat(wg, nt) * (2 * math.pi / nt)
    Y = orc.sh_basis(3, dirs)
    G = (Y * w[:, None]).T @ Y
    assert np.abs(G - np.eye(16)).max() < 1e-12


# ---------------------------------------------------------------------------
# projection closed forms

def test_ewa_unit_depth_identity_spec_example():
    """mu_cam=(0,0,1), fx=fy=1, Sigma=I -> Sigma2D = diag(1.3, 1.3) (+0.3 low-pass)."""
    cam = ident_cam(81, 81, 1.0, 40.0, 40.0)
    sc = single([0, 0, 1], [0, 0, 0], [1, 0, 0, 0], 0.0, [0.5] * 3, cam)
    p = orc.project(*planes_of(sc), cam)[0]
    assert p["visible"] == 1
    S = conic_to_cov(p)
    np.testing.assert_allclose(S, np.diag([1.3, 1.3]), rtol=1e-6, atol=1e-7)
    assert p["mx"] == 40.0 and p["my"] == 40.0
    # r = ceil(3 sqrt(1.3)) = 4 -> rect covers pixels 36..44 -> tile 2 only
    assert (p["x0"], p["x1"], p["y0"], p["y1"]) == (2, 3, 2, 3)
    assert p["depth_bits"] == np.float32(1.0).view(np.uint32)


@pytest.mark.parametrize("theta", [0.0, 0.4, 1.1])
def test_ewa_on_axis_rotated_anisotropic(theta):
    """On the optical axis J = diag(f/d, f/d): Sigma2D = (f/d)^2 R2 diag(sx^2, sy^2) R2^T + 0.3 I."""
    f, d = 200.0, 5.0
    sx, sy, sz = 0.08, 0.03, 0.05
    q = [math.cos(theta / 2), 0, 0, math.sin(theta / 2)]       # rotation about camera z
    cam = ident_cam(97, 97, f, 48.0, 48.0)
    sc = single([0, 0, d], np.log([sx, sy, sz]), q, 1.0, [0.5] * 3, cam)
    p = orc.project(*planes_of(sc), cam)[0]
    c, s = math.cos(theta), math.sin(theta)
    R2 = np.array([[c, -s], [s, c]])
    ref = (f / d) ** 2 * R2 @ np.diag([sx ** 2, sy ** 2]) @ R2.T + 0.3 * np.eye(2)
    np.testing.assert_allclose(conic_to_cov(p), ref, rtol=2e-5, atol=1e-6)
    lam = np.linalg.eigvalsh(ref).max()
    r = math.ceil(3 * math.sqrt(lam))
    assert (p["x0"], p["x1"]) == (max(0, math.floor((48 - r) / 16)), min(7, math.floor((48 + r) / 16) + 1))
    # o = sigmoid(1), t_g = -ln(255 o)
    assert abs(float(p["o"]) - 1 / (1 + math.exp(-1.0))) < 1e-7
    assert abs(float(p["t_g"]) + math.log(255 / (1 + math.exp(-1.0)))) < 2e-6


def _numeric_ewa(mu, cov3, cam):
    """Independent EWA: pixel(p) = K [R|t] p by homogeneous projection; J by central differences."""
    V = cam.viewmat.astype(np.float64)
    K = np.array([[cam.fx, 0, cam.cx], [0, cam.fy, cam.cy], [0, 0, 1.0]])
    P = K @ V[:3]

    def pix(x):
        h = P @ np.append(x, 1.0)
        return h[:2] / h[2]
    m = pix(mu)
    J = np.zeros((2, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = 1e-6
        J[:, k] = (pix(mu + e) - pix(mu - e)) / 2e-6
    return m, J @ cov3 @ J.T + 0.3 * np.eye(2)


def test_ewa_general_camera_vs_numerical_jacobian():
    cam = look_at((3.0, 1.0, 1.5), (0.1, -0.2, 0.0), 160, 120, 140.0)
    rng = np.random.default_rng(5)
    for _ in range(20):
        mu = rng.uniform(-0.5, 0.5, 3)
        ls = rng.normal(-2.5, 0.3, 3)
        q = rng.normal(size=4)
        sc = single(mu, ls, q, 0.3, [0.5] * 3, cam)
        p = orc.project(*planes_of(sc), cam)[0]
        assert p["visible"] and p["clamp_x"] == 0 and p["clamp_y"] == 0
        qn = q / np.linalg.norm(q)
        w, x, y, z = qn
        # rotation via Rodrigues from axis-angle (independent of the quaternion-matrix formula)
        ang = 2 * math.acos(np.clip(w, -1, 1))
        axis = np.array([x, y, z]) / max(math.sin(ang / 2), 1e-12)
        Kx = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
        Rm = np.eye(3) + math.sin(ang) * Kx + (1 - math.cos(ang)) * Kx @ Kx
        cov3 = Rm @ np.diag(np.exp(2 * ls)) @ Rm.T
        m, S = _numeric_ewa(mu.astype(np.float32).astype(np.float64), cov3, cam)
        assert abs(float(p["mx"]) - m[0]) < 2e-3 and abs(float(p["my"]) - m[1]) < 2e-3
        np.testing.assert_allclose(conic_to_cov(p), S, rtol=2e-4, atol=2e-4)


def test_culling_behind_and_near():
    cam = ident_cam(64, 64, 50.0, 31.5, 31.5)
    for z in (-1.0, 0.0, 0.1, 0.2):                            # z <= near -> invisible
        sc = single([0, 0, z], [-2, -2, -2], [1, 0, 0, 0], 0.0, [0.5] * 3, cam)
        assert orc.project(*planes_of(sc), cam)[0]["visible"] == 0
    sc = single([0, 0, 0.2001], [-2, -2, -2], [1, 0, 0, 0], 0.0, [0.5] * 3, cam)
    assert orc.project(*planes_of(sc), cam)[0]["visible"] == 1
    # zero quaternion -> invisible (R15); far off-screen -> empty rect -> invisible
    sc = single([0, 0, 2], [-2, -2, -2], [0, 0, 0, 0], 0.0, [0.5] * 3, cam)
    assert orc.project(*planes_of(sc), cam)[0]["visible"] == 0
    sc = single([50, 0, 2], [-6, -6, -6], [1, 0, 0, 0], 0.0, [0.5] * 3, cam)
    assert orc.project(*planes_of(sc), cam)[0]["visible"] == 0


def test_jacobian_clamp_flag():
    """R5: |x/z| beyond 1.3 tan(fov/2) clamps J only; the mean stays unclamped."""
    W, f = 64, 80.0
    cam = ident_cam(W, W, f, 31.5, 31.5)
    lim = 1.3 * 0.5 * W / f
    sc = single([0.6 * 2, 0, 2], np.log([0.5, 0.5, 0.5]), [1, 0, 0, 0], 0.0, [0.5] * 3, cam)
    p = orc.project(*planes_of(sc), cam)[0]
    assert 0.6 > lim and p["visible"] and p["clamp_x"] == 1 and p["clamp_y"] == 0
    assert abs(float(p["mx"]) - (f * 0.6 + 31.5)) < 1e-4
    # isotropic s: a = s^2 (f/z)^2 (1 + lim^2) + 0.3 with the clamped coordinate
    s2, fz = 0.25, f / 2
    a_ref = s2 * fz * fz * (1 + lim * lim) + 0.3
    c_ref = s2 * fz * fz + 0.3
    np.testing.assert_allclose(conic_to_cov(p), np.diag([a_ref, c_ref]), rtol=2e-5, atol=1e-4)


# ---------------------------------------------------------------------------
# forward closed forms (PAPER.md:189-195 + DESIGN.md R9)

SH_C0 = 1.0 / (2.0 * math.sqrt(math.pi))


def test_single_gaussian_footprint():
    f, d, s = 100.0, 4.0, 0.1
    cam = ident_cam(65, 65, f, 32.0, 32.0)
    logit, dc = 2.0, np.array([0.2, 0.6, 0.9])
    sc = single([0, 0, d], np.log([s, s, s]), [1, 0, 0, 0], logit, dc, cam)
    planes, occ = planes_of(sc)
    img, T, nc, st = orc.forward(planes, occ, 0, cam)
    o = 1 / (1 + math.exp(-logit))
    s32 = math.exp(float(np.float32(math.log(s))))             # the stored plane is fp32
    a = (f * s32 / d) ** 2 + 0.3
    jj, ii = np.mgrid[0:65, 0:65]
    power = -0.5 * ((ii - 32.0) ** 2 + (jj - 32.0) ** 2) / a
    tg = -math.log(255 * o)
    r = math.ceil(3 * math.sqrt(a))
    t0, t1 = math.floor((32 - r) / 16), math.floor((32 + r) / 16) + 1
    intile = (ii // 16 >= t0) & (ii // 16 < t1) & (jj // 16 >= t0) & (jj // 16 < t1)
    alpha = np.minimum(0.99, o * np.exp(power))
    on = (power >= tg) & intile
    rgb = SH_C0 * dc.astype(np.float32).astype(np.float64) + 0.5
    ref = alpha[None] * on[None] * rgb[:, None, None]
    safe = np.abs(power - tg) > 1e-4
    np.testing.assert_allclose(img[:, safe], ref[:, safe], atol=1e-9, rtol=1e-9)
    assert np.array_equal(nc[safe], on[safe].astype(np.int32))
    # peak alpha at the mean pixel = min(0.99, o)
    assert abs(img[0, 32, 32] - min(0.99, o) * rgb[0]) < 1e-12
    assert on.sum() > 100 and st["n_vis"] == 1 and st["K"] == (t1 - t0) ** 2


def test_termination_closed_form():
    """20 co-located Gaussians, o = 1/2 at the mean pixel: 13 composited, T = 2^-13 (R9)."""
    golden = json.load(open(os.path.join(GOLDEN, "termination.json")))
    cam = ident_cam(33, 33, 60.0, 16.0, 16.0)
    n = golden["n_gaussians"]
    sc = tiny_scene(np.tile([0, 0, 4.0], (n, 1)), [-2.5] * 3, [1, 0, 0, 0], np.zeros(n), [0.0, 0.0, 0.0], cam, 0)
    planes, occ = planes_of(sc)
    img, T, nc, _ = orc.forward(planes, occ, 0, cam)
    assert nc[16, 16] == golden["n_contrib"]
    assert T[16, 16] == np.float32(2.0 ** -golden["n_contrib"])
    np.testing.assert_allclose(img[:, 16, 16], 0.5 * (1 - 2.0 ** -13), rtol=0, atol=1e-15)


def test_two_gaussians_order():
    cam = ident_cam(33, 33, 60.0, 16.0, 16.0)
    lg = np.array([0.5, -0.3])
    o = 1 / (1 + np.exp(-lg))
    dc = np.array([[0.9, 0.1, 0.3], [0.1, 0.8, 0.6]])
    rgb = SH_C0 * dc + 0.5

    def render(z1, z2):
        mu = [[0, 0, z1], [0, 0, z2]]
        sh = dc.astype(np.float32)
        sc = tiny_scene(mu, [-3.0] * 3, [1, 0, 0, 0], lg, np.zeros(3), cam, 0)
        sc.levels[0].planes[11:14, 0, :] = sh.T
        planes, occ = planes_of(sc)
        return orc.forward(planes, occ, 0, cam)[0][:, 16, 16]
    front1 = o[0] * rgb[0] + (1 - o[0]) * o[1] * rgb[1]
    front2 = o[1] * rgb[1] + (1 - o[1]) * o[0] * rgb[0]
    np.testing.assert_allclose(render(3.0, 5.0), front1, atol=1e-12)
    np.testing.assert_allclose(render(5.0, 3.0), front2, atol=1e-12)
    np.testing.assert_allclose(render(4.0, 4.0), front1, atol=1e-12)   # equal depth: lower gid first (R8)


# ---------------------------------------------------------------------------
# binning vs brute force (R8, R11 of DESIGN.md)

def _random_tiny(seed, n=60, W=80, H=64, logit_hi=None, deg=0):
    rng = np.random.default_rng(seed)
    cam = look_at((3.0, 0.5, 1.0), (0, 0, 0), W, H, 70.0)
    mu = rng.uniform(-1, 1, (n, 3))
    ls = rng.normal(-2.2, 0.5, (n, 3))
    q = rng.normal(size=(n, 4))
    lo = rng.normal(0, 1, n) if logit_hi is None else rng.uniform(-4, logit_hi, n)
    sh = np.concatenate([rng.random((n, 3)), rng.normal(0, 0.2, (n, 3 * ((deg + 1) ** 2 - 1)))], axis=1)
    sc = tiny_scene(mu, ls[:, :], q, lo, sh, cam, deg)
    # per-Gaussian log-scales / quats (tiny_scene broadcasts; set them explicitly)
    sc.levels[0].planes[3:6, 0, :] = ls.T
    sc.levels[0].planes[6:10, 0, :] = q.T
    return sc, cam


def test_binning_equals_bruteforce():
    for seed in range(3):
        sc, cam = _random_tiny(seed)
        planes, occ = planes_of(sc)
        P = orc.project(planes, occ, cam)
        start, end, gids = orc.binning(P, cam)
        gx, gy = (cam.width + 15) // 16, (cam.height + 15) // 16
        assert P["visible"].sum() > 20
        for t in range(gx * gy):
            tx, ty = t % gx, t // gx
            members = [g for g in range(len(P)) if P[g]["visible"] and P[g]["x0"] <= tx < P[g]["x1"]
                       and P[g]["y0"] <= ty < P[g]["y1"]]
            members.sort(key=lambda g: (int(P[g]["depth_bits"]), g))
            assert list(gids[start[t]:end[t]]) == members
        assert end[-1] == P["tiles"][P["visible"] == 1].sum()
        assert np.all(start[1:] == end[:-1])


def _fma32(a, b, c):
    import math as _m
    return np.float32(_m.fsum([float(a) * float(b), float(c)]))


def test_tiled_equals_untiled_bruteforce():
    """With every o < 0.353, alpha >= 1/255 implies the pixel is within r of the mean,
    so compositing ALL Gaussians per pixel equals the tiled render."""
    sc, cam = _random_tiny(11, n=40, W=48, H=40, logit_hi=-0.7)
    planes, occ = planes_of(sc)
    P = orc.project(planes, occ, cam)
    img, T, nc, _ = orc.forward(planes, occ, 0, cam)
    vis = [g for g in range(len(P)) if P[g]["visible"]]
    order = sorted(vis, key=lambda g: (int(P[g]["depth_bits"]), g))
    dc = planes[11:14, 0, :].astype(np.float64)
    rgb = SH_C0 * dc + 0.5
    one, thr, cap = np.float32(1), np.float32(1e-4), np.float32(0.99)
    n_comp = 0
    for j in range(cam.height):
        for i in range(cam.width):
            Tb = np.float32(1.0)
            C = np.zeros(3)
            for g in order:
                p = P[g]
                dx = np.float32(p["mx"] - np.float32(i))
                dy = np.float32(p["my"] - np.float32(j))
                u = _fma32(p["nb"], dy, np.float32(p["ha"] * dx))
                power = _fma32(dx, u, np.float32(np.float32(p["hc"] * dy) * dy))
                if power > 0 or power < p["t_g"]:
                    continue
                G = orc.exp_c(np.array([power], np.float32))[0]
                a = min(cap, np.float32(p["o"] * G))
                Tn = np.float32(Tb * np.float32(one - a))
                if Tn < thr:
                    break
                C += rgb[:, g] * float(a) * float(Tb)
                Tb = Tn
                n_comp += 1
            assert Tb == T[j, i]
            np.testing.assert_allclose(img[:, j, i], C, atol=2e-6)
    assert n_comp > 500


def test_transmittance_invariants_c1():
    sc = make_scene(1)
    planes, occ = planes_of(sc)
    cam = sc.cameras[0]
    img, T, nc, st = orc.forward(planes, occ, 0, cam)
    assert T.min() >= 1e-4 and T.max() <= 1.0
    dc = planes[11:14].reshape(3, -1)
    rgb = SH_C0 * dc + 0.5
    assert img.min() >= 0.0 and np.all(img.reshape(3, -1).max(axis=1) <= rgb.max(axis=1) + 1e-9)
    assert st["n_vis"] == 4096 and st["K"] > 4096


# ---------------------------------------------------------------------------
# backward: finite differences with frozen decisions

def _fd_check(sc, cam, deg, seed, n_samples=60, mask=None):
    planes, occ = planes_of(sc)
    rng = np.random.default_rng(seed)
    w = rng.normal(size=(3, cam.height, cam.width))
    g = orc.backward(planes, occ, deg, cam, w, mask=mask)
    P = orc.project(planes, occ, cam)
    vis = np.nonzero(P["visible"])[0]
    val = planes.astype(np.float64)
    D = planes.shape[0]
    errs = []
    scale = np.abs(g).max()
    for _ in range(n_samples):
        gi = int(rng.choice(vis))
        d = int(rng.integers(D))
        x = val[d, 0, gi]
        h = 1e-5 * max(1.0, abs(x))
        vp = val.copy()
        vp[d, 0, gi] = x + h
        vm = val.copy()
        vm[d, 0, gi] = x - h
        Ip = orc.forward(planes, occ, deg, cam, val=vp)[0]
        Im = orc.forward(planes, occ, deg, cam, val=vm)[0]
        fd = float(np.sum(w * (Ip - Im)) / (2 * h))
        if mask is not None and not mask.reshape(-1)[gi]:
            fd = 0.0
        errs.append((abs(fd - g[d, 0, gi]), abs(fd), d, gi))
    for e, a, d, gi in errs:
        assert e <= 1e-6 * max(a, 1e-3 * scale), (e, a, d, gi)
    return g, P


def test_backward_fd_sh0():
    sc, cam = _random_tiny(21, n=50, W=64, H=48)
    _fd_check(sc, cam, 0, 1)


def test_backward_fd_sh3_with_clamped_jacobian():
    sc, cam = _random_tiny(22, n=40, W=64, H=48, deg=3)
    # two big Gaussians just outside the frustum on either side: J clamp active
    V = cam.viewmat.astype(np.float64)
    R, t = V[:3, :3], V[:3, 3]
    lim = 1.3 * 0.5 * cam.width / cam.fx
    pl = sc.levels[0].planes
    for k, sgn in ((0, 1.0), (1, -1.0)):
        pc = np.array([sgn * (lim + 0.08) * 2.0, 0.1, 2.0])
        pl[0:3, 0, k] = R.T @ (pc - t)
        pl[3:6, 0, k] = np.log(0.45)
        pl[10, 0, k] = 0.5
    g, P = _fd_check(sc, cam, 3, 2, n_samples=40)
    assert P["clamp_x"][0] == 1 and P["clamp_x"][1] == -1 and P["visible"][0] and P["visible"][1]
    # the clamped Gaussians themselves get exact FD agreement too
    planes, occ = planes_of(sc)
    rng = np.random.default_rng(3)
    w = rng.normal(size=(3, cam.height, cam.width))
    g = orc.backward(planes, occ, 3, cam, w)
    val = planes.astype(np.float64)
    for gi in (0, 1):
        for d in (0, 1, 2, 3, 6, 10):
            h = 1e-5 * max(1.0, abs(val[d, 0, gi]))
            vp = val.copy(); vp[d, 0, gi] += h
            vm = val.copy(); vm[d, 0, gi] -= h
            fd = float(np.sum(w * (orc.forward(planes, occ, 3, cam, val=vp)[0]
                                   - orc.forward(planes, occ, 3, cam, val=vm)[0])) / (2 * h))
            assert abs(fd - g[d, 0, gi]) <= 1e-6 * max(abs(fd), 1e-3 * np.abs(g).max())


def test_backward_single_gaussian_dc_closed_form():
    """One Gaussian: dL/d(dc_c) = C0 sum_p alpha(p) w_c(p)  (T = 1)."""
    f, d, s = 100.0, 4.0, 0.1
    cam = ident_cam(65, 65, f, 32.0, 32.0)
    logit = 0.3
    sc = single([0, 0, d], np.log([s, s, s]), [1, 0, 0, 0], logit, [0.3, 0.3, 0.3], cam)
    planes, occ = planes_of(sc)
    rng = np.random.default_rng(0)
    w = rng.normal(size=(3, 65, 65))
    g = orc.backward(planes, occ, 0, cam, w)
    o = 1 / (1 + math.exp(-float(np.float32(logit))))
    s32 = math.exp(float(np.float32(math.log(s))))
    a = (f * s32 / d) ** 2 + 0.3
    jj, ii = np.mgrid[0:65, 0:65]
    power = -0.5 * ((ii - 32.0) ** 2 + (jj - 32.0) ** 2) / a
    on = power >= -math.log(255 * o)
    alpha = o * np.exp(power) * on
    for c in range(3):
        assert abs(g[11 + c, 0, 0] - SH_C0 * np.sum(alpha * w[c])) < 1e-9
    # d/dlogit: sum_p dL/dalpha * G * o(1-o), dL/dalpha = sum_c w_c rgb_c (single layer, bg 0)
    rgb = SH_C0 * float(np.float32(0.3)) + 0.5
    dLda = rgb * w.sum(axis=0)
    ref = np.sum(dLda * np.exp(power) * on) * o * (1 - o)
    assert abs(g[10, 0, 0] - ref) < 1e-9


def test_backward_mask_freezes():
    """grad <- D_i grad."""
    sc, cam = _random_tiny(31, n=30, W=48, H=40)
    planes, occ = planes_of(sc)
    w = np.random.default_rng(1).normal(size=(3, cam.height, cam.width))
    g = orc.backward(planes, occ, 0, cam, w)
    mask = (np.arange(30) % 2).astype(np.uint8).reshape(1, 30)
    gm = orc.backward(planes, occ, 0, cam, w, mask=mask)
    assert np.all(gm[:, 0, mask[0] == 0] == 0)
    assert np.array_equal(gm[:, 0, mask[0] == 1], g[:, 0, mask[0] == 1])
    assert np.abs(g).max() > 0


# ---------------------------------------------------------------------------
# atlas packing (R15)

def test_layout_column_c2():
    place, W, H = orc.layout_column([(512, 512), (256, 256), (128, 128)])
    assert (W, H) == (768, 512)
    assert place.tolist() == [[0, 0, 0], [512, 0, 0], [512, 256, 0]]


def test_pack_rotation_by_hand():
    from synth.scenes import Level
    lv0 = Level(planes=np.arange(6, dtype=np.float32).reshape(1, 2, 3), occ=np.ones((2, 3), np.uint8),
                labels=np.ones((2, 3), np.uint8))
    # rotated 90 deg CCW at (0,0): placement is 3 tall x 2 wide, cell (r,c) -> (2-c, r)
    planes, occ, _ = orc.pack([lv0], place=np.array([[0, 0, 1]]), W=2, H=3)
    # level: [[0,1,2],[3,4,5]] -> CCW rotation: [[2,5],[1,4],[0,3]]
    assert planes[0].tolist() == [[2, 5], [1, 4], [0, 3]]
    assert occ.sum() == 6


def test_pack_c2_conservation():
    sc = make_scene(2)
    planes, occ, place = orc.pack(sc.levels)
    assert occ.sum() == 344064 and planes.shape == (23, 512, 768)
    lv = sc.levels[2]
    np.testing.assert_array_equal(planes[:, 256:384, 512:640], lv.planes)
    assert np.all(planes[:, 384:, 512:] == 0) and np.all(occ[384:, 512:] == 0)


def test_alpha_cap_and_background():
    """alpha = min(0.99, o G) (R9); C = alpha c + (1 - alpha) bg at the mean pixel; capped pairs
    carry no gradient to o or the conic (R10)."""
    cam = ident_cam(33, 33, 60.0, 16.0, 16.0)
    logit, dc, bg = 6.0, np.array([0.1, 0.5, 0.9]), (0.2, 0.5, 0.9)
    sc = single([0, 0, 4.0], [-3.0] * 3, [1, 0, 0, 0], logit, dc, cam)
    planes, occ = planes_of(sc)
    img = orc.forward(planes, occ, 0, cam, bg=bg)[0]
    rgb = SH_C0 * dc.astype(np.float32).astype(np.float64) + 0.5
    np.testing.assert_allclose(img[:, 16, 16], 0.99 * rgb + 0.01 * np.array(bg), atol=1e-12)
    w = np.zeros((3, 33, 33))
    w[:, 16, 16] = 1.0
    g = orc.backward(planes, occ, 0, cam, w, bg=bg)
    assert g[10, 0, 0] == 0.0 and np.all(g[0:10, 0, 0] == 0.0)
    np.testing.assert_allclose(g[11:14, 0, 0], SH_C0 * 0.99, atol=1e-12)


def test_backward_fd_with_background():
    sc, cam = _random_tiny(41, n=40, W=48, H=48)
    planes, occ = planes_of(sc)
    bg = (0.3, 0.1, 0.7)
    rng = np.random.default_rng(4)
    w = rng.normal(size=(3, cam.height, cam.width))
    g = orc.backward(planes, occ, 0, cam, w, bg=bg)
    P = orc.project(planes, occ, cam)
    val = planes.astype(np.float64)
    for gi in np.nonzero(P["visible"])[0][:12]:
        for d in (0, 2, 4, 7, 10, 12):
            h = 1e-5 * max(1.0, abs(val[d, 0, gi]))
            vp = val.copy(); vp[d, 0, gi] += h
            vm = val.copy(); vm[d, 0, gi] -= h
            fd = float(np.sum(w * (orc.forward(planes, occ, 0, cam, bg=bg, val=vp)[0]
                                   - orc.forward(planes, occ, 0, cam, bg=bg, val=vm)[0])) / (2 * h))
            assert abs(fd - g[d, 0, gi]) <= 1e-6 * max(abs(fd), 1e-3 * np.abs(g).max())
