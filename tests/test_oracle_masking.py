"""Pins of the oracle's covariance-aware flow masking (supp. Alg. 1)."""
import math

import numpy as np

from oracle import orc
from synth.scenes import Camera, look_at, tiny_scene
from tests.test_oracle_pins import _numeric_ewa, ident_cam, planes_of


def _single(mu, ls, q, cam):
    return planes_of(tiny_scene([mu], ls, q, 0.0, [0.5, 0.5, 0.5], cam, 0))


def test_spec_hand_example():
    """mean (10,10), Sigma2D = I + 0.3 I, mask only at (12,10): d^2 = 4/1.3 <= 9 -> dynamic."""
    cam = ident_cam(21, 21, 1.0, 10.0, 10.0)
    planes, occ = _single([0, 0, 1], [0, 0, 0], [1, 0, 0, 0], cam)
    for (i, j), expect, rmax in [((12, 10), 1, 64), ((13, 10), 1, 64), ((14, 10), 0, 64), ((10, 13), 1, 64),
                                 ((12, 10), 0, 1), ((11, 10), 1, 1)]:
        m = np.zeros((1, 21, 21), np.uint8)
        m[0, j, i] = 1
        lab = orc.label_dynamic(planes, occ, [cam], m, r_max=rmax)
        assert lab[0, 0] == expect, ((i, j), rmax, 4 / 1.3)


def test_static_cases():
    cam = ident_cam(33, 33, 40.0, 16.0, 16.0)
    m = np.ones((1, 33, 33), np.uint8)
    planes, occ = _single([0, 0, -2.0], [-2] * 3, [1, 0, 0, 0], cam)     # behind the camera
    assert orc.label_dynamic(planes, occ, [cam], m)[0, 0] == 0
    planes, occ = _single([0, 0, 0.1], [-4] * 3, [1, 0, 0, 0], cam)      # z > 0 (no near plane in Alg. 1)
    assert orc.label_dynamic(planes, occ, [cam], m)[0, 0] == 1
    planes, occ = _single([0, 0, 3.0], [-2] * 3, [1, 0, 0, 0], cam)
    assert orc.label_dynamic(planes, occ, [cam], np.zeros_like(m))[0, 0] == 0   # all-false mask


def _scene(seed, n=60):
    rng = np.random.default_rng(seed)
    cams = [look_at((3 * math.cos(a), 3 * math.sin(a), 0.8), (0, 0, 0), 72, 56, 60.0) for a in (0.0, 2.0, 4.1)]
    mu = rng.uniform(-1, 1, (n, 3))
    ls = rng.normal(-2.6, 0.4, (n, 3))
    q = rng.normal(size=(n, 4))
    sc = tiny_scene(mu, [0, 0, 0], [1, 0, 0, 0], rng.normal(size=n), np.full(3, 0.5), cams[0], 0)
    sc.levels[0].planes[3:6, 0, :] = ls.T
    sc.levels[0].planes[6:10, 0, :] = q.T
    planes, occ = planes_of(sc)
    masks = (rng.random((3, 56, 72)) < 0.004).astype(np.uint8)
    return planes, occ, cams, masks, (mu, ls, q)


def _rot(q):
    qn = q / np.linalg.norm(q)
    w, x, y, z = qn
    ang = 2 * math.acos(np.clip(w, -1, 1))
    axis = np.array([x, y, z]) / max(math.sin(ang / 2), 1e-12)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * K @ K


def test_bruteforce_full_image_equivalence():
    """equal to testing every mask pixel against the full-image Mahalanobis field
    (numerical-Jacobian EWA, no radius shortcut) for Gaussians whose 3-sigma radius <= r_max;
    pixels within 1e-3 of the d^2 = 9 boundary (fp32 vs fp64) are excluded."""
    checked = 0
    for seed in range(3):
        planes, occ, cams, masks, (mu, ls, q) = _scene(seed)
        lab = orc.label_dynamic(planes, occ, cams, masks, r_max=64)[0]
        for g in range(mu.shape[0]):
            mu32 = planes[0:3, 0, g].astype(np.float64)
            cov3 = _rot(planes[6:10, 0, g].astype(np.float64)) @ np.diag(
                np.exp(2 * planes[3:6, 0, g].astype(np.float64))) @ _rot(planes[6:10, 0, g].astype(np.float64)).T
            dyn, ambiguous = False, False
            for c, cam in enumerate(cams):
                pc = cam.viewmat.astype(np.float64) @ np.append(mu32, 1.0)
                if pc[2] <= 0:
                    continue
                m, S = _numeric_ewa(mu32, cov3, cam)
                if np.linalg.det(S) <= 1e-7 or 3 * math.sqrt(np.linalg.eigvalsh(S).max()) > 64:
                    ambiguous = True
                    continue
                Si = np.linalg.inv(S)
                jj, ii = np.nonzero(masks[c])
                d = np.stack([ii - m[0], jj - m[1]], axis=1)
                d2 = np.einsum("ni,ij,nj->n", d, Si, d)
                if np.any(np.abs(d2 - 9.0) < 1e-3 * 9):
                    ambiguous = True
                dyn |= bool(np.any(d2 <= 9.0))
            if not ambiguous:
                assert lab[g] == int(dyn), (seed, g)
                checked += 1
    assert checked > 100


def test_monotone_in_masks_and_cameras():
    planes, occ, cams, masks, _ = _scene(7)
    rng = np.random.default_rng(1)
    more = masks | (rng.random(masks.shape) < 0.01).astype(np.uint8)
    a = orc.label_dynamic(planes, occ, cams, masks)
    b = orc.label_dynamic(planes, occ, cams, more)
    assert np.all(b >= a) and b.sum() > a.sum()
    one = orc.label_dynamic(planes, occ, cams[:1], masks[:1])
    assert np.all(a >= one)
    sel = orc.label_dynamic(planes, occ, cams, masks, gids=np.arange(0, 60, 3))
    assert np.array_equal(sel[0, ::3], a[0, ::3]) and sel[0, 1::3].sum() == 0
