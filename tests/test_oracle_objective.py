"""Pins of the objective oracle (NEXT-4, oracle/objective.py).

What fixes it besides itself:
* the Gaussian window's closed form (sum 1, g5/g6 = exp(1/(2 sigma^2)));
* SSIM(x, x) = 1 and a zero SSIM gradient there (SSIM's maximum);
* closed forms for constant images: interior (2ab + C1)/(a^2 + b^2 + C1); the corner pixel's
  zero-padded window mass W gives mu = aW, var = a^2 W(1 - W);
* the window sums against scipy.signal.correlate2d (a library routine, zero fill, 'same');
* central finite differences of the loss for the analytic gradients (photo and regularisers);
* regulariser special cases (all scales below s_max -> 0; logit 0 -> alpha(1-alpha) = 1/4, zero grad).
"""
import math

import numpy as np
import pytest
from scipy.signal import correlate2d

from oracle import objective as ob


def test_window_closed_form():
    g = ob.window_1d()
    assert abs(g.sum() - 1) < 1e-15 and np.allclose(g, g[::-1], rtol=0, atol=0)
    assert math.isclose(g[5] / g[6], math.exp(1 / (2 * 1.5 ** 2)), rel_tol=1e-14)
    assert math.isclose(g[5] / g[0], math.exp(25 / (2 * 1.5 ** 2)), rel_tol=1e-12)


def test_ssim_identity_and_zero_gradient():
    rng = np.random.default_rng(0)
    x = rng.random((3, 23, 31))
    assert abs(ob.ssim(x, x) - 1) < 1e-12
    L, g = ob.photo_loss_grad(x, x, 0.2)
    assert abs(L) < 1e-12 and np.abs(g).max() < 1e-12


def test_ssim_constant_images_closed_form():
    a, b = 0.3, 0.7
    x = np.full((3, 30, 40), a)
    y = np.full((3, 30, 40), b)
    t = ob.ssim_terms(x, y)
    interior = (2 * a * b + ob.C1) / (a * a + b * b + ob.C1)
    assert np.allclose(t["ssim"][:, 5:-5, 5:-5], interior, rtol=1e-13)
    g = ob.window_1d()
    W = g[5:].sum() ** 2          # the corner pixel sees the lower-right quadrant of the window
    mx, vx, my, vy, c = a * W, a * a * W * (1 - W), b * W, b * b * W * (1 - W), a * b * W * (1 - W)
    s = (2 * mx * my + ob.C1) * (2 * c + ob.C2) / ((mx * mx + my * my + ob.C1) * (vx + vy + ob.C2))
    assert math.isclose(t["ssim"][0, 0, 0], s, rel_tol=1e-12)
    assert math.isclose(t["mx"][1, 0, 0], mx, rel_tol=1e-13)


def test_window_sums_match_scipy():
    rng = np.random.default_rng(1)
    x, y = rng.random((3, 17, 26)), rng.random((3, 17, 26))
    t = ob.ssim_terms(x, y)
    w = ob.window_2d()
    for c in range(3):
        mx = correlate2d(x[c], w, mode="same", boundary="fill")
        my = correlate2d(y[c], w, mode="same", boundary="fill")
        sxy = correlate2d(x[c] * y[c], w, mode="same", boundary="fill")
        sxx = correlate2d(x[c] ** 2, w, mode="same", boundary="fill")
        assert np.allclose(t["mx"][c], mx, rtol=1e-13, atol=1e-15)
        assert np.allclose(t["cxy"][c], sxy - mx * my, rtol=1e-9, atol=1e-14)
        assert np.allclose(t["vx"][c], sxx - mx * mx, rtol=1e-9, atol=1e-14)
        assert np.allclose(t["my"][c], my, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_photo_gradient_finite_differences(lam):
    rng = np.random.default_rng(2)
    x = rng.random((3, 14, 19))
    y = np.clip(x + rng.normal(0, 0.2, x.shape), 0, 1)
    L, g = ob.photo_loss_grad(x, y, lam)
    h = 1e-6
    idx = [(0, 0, 0), (1, 13, 18), (2, 7, 9), (0, 3, 17), (1, 0, 10), (2, 12, 1)] + \
        [tuple(int(v) for v in rng.integers(0, s)) for _ in range(20) for s in [x.shape]]
    for i in idx:
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        fd = (ob.photo_loss_grad(xp, y, lam)[0] - ob.photo_loss_grad(xm, y, lam)[0]) / (2 * h)
        assert abs(fd - g[i]) <= 1e-6 * abs(g[i]) + 1e-9, (i, fd, g[i])


def _atlas(rng, H=6, W=7, D=14):
    P = np.zeros((D, H, W), np.float32)
    P[3:6] = rng.normal(-3.0, 0.5, (3, H, W))
    P[10] = rng.normal(0, 1.5, (H, W))
    return P


def test_reg_finite_differences_and_mask():
    rng = np.random.default_rng(3)
    P = _atlas(rng)
    occ = (rng.random(P.shape[1:]) < 0.8).astype(np.uint8)
    mask = (rng.random(P.shape[1:]) < 0.6).astype(np.uint8)
    ls, lo, smax = 1e-2, 3e-2, 0.05
    for m in (None, mask):
        L, g = ob.reg_loss_grad(P, occ, ls, lo, smax, mask=m)
        sel = occ.astype(bool) if m is None else (occ & m).astype(bool)
        assert np.all(g[:, ~sel] == 0) and np.all(g[[0, 1, 2, 6, 7, 8, 9, 11, 12, 13]] == 0)
        h = 1e-5
        for d in (3, 4, 5, 10):
            for (i, j) in np.argwhere(sel)[:6]:
                Pp, Pm = P.astype(np.float64), P.astype(np.float64)
                Pp[d, i, j] += h
                Pm[d, i, j] -= h
                fd = (ob.reg_loss_grad(Pp, occ, ls, lo, smax, mask=m)[0] -
                      ob.reg_loss_grad(Pm, occ, ls, lo, smax, mask=m)[0]) / (2 * h)
                assert abs(fd - g[d, i, j]) <= 1e-6 * abs(g[d, i, j]) + 1e-12, (d, i, j, fd, g[d, i, j])


def test_reg_special_cases():
    P = np.zeros((14, 4, 5), np.float32)
    P[3:6] = math.log(0.01)
    occ = np.ones((4, 5), np.uint8)
    L, g = ob.reg_loss_grad(P, occ, 1.0, 1.0, 0.05)
    assert math.isclose(L, 0.25, rel_tol=1e-15) and np.abs(g).max() == 0     # alpha = 1/2, scales < s_max
    P[4, 0, 0] = math.log(0.15)                                                # one texel's axis 1 above s_max
    L, g = ob.reg_loss_grad(P, occ, 1.0, 0.0, 0.05)
    assert math.isclose(L, (0.15 - 0.05) ** 2 / 20, rel_tol=1e-6)
    assert g[4, 0, 0] > 0 and np.count_nonzero(g) == 1
    assert ob.reg_loss_grad(P, np.zeros_like(occ), 1.0, 1.0, 0.05)[0] == 0.0
