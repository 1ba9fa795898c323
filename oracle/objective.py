"""CPU ORACLE of the paper's training objective (NEXT-4) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` arms may
import this module.  It shares nothing with the CUDA path (paper_2602_23040_b200/).  Plain numpy,
fp64 throughout, written from PAPER.md:445-465 and the readings L1-L8 of DESIGN.md §12:

    L_photo = (1 - lambda_ssim) ||I_hat - I||_1 + lambda_ssim (1 - SSIM(I_hat, I))
    L_scale = E_i [max{0, max(s_i) - s_max}]^2
    L_opacity = E_i alpha_i (1 - alpha_i)

||.||_1 and SSIM are means over the view's 3 H W entries (L2); SSIM is Wang et al.'s index with an
11 x 11 Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero-padded 'same' windows, per
channel (L3).  The window sums are written out as the plain definition: one shifted copy of the
image per window offset, no separability.  The gradient is the chain rule of that definition,
scattered back offset by offset.
"""
from __future__ import annotations

import math

import numpy as np

WIN = 11
SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2


def window_1d():
    """g_i = exp(-(i - 5)^2 / (2 sigma^2)) / sum (DESIGN.md §12 L3)."""
    g = np.array([math.exp(-((i - WIN // 2) ** 2) / (2.0 * SIGMA * SIGMA)) for i in range(WIN)])
    return g / g.sum()


def window_2d():
    g = window_1d()
    return np.outer(g, g)


def _shift(a, dy, dx):
    """out[.., i, j] = a[.., i + dy, j + dx] (zero outside)."""
    H, W = a.shape[-2:]
    out = np.zeros_like(a)
    ys, ye = max(0, -dy), min(H, H - dy)
    xs, xe = max(0, -dx), min(W, W - dx)
    if ys < ye and xs < xe:
        out[..., ys:ye, xs:xe] = a[..., ys + dy:ye + dy, xs + dx:xe + dx]
    return out


def _window_sum(a, w):
    r = WIN // 2
    out = np.zeros_like(a)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            out += w[dy + r, dx + r] * _shift(a, dy, dx)
    return out


def ssim_terms(x, y):
    """Local statistics and the SSIM map of Wang et al. (2004) for (C, H, W) fp64 images."""
    w = window_2d()
    mx, my = _window_sum(x, w), _window_sum(y, w)
    sxx, syy, sxy = _window_sum(x * x, w), _window_sum(y * y, w), _window_sum(x * y, w)
    vx, vy, cxy = sxx - mx * mx, syy - my * my, sxy - mx * my
    n1, n2 = 2 * mx * my + C1, 2 * cxy + C2
    d1, d2 = mx * mx + my * my + C1, vx + vy + C2
    s = (n1 * n2) / (d1 * d2)
    return {"mx": mx, "my": my, "vx": vx, "vy": vy, "cxy": cxy, "n1": n1, "n2": n2, "d1": d1, "d2": d2,
            "ssim": s}


def ssim(x, y):
    """Mean SSIM of one view ((3, H, W) images)."""
    return float(ssim_terms(np.asarray(x, np.float64), np.asarray(y, np.float64))["ssim"].mean())


def photo_loss_grad(image, target, lambda_ssim):
    """One view: L_photo and dL_photo/dI_hat ((3, H, W) fp64).

    d|d|/dd = sign(d) with sign(0) = 0 (L4).  For the SSIM term, with S(p) = n1 n2 / (d1 d2):
      dS/dmu_x = 2 mu_y n2 / (d1 d2) - 2 mu_x S / d1,  dS/dvar_x = -S / d2,  dS/dcov = 2 n1 / (d1 d2);
      var_x = Sxx - mu_x^2, cov = Sxy - mu_x mu_y, so per window sum:
      A = dS/dmu_x - 2 mu_x dS/dvar_x - mu_y dS/dcov  (on mu_x),  B = dS/dvar_x  (on Sxx),  Cc = dS/dcov  (on Sxy);
      dS(p)/dx(q) = w(q - p) (A(p) + 2 B(p) x(q) + Cc(p) y(q)).
    """
    x = np.asarray(image, np.float64)
    y = np.asarray(target, np.float64)
    n = x.size
    d = x - y
    t = ssim_terms(x, y)
    s = t["ssim"]
    L = (1.0 - lambda_ssim) * np.abs(d).sum() / n + lambda_ssim * (1.0 - s.sum() / n)
    dd = t["d1"] * t["d2"]
    dS_dmx = 2 * t["my"] * t["n2"] / dd - 2 * t["mx"] * s / t["d1"]
    dS_dvx = -s / t["d2"]
    dS_dcov = 2 * t["n1"] / dd
    A = dS_dmx - 2 * t["mx"] * dS_dvx - t["my"] * dS_dcov
    B = dS_dvx
    Cc = dS_dcov
    w = window_2d()
    r = WIN // 2
    dS = np.zeros_like(x)
    for dy in range(-r, r + 1):          # scatter: q = p + (dy, dx) receives w * (A(p) + 2 B(p) x(q) + Cc(p) y(q))
        for dx in range(-r, r + 1):
            wt = w[dy + r, dx + r]
            dS += wt * (_shift(A, -dy, -dx) + 2 * _shift(B, -dy, -dx) * x + _shift(Cc, -dy, -dx) * y)
    grad = (1.0 - lambda_ssim) * np.sign(d) / n - lambda_ssim * dS / n
    return float(L), grad


def reg_loss_grad(planes, occ, lambda_scale, lambda_opacity, s_max, mask=None):
    """Scale + opacity regularisers over the occupied (and, with `mask`, dynamic) texels (L5-L7).

    planes: (D, H, W) fp32 atlas [x, y, z, ls0, ls1, ls2, q.., logit, ..].  Returns (loss, grad) with
    grad (D, H, W) fp64 holding d(lambda_s L_scale + lambda_o L_opacity) on planes 3..5 and 10."""
    P = np.asarray(planes, np.float64)
    sel = np.asarray(occ) != 0
    if mask is not None:
        sel &= np.asarray(mask) != 0
    n = int(sel.sum())
    grad = np.zeros(P.shape, np.float64)
    if n == 0:
        return 0.0, grad
    ls = P[3:6]
    s = np.exp(ls)
    am = np.argmax(ls, axis=0)                       # ties -> lowest axis (L6)
    smax = np.take_along_axis(s, am[None], 0)[0]
    h = np.maximum(0.0, smax - s_max)
    alpha = 1.0 / (1.0 + np.exp(-P[10]))
    L_scale = float((h * h)[sel].sum()) / n
    L_opac = float((alpha * (1 - alpha))[sel].sum()) / n
    gs = np.where(sel, 2.0 * h * smax / n, 0.0) * lambda_scale   # d/d ls_am of h^2 = 2 h s_am
    for a in range(3):
        grad[3 + a] = np.where(am == a, gs, 0.0)
    grad[10] = np.where(sel, (1 - 2 * alpha) * alpha * (1 - alpha) / n, 0.0) * lambda_opacity
    return lambda_scale * L_scale + lambda_opacity * L_opac, grad
