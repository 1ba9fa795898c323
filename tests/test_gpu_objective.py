"""GPU parity of the objective kernels (NEXT-4) against oracle/objective.py.

K12 (L1 + SSIM): loss within 1e-12 relative; dL/dI^ within
1e-5 |ref| + 1e-7 max|ref| (fp64 statistics on both sides, one fp32 rounding of dL on the GPU).
K13 (regularisers): loss within 1e-12 relative, gradients accumulated (+=) onto
the given planes within max(1e-3 |g|, 1e-6) like every atlas gradient (BJ.north_star)."""
import math

import numpy as np
import pytest
import torch

from oracle import objective as ob
from paper_2602_23040_b200 import puv
from synth.scenes import make_scene

pytestmark = pytest.mark.gpu


def _images(rng, V, H, W, ties=True):
    """Rendered-like image (smooth field + detail) and a U[0,1] target; some exact ties."""
    yy, xx = np.mgrid[0:H, 0:W]
    img = np.empty((V, 3, H, W), np.float32)
    for v in range(V):
        for c in range(3):
            a, b, p = rng.uniform(0.02, 0.2, 3)
            img[v, c] = 0.5 + 0.3 * np.sin(a * xx + p) * np.cos(b * yy) + rng.normal(0, 0.02, (H, W))
    tgt = rng.random((V, 3, H, W), dtype=np.float32)
    if ties:
        m = rng.random((V, 3, H, W)) < 0.02
        tgt[m] = img[m]
    return img, tgt


def _check_photo(img, tgt, lam, chunk=None):
    dev = torch.device("cuda")
    V, _, H, W = img.shape
    it, tt = torch.from_numpy(img).to(dev), torch.from_numpy(tgt).to(dev)
    dL = torch.full_like(it, float("nan"))
    loss = torch.full((1,), float("nan"), dtype=torch.float64, device=dev)
    ws = None
    if chunk is not None:
        ws = torch.empty(puv.photo_workspace_bytes(W, H, chunk), dtype=torch.uint8, device=dev)
    puv.photo_loss_grad(it, tt, dL, loss, lambda_ssim=lam, workspace=ws)
    torch.cuda.synchronize()
    g = dL.cpu().numpy().astype(np.float64)
    L_ref, err = 0.0, 0.0
    for v in range(V):
        Lv, gv = ob.photo_loss_grad(img[v], tgt[v], lam)
        L_ref += Lv
        tol = 1e-5 * np.abs(gv) + 1e-7 * np.abs(gv).max()
        bad = np.abs(g[v] - gv) > tol
        assert not bad.any(), (v, np.argwhere(bad)[:5], g[v][bad][:5], gv[bad][:5])
        err = max(err, float((np.abs(g[v] - gv) / np.maximum(np.abs(gv), 1e-30)).max()))
    assert abs(loss.item() - L_ref) <= 1e-12 * abs(L_ref) + 1e-15, (loss.item(), L_ref)
    return err


@pytest.mark.parametrize("V,H,W,lam", [(1, 16, 32, 0.2), (3, 75, 100, 0.2), (2, 37, 53, 0.0), (2, 40, 70, 1.0),
                                       (1, 1, 1, 0.2), (1, 9, 300, 0.2)])
def test_photo_loss_parity(V, H, W, lam):
    rng = np.random.default_rng(V * 1000 + H + W)
    img, tgt = _images(rng, V, H, W)
    _check_photo(img, tgt, lam)


def test_photo_loss_chunked_equals_unchunked():
    rng = np.random.default_rng(5)
    img, tgt = _images(rng, 5, 48, 64)
    _check_photo(img, tgt, 0.2, chunk=1)
    _check_photo(img, tgt, 0.2, chunk=2)


def test_photo_loss_identity():
    rng = np.random.default_rng(6)
    img, _ = _images(rng, 2, 33, 47)
    dev = torch.device("cuda")
    it = torch.from_numpy(img).to(dev)
    dL = torch.empty_like(it)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    puv.photo_loss_grad(it, it.clone(), dL, loss)
    torch.cuda.synchronize()
    assert abs(loss.item()) < 1e-12 and dL.abs().max().item() < 1e-12


def test_photo_loss_argument_errors():
    dev = torch.device("cuda")
    x = torch.zeros((1, 3, 8, 8), device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    with pytest.raises(puv.PuvError):
        puv.photo_loss_grad(x, x, x.clone(), loss, lambda_ssim=1.5)
    with pytest.raises(puv.PuvError):
        puv.photo_loss_grad(x, x, x.clone(), loss, workspace=torch.empty(16, dtype=torch.uint8, device=dev))


@pytest.mark.slow
def test_photo_loss_full_size_1080p_64_views_sampled():
    """The bench launch: 64 views of 1920 x 1080 in one call (default 8-view chunks).  Views 0 and 41
    against the oracle (dL and their one-view losses); the 64-view loss equals the sum of the 64
    one-view losses, and chunking leaves dL bit-identical."""
    dev = torch.device("cuda")
    torch.manual_seed(7)
    V, H, W = 64, 1080, 1920
    img = torch.rand((V, 3, H, W), device=dev) * 0.6 + 0.2
    tgt = torch.rand((V, 3, H, W), device=dev)
    dL = torch.empty_like(img)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    puv.photo_loss_grad(img, tgt, dL, loss)
    one = torch.empty(V, dtype=torch.float64, device=dev)
    d1 = torch.empty_like(img[:1])
    ws = torch.empty(puv.photo_workspace_bytes(W, H, 1), dtype=torch.uint8, device=dev)
    for v in range(V):
        puv.photo_loss_grad(img[v:v + 1], tgt[v:v + 1], d1, one[v:v + 1], workspace=ws)
        if v in (0, 41):
            assert torch.equal(d1[0], dL[v])
    torch.cuda.synchronize()
    assert abs(loss.item() - one.sum().item()) <= 1e-12 * loss.item()
    for v in (0, 41):
        Lv, gv = ob.photo_loss_grad(img[v].cpu().numpy(), tgt[v].cpu().numpy(), 0.2)
        assert abs(one[v].item() - Lv) <= 1e-12 * Lv
        g = dL[v].cpu().numpy().astype(np.float64)
        tol = 1e-5 * np.abs(gv) + 1e-7 * np.abs(gv).max()
        assert not (np.abs(g - gv) > tol).any()


# ---- K13 regularisers -------------------------------------------------------------------------------

def _reg_case(rng, D, H, W, holes=True):
    P = np.zeros((D, H, W), np.float32)
    P[0:3] = rng.normal(0, 1, (3, H, W))
    P[3:6] = rng.normal(-3.0, 0.6, (3, H, W))
    P[6:10] = rng.normal(0, 1, (4, H, W))
    P[10] = rng.normal(0, 1.5, (H, W))
    P[11:] = rng.normal(0, 0.1, (D - 11, H, W))
    P[4, 0, :3] = P[3, 0, :3]          # exact ties of the max axis
    occ = (rng.random((H, W)) < (0.85 if holes else 1.0)).astype(np.uint8)
    return P, occ


@pytest.mark.parametrize("mask_on", [False, True])
def test_reg_loss_parity(mask_on):
    rng = np.random.default_rng(11 + mask_on)
    lay = puv.layout_for_levels([(37, 53)], 1)
    P, occ = _reg_case(rng, lay.planes, 37, 53)
    mask = (rng.random((37, 53)) < 0.4).astype(np.uint8) if mask_on else None
    dev = torch.device("cuda")
    g0 = rng.normal(0, 1e-3, P.shape).astype(np.float32)
    grad = torch.from_numpy(g0).to(dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ls, lo, smax = 0.5, 0.25, 0.06
    puv.reg_loss_grad(lay, torch.from_numpy(P).to(dev), torch.from_numpy(occ).to(dev), grad, loss, ls, lo, smax,
                      mask=None if mask is None else torch.from_numpy(mask).to(dev))
    torch.cuda.synchronize()
    L_ref, g_ref = ob.reg_loss_grad(P, occ, ls, lo, smax, mask=mask)
    assert abs(loss.item() - L_ref) <= 1e-12 * abs(L_ref)
    exp = g0.astype(np.float64) + g_ref
    got = grad.cpu().numpy().astype(np.float64)
    tol = np.maximum(1e-3 * np.abs(exp), 1e-6)
    assert not (np.abs(got - exp) > tol).any()
    untouched = [d for d in range(lay.planes) if d not in (3, 4, 5, 10)]
    assert np.array_equal(got[untouched], g0[untouched].astype(np.float64))


def test_reg_loss_c3_atlas_paper_lambdas():
    """C3's atlas (1M texels, SH3) with the paper's lambdas (1e-4); s_max = 0.05 (L5)."""
    sc = make_scene(3, views=1)
    lv = sc.levels[0]
    lay = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    dev = torch.device("cuda")
    atlas = torch.from_numpy(lv.planes).to(dev)
    occ = torch.from_numpy(lv.occ).to(dev)
    grad = torch.zeros_like(atlas)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    puv.reg_loss_grad(lay, atlas, occ, grad, loss, 1e-4, 1e-4, 0.05)
    torch.cuda.synchronize()
    L_ref, g_ref = ob.reg_loss_grad(lv.planes, lv.occ, 1e-4, 1e-4, 0.05)
    assert abs(loss.item() - L_ref) <= 1e-12 * abs(L_ref)
    got = grad.cpu().numpy()
    for d in (3, 4, 5, 10):
        tol = np.maximum(1e-3 * np.abs(g_ref[d]), 1e-6)
        assert not (np.abs(got[d] - g_ref[d]) > tol).any()
    assert np.count_nonzero(got[3:6]) > 0


def test_reg_loss_empty_selection():
    lay = puv.layout_for_levels([(8, 8)], 0)
    dev = torch.device("cuda")
    P = torch.zeros((lay.planes, 8, 8), device=dev)
    grad = torch.zeros_like(P)
    loss = torch.full((1,), 7.0, dtype=torch.float64, device=dev)
    puv.reg_loss_grad(lay, P, torch.zeros((8, 8), dtype=torch.uint8, device=dev), grad, loss, 1.0, 1.0, 0.05)
    torch.cuda.synchronize()
    assert loss.item() == 0.0 and grad.abs().max().item() == 0.0
