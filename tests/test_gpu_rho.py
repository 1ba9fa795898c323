"""GPU parity of the paper-native atlas (NEXT-1): the K-level pyramid layout with
odd levels rotated, UV-ray planes (PAPER.md eq. uvgs2) and rho storage
(mu = c + rho ray) rendered forward and backward through the C ABI, against the
oracle rendering the materialised positions.

Bit-exact: pack (incl. rotations), ray planes, depth keys / tile lists / pixel state.  Images within
1e-4.  Gradients within max(1e-3 |g|, 1e-6) per component, d rho included: it is compared with the
oracle's ray . d mu (orc.rho_grad) at max(1e-3 |d rho|, 1e-6) (reading N5; round 1 used the looser
max(1e-3 sum_i |ray_i d mu_i|, 1e-6), the xyz tolerance carried through the dot product)."""
import math

import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import look_at, ring, rho_scene
from tests.gpu_common import GRAD_ATOL, GRAD_RTOL, IMG_ATOL, describe_violations, grad_violations

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint32)


def _run_rho(S, K, sh, cams, cfg, centre, views_checked, full_check=True, sample=None):
    dev = torch.device("cuda")
    rows, cols, place, W, H = orc.layout_paper(S, K)
    sc = rho_scene(cfg, list(zip(rows.tolist(), cols.tolist())), sh, cams, centre)
    # ---- GPU: paper layout, pack, rays, rho-mode render + backward
    lay_x = puv.layout_paper(S, K, sh)
    lay = puv.with_rho(lay_x, centre)
    lp = [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels]
    lo = [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels]
    atlas, occ_t = puv.pack_atlas(lay, lp, lo)
    rays_t = puv.ray_planes(lay)
    table = puv.rho_plane_table(atlas, rays_t)
    cam_arr = puv.cameras(sc.cameras)
    R = puv.Renderer(lay, cam_arr, device=dev)
    img = R.forward(table, occ_t).cpu().numpy()
    # ---- oracle: same layout, pack, rays; positions materialised
    planes, occ, _ = orc.pack(sc.levels, place=place, W=W, H=H)
    rays = orc.ray_dirs(rows, cols, place, W, H)
    assert np.array_equal(_bits(atlas.cpu().numpy()), _bits(planes)), "pack (with rotated levels) differs"
    assert np.array_equal(occ_t.cpu().numpy(), occ)
    assert np.array_equal(_bits(rays_t.cpu().numpy()), _bits(rays)), "ray planes differ"
    mat = planes.copy()
    mat[0:3] = orc.positions_from_rho(planes[0], rays, centre)
    dls = []
    for vi in range(len(sc.cameras)):
        cam = sc.cameras[vi]
        ref, T, nc, st = orc.forward(mat, occ, sh, cam)
        if vi in views_checked:
            dbg = puv.debug_tensors(lay, cam_arr, R.state, R.arena, vi)
            P = orc.project(mat, occ, cam)
            ref_depth = np.where(P["visible"] == 1, P["depth_bits"], np.uint32(0xFFFFFFFF)).astype(np.uint32)
            assert np.array_equal(dbg["depth_key"].cpu().numpy().view(np.uint32), ref_depth)
            if full_check:
                start, end, gids = orc.binning(P, cam)
                assert np.array_equal(dbg["keys_gid"].cpu().numpy().view(np.uint32), gids)
                assert np.array_equal(dbg["tile_start"].cpu().numpy().view(np.uint32), start)
            assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T))
            assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc)
        assert np.abs(img[vi] - ref).max() <= IMG_ATOL
        dls.append(orc.l2_loss_grad(ref, sc.target(vi))[1].astype(np.float32).astype(np.float64))
    dL = torch.from_numpy(np.stack(dls).astype(np.float32)).to(dev)
    grad = R.backward(table, occ_t, dL)
    torch.cuda.synchronize()
    grad = grad.cpu().numpy()
    g_ref = np.zeros(mat.shape, np.float64)
    for vi, dl in enumerate(dls):
        orc.backward(mat, occ, sh, sc.cameras[vi], dl, grad=g_ref)
    bad = grad_violations(grad[3:], g_ref[3:])
    assert not bad.any(), f"{bad.sum()} attribute components outside tolerance: " + \
        describe_violations(grad[3:], g_ref[3:], bad)
    assert np.all(grad[1:3] == 0), "planes 1, 2 are unused in rho mode"
    g_rho = orc.rho_grad(rays, g_ref[0:3])
    tol = np.maximum(GRAD_RTOL * np.abs(g_rho), GRAD_ATOL)   # the north_star bar on d rho itself (N5)
    badr = np.abs(grad[0] - g_rho) > tol
    assert not badr.any(), f"{badr.sum()} d rho outside tolerance: " + describe_violations(grad[0], g_rho, badr)
    assert np.all(grad[:, occ == 0] == 0)
    assert np.abs(g_rho).max() > 0
    return sc, grad, g_rho


def test_rho_paper_k8_small_parity():
    """S = 64, K = 8 (the paper's level count on a 96 x 96 atlas), 3 views 160 x 120 around c."""
    centre = (0.1, -0.2, 0.3)
    cams = ring(3, 3.0, 0.8, 160, 120, 140.0, target=centre)
    _run_rho(64, 8, 1, cams, 61, centre, views_checked=(0, 1, 2))


def test_rho_ragged_sh3_offcentre():
    """S = 32, K = 5, SH degree 3, a ragged 100 x 75 image and a camera inside the shell."""
    centre = (0.0, 0.0, 0.0)
    cams = ring(2, 3.0, 0.5, 100, 75, 80.0, target=centre) + [look_at((0.0, 0.0, 0.0), (1.0, 0.2, 0.1), 100, 75,
                                                                      60.0)]
    _run_rho(32, 5, 3, cams, 62, centre, views_checked=(0, 1, 2))


def test_rho_matches_xyz_mode_render():
    """Rendering a rho atlas equals rendering the xyz atlas of its materialised positions, bit for bit
    (same fp32 mu either way), through the same ABI."""
    dev = torch.device("cuda")
    S, K, sh = 64, 8, 0
    centre = (0.0, 0.0, 0.0)
    rows, cols, place, W, H = orc.layout_paper(S, K)
    sc = rho_scene(63, list(zip(rows.tolist(), cols.tolist())), sh, ring(2, 3.0, 0.5, 128, 96, 120.0), centre)
    lay_x = puv.layout_paper(S, K, sh)
    lay = puv.with_rho(lay_x, centre)
    lp = [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels]
    atlas, occ_t = puv.pack_atlas(lay, lp, [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    rays = puv.ray_planes(lay)
    cams = puv.cameras(sc.cameras)
    img_r = puv.Renderer(lay, cams, device=dev).forward(puv.rho_plane_table(atlas, rays), occ_t)
    planes, occ, _ = orc.pack(sc.levels, place=place, W=W, H=H)
    mat = planes.copy()
    mat[0:3] = orc.positions_from_rho(planes[0], orc.ray_dirs(rows, cols, place, W, H), centre)
    img_x = puv.Renderer(lay_x, cams, device=dev).forward(torch.from_numpy(mat).to(dev), occ_t)
    assert torch.equal(img_r, img_x)


@pytest.mark.slow
def test_rho_paper_full_size_s1024_k8():
    """The paper's atlas at full size: S = 1024, K = 8 (2,088,960 texels on 1536 x 1536),
    SH3, C3's 64-view 1920 x 1080 rig in one call (the NEXT-1 bench launch); bit-exact depth keys and
    pixel state + image tolerance on views 0 and 33; gradients of a 2-view call vs the oracle."""
    dev = torch.device("cuda")
    S, K, sh = 1024, 8, 3
    centre = (0.0, 0.0, 0.0)
    cams = ring(32, 3.5, 1.0, 1920, 1080, 1400.0) + ring(32, 3.5, 2.0, 1920, 1080, 1400.0, offset=math.pi / 32)
    rows, cols, place, W, H = orc.layout_paper(S, K)
    sc = rho_scene(64, list(zip(rows.tolist(), cols.tolist())), sh, cams, centre)
    lay = puv.with_rho(puv.layout_paper(S, K, sh), centre)
    atlas, occ_t = puv.pack_atlas(lay, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                                  [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    table = puv.rho_plane_table(atlas, puv.ray_planes(lay))
    cam_arr = puv.cameras(cams)
    R = puv.Renderer(lay, cam_arr, device=dev)
    img = R.forward(table, occ_t).cpu().numpy()
    planes, occ, _ = orc.pack(sc.levels, place=place, W=W, H=H)
    mat = planes.copy()
    mat[0:3] = orc.positions_from_rho(planes[0], orc.ray_dirs(rows, cols, place, W, H), centre)
    for v in (0, 33):
        dbg = puv.debug_tensors(lay, cam_arr, R.state, R.arena, v)
        P = orc.project(mat, occ, cams[v])
        ref_depth = np.where(P["visible"] == 1, P["depth_bits"], np.uint32(0xFFFFFFFF)).astype(np.uint32)
        assert np.array_equal(dbg["depth_key"].cpu().numpy().view(np.uint32), ref_depth)
        start, end, gids = orc.binning(P, cams[v])
        assert np.array_equal(dbg["keys_gid"].cpu().numpy().view(np.uint32), gids)
        ref, T, nc, _ = orc.forward(mat, occ, sh, cams[v])
        assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T))
        assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc)
        assert np.abs(img[v] - ref).max() <= IMG_ATOL
    del R, img, table, atlas
    torch.cuda.empty_cache()
    _run_rho(S, K, sh, [cams[0], cams[33]], 64, centre, views_checked=(0,), full_check=False)
