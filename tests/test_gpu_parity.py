"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same
seeded inputs.  Bit-exact for everything integer (depth keys, visibility, tile
ranges, sorted lists, composited counts) and for the fp32-contract
transmittance; images within 1e-4 absolute; gradients within
max(1e-3 |g|, 1e-6) per component (BJ.north_star)."""
import math

import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import Camera, Level, Scene, look_at, make_scene, tiny_scene
from tests.gpu_common import (IMG_ATOL, describe_violations, gpu_scene, grad_violations, oracle_scene)

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint32)


# ---------------------------------------------------------------------------------------------
# contract functions: GPU == oracle bit for bit

def test_contract_exp_log_bitexact_exhaustive():
    """exp_c and log_c (R13) on the GPU equal the oracle's bit for bit on EVERY fp32 bit
    pattern (2^32 inputs each; NaN results compare as NaN).  This covers the whole used domains:
    exp_c of log-scales, -logits and the compositing exponents power in [t_g, 0]; log_c of
    255 o in (0, 255] (t_g = -log_c(255 o), R13 U5)."""
    step = 1 << 28
    for op in ("exp_c", "log_c"):
        f = orc.exp_c if op == "exp_c" else orc.log_c
        for lo in range(0, 1 << 32, step):
            x = np.arange(lo, lo + step, dtype=np.uint64).astype(np.uint32).view(np.float32)
            ref = f(x)
            got = puv.debug_contract(op, torch.from_numpy(x).cuda()).cpu().numpy()
            same = (_bits(got) == _bits(ref)) | (np.isnan(got) & np.isnan(ref))
            if not same.all():
                bad = np.flatnonzero(~same)[:5]
                raise AssertionError((op, hex(lo), x[bad], got[bad], ref[bad]))


# ---------------------------------------------------------------------------------------------

def _parity_view(sc, g, planes, occ, vi, view, img_gpu, check_bins=True, val=None):
    """Bit-exact binning / pixel state and image tolerance for one view. Returns oracle image."""
    cam = sc.cameras[view]
    P = orc.project(planes, occ, cam)
    dbg = puv.debug_tensors(g["layout"], g["cams"], g["R"].state, g["R"].arena, vi)
    ref_depth = np.where(P["visible"] == 1, P["depth_bits"], np.uint32(0xFFFFFFFF)).astype(np.uint32)
    got_depth = dbg["depth_key"].cpu().numpy().view(np.uint32)
    assert np.array_equal(got_depth, ref_depth), "depth keys / visibility differ"
    assert dbg["n_visible"] == int(P["visible"].sum())
    if check_bins:
        start, end, gids = orc.binning(P, cam)
        assert dbg["n_keys"] == gids.size
        assert np.array_equal(dbg["tile_start"].cpu().numpy().view(np.uint32), start)
        assert np.array_equal(dbg["tile_end"].cpu().numpy().view(np.uint32), end)
        assert np.array_equal(dbg["keys_gid"].cpu().numpy().view(np.uint32), gids), "sorted tile lists differ"
    ref_img, T, nc, st = orc.forward(planes, occ, sc.sh_degree, cam, val=val)
    assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T)), "T_final differs"
    assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc), "n_contrib differs"
    err = np.abs(img_gpu - ref_img).max()
    assert err <= IMG_ATOL, err
    return ref_img


def _grad_check(sc, planes, occ, views, dls_ref, grad_gpu, mask=None, bg=(0.0, 0.0, 0.0)):
    g_ref = np.zeros(planes.shape, np.float64)
    for v, dl in zip(views, dls_ref):
        orc.backward(planes, occ, sc.sh_degree, sc.cameras[v], dl, mask=mask, bg=bg, grad=g_ref)
    bad = grad_violations(grad_gpu, g_ref)
    frac = bad.mean()
    assert not bad.any(), f"{bad.sum()} of {bad.size} components ({frac:.2e}) outside tolerance: " + \
        describe_violations(grad_gpu, g_ref, bad)
    return g_ref


def _run(sc, views, dls=None, bg=(0.0, 0.0, 0.0), mask=None, arena_bytes=None):
    """GPU forward (+ its own L2 loss) and backward.  The backward consumes `dls` (the oracle's
    dL/dImage, fp64 -> fp32) when given, so gradient parity compares the two backwards on the
    same input; otherwise the GPU's own dL."""
    g = gpu_scene(sc, views, bg=bg, arena_bytes=arena_bytes)
    img = g["R"].forward(g["atlas"], g["occ"])
    tg = torch.from_numpy(np.stack([sc.target(v) for v in g["views"]])).cuda()
    dL = torch.empty_like(img)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    puv.l2_loss_grad(img, tg, dL, loss)
    if dls is not None:
        dL = torch.from_numpy(np.stack(dls).astype(np.float32)).cuda()
    m = None if mask is None else torch.from_numpy(mask).cuda()
    grad = g["R"].backward(g["atlas"], g["occ"], dL, mask=m)
    torch.cuda.synchronize()
    return g, img.cpu().numpy(), loss.item(), grad.cpu().numpy()


def _oracle_dls(sc, planes, occ, views, bg=(0.0, 0.0, 0.0)):
    """Oracle images and dL/dImage = I_hat - I (R11), rounded to the fp32 the GPU consumes."""
    imgs, dls = [], []
    for v in views:
        ref = orc.forward(planes, occ, sc.sh_degree, sc.cameras[v], bg=bg)[0]
        imgs.append(ref)
        dls.append(orc.l2_loss_grad(ref, sc.target(v))[1].astype(np.float32).astype(np.float64))
    return imgs, dls


def test_c1_full_parity():
    sc = make_scene(1)
    planes, occ, _ = oracle_scene(sc)
    refs, dls = _oracle_dls(sc, planes, occ, [0])
    g, img, loss, grad = _run(sc, [0], dls=dls)
    assert np.array_equal(_bits(g["atlas"].cpu().numpy()), _bits(planes)), "pack differs"
    _parity_view(sc, g, planes, occ, 0, 0, img[0])
    L_ref = orc.l2_loss_grad(refs[0], sc.target(0))[0]
    assert abs(loss - L_ref) <= 1e-6 * L_ref
    _grad_check(sc, planes, occ, [0], dls, grad)


def test_c2_parity_two_views():
    sc = make_scene(2)
    views = [0, 5]
    planes, occ, _ = oracle_scene(sc)
    refs, dls = _oracle_dls(sc, planes, occ, views)
    g, img, loss, grad = _run(sc, views, dls=dls)
    assert np.array_equal(_bits(g["atlas"].cpu().numpy()), _bits(planes))
    assert np.array_equal(g["occ"].cpu().numpy(), occ)
    for vi, v in enumerate(views):
        _parity_view(sc, g, planes, occ, vi, v, img[vi])
    _grad_check(sc, planes, occ, views, dls, grad)


@pytest.mark.parametrize("deg", [2, 3])
def test_sh_degree_parity_small(deg):
    """SH degrees 2 and 3 on a small two-level atlas (K1 / K7 instantiations with the fp64 SH staging),
    3 views of a ragged 150x110 image: bit-exact binning and pixel state, images and gradients."""
    from synth.scenes import _fill_levels, ring
    rng = np.random.default_rng(np.random.SeedSequence([2602, 23040, 90 + deg]))
    shapes = [(40, 36), (20, 18)]
    n = sum(r * c for r, c in shapes)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pos = d * rng.uniform(0.7, 1.1, size=(n, 1))
    levels = _fill_levels(rng, pos, deg, shapes, (0, 0, 0))
    sc = Scene(90 + deg, deg, levels, ring(3, 3.0, 0.4, 150, 110, 140.0), f"SH{deg} small")
    views = [0, 1, 2]
    planes, occ, _ = oracle_scene(sc)
    _, dls = _oracle_dls(sc, planes, occ, views)
    g, img, loss, grad = _run(sc, views, dls=dls)
    for vi in views:
        _parity_view(sc, g, planes, occ, vi, vi, img[vi])
    _grad_check(sc, planes, occ, views, dls, grad)


@pytest.mark.parametrize("wh", [(1, 1), (17, 3)])
def test_degenerate_tiny_images_and_empty_atlas(wh):
    """Degenerate sizes: a 1x1 image (one partial tile, one pixel) and a 17x3 one (two partial
    tiles), with pixels that terminate (T < 1e-4) and pixels that exhaust their list; then the same
    scene with every texel unoccupied (nothing visible: zero image, T_final = 1, n_contrib = 0 and
    an exactly zero gradient)."""
    W, H = wh
    rng = np.random.default_rng(7)
    n = 300
    mu = rng.uniform(-0.3, 0.3, (n, 3))
    sh = rng.random((n, 3))
    logit = rng.normal(0, 1, n)
    f = 2.0 * max(W, H)
    cams = [look_at((2.0, 0.2, 0.3), (0, 0, 0), W, H, f), look_at((-1.5, 1.5, 0.5), (0, 0, 0), W, H, f)]
    for empty in (False, True):
        sc = tiny_scene(mu, [-2.0] * 3, [1, 0, 0, 0], logit, sh, cams[0], 0)
        sc.cameras = cams
        sc.cfg = 97
        if empty:
            sc.levels[0].occ[:] = 0
        planes, occ, _ = oracle_scene(sc)
        _, dls = _oracle_dls(sc, planes, occ, [0, 1])
        g, img, loss, grad = _run(sc, [0, 1], dls=dls)
        for vi in (0, 1):
            _parity_view(sc, g, planes, occ, vi, vi, img[vi])
        _grad_check(sc, planes, occ, [0, 1], dls, grad)
        if empty:
            assert not img.any() and not grad.any()
            dbg = puv.debug_tensors(g["layout"], g["cams"], g["R"].state, g["R"].arena, 0)
            assert dbg["n_visible"] == 0 and dbg["n_keys"] == 0
            assert (dbg["t_final"].cpu().numpy() == 1.0).all() and not dbg["n_contrib"].cpu().numpy().any()


def test_edge_ragged_multiview_empty_views_bg_mask():
    """Ragged image (100x75, partial tiles), 18 views (> one camera batch), views that see nothing,
    a background colour and a dynamic mask."""
    rng = np.random.default_rng(7)
    n = 37 * 23
    mu = rng.uniform(-1, 1, (n, 3))
    sh = np.concatenate([rng.random((n, 3)), rng.normal(0, 0.1, (n, 9))], axis=1)
    cams = []
    for i in range(18):
        a = 2 * math.pi * i / 18
        if i in (4, 11):   # looking away from the scene: nothing visible
            cams.append(look_at((3 * math.cos(a), 3 * math.sin(a), 0.5), (6 * math.cos(a), 6 * math.sin(a), 0.5),
                                100, 75, 80.0))
        else:
            cams.append(look_at((3 * math.cos(a), 3 * math.sin(a), 0.5), (0, 0, 0), 100, 75, 80.0))
    sc = tiny_scene(mu, [-2.5] * 3, [1, 0, 0, 0], rng.normal(0, 1, n), sh, cams[0], 1)
    lv = sc.levels[0]
    lv.planes[3:6] = rng.normal(-2.6, 0.4, (3, 1, n)).astype(np.float32)
    lv.planes[6:10] = rng.normal(size=(4, 1, n)).astype(np.float32)
    lv.occ[0, ::13] = 0    # holes
    # reshape the 1 x n level into 37 x 23 so the atlas is 2-D
    sc.levels = [Level(planes=np.ascontiguousarray(lv.planes.reshape(-1, 37, 23)),
                       occ=np.ascontiguousarray(lv.occ.reshape(37, 23)),
                       labels=np.ascontiguousarray(lv.labels.reshape(37, 23)))]
    sc.cameras = cams
    sc.cfg = 99
    bg = (0.25, 0.5, 0.75)
    mask = (rng.random((37, 23)) < 0.5).astype(np.uint8)
    views = list(range(18))
    planes, occ, _ = oracle_scene(sc)
    _, dls = _oracle_dls(sc, planes, occ, views, bg=bg)
    g, img, loss, grad = _run(sc, views, dls=dls, bg=bg, mask=mask)
    for vi in views:
        cam = sc.cameras[vi]
        P = orc.project(planes, occ, cam)
        ref, T, nc, st = orc.forward(planes, occ, 1, cam, bg=bg)
        dbg = puv.debug_tensors(g["layout"], g["cams"], g["R"].state, g["R"].arena, vi)
        start, end, gids = orc.binning(P, cam)
        assert np.array_equal(dbg["keys_gid"].cpu().numpy().view(np.uint32), gids)
        assert np.array_equal(dbg["tile_start"].cpu().numpy().view(np.uint32), start)
        assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc)
        assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T))
        assert np.abs(img[vi] - ref).max() <= IMG_ATOL
        if vi in (4, 11):
            assert st["n_vis"] == 0 and dbg["n_keys"] == 0
            assert np.allclose(img[vi], np.array(bg)[:, None, None])
    _grad_check(sc, planes, occ, views, dls, grad, mask=mask, bg=bg)
    assert np.all(grad[:, mask == 0] == 0)


def test_high_opacity_alpha_cap_parity():
    """Opacity logits ~ N(4, 2): a third of the Gaussians have o >= 0.99, so the alpha cap (R9) is
    active on many pairs (zero gradient through o and the conic there, R10), mixed with uncapped
    pairs of the same Gaussians; 2 views, ragged 120x90 image, SH degree 1."""
    rng = np.random.default_rng(11)
    n = 40 * 30
    mu = rng.uniform(-1, 1, (n, 3))
    sh = np.concatenate([rng.random((n, 3)), rng.normal(0, 0.1, (n, 9))], axis=1)
    cams = [look_at((3.0, 0.3, 0.8), (0, 0, 0), 120, 90, 110.0), look_at((-0.5, 3.0, 1.2), (0, 0, 0), 120, 90, 110.0)]
    sc = tiny_scene(mu, [-2.4] * 3, [1, 0, 0, 0], rng.normal(4.0, 2.0, n), sh, cams[0], 1)
    lv = sc.levels[0]
    lv.planes[3:6] = rng.normal(-2.4, 0.3, (3, 1, n)).astype(np.float32)
    lv.planes[6:10] = rng.normal(size=(4, 1, n)).astype(np.float32)
    sc.levels = [Level(planes=np.ascontiguousarray(lv.planes.reshape(-1, 40, 30)),
                       occ=np.ascontiguousarray(lv.occ.reshape(40, 30)),
                       labels=np.ascontiguousarray(lv.labels.reshape(40, 30)))]
    sc.cameras = cams
    sc.cfg = 98
    views = [0, 1]
    planes, occ, _ = oracle_scene(sc)
    o = 1.0 / (1.0 + np.exp(-planes[10].astype(np.float64)))
    assert (o >= 0.99).mean() > 0.2
    _, dls = _oracle_dls(sc, planes, occ, views)
    g, img, loss, grad = _run(sc, views, dls=dls)
    for vi in views:
        _parity_view(sc, g, planes, occ, vi, vi, img[vi])
    _grad_check(sc, planes, occ, views, dls, grad)


def test_binning_dense_overlap_many_segments():
    """Adversarial binning: 12,000 large Gaussians in front of a 200x136 camera (13 x 9 tiles,
    ragged), each covering most of the image, so every 4x4-tile super-tile holds ~12k ranks
    (~24 level-2 segments of 512) and every tile list ~10k entries.  Lists, ranges, visibility,
    n_contrib, T_final bit-exact; image within tolerance.  Opacities are low (logit ~ N(-3, 0.5)),
    so pixels composite up to ~11k entries: the backward walks ~175 staged batches per tile and
    its fp64 T / Sd recurrences run ~11k steps; gradients checked at the north-star tolerance."""
    rng = np.random.default_rng(5)
    n = 120 * 100
    mu = np.stack([rng.uniform(-0.4, 0.4, n), rng.uniform(-0.4, 0.4, n), rng.uniform(-0.3, 0.3, n)], 1)
    cam = look_at((2.0, 0.0, 0.0), (0.0, 0.0, 0.0), 200, 136, 170.0)
    sc = tiny_scene(mu, [-1.2] * 3, [1, 0, 0, 0], rng.normal(-3.0, 0.5, n), np.full((n, 3), 0.4), cam, 0)
    lv = sc.levels[0]
    lv.planes[3:6] = rng.normal(-1.2, 0.2, (3, 1, n)).astype(np.float32)
    lv.planes[6:10] = rng.normal(size=(4, 1, n)).astype(np.float32)
    sc.levels = [Level(planes=np.ascontiguousarray(lv.planes.reshape(-1, 120, 100)),
                       occ=np.ascontiguousarray(lv.occ.reshape(120, 100)),
                       labels=np.ascontiguousarray(lv.labels.reshape(120, 100)))]
    sc.cfg = 97
    planes, occ, _ = oracle_scene(sc)
    P = orc.project(planes, occ, cam)
    vis = P[P["visible"] == 1]
    assert vis.size > 10000 and vis["tiles"].mean() > 60     # most of the 117 tiles per Gaussian
    _, dls = _oracle_dls(sc, planes, occ, [0])
    g, img, loss, grad = _run(sc, [0], dls=dls)
    _parity_view(sc, g, planes, occ, 0, 0, img[0])
    dbg = puv.debug_tensors(g["layout"], g["cams"], g["R"].state, g["R"].arena, 0)
    assert int(dbg["n_contrib"].max().item()) > 5000
    _grad_check(sc, planes, occ, [0], dls, grad)


def test_more_views_than_a_camera_batch():
    """70 views in one call (> kCamBatch = 64: two K1 / K7 launches, grid.y = 70 in K6): C1's
    4,096 Gaussians seen from a ring of 70 cameras at 96 x 80 px; every view's binning, pixel state
    and image, and the 70-view gradient sum, against the oracle."""
    sc = make_scene(1)
    cams = []
    for i in range(70):
        a = 2 * math.pi * i / 70
        cams.append(look_at((4 * math.cos(a), 4 * math.sin(a), 0.6 * math.sin(3 * a)), (0, 0, 0), 96, 80, 110.0))
    sc.cameras = cams
    sc.cfg = 96
    views = list(range(70))
    planes, occ, _ = oracle_scene(sc)
    _, dls = _oracle_dls(sc, planes, occ, views)
    g, img, loss, grad = _run(sc, views, dls=dls)
    for vi in (0, 1, 33, 63, 64, 69):
        _parity_view(sc, g, planes, occ, vi, vi, img[vi])
    for vi in views:
        ref = orc.forward(planes, occ, sc.sh_degree, sc.cameras[vi])[0]
        assert np.abs(img[vi] - ref).max() <= IMG_ATOL
    _grad_check(sc, planes, occ, views, dls, grad)


def test_arena_overflow_flag_and_retry():
    sc = make_scene(1)
    g = gpu_scene(sc, [0], arena_bytes=4096)
    R = g["R"]
    img = torch.empty(R.image_shape, dtype=torch.float32, device="cuda")
    puv.render_views(R.layout, g["atlas"], g["occ"], R.cams, R.opts, img, R.state, R.arena)
    ov, need = puv.check_overflow(R.state, 1)
    planes, occ, _ = oracle_scene(sc)
    P = orc.project(planes, occ, sc.cameras[0])
    vis = P[P["visible"] == 1]
    K = int(vis["tiles"].sum())
    # + the level-1 keys of the binning: super-tiles of 4 x 4 tiles (include/puv.h)
    K1 = int((((vis["x1"] + 3) // 4 - vis["x0"] // 4) * ((vis["y1"] + 3) // 4 - vis["y0"] // 4)).sum())
    assert ov and need == 4 * (K + K1)
    assert torch.all(img == 0)     # overflowed view renders only the (black) background
    img2 = R.forward(g["atlas"], g["occ"])   # grows the arena and re-renders
    assert R.arena.numel() >= 4 * K
    ref, _, _, _ = orc.forward(planes, occ, 0, sc.cameras[0])
    assert np.abs(img2.cpu().numpy()[0] - ref).max() <= IMG_ATOL


def test_pack_rotated_levels_and_unpack_roundtrip():
    rng = np.random.default_rng(3)
    D = 14
    lv = [Level(planes=rng.random((D, 5, 3)).astype(np.float32), occ=np.ones((5, 3), np.uint8),
                labels=np.ones((5, 3), np.uint8)),
          Level(planes=rng.random((D, 2, 4)).astype(np.float32), occ=(rng.random((2, 4)) < 0.5).astype(np.uint8),
                labels=np.ones((2, 4), np.uint8))]
    place = np.array([[0, 0, 1], [5, 0, 0]], np.int32)   # level 0 rotated: 3 tall x 5 wide
    ref_planes, ref_occ, _ = orc.pack(lv, place=place, W=9, H=3)
    layout = puv.layout_for_levels([(5, 3), (2, 4)], 0)
    layout.atlas_w, layout.atlas_h = 9, 3
    for k, (x, y, r) in enumerate(place):
        layout.level[k].x, layout.level[k].y, layout.level[k].rot90ccw = int(x), int(y), int(r)
    atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(l.planes).cuda() for l in lv],
                                [torch.from_numpy(l.occ).cuda() for l in lv])
    assert np.array_equal(atlas.cpu().numpy(), ref_planes) and np.array_equal(occ.cpu().numpy(), ref_occ)
    back = puv.unpack_levels(layout, atlas)
    for b, l in zip(back, lv):
        assert np.array_equal(b.cpu().numpy(), l.planes)


@pytest.mark.slow
def test_c3_full_size_64_view_parity():
    """C3 at full size in the bench's launch configuration (all 64 views in one render call and one
    backward call): for EVERY view bit-exact depth keys / visibility, T_final and n_contrib and the
    image within 1e-4; bit-exact sorted tile lists on views 0, 33 and every 8th view; then the
    gradient of the 64-view backward launch over ALL 1,048,576 x 59 texel components against the
    oracle summed over the 64 views, on the same dL/dImage (the oracle's, rounded to fp32)."""
    sc = make_scene(3)
    planes, occ, _ = oracle_scene(sc)
    val = planes.astype(np.float64)
    orc.set_threads(0)
    g = gpu_scene(sc, None)
    img = g["R"].forward(g["atlas"], g["occ"])
    imgs = img.cpu().numpy()
    del img
    n = len(sc.cameras)
    assert n == 64
    H, W = sc.cameras[0].height, sc.cameras[0].width
    dls = np.empty((n, 3, H, W), np.float32)
    g_ref = np.zeros(planes.shape, np.float64)
    for v in range(n):
        ref = _parity_view(sc, g, planes, occ, v, v, imgs[v], check_bins=(v % 8 == 1 or v in (0, 33)), val=val)
        dls[v] = orc.l2_loss_grad(ref, sc.target(v))[1]
        orc.backward(planes, occ, sc.sh_degree, sc.cameras[v], dls[v].astype(np.float64), val=val, grad=g_ref)
    grad = g["R"].backward(g["atlas"], g["occ"], torch.from_numpy(dls).cuda())
    torch.cuda.synchronize()
    got = grad.cpu().numpy()
    bad = grad_violations(got, g_ref)
    assert not bad.any(), f"{bad.sum()} of {bad.size} components outside tolerance: " + \
        describe_violations(got, g_ref, bad)
