"""GPU parity on the remaining BASELINE.json configs (sampled: the oracle is slow at these sizes).

C4 (BJ.configs[3]): a frame sequence of 1024^2 atlases sharing 56 constant planes (plane-pointer
tables, no copies), dynamic texels moved by a smooth flow field, gradient freezing with the
dynamic labels.  C5 (BJ.configs[4]): 2048^2 + 1024^2 levels at 3840x2160.
Bit-exact binning / pixel state, images within 1e-4, gradients within max(1e-3|g|, 1e-6)."""
import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import frame_positions, make_scene
from tests.gpu_common import IMG_ATOL, describe_violations, grad_violations

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint32)


def _check_view(dbg, planes, occ, sh_degree, cam, img, bg=(0.0, 0.0, 0.0)):
    P = orc.project(planes, occ, cam)
    start, end, gids = orc.binning(P, cam)
    assert np.array_equal(dbg["tile_start"].cpu().numpy().view(np.uint32), start)
    assert np.array_equal(dbg["tile_end"].cpu().numpy().view(np.uint32), end)
    assert np.array_equal(dbg["keys_gid"].cpu().numpy().view(np.uint32), gids)
    ref, T, nc, _ = orc.forward(planes, occ, sh_degree, cam, bg=bg)
    assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T))
    assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc)
    assert np.abs(img - ref).max() <= IMG_ATOL
    return ref


def test_c4_frames_shared_planes_and_freezing():
    sc = make_scene(4)
    dev = torch.device("cuda")
    lv = sc.levels[0]
    layout = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    base = torch.from_numpy(lv.planes).to(dev)            # frame-independent planes 3..58 live here
    occ_t = torch.from_numpy(lv.occ).to(dev)
    mask = lv.labels.astype(np.uint8)
    mask_t = torch.from_numpy(mask).to(dev)
    views = [0, 27]
    cams = puv.cameras([sc.cameras[v] for v in views])
    for frame in (0, 29):
        pos = torch.from_numpy(frame_positions(sc, frame)).to(dev)
        planes_t = [pos[0], pos[1], pos[2]] + [base[d] for d in range(3, layout.planes)]
        R = puv.Renderer(layout, cams, device=dev)
        img = R.forward(planes_t, occ_t).cpu().numpy()
        planes = lv.planes.copy()
        planes[0:3] = frame_positions(sc, frame)
        occ = lv.occ
        dls = []
        for vi, v in enumerate(views):
            dbg = puv.debug_tensors(layout, cams, R.state, R.arena, vi)
            ref = _check_view(dbg, planes, occ, 3, sc.cameras[v], img[vi])
            dls.append(orc.l2_loss_grad(ref, sc.target(v))[1].astype(np.float32).astype(np.float64))
        grad = R.backward(planes_t, occ_t, torch.from_numpy(np.stack(dls).astype(np.float32)).to(dev),
                          mask=mask_t).cpu().numpy()
        g_ref = np.zeros(planes.shape)
        for v, dl in zip(views, dls):
            orc.backward(planes, occ, 3, sc.cameras[v], dl, mask=mask, grad=g_ref)
        bad = grad_violations(grad, g_ref)
        assert not bad.any(), describe_violations(grad, g_ref, bad)
        assert np.all(grad[:, mask == 0] == 0)       # static texels frozen
        del R
        torch.cuda.empty_cache()


def test_c5_one_view_4k():
    sc = make_scene(5)
    dev = torch.device("cuda")
    layout = puv.layout_for_levels([(l.rows, l.cols) for l in sc.levels], 3)
    atlas, occ_t = puv.pack_atlas(layout, [torch.from_numpy(l.planes).to(dev) for l in sc.levels],
                                  [torch.from_numpy(l.occ).to(dev) for l in sc.levels])
    planes, occ, _ = orc.pack(sc.levels)
    assert np.array_equal(_bits(atlas.cpu().numpy()), _bits(planes))
    v = 7
    cams = puv.cameras([sc.cameras[v]])
    R = puv.Renderer(layout, cams, device=dev)
    img = R.forward(atlas, occ_t).cpu().numpy()
    dbg = puv.debug_tensors(layout, cams, R.state, R.arena, 0)
    ref = _check_view(dbg, planes, occ, 3, sc.cameras[v], img[0])
    dl = orc.l2_loss_grad(ref, sc.target(v))[1].astype(np.float32).astype(np.float64)
    grad = R.backward(atlas, occ_t, torch.from_numpy(dl.astype(np.float32))[None].to(dev)).cpu().numpy()
    g_ref = orc.backward(planes, occ, 3, sc.cameras[v], dl)
    bad = grad_violations(grad, g_ref)
    assert not bad.any(), describe_violations(grad, g_ref, bad)


def test_c4_frame_step_equals_per_frame_steps_and_oracle():
    """FrameStep (the C4 bench path): (frame, view) pairs of frames {0, 29} x views {0, 27, 54} in one
    step, each frame's gradient frozen by the dynamic labels.  Each frame's gradient equals a
    separate puv_train_step of that frame (up to fp64 atomic order) and the oracle's on the same
    dL/dImage; static texels are exactly zero; the loss is the sum of the frames'."""
    from paper_2602_23040_b200.shard import FrameStep
    sc = make_scene(4)
    dev = torch.device("cuda")
    lv = sc.levels[0]
    layout = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    base = torch.from_numpy(lv.planes).to(dev)
    occ_t = torch.from_numpy(lv.occ).to(dev)
    mask = lv.labels.astype(np.uint8)
    mask_t = torch.from_numpy(mask).to(dev)
    frames, views = [0, 29], [0, 27, 54]
    cams_all = [sc.cameras[v] for v in views]
    pos = [torch.from_numpy(frame_positions(sc, f)).to(dev) for f in frames]
    tables = [[p[0], p[1], p[2]] + [base[d] for d in range(3, layout.planes)] for p in pos]
    fs = FrameStep(layout, cams_all, len(frames), device=dev, dynamic=mask_t)
    idx = fs.local_targets_index()
    tg = torch.from_numpy(np.stack([sc.target(views[v], frame=frames[f]) for f, v in idx])).to(dev)
    grads = torch.full((2, layout.planes, lv.rows, lv.cols), 3.0, device=dev)   # OVERWRITTEN
    loss = fs.step(tables, occ_t, tg, grads, mask=mask_t).item()
    G = grads.cpu().numpy().astype(np.float64)
    assert np.all(G[:, :, mask == 0] == 0)
    orc.set_threads(0)
    L_sum = 0.0
    for fi, f in enumerate(frames):
        st = puv.StepState(layout, puv.cameras(cams_all), dev)
        g1 = torch.empty_like(base)
        puv.train_step(layout, tables[fi], occ_t, puv.cameras(cams_all), tg[3 * fi:3 * fi + 3], g1, st, mask=mask_t)
        torch.cuda.synchronize()
        L_sum += st.loss.item()
        a = g1.cpu().numpy().astype(np.float64)
        assert np.all(np.abs(G[fi] - a) <= 1e-6 * np.abs(a) + 1e-30)
        planes = lv.planes.copy()
        planes[0:3] = frame_positions(sc, f)
        val = planes.astype(np.float64)
        dL = st.dL.cpu().numpy().astype(np.float64)
        g_ref = np.zeros(planes.shape)
        for vi, v in enumerate(views):
            orc.backward(planes, lv.occ, 3, sc.cameras[v], dL[vi], mask=mask, val=val, grad=g_ref)
        bad = grad_violations(a, g_ref)
        assert not bad.any(), describe_violations(a, g_ref, bad)
    assert abs(loss - L_sum) <= 1e-12 * L_sum
