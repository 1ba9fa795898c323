"""GPU: the sharded step (row a10) and its end-to-end form from host inputs.

`ShardedStep.step_host` copies the atlas and the targets from pinned host memory (targets on a
side stream, overlapped with the forward) and must produce the same loss and gradient as `step`
on device-resident inputs; both must match the oracle's L2 loss on the same views."""
import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from paper_2602_23040_b200.shard import ShardedStep
from synth.scenes import make_scene
from tests.gpu_common import GRAD_ATOL, oracle_scene

pytestmark = pytest.mark.gpu


def test_step_host_equals_step_c2():
    sc = make_scene(2, views=4)
    dev = torch.device("cuda")
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                                [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    st = ShardedStep(layout, sc.cameras, device=dev)
    tg_host = torch.from_numpy(np.stack([sc.target(v) for v in st.views])).pin_memory()
    grad = torch.zeros_like(atlas)
    loss = st.step(atlas, occ, tg_host.to(dev), grad, check_overflow=True).item()
    g_dev = grad.clone()
    atlas_host = atlas.cpu().pin_memory()
    a_dev, t_dev = torch.empty_like(atlas), torch.empty(tuple(tg_host.shape), dtype=torch.float32, device=dev)
    loss_host = torch.zeros(1, dtype=torch.float64).pin_memory()
    for _ in range(2):   # twice: the second step reuses the copy stream and the device buffers
        grad.zero_()
        st.step_host(atlas_host, occ, tg_host, grad, a_dev, t_dev, loss_host)
        torch.cuda.synchronize()
        assert abs(loss_host.item() - loss) <= 1e-12 * loss   # fp64 partial sums, atomic order
        g = grad.cpu().numpy()
        ref = g_dev.cpu().numpy()
        assert np.all(np.abs(g - ref) <= np.maximum(1e-6 * np.abs(ref), GRAD_ATOL))
    planes, aocc, _ = oracle_scene(sc)
    L_ref = sum(orc.l2_loss_grad(orc.forward(planes, aocc, sc.sh_degree, sc.cameras[v])[0], sc.target(v))[0]
                for v in st.views)
    assert abs(loss - L_ref) <= 1e-6 * L_ref


def test_fused_l2_step_equals_separate_calls_c2():
    """puv_render_l2_step (per-view loss + composite backward on a second stream, overlapping later
    views) against render_views + l2_loss_grad + render_backward: images, T_final, n_contrib and the
    tile lists bit-identical, loss and gradients up to fp64 atomic-order rounding; and the oracle."""
    sc = make_scene(2, views=6)
    dev = torch.device("cuda")
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                                [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    cams = puv.cameras(sc.cameras)
    tg = torch.from_numpy(np.stack([sc.target(v) for v in range(6)])).to(dev)
    R = puv.Renderer(layout, cams, device=dev)
    img = R.forward(atlas, occ)
    dL = torch.empty_like(img)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    puv.l2_loss_grad(img, tg, dL, loss)
    grad = R.backward(atlas, occ, dL)
    torch.cuda.synchronize()
    ref = {v: {k: t.clone() for k, t in puv.debug_tensors(layout, cams, R.state, R.arena, v).items()
               if isinstance(t, torch.Tensor)} for v in range(6)}
    img_f, dL_f = torch.empty_like(img), torch.empty_like(img)
    loss_f = torch.zeros(1, dtype=torch.float64, device=dev)
    grad_f = torch.zeros_like(atlas)
    for _ in range(2):
        grad_f.zero_()
        puv.render_l2_step(layout, atlas, occ, cams, R.opts, img_f, tg, dL_f, loss_f, None, R.state, R.arena, grad_f)
        torch.cuda.synchronize()
        assert torch.equal(img_f, img)
        assert torch.equal(dL_f, dL)
        assert abs(loss_f.item() - loss.item()) <= 1e-12 * loss.item()
        for v in range(6):
            d = puv.debug_tensors(layout, cams, R.state, R.arena, v)
            for k in ("t_final", "n_contrib", "tile_start", "tile_end", "depth_key", "keys_gid"):
                assert torch.equal(d[k], ref[v][k]), (v, k)
        g, r = grad_f.cpu().numpy(), grad.cpu().numpy()
        assert np.all(np.abs(g - r) <= np.maximum(1e-6 * np.abs(r), GRAD_ATOL))
    planes, aocc, _ = oracle_scene(sc)
    L_ref = sum(orc.l2_loss_grad(orc.forward(planes, aocc, sc.sh_degree, sc.cameras[v])[0], sc.target(v))[0]
                for v in range(6))
    assert abs(loss_f.item() - L_ref) <= 1e-6 * L_ref
