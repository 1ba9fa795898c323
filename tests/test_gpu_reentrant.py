"""GPU: puv_render_backward is re-entrant (include/puv.h): k backward calls after one render add
exactly k times the gradient of one call (the per-(view, Gaussian) moment slots
used to be zeroed by the forward only, so a second backward double-counted them)."""
import numpy as np
import pytest
import torch

from paper_2602_23040_b200 import puv
from synth.scenes import make_scene
from tests.gpu_common import gpu_scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,views", [(1, None), (2, [0, 5, 9])])
def test_backward_twice_is_twice(cfg, views):
    sc = make_scene(cfg)
    g = gpu_scene(sc, views=views)
    R = g["R"]
    img = R.forward(g["atlas"], g["occ"])
    tg = torch.from_numpy(np.stack([sc.target(v) for v in g["views"]])).cuda()
    dL = torch.empty_like(img)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    puv.l2_loss_grad(img, tg, dL, loss)
    g1 = R.backward(g["atlas"], g["occ"], dL)
    g2 = torch.zeros_like(g1)
    R.backward(g["atlas"], g["occ"], dL, grad=g2)
    R.backward(g["atlas"], g["occ"], dL, grad=g2)
    torch.cuda.synchronize()
    a, b = g1.cpu().numpy().astype(np.float64), g2.cpu().numpy().astype(np.float64)
    assert np.abs(a).max() > 0
    # each call rounds its fp64 texel sum once onto the fp32 accumulator: 2 g1 up to that rounding
    # (and the fp64 atomic order of the moments)
    assert np.all(np.abs(b - 2 * a) <= 1e-6 * np.abs(a) + 1e-12), np.abs(b - 2 * a).max()


def test_view_counts_match_debug_view_and_check_the_index():
    sc = make_scene(2)
    g = gpu_scene(sc, views=[0, 3])
    g["R"].forward(g["atlas"], g["occ"])
    for i in range(2):
        c = puv.view_counts(g["R"].state, i)
        d = puv.debug_view(g["layout"], g["cams"], g["R"].state, g["R"].arena, i)
        assert (c["n_vis"], c["K"], c["examined"], c["composited"]) == (d.n_visible, d.n_keys, d.n_examined,
                                                                         d.n_composited)
        assert c["K"] > 0 and c["composited"] > 0 and not c["overflow"]
    with pytest.raises(puv.PuvError):
        puv.view_counts(g["R"].state, 2)
