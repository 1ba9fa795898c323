"""GPU parity of the flow-masking kernel (supp. Alg. 1): labels bit-exact vs the
oracle's plain window scan, including the r_max clamp, empty masks, cameras seeing nothing, and a
C4-size atlas (1M Gaussians x 55 cameras) on sampled texels."""
import math

import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import look_at, make_scene, motion_masks
from tests.test_oracle_masking import _scene

pytestmark = pytest.mark.gpu


def _gpu_labels(planes, occ, cams_list, masks, r_max, shapes=None):
    dev = torch.device("cuda")
    D, HA, WA = planes.shape
    layout = puv.layout_for_levels([(HA, WA)], {14: 0, 23: 1, 59: 3}[D])
    cams = puv.cameras(cams_list)
    return puv.label_dynamic(layout, torch.from_numpy(np.ascontiguousarray(planes)).to(dev),
                             torch.from_numpy(np.ascontiguousarray(occ)).to(dev), cams,
                             torch.from_numpy(np.ascontiguousarray(masks)).to(dev), r_max=r_max).cpu().numpy()


@pytest.mark.parametrize("r_max", [64, 3, 0])
def test_tiny_scenes_bitexact(r_max):
    for seed in range(4):
        planes, occ, cams, masks, _ = _scene(seed, n=200)
        ref = orc.label_dynamic(planes, occ, cams, masks, r_max=r_max)
        got = _gpu_labels(planes, occ, cams, masks, r_max)
        assert np.array_equal(got, ref), (seed, np.nonzero(got != ref))
    # empty masks: all static
    got = _gpu_labels(planes, occ, cams, np.zeros_like(masks), 64)
    assert got.sum() == 0


def test_c2_all_views_bitexact():
    sc = make_scene(2)
    planes, occ, _ = orc.pack(sc.levels)
    views = list(range(16))
    masks = motion_masks(sc, views)
    ref = orc.label_dynamic(planes, occ, sc.cameras, masks)
    got = _gpu_labels(planes, occ, sc.cameras, masks, 64)
    assert np.array_equal(got, ref)
    assert 0 < got.sum() < occ.sum()


@pytest.mark.slow
def test_c4_size_sampled_bitexact():
    sc = make_scene(4)
    planes, occ, _ = orc.pack(sc.levels)
    masks = motion_masks(sc, list(range(len(sc.cameras))))
    got = _gpu_labels(planes, occ, sc.cameras, masks, 64)
    rng = np.random.default_rng(0)
    gids = rng.choice(planes.shape[1] * planes.shape[2], size=3000, replace=False)
    ref = orc.label_dynamic(planes, occ, sc.cameras, masks, gids=gids)
    assert np.array_equal(got.reshape(-1)[gids], ref.reshape(-1)[gids])
    frac = got.mean()
    assert 0.01 < frac < 0.99, frac
