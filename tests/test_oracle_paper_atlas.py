"""Pins of the paper-native atlas (NEXT-1): the K=8 pyramid layout and the UV rays of rho storage.

* 88.5 % packing efficiency is the number the paper prints, reproduced exactly by the
  SPEC.md:257 placement (2,088,960 / 2,359,296 = 0.8854) — golden/paper_atlas.json.
* Rays invert PAPER.md eq. (uvgs2): re-projecting a texel's ray gives back its (u, v).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import orc
from synth.scenes import Level

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_atlas.json")


def test_paper_layout_efficiency_golden():
    g = json.load(open(GOLDEN))
    rows, cols, place, W, H = orc.layout_paper(g["S"], g["K"])
    assert (W, H) == tuple(g["atlas"])
    used = int((rows.astype(np.int64) * cols).sum())
    assert used == g["used_texels"]
    assert abs(used / (W * H) - g["efficiency"]) < 5e-5
    # the schedule of PAPER.md:250-258: odd k halves N, even k halves M
    for k in range(1, len(rows)):
        if k % 2:
            assert (cols[k], rows[k]) == (cols[k - 1], rows[k - 1] // 2)
        else:
            assert (cols[k], rows[k]) == (cols[k - 1] // 2, rows[k - 1])


@pytest.mark.parametrize("S,K", [(1024, 8), (64, 8), (32, 5), (16, 2), (16, 1)])
def test_paper_layout_disjoint_in_bounds(S, K):
    rows, cols, place, W, H = orc.layout_paper(S, K)
    cover = np.zeros((H, W), np.int32)
    for k in range(K):
        x, y, rot = place[k]
        w, h = (rows[k], cols[k]) if rot else (cols[k], rows[k])
        assert 0 <= x and x + w <= W and 0 <= y and y + h <= H
        cover[y:y + h, x:x + w] += 1
    assert cover.max() == 1
    if K == 1:
        assert cover.sum() == W * H


def test_rays_invert_uv_projection():
    S, K = 64, 8
    rows, cols, place, W, H = orc.layout_paper(S, K)
    rays = orc.ray_dirs(rows, cols, place, W, H)
    levels = []
    for k in range(K):   # a level whose single plane stores the linear cell id, to locate cells after packing
        ids = (np.arange(rows[k] * cols[k], dtype=np.float32) + 1).reshape(1, rows[k], cols[k])
        levels.append(Level(planes=ids, occ=np.ones((rows[k], cols[k]), np.uint8),
                            labels=np.ones((rows[k], cols[k]), np.uint8)))
    packed, occ, _ = orc.pack(levels, place=place, W=W, H=H)
    n = np.linalg.norm(rays.astype(np.float64), axis=0)
    assert np.all(np.abs(n[occ == 1] - 1) < 3e-7) and np.all(n[occ == 0] == 0)
    for k in range(K):
        x, y, rot = place[k]
        w, h = (rows[k], cols[k]) if rot else (cols[k], rows[k])
        ids = packed[0, y:y + h, x:x + w].astype(np.int64) - 1
        r = rays[:, y:y + h, x:x + w].reshape(3, -1).astype(np.float64)
        theta = np.arctan2(r[1], r[0])
        phi = np.arccos(np.clip(r[2], -1, 1))
        u = np.floor((math.pi + theta) / (2 * math.pi) * cols[k]).astype(np.int64)
        v = np.floor(phi / math.pi * rows[k]).astype(np.int64)
        assert np.array_equal(v * cols[k] + u, ids.reshape(-1))


def test_spec_ray_example_and_rho_positions():
    """(u, v) = (0, 0) on a 2 x 2 grid -> theta = -pi/2, phi = pi/4; mu = c + rho ray."""
    rays = orc.ray_dirs(np.array([2]), np.array([2]), np.array([[0, 0, 0]]), 2, 2)
    th, ph = -math.pi / 2, math.pi / 4
    np.testing.assert_allclose(rays[:, 0, 0], [math.sin(ph) * math.cos(th), math.sin(ph) * math.sin(th),
                                               math.cos(ph)], atol=1e-7)
    rho = np.full((2, 2), 2.0, np.float32)
    mu = orc.positions_from_rho(rho, rays, [5.0, 5.0, 5.0])
    d = mu.astype(np.float64) - 5.0
    np.testing.assert_allclose(np.linalg.norm(d, axis=0), 2.0, rtol=1e-6)
    g = np.random.default_rng(0).normal(size=(3, 2, 2))
    np.testing.assert_allclose(orc.rho_grad(rays, g), np.einsum("kij,kij->ij", rays.astype(np.float64), g))
