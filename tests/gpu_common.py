"""Shared helpers of the GPU parity tests: run a scene through the C ABI and
through the oracle on the same seeded inputs (synth/)."""
import numpy as np
import torch

from oracle import orc
from paper_2602_23040_b200 import puv

GRAD_RTOL = 1e-3     # BJ.north_star: gradients within 1e-3 relative ...
GRAD_ATOL = 1e-6     # ... with 1e-6 absolute below that magnitude
IMG_ATOL = 1e-4      # BJ.north_star: images within 1e-4 absolute


def gpu_scene(scene, views=None, bg=(0.0, 0.0, 0.0), arena_bytes=None):
    """Pack on the GPU, render the selected views. Returns dict of tensors/objects."""
    dev = torch.device("cuda")
    shapes = [(lv.rows, lv.cols) for lv in scene.levels]
    layout = puv.layout_for_levels(shapes, scene.sh_degree)
    lp = [torch.from_numpy(lv.planes).to(dev) for lv in scene.levels]
    lo = [torch.from_numpy(lv.occ).to(dev) for lv in scene.levels]
    atlas, occ = puv.pack_atlas(layout, lp, lo)
    vids = list(range(len(scene.cameras))) if views is None else list(views)
    cams = puv.cameras([scene.cameras[v] for v in vids])
    R = puv.Renderer(layout, cams, bg=bg, device=dev, arena_bytes=arena_bytes)
    return {"layout": layout, "atlas": atlas, "occ": occ, "cams": cams, "R": R, "views": vids}


def oracle_scene(scene):
    planes, occ, place = orc.pack(scene.levels)
    return planes, occ, place


def grad_violations(g_gpu, g_ref, rtol=GRAD_RTOL, atol=GRAD_ATOL):
    """Boolean mask of components outside max(rtol |ref|, atol)."""
    tol = np.maximum(rtol * np.abs(g_ref), atol)
    return np.abs(g_gpu - g_ref) > tol


def describe_violations(g_gpu, g_ref, bad, limit=8):
    idx = np.argwhere(bad)[:limit]
    return "; ".join(f"{tuple(i)}: gpu={g_gpu[tuple(i)]:.6g} ref={g_ref[tuple(i)]:.6g}" for i in idx)
