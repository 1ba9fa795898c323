"""Measurements of the "next" rows on one GPU; one JSON line per row.

  label: supp. Alg. 1 flow masking on C4 (1,048,576 Gaussians x 55 cameras, 1080p seeded motion masks):
         (Gaussian, camera) tests per second, CUDA events, warm-up 2, 5 timed calls.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_23040_b200 import puv  # noqa: E402
from synth.scenes import make_scene, motion_masks  # noqa: E402


def bench_label(steps=5, warmup=2):
    sc = make_scene(4)
    dev = torch.device("cuda")
    lv = sc.levels[0]
    layout = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    atlas = torch.from_numpy(lv.planes).to(dev)
    occ = torch.from_numpy(lv.occ).to(dev)
    cams = puv.cameras(sc.cameras)
    masks = torch.from_numpy(motion_masks(sc, list(range(len(sc.cameras))))).to(dev)
    ws = torch.empty(puv.label_workspace_bytes(cams[0].width, cams[0].height), dtype=torch.uint8, device=dev)
    labels = torch.empty((lv.rows, lv.cols), dtype=torch.uint8, device=dev)
    for _ in range(warmup):
        puv.label_dynamic(layout, atlas, occ, cams, masks, labels=labels, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = puv.kernel_launches()
    e0.record()
    for _ in range(steps):
        puv.label_dynamic(layout, atlas, occ, cams, masks, labels=labels, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    n = lv.rows * lv.cols
    tests = n * len(sc.cameras)
    return {"row": "NEXT-3 flow masking (supp. Alg. 1)", "metric": "(Gaussian, camera) tests/s",
            "value": tests / (ms / 1e3), "ms_per_call": ms, "gaussians": n, "cameras": len(sc.cameras),
            "dynamic_fraction": float(labels.float().mean().item()),
            "mask_fraction": float(masks.float().mean().item()),
            "gpu_launches_per_call": (puv.kernel_launches() - l0) // steps,
            "workload": "C4 atlas 1024^2 SH3, 55 dome cameras 1920x1080, seeded disc motion masks"}


if __name__ == "__main__":
    which = sys.argv[1:] or ["label"]
    for w in which:
        print(json.dumps({"label": bench_label}[w]()), flush=True)
