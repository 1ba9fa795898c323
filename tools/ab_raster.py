"""A/B timing of the raster kernels: C3 (64 views, 1080p), one forward to size the arena, then
`--reps` timed forwards and backwards (CUDA events on the current stream, median).  Run once per
library build (PUV_LIB=...), interleaved, to compare kernel variants on the same box."""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_23040_b200 import puv  # noqa: E402
from synth.scenes import make_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--tag", default=os.environ.get("PUV_LIB", "default"))
ap.add_argument("--fused", action="store_true", help="also time the fused puv_render_l2_step")
a = ap.parse_args()
sc = make_scene(3, views=a.views)
dev = torch.device("cuda")
layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                            [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
cams = puv.cameras(sc.cameras)
R = puv.Renderer(layout, cams, device=dev)
img = R.forward(atlas, occ)
tg = torch.from_numpy(np.stack([sc.target(v) for v in range(a.views)])).to(dev)
dL = torch.empty_like(img)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
puv.l2_loss_grad(img, tg, dL, loss)
grad = torch.zeros_like(atlas)
R.backward(atlas, occ, dL, grad=grad)
torch.cuda.synchronize()
fw, bw = [], []
for _ in range(a.reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    puv.render_views(R.layout, atlas, occ, R.cams, R.opts, img, R.state, R.arena)
    e[1].record()
    R.backward(atlas, occ, dL, grad=grad)
    e[2].record()
    torch.cuda.synchronize()
    fw.append(e[0].elapsed_time(e[1]))
    bw.append(e[1].elapsed_time(e[2]))
sep, fus = [], []
for _ in range(a.reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    puv.render_views(R.layout, atlas, occ, R.cams, R.opts, img, R.state, R.arena)
    puv.l2_loss_grad(img, tg, dL, loss)
    R.backward(atlas, occ, dL, grad=grad)
    e[1].record()
    torch.cuda.synchronize()
    sep.append(e[0].elapsed_time(e[1]))
    if a.fused:
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        puv.render_l2_step(R.layout, atlas, occ, R.cams, R.opts, img, tg, dL, loss, None, R.state, R.arena, grad)
        e[1].record()
        torch.cuda.synchronize()
        fus.append(e[0].elapsed_time(e[1]))
out = {"tag": a.tag, "views": a.views, "fwd_ms": statistics.median(fw), "bwd_ms": statistics.median(bw),
       "step_sep_ms": statistics.median(sep), "fwd_all": fw, "bwd_all": bw}
if fus:
    out["step_fused_ms"] = statistics.median(fus)
print(json.dumps(out), flush=True)
