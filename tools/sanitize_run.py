"""One fwd + L2 + bwd of a small config through the C ABI, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  usage: sanitize_run.py CONFIG [VIEWS]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_23040_b200 import puv  # noqa: E402
from synth.scenes import make_scene  # noqa: E402

cfg = int(sys.argv[1])
views = int(sys.argv[2]) if len(sys.argv) > 2 else None
sc = make_scene(cfg, views=views)
dev = torch.device("cuda")
layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                            [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
cams = puv.cameras(sc.cameras)
R = puv.Renderer(layout, cams, device=dev)
img = R.forward(atlas, occ)
tg = torch.from_numpy(np.stack([sc.target(v) for v in range(len(sc.cameras))])).to(dev)
dL = torch.empty_like(img)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
puv.l2_loss_grad(img, tg, dL, loss)
grad = R.backward(atlas, occ, dL)
torch.cuda.synchronize()
print(f"config {cfg}: views {len(sc.cameras)}, loss {loss.item():.6f}, |grad|max {grad.abs().max().item():.4g}")
