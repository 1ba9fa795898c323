"""Timeline of one C3 training step (stage instances with start/end ms) -> gpurun_out/timeline.json,
plus a summary: per-view gap between consecutive forward composites and when each view's binning
ended relative to its composite start."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_23040_b200 import puv  # noqa: E402
from paper_2602_23040_b200.shard import ShardedStep  # noqa: E402
from synth.scenes import make_scene  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
every = int(sys.argv[2]) if len(sys.argv) > 2 else 1   # views v with v % every == 0 (one rank of `every`)
sc = make_scene(cfg)
sc.cameras = [c for v, c in enumerate(sc.cameras) if v % every == 0]
dev = torch.device("cuda")
layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                            [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
st = ShardedStep(layout, sc.cameras, device=dev)
tg = torch.from_numpy(np.stack([sc.target(v) for v in st.views])).to(dev)
grad = torch.empty_like(atlas)
for w in range(3):
    st.step(atlas, occ, tg, grad, check_overflow=(w == 0))
torch.cuda.synchronize()
puv.profile_read(reset=True)
puv.profile_enable(True)
st.step(atlas, occ, tg, grad, check_overflow=False)
torch.cuda.synchronize()
puv.profile_enable(False)
tl = puv.profile_timeline()
puv.profile_read(reset=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(tl, open(os.path.join(ROOT, "gpurun_out", "timeline.json"), "w"))
fw = [(a, b) for s, a, b in tl if s == "raster_fwd"]
bins = [(a, b) for s, a, b in tl if s == "bin"]
ds = [(a, b) for s, a, b in tl if s == "depth_sort"]
end = max(b for _, _, b in tl)
print("step span ms", round(end, 2))
for s in ("project", "raster_fwd", "loss", "raster_bwd", "project_bwd", "depth_sort", "bin"):
    iv = [(a, b) for ss, a, b in tl if ss == s]
    if iv:
        print(f"{s:12s} n={len(iv):3d} first start {iv[0][0]:8.2f} last end {iv[-1][1]:8.2f} sum {sum(b - a for a, b in iv):8.2f}")
gaps = [fw[i + 1][0] - fw[i][1] for i in range(len(fw) - 1)]
print("fwd gaps: total", round(sum(gaps), 2), "max", round(max(gaps), 3), "n>0.05ms", sum(g > 0.05 for g in gaps))
late = [round(bins[i][1] - fw[i][0], 3) for i in range(min(len(bins), len(fw)))]
print("bin end - fwd start per view (<=0: binning was ready):", late[:16], "...")
print("binning span per view (ds start -> bin end):", [round(bins[i][1] - ds[i][0], 2) for i in range(min(12, len(ds)))])
