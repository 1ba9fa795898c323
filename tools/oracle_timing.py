"""CPU oracle timing on the host cores (SURVEY §8(d) oracle plan): C1 and C2 in full and C3 on two
views, fwd+bwd, on all cores (OpenMP) and on one thread; nproc + lscpu model.  Writes one JSON
line (the reported CPU baseline; not an optimisation target)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import host_cpu  # noqa: E402
from oracle import orc  # noqa: E402
from synth.scenes import make_scene  # noqa: E402


def run(cfg, views, threads):
    sc = make_scene(cfg)
    planes, occ, _ = orc.pack(sc.levels)
    val = planes.astype(np.float64)
    used = orc.set_threads(threads)
    t0 = time.perf_counter()
    for v in views:
        img = orc.forward(planes, occ, sc.sh_degree, sc.cameras[v], val=val)[0]
        _, dl = orc.l2_loss_grad(img, sc.target(v))
        orc.backward(planes, occ, sc.sh_degree, sc.cameras[v], dl, val=val)
    dt = time.perf_counter() - t0
    return {"config": f"C{cfg}", "views": len(views), "threads": used, "seconds": round(dt, 3),
            "views_per_s": len(views) / dt}


out = {"host": host_cpu(), "runs": []}
for cfg, views, single in ((1, [0], [0]), (2, list(range(16)), [0]), (3, [0, 33], [0])):
    out["runs"].append(run(cfg, views, 0))
    out["runs"].append(run(cfg, single, 1))
print(json.dumps(out))
