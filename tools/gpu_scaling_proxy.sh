# Per-rank step time at 64/N views (the work one rank of an N-GPU run does on C3, round-robin views
# r, r+N, ...) on one B200: a proxy for the strong-scaling curve when only one GPU is available.
set -u
mkdir -p gpurun_out
make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
python - <<'PY' > gpurun_out/scaling_proxy.json
import json, sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2602_23040_b200 import puv
from paper_2602_23040_b200.shard import ShardedStep
from synth.scenes import make_scene
sc = make_scene(3)
dev = torch.device("cuda")
layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                            [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
out = {}
for n in (1, 2, 4, 8):
    st = ShardedStep(layout, sc.cameras, rank=0, world=1, device=dev)   # world 1: no exchange here
    views = [v for v in range(64) if v % n == 0]
    st = ShardedStep(layout, [sc.cameras[v] for v in views], device=dev)
    tg = torch.from_numpy(np.stack([sc.target(v) for v in views])).to(dev)
    g = torch.empty_like(atlas)
    for w in range(3):
        st.step(atlas, occ, tg, g, check_overflow=(w == 0))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        st.step(atlas, occ, tg, g, check_overflow=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[n] = {"views_per_rank": len(views), "ms_per_step_one_rank": ms}
    del st, tg, g
    torch.cuda.empty_cache()
t1 = out[1]["ms_per_step_one_rank"]
for n in out:
    # + the ring all-reduce lower bound of the 247.5 MB gradient at 900 GB/s per direction
    ar = 0.0 if n == 1 else 2 * (n - 1) / n * 247.5e6 / 900e9 * 1e3
    out[n]["allreduce_ms_lower_bound"] = ar
    out[n]["predicted_efficiency"] = t1 / (n * (out[n]["ms_per_step_one_rank"] + ar))
print(json.dumps(out))
PY
cat gpurun_out/scaling_proxy.json
