import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import make_scene
from tests.gpu_common import gpu_scene, grad_violations
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
views = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [0]
sc = make_scene(cfg)
g = gpu_scene(sc, views)
img = g['R'].forward(g['atlas'], g['occ'])
tg = torch.from_numpy(np.stack([sc.target(v) for v in views])).cuda()
dL = torch.empty_like(img); loss = torch.zeros(1, dtype=torch.float64, device='cuda')
puv.l2_loss_grad(img, tg, dL, loss)
planes, occ, _ = orc.pack(sc.levels)
gref = np.zeros(planes.shape)
dls = []
for vi, v in enumerate(views):
    ref = orc.forward(planes, occ, sc.sh_degree, sc.cameras[v])[0]
    dl = orc.l2_loss_grad(ref, sc.target(v))[1].astype(np.float32).astype(np.float64)
    dls.append(dl)
    orc.backward(planes, occ, sc.sh_degree, sc.cameras[v], dl, grad=gref)
grad = g['R'].backward(g['atlas'], g['occ'], torch.from_numpy(np.stack(dls).astype(np.float32)).cuda()).cpu().numpy()
bad = grad_violations(grad, gref)
print('violations', bad.sum(), 'of', bad.size, 'per plane', bad.sum(axis=(1, 2)))
rel = np.abs(grad - gref) / np.maximum(np.abs(gref), 1e-6)
for idx in np.argwhere(bad)[:12]:
    t = tuple(idx)
    print(t, 'gpu', grad[t], 'ref', gref[t], 'rel', rel[t])
# overall error stats per plane
for d in range(planes.shape[0]):
    m = np.abs(gref[d]) > 1e-6
    print(d, 'max rel', rel[d][m].max() if m.any() else 0, 'p99.9', np.quantile(rel[d][m], 0.999) if m.any() else 0)
