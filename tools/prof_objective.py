"""One L1+SSIM call on 8 views of 1920x1080 (one chunk), for ncu captures of K12."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_23040_b200 import puv  # noqa: E402

dev = torch.device("cuda")
V, H, W = 8, 1080, 1920
img = torch.rand((V, 3, H, W), device=dev) * 0.6 + 0.2
tgt = torch.rand((V, 3, H, W), device=dev)
dL = torch.empty_like(img)
loss = torch.empty(1, dtype=torch.float64, device=dev)
ws = torch.empty(puv.photo_workspace_bytes(W, H, 8), dtype=torch.uint8, device=dev)
for _ in range(2):
    puv.photo_loss_grad(img, tgt, dL, loss, 0.2, workspace=ws)
torch.cuda.synchronize()
print("ok", loss.item())
