"""View sharding over torch.distributed (row a10 of DESIGN.md §1).

Cameras shard naturally across GPUs (BJ.north_star): rank r renders views
v = r, r + n, r + 2n, ... (round-robin mixes the two camera rings of C3 so the
per-rank key counts balance), accumulates its local atlas gradient with
`render_backward` (+=), and the gradient planes are summed with ONE
all-reduce over NCCL (NVLink 5 / NVSwitch).  The atlas is replicated.  The
loss is summed the same way.  Everything here is orchestration: the render
runs in libpuv's kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import puv


def local_views(n_views: int, rank: int, world: int) -> list[int]:
    return [v for v in range(n_views) if v % world == rank]


def reduce_gradients(grad: torch.Tensor, loss: torch.Tensor, world: int, group=None) -> None:
    """The one exchange of the path (row a10): sum the atlas gradient planes and the loss over ranks."""
    if world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)


class ShardedStep:
    """One fwd + loss + bwd step over this rank's views, then the gradient all-reduce."""

    def __init__(self, layout, cameras, rank=0, world=1, device="cuda", bg=(0.0, 0.0, 0.0), arena_bytes=None,
                 group=None):
        self.rank, self.world, self.group = rank, world, group
        self.views = local_views(len(cameras), rank, world)
        if not self.views:
            raise ValueError(f"rank {rank} of {world} has no views (n_views={len(cameras)})")
        self.device = torch.device(device)
        self.cams = puv.cameras([cameras[v] for v in self.views])
        self.R = puv.Renderer(layout, self.cams, bg=bg, device=self.device, arena_bytes=arena_bytes)
        self.images = torch.empty(self.R.image_shape, dtype=torch.float32, device=self.device)
        self.dL = torch.empty_like(self.images)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)

    def step(self, atlas, occ, targets, grad, mask=None, check_overflow=True):
        """targets: (n_local, 3, H, W) fp32 on device; grad: (D, H_A, W_A) fp32, zeroed by the caller.
        Returns the (device) loss, summed over ranks when world > 1.

        check_overflow (default on): after the forward, read the key-arena overflow flag (one host
        sync) and, if a view did not fit, grow the arena and re-render before the loss and the
        backward, so an overflowed view can never contribute a wrong gradient.  Callers that have
        sized the arena already (the bench, after its first warm-up step) opt out explicitly and
        check `overflowed()` after their timed region."""
        # The separate calls, not the fused puv_render_l2_step: the fused pipeline measured the same
        # step time on C3 (118.7 ms both, the GPU is already saturated by the compositing and the
        # binning streams), and the separate calls keep each stage alone on its stream, so the
        # per-stage CUDA-event times the bench reports are not shared with concurrent stages.
        if check_overflow:   # sizes the key arena (grow and re-render)
            self.R.forward(atlas, occ, images=self.images, check=True)
        else:
            puv.render_views(self.R.layout, atlas, occ, self.cams, self.R.opts, self.images, self.R.state,
                             self.R.arena)
        puv.l2_loss_grad(self.images, targets, self.dL, self.loss)
        self.R.backward(atlas, occ, self.dL, grad=grad, mask=mask)
        reduce_gradients(grad, self.loss, self.world, self.group)
        return self.loss

    def step_host(self, atlas_host, occ, targets_host, grad, atlas_dev, targets_dev, loss_host, mask=None):
        """The same step from HOST inputs (the end-to-end call): the atlas is copied in first on the
        current stream (K1 reads all of it), the targets on a side copy stream so that their
        host->device transfer overlaps the render; the loss kernel waits for them.  The
        (rank-summed) loss is read back into `loss_host`.  Host tensors must be pinned for the
        copies to be asynchronous."""
        cur = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(device=self.device)
            self._targets_ready = torch.cuda.Event()
        self._copy_stream.wait_stream(cur)          # targets_dev is free once the previous step's loss ran
        with torch.cuda.stream(self._copy_stream):
            targets_dev.copy_(targets_host, non_blocking=True)
            self._targets_ready.record(self._copy_stream)
        atlas_dev.copy_(atlas_host, non_blocking=True)
        puv.render_views(self.R.layout, atlas_dev, occ, self.cams, self.R.opts, self.images, self.R.state,
                         self.R.arena)
        cur.wait_event(self._targets_ready)
        puv.l2_loss_grad(self.images, targets_dev, self.dL, self.loss)
        self.R.backward(atlas_dev, occ, self.dL, grad=grad, mask=mask)
        reduce_gradients(grad, self.loss, self.world, self.group)
        loss_host.copy_(self.loss, non_blocking=True)
        return loss_host

    def overflowed(self) -> bool:
        return puv.check_overflow(self.R.state, len(self.views))[0]
