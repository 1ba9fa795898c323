"""View sharding over torch.distributed (row a10 of DESIGN.md §1).

Cameras shard naturally across GPUs (BJ.north_star): rank r renders views
v = r, r + n, r + 2n, ... (round-robin mixes the two camera rings of C3 so the
per-rank key counts balance), forms its local atlas gradient with one
`puv_train_step` (render, L2 loss gradient, backward; in chunks of
`views_per_call` views so a large rig fits HBM), and the gradient planes are
summed with ONE all-reduce over NCCL (NVLink 5 / NVSwitch).  The atlas is
replicated.  The loss is summed the same way.

`FrameStep` is the temporal workload C4 (BJ.configs[3]): the (frame, view)
pairs of a frame sequence are dealt round-robin over the ranks, each frame has
its own atlas (plane table: per-frame position planes + shared constant
planes) and its own gradient, and the frames' gradients are exchanged in one
all-reduce restricted to the dynamic texels (static texels are frozen,
PAPER.md:410-414, so their gradient is exactly zero on every rank).

Everything here is orchestration: the render runs in libpuv's kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import puv


def local_views(n_views: int, rank: int, world: int) -> list[int]:
    return [v for v in range(n_views) if v % world == rank]


def local_pairs(n_frames: int, n_views: int, rank: int, world: int) -> list[tuple[int, int]]:
    """C4: (frame, view) pairs p = frame * n_views + view with p mod world == rank."""
    return [(p // n_views, p % n_views) for p in range(n_frames * n_views) if p % world == rank]


def reduce_gradients(grad: torch.Tensor, loss: torch.Tensor, world: int, group=None) -> None:
    """The one exchange of the path (row a10): sum the atlas gradient planes and the loss over ranks."""
    if world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)


def reduce_frame_gradients(grads: torch.Tensor, loss: torch.Tensor, world: int, dyn=None, group=None) -> None:
    """C4's exchange: sum the per-frame gradients (n_frames, D, H_A, W_A) and the loss over ranks.
    With `dyn` (flattened ids of the dynamic texels) only those texels are exchanged: gradient
    freezing makes every static texel's gradient exactly zero on every rank, so
    the compacted exchange is lossless and moves |dyn| / (H_A W_A) of the bytes (~25 % on C4)."""
    if world <= 1:
        return
    if dyn is None:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    else:
        flat = grads.view(grads.shape[0], grads.shape[1], -1)
        buf = flat.index_select(2, dyn)
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        flat.index_copy_(2, dyn, buf)
    dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)


class ShardedStep:
    """One fwd + loss + bwd step over this rank's views (puv_train_step), then the all-reduce."""

    def __init__(self, layout, cameras, rank=0, world=1, device="cuda", bg=(0.0, 0.0, 0.0), arena_bytes=None,
                 group=None, views_per_call=None):
        self.layout = layout
        self.rank, self.world, self.group = rank, world, group
        self.views = local_views(len(cameras), rank, world)
        if not self.views:
            raise ValueError(f"rank {rank} of {world} has no views (n_views={len(cameras)})")
        self.device = torch.device(device)
        self.cams = puv.cameras([cameras[v] for v in self.views])
        vpc = min(views_per_call or len(self.views), len(self.views))
        self.views_per_call = vpc
        self.st = puv.StepState(layout, puv.cameras([cameras[v] for v in self.views[:vpc]]), self.device,
                                arena_bytes=arena_bytes, bg=bg)

    @property
    def loss(self):
        return self.st.loss

    def step(self, atlas, occ, targets, grad, mask=None, check_overflow=True):
        """targets: (n_local, 3, H, W) fp32 on device; grad: (D, H_A, W_A) fp32, OVERWRITTEN with the
        gradient summed over all ranks' views.  Returns the (device) loss, summed over ranks.

        check_overflow (default on): after the step, read the key-arena overflow flag (one host
        sync) and, if a view chunk did not fit, grow the arena and re-run the step, so an
        overflowed view can never contribute a wrong gradient.  Callers that have sized the arena
        already (the bench, after its first warm-up step) opt out explicitly and check
        `overflowed()` after their timed region."""
        while True:
            puv.train_step(self.layout, atlas, occ, self.cams, targets, grad, self.st, mask=mask)
            if not check_overflow:
                break
            ov, need = self.st.overflow()
            if not ov:
                break
            self.st.grow(need)
        reduce_gradients(grad, self.st.loss, self.world, self.group)
        return self.st.loss

    def step_host(self, atlas_host, occ, targets_host, grad, atlas_dev, targets_dev, grad_host, loss_host,
                  mask=None):
        """The same step from HOST inputs, end to end (puv_train_step_host): the atlas is uploaded
        first (K1 reads all of it), the targets on the library's copy stream overlapping the
        render, and the result -- the gradient planes and the loss -- is copied back into
        `grad_host` / `loss_host`.  With world > 1 the download follows the all-reduce.  Host
        tensors should be pinned (asynchronous copies).  Synchronise before reading the results."""
        if self.world == 1:   # uploads and downloads in texel chunks overlapping K1 / K7
            puv.train_step_host_atlas(self.layout, atlas_dev, atlas_host, occ, self.cams, targets_host, targets_dev,
                                      grad, grad_host, loss_host, self.st, mask=mask)
            return loss_host
        puv.train_step_host(self.layout, atlas_dev, occ, self.cams, targets_host, targets_dev, grad, self.st,
                            uploads=[(atlas_host, atlas_dev)], downloads=[], mask=mask)
        if self.world > 1:
            reduce_gradients(grad, self.st.loss, self.world, self.group)
            grad_host.copy_(grad, non_blocking=True)
            loss_host.copy_(self.st.loss, non_blocking=True)
        return loss_host

    def overflowed(self) -> bool:
        """Whether any view chunk of the last step overflowed the key arena (synchronises)."""
        return self.st.overflow()[0]


class FrameStep:
    """C4 (BJ.configs[3]): one step renders every (frame, view) pair of a frame sequence fwd + bwd.

    Pairs are dealt round-robin over the ranks; per frame the local views run as one
    puv_train_step (chunks of `views_per_call`) into that frame's gradient, with gradient
    freezing by the dynamic labels.  Then ONE all-reduce sums the frames'
    gradients over the dynamic texels only (the static ones are zero on every rank), and the
    frames' losses are summed."""

    def __init__(self, layout, cameras, n_frames, rank=0, world=1, device="cuda", dynamic=None, bg=(0.0, 0.0, 0.0),
                 arena_bytes=None, group=None, views_per_call=None):
        self.layout = layout
        self.rank, self.world, self.group = rank, world, group
        self.n_frames, self.n_views = n_frames, len(cameras)
        self.device = torch.device(device)
        self.pairs = local_pairs(n_frames, len(cameras), rank, world)
        if not self.pairs:
            raise ValueError(f"rank {rank} of {world} has no (frame, view) pairs")
        self.frames = {}
        for f, v in self.pairs:
            self.frames.setdefault(f, []).append(v)
        self.cams = {f: puv.cameras([cameras[v] for v in vs]) for f, vs in self.frames.items()}
        vmax = max(len(vs) for vs in self.frames.values())
        vpc = min(views_per_call or vmax, vmax)
        self.views_per_call = vpc
        self.st = puv.StepState(layout, puv.cameras([cameras[0]] * vpc), self.device, arena_bytes=arena_bytes, bg=bg)
        self.losses = torch.zeros(n_frames, dtype=torch.float64, device=self.device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)
        # dynamic texel ids (flattened atlas index) for the compacted exchange; None = all texels
        self.dyn = None if dynamic is None else torch.nonzero(dynamic.reshape(-1)).reshape(-1).to(self.device)

    def local_targets_index(self):
        """[(frame, view)] in the order `step` expects the targets: frame-major, local views."""
        return [(f, v) for f in sorted(self.frames) for v in self.frames[f]]

    def step(self, frame_planes, occ, targets, grads, mask=None, check_overflow=True):
        """frame_planes: per frame a plane table (D CUDA planes; constant planes may be shared);
        targets: (n_local_pairs, 3, H, W) fp32 in `local_targets_index()` order; grads:
        (n_frames, D, H_A, W_A) fp32, OVERWRITTEN with each frame's gradient summed over ranks;
        mask: the dynamic labels D_i (H_A, W_A) uint8 (gradient freezing).  Returns the loss."""
        off = 0
        self.losses.zero_()
        for f in range(self.n_frames):
            vs = self.frames.get(f)
            if not vs:
                grads[f].zero_()   # no local view of this frame: it contributes nothing on this rank
                continue
            tg = targets[off:off + len(vs)]
            off += len(vs)
            while True:
                puv.train_step(self.layout, frame_planes[f], occ, self.cams[f], tg, grads[f], self.st, mask=mask)
                if not check_overflow:
                    break
                ov, need = self.st.overflow()
                if not ov:
                    break
                self.st.grow(need)
            self.losses[f:f + 1].copy_(self.st.loss)
        torch.sum(self.losses, dim=0, keepdim=True, out=self.loss)
        reduce_frame_gradients(grads, self.loss, self.world, self.dyn, self.group)
        return self.loss

    def overflowed(self) -> bool:
        return self.st.overflow()[0]
