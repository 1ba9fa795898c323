"""One rank of the 2-process sharded-step GPU test (tests/test_gpu_shard.py), launched as a
subprocess with RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in the environment.  Both ranks
share the one B200 (cuda:0); the exchange is gloo over CUDA tensors (NCCL refuses two ranks on
one device).  Writes its per-view digests, its local (pre-exchange) gradient and the exchanged
gradient and loss to <outdir>/rank<r>.npz."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_23040_b200 import puv  # noqa: E402
from paper_2602_23040_b200.shard import ShardedStep  # noqa: E402
from synth.scenes import make_scene  # noqa: E402


def digests(layout, cams, st, n):
    """sha256 of each view's image, depth keys, tile ranges, tile lists, T_final and n_contrib."""
    out = []
    for i in range(n):
        d = puv.debug_tensors(layout, cams, st.state, st.arena, i)
        h = hashlib.sha256()
        h.update(st.images[i].cpu().numpy().tobytes())
        for k in ("depth_key", "tile_start", "tile_end", "keys_gid", "t_final", "n_contrib"):
            h.update(d[k].cpu().numpy().tobytes())
        out.append(h.hexdigest())
    return out


def scene_views(cfg, views):
    sc = make_scene(cfg)
    if views is not None:
        sc.cameras = [sc.cameras[v] for v in views]
    return sc


def frame_setup(dev):
    """C4 frames {0, 29} x views {0, 27, 54} (FrameStep): layout, per-frame plane tables, labels, targets."""
    from synth.scenes import frame_positions
    sc = make_scene(4)
    lv = sc.levels[0]
    layout = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    base = torch.from_numpy(lv.planes).to(dev)
    occ = torch.from_numpy(lv.occ).to(dev)
    labels = torch.from_numpy(lv.labels).to(dev)
    frames, views = [0, 29], [0, 27, 54]
    pos = [torch.from_numpy(frame_positions(sc, f)).to(dev) for f in frames]
    tables = [[p[0], p[1], p[2]] + [base[d] for d in range(3, layout.planes)] for p in pos]
    return sc, layout, occ, labels, frames, views, tables, pos


def frame_targets(sc, frames, views, idx, dev):
    return torch.from_numpy(np.stack([sc.target(views[v], frame=frames[f]) for f, v in idx])).to(dev)


def main_frames(outdir, rank, world, dev):
    from paper_2602_23040_b200.shard import FrameStep
    sc, layout, occ, labels, frames, views, tables, pos = frame_setup(dev)
    fs = FrameStep(layout, [sc.cameras[v] for v in views], len(frames), rank, world, dev, dynamic=labels)
    tg = frame_targets(sc, frames, views, fs.local_targets_index(), dev)
    grads = torch.empty((2, layout.planes, layout.atlas_h, layout.atlas_w), dtype=torch.float32, device=dev)
    fs.world = 1                                   # the local gradients, before the exchange
    fs.step(tables, occ, tg, grads, mask=labels)
    torch.cuda.synchronize()
    local = grads.cpu().numpy()
    fs.world = world
    loss = fs.step(tables, occ, tg, grads, mask=labels)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"frames_rank{rank}.npz"), local=local, grad=grads.cpu().numpy(),
             loss=np.array([loss.item()]), pairs=np.array(fs.pairs))


def main():
    cfg = int(sys.argv[1])
    views = None if sys.argv[2] == "all" else [int(x) for x in sys.argv[2].split(",")]
    outdir = sys.argv[3]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if cfg == 4:
        main_frames(outdir, rank, world, dev)
        dist.barrier()
        dist.destroy_process_group()
        return
    sc = scene_views(cfg, views)
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                                [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    stp = ShardedStep(layout, sc.cameras, rank, world, dev)
    tg = torch.from_numpy(np.stack([sc.target(v) for v in stp.views])).to(dev)
    grad = torch.empty_like(atlas)
    # the local gradient before the exchange (world 1 call on this rank's views) ...
    puv.train_step(layout, atlas, occ, stp.cams, tg, grad, stp.st)
    torch.cuda.synchronize()
    local = grad.cpu().numpy()
    # ... then the sharded step itself (render, backward, all-reduce)
    loss = stp.step(atlas, occ, tg, grad)
    torch.cuda.synchronize()
    dg = digests(layout, stp.cams, stp.st, len(stp.views))
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), views=np.array(stp.views), digests=np.array(dg),
             local=local, grad=grad.cpu().numpy(), loss=np.array([loss.item()]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
