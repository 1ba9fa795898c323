"""GPU: the sharded step (row a10) and its end-to-end form from host inputs.

* 2 ranks on the one B200 (subprocesses, gloo over CUDA tensors: NCCL refuses two ranks on one
  device; the exchange is the same `reduce_gradients` call the bench makes over NCCL):
  every rank's per-view images, depth keys, tile ranges, tile lists, T_final and n_contrib are
  bit-identical to the world-1 run (the forward has no atomics); the exchanged
  gradient is the fp32 sum of the two ranks' local gradients; it equals the world-1 gradient up
  to that summation order and the oracle's at the north_star tolerance (+ the same allowance).
* `step_host` (puv_train_step_host_atlas: host atlas and targets in, gradient + loss out, the
  copies overlapping K1 / K7 in texel chunks) and the generic puv_train_step_host equal `step`.
* View chunks (views_per_call) equal one call up to the fp32 rounding of each chunk's sum."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from paper_2602_23040_b200.shard import ShardedStep, local_views
from synth.scenes import make_scene
from tests.gpu_common import GRAD_ATOL, GRAD_RTOL, oracle_scene
from tests.shard_worker import digests, frame_setup, frame_targets, scene_views

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U32 = 2.0 ** -23   # fp32 unit roundoff x 2 (one ulp relative)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gpu_atlas(sc, dev):
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    atlas, occ = puv.pack_atlas(layout, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                                [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    return layout, atlas, occ


@pytest.mark.parametrize("cfg,views", [(2, None), (3, [0, 1, 32, 33])])
def test_two_ranks_equal_world_one_and_oracle(cfg, views, tmp_path):
    sc = scene_views(cfg, views)
    dev = torch.device("cuda")
    layout, atlas, occ = _gpu_atlas(sc, dev)
    # world 1: every view in one call
    st1 = ShardedStep(layout, sc.cameras, 0, 1, dev)
    tg = torch.from_numpy(np.stack([sc.target(v) for v in range(len(sc.cameras))])).to(dev)
    g_all = torch.empty_like(atlas)
    loss_all = st1.step(atlas, occ, tg, g_all).item()
    torch.cuda.synchronize()
    dg1 = digests(layout, st1.cams, st1.st, len(sc.cameras))
    dL = st1.st.dL.cpu().numpy().astype(np.float64)
    g_all = g_all.cpu().numpy().astype(np.float64)
    del st1, atlas, occ, tg
    torch.cuda.empty_cache()
    # world 2
    port = _port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LOCAL_RANK="0")
        vs = "all" if views is None else ",".join(map(str, views))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "shard_worker.py"), str(cfg), vs,
                                       str(tmp_path)], env=env, cwd=ROOT, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    for p in procs:
        out, _ = p.communicate(timeout=900)
        assert p.returncode == 0, out.decode()[-3000:]
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    n = len(sc.cameras)
    for r in range(2):
        assert list(res[r]["views"]) == local_views(n, r, 2)
        for i, v in enumerate(res[r]["views"]):
            assert res[r]["digests"][i] == dg1[v], f"rank {r} view {v}: forward outputs differ from world 1"
    g0, g1 = res[0]["grad"].astype(np.float64), res[1]["grad"].astype(np.float64)
    assert np.array_equal(res[0]["grad"], res[1]["grad"]), "ranks hold different exchanged gradients"
    l0, l1 = res[0]["local"].astype(np.float64), res[1]["local"].astype(np.float64)
    part = np.abs(l0) + np.abs(l1)
    # the exchange is the fp32 sum of the local gradients (up to 1-ulp fp64 atomic-order noise of the
    # step's second backward)
    s32 = (res[0]["local"] + res[1]["local"]).astype(np.float64)
    assert np.all(np.abs(g0 - s32) <= 2 * U32 * part + 1e-30)
    # world 2 == world 1 up to the order of the sum (each rank's partial rounded to fp32 once)
    assert np.all(np.abs(g0 - g_all) <= 4 * U32 * (part + np.abs(g_all)) + 1e-30)
    assert abs(res[0]["loss"][0] - loss_all) <= 1e-12 * loss_all and res[0]["loss"][0] == res[1]["loss"][0]
    # and the oracle's gradient on the same dL/dImage, at the north_star tolerance + that allowance
    planes, aocc, _ = oracle_scene(sc)
    val = planes.astype(np.float64)
    g_ref = np.zeros(planes.shape, np.float64)
    orc.set_threads(0)
    for v in range(n):
        orc.backward(planes, aocc, sc.sh_degree, sc.cameras[v], dL[v], val=val, grad=g_ref)
    tol = np.maximum(GRAD_RTOL * np.abs(g_ref), GRAD_ATOL) + 4 * U32 * part
    bad = np.abs(g0 - g_ref) > tol
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside tolerance"


def test_step_host_equals_step_c2():
    sc = make_scene(2, views=4)
    dev = torch.device("cuda")
    layout, atlas, occ = _gpu_atlas(sc, dev)
    st = ShardedStep(layout, sc.cameras, device=dev)
    tg_host = torch.from_numpy(np.stack([sc.target(v) for v in st.views])).pin_memory()
    grad = torch.empty_like(atlas)
    loss = st.step(atlas, occ, tg_host.to(dev), grad).item()
    g_dev = grad.cpu().numpy()
    atlas_host = atlas.cpu().pin_memory()
    a_dev, t_dev = torch.empty_like(atlas), torch.empty(tuple(tg_host.shape), dtype=torch.float32, device=dev)
    grad_host = torch.empty(tuple(atlas.shape), dtype=torch.float32).pin_memory()
    loss_host = torch.zeros(1, dtype=torch.float64).pin_memory()
    for _ in range(2):   # twice: the second step reuses the device buffers and the copy stream
        grad.fill_(7.0)  # OVERWRITTEN by the step
        grad_host.zero_()
        st.step_host(atlas_host, occ, tg_host, grad, a_dev, t_dev, grad_host, loss_host)
        torch.cuda.synchronize()
        assert abs(loss_host.item() - loss) <= 1e-12 * loss   # fp64 partial sums, atomic order
        g = grad_host.numpy()
        assert np.all(np.abs(g - g_dev) <= np.maximum(1e-6 * np.abs(g_dev), 1e-12))
    # the generic host-buffer call (upload / download lists) gives the same
    grad_host.zero_()
    loss_host.zero_()
    puv.train_step_host(layout, a_dev, occ, st.cams, tg_host, t_dev, grad, st.st, uploads=[(atlas_host, a_dev)],
                        downloads=[(grad, grad_host), (st.st.loss, loss_host)])
    torch.cuda.synchronize()
    assert abs(loss_host.item() - loss) <= 1e-12 * loss
    assert np.all(np.abs(grad_host.numpy() - g_dev) <= np.maximum(1e-6 * np.abs(g_dev), 1e-12))
    planes, aocc, _ = oracle_scene(sc)
    L_ref = sum(orc.l2_loss_grad(orc.forward(planes, aocc, sc.sh_degree, sc.cameras[v])[0], sc.target(v))[0]
                for v in st.views)
    assert abs(loss - L_ref) <= 1e-6 * L_ref


def test_view_chunks_equal_one_call_c2():
    """views_per_call = 5 over 16 views (chunks 5, 5, 5, 1) against one call: the loss up to fp64
    order; the gradient up to the fp32 rounding of each chunk's partial sum (bound from the
    chunks' own gradients); the overflow flags of every chunk are accumulated."""
    sc = make_scene(2)
    dev = torch.device("cuda")
    layout, atlas, occ = _gpu_atlas(sc, dev)
    tg = torch.from_numpy(np.stack([sc.target(v) for v in range(16)])).to(dev)
    one = ShardedStep(layout, sc.cameras, device=dev)
    g1 = torch.empty_like(atlas)
    L1 = one.step(atlas, occ, tg, g1).item()
    ch = ShardedStep(layout, sc.cameras, device=dev, views_per_call=5)
    gc = torch.empty_like(atlas)
    Lc = ch.step(atlas, occ, tg, gc).item()
    assert abs(L1 - Lc) <= 1e-12 * L1
    parts = np.zeros(tuple(atlas.shape))
    for c0 in range(0, 16, 5):
        vs = list(range(c0, min(c0 + 5, 16)))
        s = ShardedStep(layout, [sc.cameras[v] for v in vs], device=dev)
        gp = torch.empty_like(atlas)
        s.step(atlas, occ, tg[vs[0]:vs[-1] + 1], gp)
        parts += np.abs(gp.cpu().numpy())
    a, b = g1.cpu().numpy().astype(np.float64), gc.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(a - b) <= 4 * U32 * (parts + np.abs(a)) + 1e-30)
    # a too-small arena: every chunk overflows, the flag and the needed size come back, and the
    # default checked step grows the arena and re-runs to the same result
    small = ShardedStep(layout, sc.cameras, device=dev, views_per_call=5, arena_bytes=4096)
    puv.train_step(layout, atlas, occ, small.cams, tg, gc, small.st)
    ov, need = small.st.overflow()
    assert ov and need > 4096
    Ls = small.step(atlas, occ, tg, gc).item()
    assert not small.overflowed() and abs(Ls - L1) <= 1e-12 * L1


def test_two_ranks_frame_step_c4(tmp_path):
    """C4's FrameStep at world size 2 on the one GPU: the 6 (frame, view) pairs of frames {0, 29} x
    views {0, 27, 54} dealt round-robin, each rank's per-frame gradients frozen on static texels,
    then the compacted exchange over the dynamic texels: every rank ends with the fp32 sum of the
    two ranks' local gradients (up to atomic-order noise), = the world-1 FrameStep up to that
    summation order, static texels exactly zero, and the loss = the world-1 loss."""
    from paper_2602_23040_b200.shard import FrameStep, local_pairs
    dev = torch.device("cuda")
    sc, layout, occ, labels, frames, views, tables, pos = frame_setup(dev)
    fs = FrameStep(layout, [sc.cameras[v] for v in views], len(frames), 0, 1, dev, dynamic=labels)
    tg = frame_targets(sc, frames, views, fs.local_targets_index(), dev)
    g1 = torch.empty((2, layout.planes, layout.atlas_h, layout.atlas_w), dtype=torch.float32, device=dev)
    L1 = fs.step(tables, occ, tg, g1, mask=labels).item()
    g1 = g1.cpu().numpy().astype(np.float64)
    del fs, tg
    torch.cuda.empty_cache()
    port = _port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "shard_worker.py"), "4", "all",
                                       str(tmp_path)], env=env, cwd=ROOT, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    for p in procs:
        out, _ = p.communicate(timeout=900)
        assert p.returncode == 0, out.decode()[-3000:]
    res = [np.load(tmp_path / f"frames_rank{r}.npz") for r in range(2)]
    for r in range(2):
        assert [tuple(x) for x in res[r]["pairs"]] == local_pairs(2, 3, r, 2)
    assert np.array_equal(res[0]["grad"], res[1]["grad"])
    g = res[0]["grad"].astype(np.float64)
    l0, l1 = res[0]["local"].astype(np.float64), res[1]["local"].astype(np.float64)
    part = np.abs(l0) + np.abs(l1)
    s32 = (res[0]["local"] + res[1]["local"]).astype(np.float64)
    assert np.all(np.abs(g - s32) <= 2 * U32 * part + 1e-30)
    assert np.all(np.abs(g - g1) <= 4 * U32 * (part + np.abs(g1)) + 1e-30)
    static = labels.cpu().numpy() == 0
    assert np.all(g[:, :, static] == 0) and np.abs(g).max() > 0
    assert abs(res[0]["loss"][0] - L1) <= 1e-12 * L1 and res[0]["loss"][0] == res[1]["loss"][0]
