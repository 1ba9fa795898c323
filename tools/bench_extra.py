"""Measurements of the "next" rows on one GPU; one JSON line per row.

  label: supp. Alg. 1 flow masking on C4 (1,048,576 Gaussians x 55 cameras, 1080p seeded motion masks):
         (Gaussian, camera) tests per second, CUDA events, warm-up 2, 5 timed calls.
  rho:   the paper-native atlas (NEXT-1): S = 1024, K = 8 pyramid (2,088,960 texels, 1536^2 atlas), SH3,
         rho positions on UV rays, C3's 64-view 1080p rig; fwd + L2 + bwd views/s, and the same Gaussians
         rendered from a materialised xyz atlas (the cost of the ray representation).
  lpo:   NEXT-2 on C3: per step quant_fit + quantize (16-bit xyz, 8-bit rest) + the proxy render fwd + L2 +
         bwd into the master gradient (STE), views/s vs the plain step; the quantiser's HBM GB/s.
  objective: NEXT-4 on C3's shapes: L1+SSIM loss + dL over 64 views of 1920x1080 (vs the L2 harness
         loss), and the regularisers over the 1024^2 atlas; CUDA events, warm-up 3, 10 timed calls.
"""
import math
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_23040_b200 import puv  # noqa: E402
from synth.scenes import make_scene, motion_masks, moving_region_masks, ring, rho_scene  # noqa: E402


def bench_label(steps=5, warmup=2, region=True, radius=None):
    """region=True: the motion masks of a spatially coherent moving part (a 0.6 m ball around the
    scene point nearest to the densest texel neighbourhood, synth.moving_region_masks); False: the
    round-1 seeded disc masks (unstructured: their OR over 55 cameras labels ~97 % dynamic)."""
    sc = make_scene(4)
    dev = torch.device("cuda")
    lv = sc.levels[0]
    layout = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    atlas = torch.from_numpy(lv.planes).to(dev)
    occ = torch.from_numpy(lv.occ).to(dev)
    cams = puv.cameras(sc.cameras)
    if region:
        mu = lv.planes[0:3].reshape(3, -1).T
        rng = np.random.default_rng(np.random.SeedSequence([2602, 23040, 4, 5]))
        cand = mu[rng.choice(mu.shape[0], 64, replace=False)]
        # the candidate with the most texels within 0.6 m: a moving part inside one of the blobs
        counts = [(np.linalg.norm(mu[::16] - c, axis=1) <= 0.6).sum() for c in cand]
        centre = cand[int(np.argmax(counts))]
        radius = LABEL_RADIUS if radius is None else radius
        masks_np = moving_region_masks(sc, list(range(len(sc.cameras))), centre, radius)
        inside = float((np.linalg.norm(mu - centre, axis=1) <= radius).mean())
    else:
        masks_np = motion_masks(sc, list(range(len(sc.cameras))))
    masks = torch.from_numpy(masks_np).to(dev)
    ws = torch.empty(puv.label_workspace_bytes(cams[0].width, cams[0].height), dtype=torch.uint8, device=dev)
    labels = torch.empty((lv.rows, lv.cols), dtype=torch.uint8, device=dev)
    for _ in range(warmup):
        puv.label_dynamic(layout, atlas, occ, cams, masks, labels=labels, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = puv.kernel_launches()
    e0.record()
    for _ in range(steps):
        puv.label_dynamic(layout, atlas, occ, cams, masks, labels=labels, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    n = lv.rows * lv.cols
    tests = n * len(sc.cameras)
    return {"row": "NEXT-3 flow masking (supp. Alg. 1)", "metric": "(Gaussian, camera) tests/s",
            "value": tests / (ms / 1e3), "ms_per_call": ms, "gaussians": n, "cameras": len(sc.cameras),
            "dynamic_fraction": float(labels.float().mean().item()),
            "mask_fraction": float(masks.float().mean().item()),
            "gpu_launches_per_call": (puv.kernel_launches() - l0) // steps,
            "moving_ball_fraction": inside if region else None,
            "workload": "C4 atlas 1024^2 SH3, 55 dome cameras 1920x1080, " +
                        (f"masks of a moving {radius} m ball (synth.moving_region_masks)" if region else
                         "seeded disc motion masks")}


# radius of the moving ball of the NEXT-3 row: chosen with label_sweep so that Alg. 1 labels about
# the 25 % dynamic texels of BJ.configs[3] (the OR over 55 dome cameras labels every Gaussian on a
# ray through the ball in any view, so the labelled fraction grows much faster than the ball)
LABEL_RADIUS = 0.6


def bench_label_sweep():
    """Labelled (dynamic) fraction and throughput of Alg. 1 against the moving-ball radius."""
    return [bench_label(steps=2, warmup=1, radius=r) for r in (0.05, 0.1, 0.15, 0.2, 0.3, 0.45, 0.6)]


def _time_steps(R, planes, occ, targets, steps, warmup):
    img = torch.empty(R.image_shape, dtype=torch.float32, device=targets.device)
    dL = torch.empty_like(img)
    loss = torch.zeros(1, dtype=torch.float64, device=targets.device)
    grad = torch.zeros((R.layout.planes,) + tuple(occ.shape), dtype=torch.float32, device=targets.device)
    R.forward(planes, occ, images=img, check=True)

    def step():
        grad.zero_()
        puv.render_views(R.layout, planes, occ, R.cams, R.opts, img, R.state, R.arena)
        puv.l2_loss_grad(img, targets, dL, loss)
        R.backward(planes, occ, dL, grad=grad)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    puv.profile_read(reset=True)
    puv.profile_enable(True)
    l0 = puv.kernel_launches()
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    puv.profile_enable(False)
    prof = puv.profile_read(reset=True)
    ms = e0.elapsed_time(e1) / steps
    return ms, {k: round(v / steps, 3) for k, v in prof["ms"].items()}, (puv.kernel_launches() - l0) // steps


def bench_rho(steps=5, warmup=3):
    dev = torch.device("cuda")
    S, K, sh = 1024, 8, 3
    cams = ring(32, 3.5, 1.0, 1920, 1080, 1400.0) + ring(32, 3.5, 2.0, 1920, 1080, 1400.0, offset=math.pi / 32)
    lay_x = puv.layout_paper(S, K, sh)
    shapes = [(lay_x.level[k].rows, lay_x.level[k].cols) for k in range(K)]
    sc = rho_scene(64, shapes, sh, cams)
    lay = puv.with_rho(lay_x, (0.0, 0.0, 0.0))
    atlas, occ = puv.pack_atlas(lay, [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels],
                                [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels])
    rays = puv.ray_planes(lay)
    table = puv.rho_plane_table(atlas, rays)
    cam_arr = puv.cameras(cams)
    targets = torch.from_numpy(np.stack([sc.target(v) for v in range(len(cams))])).to(dev)
    R = puv.Renderer(lay, cam_arr, device=dev)
    ms, stages, launches = _time_steps(R, table, occ, targets, steps, warmup)
    n_vis = sum(puv.debug_view(lay, cam_arr, R.state, R.arena, v).n_visible for v in range(len(cams)))
    del R
    # the same Gaussians from an xyz atlas (positions materialised by the library's own K1 arithmetic:
    # mu = c + rho ray, computed here with torch fp32 ops, non-fused, only to build the comparison input)
    xyz = atlas.clone()
    xyz[0:3] = rays * atlas[0:1]
    Rx = puv.Renderer(lay_x, cam_arr, device=dev)
    ms_x, stages_x, _ = _time_steps(Rx, xyz, occ, targets, steps, warmup)
    n = sum(r * c for r, c in shapes)
    return {"row": "NEXT-1 paper-native atlas (rho on UV rays, K=8 pyramid)", "metric": "views/s fwd+bwd",
            "value": len(cams) / (ms / 1e3), "ms_per_step": ms, "stage_ms_per_step": stages,
            "gpu_launches_per_step": launches, "xyz_atlas_views_per_s": len(cams) / (ms_x / 1e3),
            "xyz_stage_ms_per_step": stages_x, "gaussians": n, "atlas": [lay.atlas_w, lay.atlas_h],
            "visible_per_view": n_vis / len(cams),
            "workload": "S=1024 K=8 rho atlas SH3 (2,088,960 G), C3 64-view ring rig 1920x1080, synthetic shell"}


def _events_ms(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def bench_objective(steps=10, warmup=3):
    dev = torch.device("cuda")
    V, H, W = 64, 1080, 1920
    g = torch.Generator(device=dev).manual_seed(3)
    img = torch.rand((V, 3, H, W), device=dev, generator=g) * 0.6 + 0.2
    tgt = torch.rand((V, 3, H, W), device=dev, generator=g)
    dL = torch.empty_like(img)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ws = torch.empty(puv.photo_workspace_bytes(W, H, 8), dtype=torch.uint8, device=dev)
    l0 = puv.kernel_launches()
    ms_photo = _events_ms(lambda: puv.photo_loss_grad(img, tgt, dL, loss, 0.2, workspace=ws), steps, warmup)
    launches = (puv.kernel_launches() - l0) // (steps + warmup)
    ms_l2 = _events_ms(lambda: puv.l2_loss_grad(img, tgt, dL, loss), steps, warmup)
    sc = make_scene(3, views=1)
    lv = sc.levels[0]
    lay = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    atlas = torch.from_numpy(lv.planes).to(dev)
    occ = torch.from_numpy(lv.occ).to(dev)
    grad = torch.zeros_like(atlas)
    rws = torch.empty(puv.reg_workspace_bytes(), dtype=torch.uint8, device=dev)
    ms_reg = _events_ms(lambda: puv.reg_loss_grad(lay, atlas, occ, grad, loss, 1e-4, 1e-4, 0.05, workspace=rws),
                        steps, warmup)
    n = V * 3 * H * W
    return {"row": "NEXT-4 paper objective (L1 + SSIM, scale/opacity regularisers)", "metric": "views/s (loss + dL)",
            "value": V / (ms_photo / 1e3), "ms_per_call_64_views": ms_photo, "l2_ms_per_call_64_views": ms_l2,
            "photo_gpix_ch_per_s": n / (ms_photo / 1e3) / 1e9, "gpu_launches_per_call": launches,
            "reg_ms_per_call_1M_texels": ms_reg,
            "workload": "64 views 1920x1080x3 fp32 (C3 image shapes), lambda_ssim 0.2, 8-view chunks; "
                        "regularisers on C3's 1024^2 SH3 atlas, lambdas 1e-4, s_max 0.05"}


def bench_lpo(steps=5, warmup=3):
    dev = torch.device("cuda")
    sc = make_scene(3)
    lv = sc.levels[0]
    layout = puv.layout_for_levels([(lv.rows, lv.cols)], 3)
    atlas = torch.from_numpy(lv.planes).to(dev)
    occ = torch.from_numpy(lv.occ).to(dev)
    cams = puv.cameras(sc.cameras)
    targets = torch.from_numpy(np.stack([sc.target(v) for v in range(len(sc.cameras))])).to(dev)
    R = puv.Renderer(layout, cams, device=dev)
    spec = puv.quant_fit(layout, atlas, occ)
    proxy, _ = puv.quantize(layout, atlas, occ, spec)
    img = torch.empty(R.image_shape, dtype=torch.float32, device=dev)
    dL = torch.empty_like(img)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    grad = torch.zeros_like(atlas)
    R.forward(proxy, occ, images=img, check=True)

    fused_opts = puv.opts(lpo=(spec, 16, 8))

    def step(lpo):
        grad.zero_()
        src, o = atlas, R.opts
        if lpo == "proxy":        # refit + materialise the proxy atlas, render it
            puv.quant_fit(layout, atlas, occ, spec=spec)
            puv.quantize(layout, atlas, occ, spec, proxy=proxy)
            src = proxy
        elif lpo == "fused":      # refit, then the render reads the masters through the quantiser
            puv.quant_fit(layout, atlas, occ, spec=spec)
            o = fused_opts
        puv.render_views(layout, src, occ, R.cams, o, img, R.state, R.arena)
        puv.l2_loss_grad(img, targets, dL, loss)
        puv.render_backward(layout, src, occ, R.cams, o, dL, None, R.state, R.arena, grad)

    out = {}
    for lpo in ("proxy", "fused", False):
        for _ in range(warmup):
            step(lpo)
        torch.cuda.synchronize()
        puv.profile_read(reset=True)
        puv.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step(lpo)
        e1.record()
        torch.cuda.synchronize()
        puv.profile_enable(False)
        prof = puv.profile_read(reset=True)
        out[lpo] = (e0.elapsed_time(e1) / steps, {k: round(v / steps, 3) for k, v in prof["ms"].items()})
    # the quantiser alone: reads D fp32 planes, writes D fp32 proxy planes (+ occ)
    qms = _events_ms(lambda: puv.quantize(layout, atlas, occ, spec, proxy=proxy), 20, 3)
    n = lv.rows * lv.cols
    qbytes = n * (layout.planes * 8 + 1)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    ms_f, st_f = out["fused"]
    ms_l, _ = out["proxy"]
    ms_p, _ = out[False]
    return {"row": "NEXT-2 LPO (16-bit xyz / 8-bit attributes fake quantiser, STE)", "metric": "views/s fwd+bwd",
            "value": len(sc.cameras) / (ms_l / 1e3), "ms_per_step": ms_l,
            "mode": "range refit + materialised proxy atlas every step (the faster path)",
            "fused_views_per_s": len(sc.cameras) / (ms_f / 1e3),
            "fused_mode": "PUV_RENDER_LPO: K1/K7 read the masters through the quantiser (no proxy atlas)",
            "plain_views_per_s": len(sc.cameras) / (ms_p / 1e3), "fused_stage_ms_per_step": st_f, "quantize_ms": qms,
            "quantize_roofline": {"bound": "hbm", "achieved": qbytes / (qms / 1e3) / 1e9, "peak": hbm,
                                  "unit": "GB/s", "frac": qbytes / (qms / 1e3) / 1e9 / hbm,
                                  "bytes_per_launch": qbytes},
            "workload": "C3 1024^2 SH3 atlas, 64 views 1920x1080, range refit every step"}


if __name__ == "__main__":
    which = sys.argv[1:] or ["label", "rho", "objective", "lpo"]
    rows = {"label": bench_label, "label_sweep": bench_label_sweep, "rho": bench_rho, "objective": bench_objective, "lpo": bench_lpo}
    for w in which:
        print(json.dumps(rows[w]()), flush=True)
