"""Benchmark: views/s of the fwd+bwd render of UV-atlas Gaussians @1080p (BASELINE.json `metric`).

One step = the whole hot path (DESIGN.md §1 rows a1-a10) over one batch: every
view of the workload is projected, binned, composited, the L2 loss gradient is
formed, the backward scatters gradients onto the atlas texels, and (N > 1) the
gradient planes are all-reduced over NCCL.  Default workload: BJ.configs[2]
(C3: 1,048,576 Gaussians, SH degree 3, 64 views at 1920x1080), all 64 views per
step (strong scaling over N GPUs: rank r renders views r, r+N, ...).
--config 4: the C4 frame sequence (30 frames x 55 views = 1650 view-renders per
step, gradient freezing); --config 5: C5 (5.24M Gaussians, 88 views at 4K, in
view chunks that fit HBM).

    python bench.py [--gpus N --steps K --warmup W] [--config 3] [--impl reference]

Prints ONE JSON line (rank 0).  The oracle (oracle/, CPU) is only executed by
the `cpu_baseline` leg and by `--impl reference`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "views/sec fwd+bwd render of UV-atlas Gaussians @1080p, 1/2/4/8 GPUs"
UNIT = "views/s"
WORKLOADS = {1: "BJ.configs[0] C1: 64x64 atlas (4096 G, SH0), 1 view 128x128",
             2: "BJ.configs[1] C2: 512^2+256^2+128^2 levels (344,064 G, SH1), 16 views 1024x768",
             3: "BJ.configs[2] C3: 1024^2 atlas (1,048,576 G, SH3), 64 views 1920x1080",
             4: "BJ.configs[3] C4: 30 frames of a 1024^2 atlas (SH3, 25% dynamic texels, gradient freezing), "
                "55 views 1920x1080: 1650 view-renders per step",
             5: "BJ.configs[4] C5: 2048^2+1024^2 levels (5,242,880 G, SH3), 88 views 3840x2160"}
THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--views", type=int, default=None, help="use only the first V views of the config")
    ap.add_argument("--frames", type=int, default=None, help="C4: use only the first F frames")
    ap.add_argument("--views-per-call", type=int, default=None, help="view chunk of one render call")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-serial", action="store_true", help="skip the serialised per-stage profile step")
    ap.add_argument("--cpu-sample-views", type=int, default=2)
    return ap.parse_args()


# ----------------------------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"puv_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], 0
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                reasons |= int(parts[3], 16)
            except ValueError:
                continue
        names = sorted(v for k, v in THROTTLE_BITS.items() if reasons & k and v != "gpu_idle")
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": names, "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)


def host_cpu():
    model = "unknown"
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


def oracle_views_per_s(scene, views, threads=0):
    """Time the CPU oracle (as it stands) doing fwd+bwd of `views` with `threads` OpenMP threads
    (0 = all host cores); returns (views/s, seconds, threads used)."""
    from oracle import orc
    planes, occ, _ = orc.pack(scene.levels)
    val = planes.astype(np.float64)
    used = orc.set_threads(threads)
    t0 = time.perf_counter()
    for v in views:
        cam = scene.cameras[v]
        img = orc.forward(planes, occ, scene.sh_degree, cam, val=val)[0]
        _, dl = orc.l2_loss_grad(img, scene.target(v))
        orc.backward(planes, occ, scene.sh_degree, cam, dl, val=val)
    dt = time.perf_counter() - t0
    orc.set_threads(0)
    return len(views) / dt, dt, used


def run_reference(args):
    """--impl reference: the CPU oracle (all host cores) is this tier's reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.scenes import make_scene
    cfg = args.config if args.config != 4 else 3   # C4 frames are C3-sized atlases; sample on C3's views
    sc = make_scene(cfg, views=args.views)
    nv = 1   # one full-resolution view fwd+bwd per step keeps the driver's 20-step run to minutes
    times, used = [], 0
    for s in range(args.steps):
        _, dt, used = oracle_views_per_s(sc, [(s * nv + i) % len(sc.cameras) for i in range(nv)])
        times.append(dt)
    t = sum(times) / len(times)
    value = nv / t
    hc = host_cpu()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, str(args.config)), "views_per_step": nv,
                       "parallelism": f"CPU oracle, OpenMP over pixel rows on {used} threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "oracle",
                             "sample": f"{nv} view(s) (of {len(sc.cameras)}) fwd+bwd per step, full resolution",
                             **hc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
# roofline bookkeeping (DESIGN.md §6 / SURVEY.md §8(d): algorithmic work per unit)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


# SURVEY.md §8(d) FP32-pipe instruction counts of the compositing kernels (per (pixel, entry) pair)
K5_PER_EXAMINED, K5_PER_COMPOSITED = 8, 11
K6_PER_EXAMINED, K6_PER_COMPOSITED = 8, 45


def stage_work(stage, c, D):
    """Algorithmic work of the per-view share of `stage` for the per-view counts c:
    ('hbm', bytes) or ('alu_fp32', FP32 lane-instructions)."""
    N, nv, K, E, P = c["N"], c["n_vis"], c["K"], c["examined"], c["composited"]
    sh = 4 * (D - 11)
    if stage == "project":          # 44 B geometry + SH of a visible G, ~56 B record out
        return "hbm", 44 * N / c["views"] + (sh + 56) * nv
    if stage == "depth_sort":       # read the depth key of every texel, write the depth order
        return "hbm", 4 * N + 4 * nv
    if stage == "bin":              # 12 B per key written (+ rank rects, ranges)
        return "hbm", 8 * nv + 12 * K + 8 * c["ntiles"]
    if stage == "raster_fwd":       # 8 FP32 instr per examined pair, +11 per composited pair
        return "alu_fp32", K5_PER_EXAMINED * E + K5_PER_COMPOSITED * P
    if stage == "raster_bwd":       # ~8 per evaluated pair, ~45 per composited pair
        return "alu_fp32", K6_PER_EXAMINED * E + K6_PER_COMPOSITED * P
    if stage == "project_bwd":      # 9 moments per visible (view, G) + every (view, texel) depth key; the texel's
        # parameters once per call and its gradient written once (train step: overwrite mode)
        return "hbm", 72 * nv + 4 * N + (44 + sh + 4 * D) * N / c["views"]
    if stage == "loss":
        return "hbm", 12 * 3 * c["HW"]
    return "hbm", 0


def roofline(stage, per_view, D, views_in_stage, stage_ms, calls, peaks, nsm, fp64_secondary=True):
    kind, work = stage_work(stage, per_view, D)
    avg_launch_s = stage_ms / 1000.0 / max(calls, 1)
    work_per_launch = work * views_in_stage / max(calls, 1)
    if kind == "hbm":
        achieved = work_per_launch / avg_launch_s / 1e9
        r = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
             "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_source": peaks["source"]}
    else:
        peak = nsm * 128 * peaks["sm_max_mhz"] * 1e6 / 1e12
        achieved = work_per_launch / avg_launch_s / 1e12
        r = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "T FP32 lane-instr/s",
             "frac": achieved / peak, "traffic": None,
             "peak_source": f"derived: {nsm} SMs x 128 FP32 lanes x {peaks['sm_max_mhz']:.0f} MHz "
                            "(B200_PROFILING.md unit counts; DESIGN.md §6)",
             "work": {"raster_fwd": f"SURVEY §8(d): {K5_PER_EXAMINED} FP32 instr per examined (pixel, entry) pair "
                                    f"+ {K5_PER_COMPOSITED} per composited pair",
                      "raster_bwd": f"SURVEY §8(d): {K6_PER_EXAMINED} per examined + {K6_PER_COMPOSITED} per "
                                    "composited pair"}[stage]}
        if stage in ("raster_fwd", "raster_bwd"):
            # this design's own algorithmic work (DESIGN.md §6/§14): the fp32 contract per composited pair
            # (exp_c, cap, transmittance, termination: ~20 in K5; K6 replays decisions from K5's bits) plus
            # its fp64 value path at two fp32 lanes per fp64 lane-op
            e, p_ = per_view["examined"], per_view["composited"]
            own = ((8 * e + 20 * p_ + 2 * 18 * p_) if stage == "raster_fwd" else (2 * 32 * p_)) \
                * views_in_stage / max(calls, 1)
            r["design_work"] = {"achieved": own / avg_launch_s / 1e12, "peak": peak,
                                "frac": own / avg_launch_s / 1e12 / peak, "unit": "T FP32-equivalent lane-instr/s",
                                "work": ("8 fp32 per examined pair + (20 fp32 contract + 2 x 18 fp64) per composited pair"
                                         if stage == "raster_fwd" else "2 x 32 fp64 per composited pair")}
        if fp64_secondary:
            # the build's own value path: fp64 lane-ops per composited pair vs 64 FP64 lanes/SM
            n64 = {"raster_fwd": 18, "raster_bwd": 32}[stage] * per_view["composited"] * views_in_stage / max(calls, 1)
            p64 = nsm * 64 * peaks["sm_max_mhz"] * 1e6 / 1e12
            r["fp64_value_path"] = {"achieved": n64 / avg_launch_s / 1e12, "peak": p64,
                                    "frac": n64 / avg_launch_s / 1e12 / p64, "unit": "T FP64 lane-ops/s",
                                    "work": f"{ {'raster_fwd': 18, 'raster_bwd': 32}[stage]} fp64 ops per "
                                            "composited pair (DESIGN.md §6)"}
    r["kernel"] = stage
    r["avg_launch_ms"] = avg_launch_s * 1000.0
    return r


# ----------------------------------------------------------------------------------------------


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2602_23040_b200 import puv
    from paper_2602_23040_b200.shard import FrameStep, ShardedStep
    from synth.scenes import frame_positions, make_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    puv.lib()

    cfg = args.config
    sc = make_scene(cfg, views=args.views)
    n_views = len(sc.cameras)
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    lp = [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels]
    lo = [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels]
    atlas, occ = puv.pack_atlas(layout, lp, lo)
    del lp, lo
    D = layout.planes
    N = layout.atlas_w * layout.atlas_h
    W, H = sc.cameras[0].width, sc.cameras[0].height

    vpc = args.views_per_call
    if vpc is None and cfg == 5:
        # C5 does not fit one call at 88 views: chunk so that state + key arena use
        # about half of the free HBM (arena estimate: 1.3 x the library's first guess per view)
        free = torch.cuda.mem_get_info(dev)[0]
        sb1, ah1 = puv.query_sizes(layout, puv.cameras(sc.cameras[:1]))
        per_view = sb1 + 1.3 * ah1
        local_n = len(range(rank, n_views, world))
        chunks = max(1, int(np.ceil(local_n * per_view / (0.5 * free))))
        vpc = int(np.ceil(local_n / chunks))

    frames = None
    if cfg == 4:
        n_frames = args.frames or sc.meta["frames"]
        labels = torch.from_numpy(sc.levels[0].labels).to(dev)
        stepper = FrameStep(layout, sc.cameras, n_frames, rank, world, dev, dynamic=labels, views_per_call=vpc)
        pos = [torch.from_numpy(frame_positions(sc, f)).to(dev) for f in range(n_frames)]
        frames = [[pos[f][0], pos[f][1], pos[f][2]] + [atlas[d] for d in range(3, D)] for f in range(n_frames)]
        idx = stepper.local_targets_index()
        tg_host = torch.empty((len(idx), 3, H, W), dtype=torch.float32).pin_memory()
        for i, (f, v) in enumerate(idx):
            tg_host[i].copy_(torch.from_numpy(sc.target(v, frame=f)))
        targets = tg_host.to(dev)
        grad = torch.zeros((n_frames, D, layout.atlas_h, layout.atlas_w), dtype=torch.float32, device=dev)
        mask = labels
        renders_per_step = n_frames * n_views
        local_renders = len(idx)

        def step(check=False):
            return stepper.step(frames, occ, targets, grad, mask=mask, check_overflow=check)
    else:
        stepper = ShardedStep(layout, sc.cameras, rank, world, dev, views_per_call=vpc)
        tg_host = torch.from_numpy(np.stack([sc.target(v) for v in stepper.views])).pin_memory()
        targets = tg_host.to(dev)
        grad = torch.zeros_like(atlas)
        mask = None
        renders_per_step = n_views
        local_renders = len(stepper.views)

        def step(check=False):
            return stepper.step(atlas, occ, targets, grad, check_overflow=check)
    torch.cuda.synchronize()

    # ---- warm-up (the first step checks the key arena and grows it if needed) ----
    for w in range(max(args.warmup, 1)):
        step(check=(w == 0))
    torch.cuda.synchronize()

    # ---- timed region: inputs resident in HBM (larger than L2: no flush needed) ----
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = puv.kernel_launches()
    puv.profile_read(reset=True)
    puv.profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            loss = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    puv.profile_enable(False)
    prof = puv.profile_read(reset=True)
    launches = puv.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    overflow = stepper.overflowed()
    value = renders_per_step / (ms_max / 1000.0)
    loss_value = float(loss.item())

    # ---- serialised per-stage times: one extra (untimed) step with binning on the main stream ----
    serial = None
    if not args.no_serial:
        puv.profile_serial(True)
        puv.profile_enable(True)
        step()
        torch.cuda.synchronize()
        puv.profile_enable(False)
        puv.profile_serial(False)
        sp = puv.profile_read(reset=True)
        serial = {k: round(v / local_renders, 4) for k, v in sp["ms"].items() if v > 0}

    # ---- e2e: the same step through the C ABI with HOST buffers (puv_train_step_host): inputs
    # copied in from pinned memory and the step's result (gradient planes + loss) copied back ----
    e2e = None
    if not args.no_e2e:
        grad_host = torch.empty(tuple(grad.shape), dtype=torch.float32).pin_memory()
        loss_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        if cfg == 4:
            pos_host = [p.cpu().pin_memory() for p in pos]
            shared_host = atlas[3:].cpu().pin_memory()
            a_dev = torch.empty_like(atlas)
            p_dev = [torch.empty_like(p) for p in pos]
            fr_dev = [[p_dev[f][0], p_dev[f][1], p_dev[f][2]] + [a_dev[d] for d in range(3, D)]
                      for f in range(len(pos))]
            t_dev = torch.empty_like(targets)

            def e2e_step():
                off = 0
                for f in range(len(pos)):
                    vs = stepper.frames.get(f, [])
                    if not vs:
                        grad[f].zero_()
                        continue
                    up = [(pos_host[f], p_dev[f])] + ([(shared_host, a_dev[3:])] if off == 0 else [])
                    puv.train_step_host(layout, fr_dev[f], occ, stepper.cams[f], tg_host[off:off + len(vs)],
                                        t_dev[off:off + len(vs)], grad[f], stepper.st, uploads=up,
                                        downloads=[(grad[f], grad_host[f])] if world == 1 else [], mask=mask)
                    stepper.losses[f:f + 1].copy_(stepper.st.loss)
                    off += len(vs)
                torch.sum(stepper.losses, dim=0, keepdim=True, out=stepper.loss)
                if world > 1:
                    dist.all_reduce(grad)
                    dist.all_reduce(stepper.loss)
                    grad_host.copy_(grad, non_blocking=True)
                loss_host.copy_(stepper.loss, non_blocking=True)
            h2d = sum(p.nbytes for p in pos_host) + shared_host.nbytes + tg_host.nbytes
        else:
            atlas_host = atlas.cpu().pin_memory()
            a_dev = torch.empty_like(atlas)
            t_dev = torch.empty_like(targets)

            def e2e_step():
                stepper.step_host(atlas_host, occ, tg_host, grad, a_dev, t_dev, grad_host, loss_host)
            h2d = atlas_host.nbytes + tg_host.nbytes

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": renders_per_step / (float(te.item()) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(grad_host.nbytes + loss_host.nbytes),
               "api": "puv_train_step_host_atlas (C ABI, host buffers)" if cfg != 4 and world == 1 else "puv_train_step_host (C ABI, host buffers)"}

    # ---- per-view counts of the last render call on the state (deterministic; read after timing) ----
    st = stepper.st
    if cfg == 4:
        last_views = stepper.frames[max(stepper.frames)]
    else:
        last_views = stepper.views
    k0 = (len(last_views) - 1) // st.views_per_call * st.views_per_call
    chunk_cams = puv.cameras([sc.cameras[v] for v in last_views[k0:]])
    counts = [puv.view_counts(st.state, i) for i in range(len(chunk_cams))]
    c_tot = {k2: sum(c[k2] for c in counts) / len(counts) for k2 in ("n_vis", "K", "examined", "composited")}

    # ---- roofline of the dominant compositing kernel (SURVEY §8(d) basis) ----
    peaks = load_peaks()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    stage_ms = {s: prof["ms"][s] / args.steps for s in prof["ms"]}
    gx, gy = (W + 15) // 16, (H + 15) // 16
    per_view = {"N": N, "views": max(st.views_per_call, 1), "HW": W * H, "ntiles": gx * gy, **c_tot}
    rf = {}
    for s_ in ("raster_fwd", "raster_bwd"):
        rf[s_] = roofline(s_, per_view, D, local_renders, stage_ms[s_], prof["calls"][s_] / args.steps, peaks, nsm)
    dom = max(rf, key=lambda k2: stage_ms[k2])
    roof = dict(rf[dom])
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and cfg == 3:
        tj = json.load(open(tp))
        if dom in tj.get("bytes_per_launch", {}):
            vpl = local_renders / max(prof["calls"][dom] / args.steps, 1)
            roof["traffic"] = tj["bytes_per_launch"][dom] / tj["views_per_launch"][dom] * vpl
            roof["traffic_unit"] = "bytes/launch (ncu dram read+write, profiles/traffic.json)"
    other = "raster_bwd" if dom == "raster_fwd" else "raster_fwd"
    roof["other_raster_kernel"] = {k2: rf[other][k2] for k2 in ("kernel", "achieved", "frac", "avg_launch_ms")}
    hbm_stages = {}
    for s_ in ("project", "project_bwd", "loss"):
        # the loss runs on the second stream beside the compositing: its event span is not its duration,
        # so it is rated on the serialised step's time (one launch per view there)
        ms_, calls_ = stage_ms.get(s_, 0), prof["calls"][s_] / args.steps if s_ in prof["calls"] else 0
        if s_ == "loss":
            ms_ = serial.get("loss", 0) * local_renders if serial else 0
            calls_ = local_renders
        if ms_ > 0:
            r = roofline(s_, per_view, D, local_renders, ms_, calls_, peaks, nsm)
            hbm_stages[s_] = {"achieved_gbs": round(r["achieved"], 1), "frac": round(r["frac"], 3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        csc = sc if cfg != 4 else make_scene(3)
        nv = args.cpu_sample_views
        if cfg == 5:
            nv = 1   # a 4K view of 5.2M Gaussians: one view at all cores is the bounded sample
        vps, dt, used = oracle_views_per_s(csc, list(range(nv)), threads=0)
        single = None
        if cfg != 5:
            vps1, dt1, _ = oracle_views_per_s(csc, [0], threads=1)
            single = {"value": vps1, "unit": UNIT, "sample": f"1 view ({dt1:.1f} s)"}
        cpu = {"value": vps, "unit": UNIT, "cores": used, "kind": "oracle",
               "sample": f"{nv} view(s) of {len(csc.cameras)} ({'C3 views for the C4 frames' if cfg == 4 else 'this config'}), "
                         f"full resolution fwd+bwd, OpenMP over pixel rows ({dt:.1f} s)",
               "single_thread": single, **host_cpu()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32 decisions (bit-exact contract), f64 composite values",
                "data": "synthetic",
                "config": {"workload": WORKLOADS.get(cfg, str(cfg)), "view_renders_per_step": renders_per_step,
                           "view_renders_per_gpu": local_renders, "views_per_call": st.views_per_call,
                           "parallelism": f"view-sharded dp{world}",
                           "l2": "inputs larger than L2 (atlas >= 247.5 MB, per-call state > 3 GB)"},
                "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches, "roofline": roof,
                "hbm_stages": hbm_stages, "cpu_baseline": cpu,
                "stage_ms_per_step": {k2: round(v, 4) for k2, v in stage_ms.items() if v > 0},
                "overlapped_stages": ["depth_sort", "bin", "loss"],
                "stage_ms_per_view_serialised": serial,
                "counts_per_view": c_tot, "overflow": overflow, "loss": loss_value}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
