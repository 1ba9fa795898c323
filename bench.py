"""Benchmark: views/s of the fwd+bwd render of UV-atlas Gaussians @1080p (BASELINE.json `metric`).

One step = the whole hot path (DESIGN.md §1 rows a1-a10) over one batch: every
view of the workload is projected, binned, composited, the L2 loss gradient is
formed, the backward scatters gradients onto the atlas texels, and (N > 1) the
gradient planes are all-reduced over NCCL.  Default workload: BJ.configs[2]
(C3: 1,048,576 Gaussians, SH degree 3, 64 views at 1920x1080), all 64 views per
step (strong scaling over N GPUs: rank r renders views r, r+N, ...).

    python bench.py [--gpus N --steps K --warmup W] [--config 3] [--impl reference]

Prints ONE JSON line (rank 0).  The oracle (oracle/, CPU) is only executed by
the `cpu_baseline` leg and by `--impl reference`.
"""
from __future__ import annotations

import argparse
import json
import math
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
             3: "BJ.configs[2] C3: 1024^2 atlas (1,048,576 G, SH3), 64 views 1920x1080"}
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
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-views", type=int, default=1)
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


def oracle_views_per_s(scene, views, targets=None):
    """Time the CPU oracle (as it stands) doing fwd+bwd of `views`; returns (views/s, seconds, cores)."""
    from oracle import orc
    planes, occ, _ = orc.pack(scene.levels)
    t0 = time.perf_counter()
    for v in views:
        cam = scene.cameras[v]
        img = orc.forward(planes, occ, scene.sh_degree, cam)[0]
        tg = scene.target(v) if targets is None else targets[v]
        _, dl = orc.l2_loss_grad(img, tg)
        orc.backward(planes, occ, scene.sh_degree, cam, dl)
    dt = time.perf_counter() - t0
    return len(views) / dt, dt, 1


def run_reference(args):
    """--impl reference: the CPU oracle is this tier's reference arm (runs on rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.scenes import make_scene
    sc = make_scene(args.config, views=args.views)
    nv = max(1, args.cpu_sample_views)
    sample = list(range(nv))
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up effects worth paying minutes for; see DESIGN.md §6
    times = []
    for s in range(args.steps):
        vps, dt, cores = oracle_views_per_s(sc, [sample[s % nv]])
        times.append(dt)
    t = sum(times) / len(times)
    value = 1.0 / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, str(args.config)), "views_per_step": 1,
                       "parallelism": "single CPU thread (oracle)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"1 view (of {len(sc.cameras)}) fwd+bwd per step, full resolution"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
# roofline bookkeeping (algorithmic work per unit)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


def stage_work(stage, c, D):
    """Algorithmic work of ONE launch-set of `stage` for the per-view counts c."""
    N, nv, K, E, P = c["N"], c["n_vis"], c["K"], c["examined"], c["composited"]
    if stage == "project":          # per view share of K1: texel read (once per call) + records written
        return "hbm", (D * 4 * N) / c["views"] + 212 * nv + 4 * (N - nv)
    if stage == "depth_sort":       # read the depth key of every texel, write the depth order
        return "hbm", 4 * N + 4 * nv
    if stage == "bin":              # read rank rects, write every key once, ranges
        return "hbm", 8 * nv + 4 * K + 8 * c["ntiles"]
    if stage == "raster_fwd":       # fp64-equivalent lane-ops: 18 fp64 per composited pair, plus the
        # fp32 contract work at half weight (the fp32 pipe is twice as wide): 8 per examined pair (skip
        # test), 19 per composited pair (exp_c, alpha cap, transmittance, termination test)
        return "alu_fp64", 18 * P + 0.5 * (8 * E + 19 * P)
    if stage == "raster_bwd":       # fp64 lane-ops per composited pair: 32
        return "alu_fp64", 32 * P
    if stage == "project_bwd":      # read 2D grads + params, RMW texel grads
        return "hbm", 72 * nv + (D * 4 * 3 * N) / c["views"]
    if stage == "loss":
        return "hbm", 12 * 3 * c["HW"]
    return "hbm", 0


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2602_23040_b200 import puv
    from paper_2602_23040_b200.shard import ShardedStep
    from synth.scenes import make_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    puv.lib()

    sc = make_scene(args.config, views=args.views)
    n_views = len(sc.cameras)
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    lp = [torch.from_numpy(lv.planes).to(dev) for lv in sc.levels]
    lo = [torch.from_numpy(lv.occ).to(dev) for lv in sc.levels]
    atlas, occ = puv.pack_atlas(layout, lp, lo)
    del lp, lo
    stepper = ShardedStep(layout, sc.cameras, rank, world, dev)
    mine = stepper.views
    tg_host = torch.from_numpy(np.stack([sc.target(v) for v in mine])).pin_memory()
    targets = tg_host.to(dev)
    grad = torch.zeros_like(atlas)
    torch.cuda.synchronize()

    # ---- warm-up (first step checks the key arena and grows it if needed) ----
    for w in range(max(args.warmup, 1)):
        grad.zero_()
        stepper.step(atlas, occ, targets, grad, check_overflow=(w == 0))
    torch.cuda.synchronize()

    # ---- timed region: inputs resident in HBM ----
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
            grad.zero_()
            loss = stepper.step(atlas, occ, targets, grad)
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
    value = n_views / (ms_max / 1000.0)

    # ---- e2e: the same step through the public API with HOST inputs (pinned), H2D + D2H inside ----
    e2e = None
    if not args.no_e2e:
        atlas_host = atlas.cpu().pin_memory()
        loss_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        a_dev = torch.empty_like(atlas)
        t_dev = torch.empty_like(targets)

        def e2e_step():
            grad.zero_()
            stepper.step_host(atlas_host, occ, tg_host, grad, a_dev, t_dev, loss_host)

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
        e2e = {"value": n_views / (float(te.item()) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(atlas_host.numel() * 4 + tg_host.numel() * 4),
               "d2h_bytes_per_step": 8}

    # ---- per-view counts (deterministic; read after timing) ----
    counts = []
    for i in range(len(mine)):
        d = puv.debug_view(layout, stepper.cams, stepper.R.state, stepper.R.arena, i)
        counts.append({"n_vis": d.n_visible, "K": d.n_keys, "examined": d.n_examined, "composited": d.n_composited})
    HW = sc.cameras[0].width * sc.cameras[0].height
    c_tot = {k: sum(c[k] for c in counts) for k in ("n_vis", "K", "examined", "composited")}

    # ---- roofline of the dominant stage ----
    peaks = load_peaks()
    sm_mhz = peaks["sm_max_mhz"]
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    stage_ms = {s: prof["ms"][s] / args.steps for s in prof["ms"]}
    # depth_sort and bin run on the library's binning streams, overlapped with the compositing of
    # earlier views: their event intervals include time-sharing, so they are not candidates for the
    # dominant kernel (the ncu launch list in profiles/ gives their serialised share).
    overlapped = ("depth_sort", "bin")
    dom = max((s for s in stage_ms if s not in overlapped), key=lambda s: stage_ms[s])
    per_view = {"N": atlas.shape[1] * atlas.shape[2], "views": len(mine), "HW": HW, "ntiles": 0,
                "n_vis": c_tot["n_vis"] / len(mine), "K": c_tot["K"] / len(mine),
                "examined": c_tot["examined"] / len(mine), "composited": c_tot["composited"] / len(mine)}
    gx = (sc.cameras[0].width + 15) // 16
    gy = (sc.cameras[0].height + 15) // 16
    per_view["ntiles"] = gx * gy
    calls = max(prof["calls"][dom] / args.steps, 1)
    units = len(mine) if dom not in ("loss",) else 1
    kind, work = stage_work(dom, per_view, layout.planes)
    avg_launch_s = stage_ms[dom] / 1000.0 / calls
    work_per_launch = work * units / calls
    if kind == "hbm":
        achieved = work_per_launch / avg_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "peak_source": peaks["source"]}
    else:
        lanes = 128 if kind == "alu_fp32" else 64
        peak = nsm * lanes * sm_mhz * 1e6 / 1e12
        achieved = work_per_launch / avg_launch_s / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak,
                "unit": "T lane-ops/s (" + ("fp32" if kind == "alu_fp32" else "fp64") + ")",
                "frac": achieved / peak, "traffic": None,
                "peak_source": f"derived: {nsm} SMs x {lanes} {kind[4:]} lanes x {sm_mhz:.0f} MHz (DESIGN.md §6)"}
    roof["kernel"] = dom
    roof["work"] = {"raster_fwd": "18 fp64 lane-ops per composited pair + fp32 contract work at half weight "
                                  "(8 per examined, 19 per composited pair)",
                    "raster_bwd": "32 fp64 lane-ops per composited pair"}.get(dom, "algorithmic bytes, DESIGN.md §6")
    roof["avg_launch_ms"] = avg_launch_s * 1000.0
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and args.config == 3:
        tj = json.load(open(tp))
        if dom in tj.get("bytes_per_launch", {}):
            # ncu capture of the same kernel on C3, scaled to this run's views per launch
            roof["traffic"] = tj["bytes_per_launch"][dom] / tj["views_per_launch"][dom] * (units / calls)
            roof["traffic_unit"] = "bytes/launch (ncu dram read+write)"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        vps, dt, cores = oracle_views_per_s(sc, list(range(args.cpu_sample_views)))
        cpu = {"value": vps, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{args.cpu_sample_views} view(s) of {n_views}, full resolution fwd+bwd ({dt:.1f} s)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32 decisions+forward / f64 backward values", "data": "synthetic",
                "config": {"workload": WORKLOADS.get(args.config, str(args.config)), "views_per_step": n_views,
                           "views_per_gpu": len(mine), "parallelism": f"view-sharded dp{world}",
                           "l2": "inputs larger than L2 (atlas 247.5 MB, per-step state > 10 GB)"},
                "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches, "roofline": roof,
                "cpu_baseline": cpu,
                "stage_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
                "overlapped_stages": list(overlapped),
                "counts_per_view": {k: v / len(mine) for k, v in c_tot.items()},
                "overflow": overflow, "loss": float(loss.item())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
