"""Benchmark: 1080p training iterations/s and render FPS, 3M Gaussians SH3 (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE configs[2], "c3"): the SURVEY §8(d) frustum generator,
3,000,000 Gaussians, SH degree 3, one 1920x1080 camera; a step is one
training iteration: project -> bin/sort -> forward blend -> L1+D-SSIM loss
(lambda 0.2) -> backward blend -> backward preprocess (+densify stats) ->
fused Adam.  Multi-GPU (torchrun): one process per GPU, each rank trains on
its own view of the replicated scene per step, gradients are summed with an
NCCL all-reduce, every rank runs the identical Adam (weak scaling).

The reference arm (--impl reference) times the float64 C oracle port of the
reference hot path (oracle/, pinned to splatlab's own outputs) on the host
cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "1080p render FPS + fwd/bwd train iters/sec, 3M Gaussians SH3, 1/2/4/8 B200"
UNIT = "train_iters/s"
N_GAUSS = 3_000_000
WIDTH, HEIGHT = 1920, 1080
DEGREE = 3
LAMBDA_DSSIM = 0.2


def peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 20 ms) during the
    timed region: the same fields as the recipe's nvidia-smi clocks line."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self._err = None

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(name for bit, name in self.REASONS.items() if mask & bit)
                self._stop.wait(0.02)
        except Exception as exc:  # pragma: no cover - depends on the box
            self._err = repr(exc)

    def start(self):
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=5)
        out = {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self._err:
            out["error"] = self._err
        return out


# ---------------------------------------------------------------------------
# our arm

def check_binned(k_infos: list) -> None:
    """Every async binning of the run stayed within its instance capacity and
    raised no error flag (K and flags stay on the device until here)."""
    import torch
    if k_infos:
        flags = torch.stack(k_infos)[:, 1]
        if bool((flags != 0).any()):
            raise RuntimeError(f"async binning flagged an error/overflow: flags {flags.unique().tolist()}")
    k_infos.clear()


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2308_04079_b200 import _lib, synthetic
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.camera import Camera
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.loss import l1_dssim_loss
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    from paper_2308_04079_b200.profiling import StageTimer, evaluated_pairs, measure_fp32_peak

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _lib.load()
    n = args.n_gaussians
    cloud_np, cam0 = synthetic.frustum_scene(n, WIDTH, HEIGHT, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np, device=dev)
    del cloud_np
    # the e2e arm starts from the same initial scene as the device loop (the
    # loop trains `cloud` in place)
    initial = {g: getattr(cloud, g).clone() for g in ("means", "rotations", "log_scales", "opacity_logits", "sh")}
    # each rank renders its own view: the frustum camera panned by a small per-rank offset
    def view_for(r: int) -> Camera:
        return Camera(np.eye(3), np.array([0.02 * r, -0.01 * r, 0.0]), cam0.fx, cam0.fy, cam0.cx, cam0.cy,
                      WIDTH, HEIGHT, cam0.near)
    cam = view_for(rank)
    # target image: render of the same generator with seed 1
    tgt_np, _ = synthetic.frustum_scene(n, WIDTH, HEIGHT, seed=1)
    target_cloud = GaussianCloud.from_numpy(**tgt_np, device=dev)
    del tgt_np
    bg = (0.0, 0.0, 0.0)
    with torch.no_grad():
        target, _, _ = R.render_view(target_cloud, cam, bg, DEGREE)
    target = target.image.contiguous()
    del target_cloud
    torch.cuda.synchronize()

    config = TrainConfig(lambda_dssim=LAMBDA_DSSIM)
    stats = R.DensifyStats.zeros(n, dev)
    sharded = None
    if world > 1:
        # ZeRO-1 style: gradients reduce-scattered by Gaussian range, Adam on
        # this rank's shard only, parameters all-gathered (distributed.ShardedAdam)
        from paper_2308_04079_b200.distributed import ShardedAdam
        sharded = ShardedAdam(cloud)
        grads = sharded.grads
    else:
        adam = DeviceAdam(cloud)
        grads = R.GaussianGrads.zeros(n, dev)
    timer = StageTimer(enabled=True)
    iteration = [0]
    prev_order = [None]

    def train_step(gt: torch.Tensor, timed: bool) -> torch.Tensor:
        iteration[0] += 1
        tm = timer if timed else None
        params = cloud.c_params()
        with StageTimer.stage(tm, "preprocess_fwd"):
            splats = R._project_tensors(params, n, dev, cam, DEGREE)
        with StageTimer.stage(tm, "bin_and_sort"):
            # sync-free binning: K stays on the device, checked after the loop
            binning = R.bin_and_sort_async(splats, WIDTH, HEIGHT)
        binnings.append(binning.k_info)
        with StageTimer.stage(tm, "blend_fwd"):
            # tiles in the previous backward's longest-first order (same view)
            out = R.render_forward(splats, binning, WIDTH, HEIGHT, bg, training=True, tile_order=prev_order[0])
        with StageTimer.stage(tm, "loss"):
            loss, d_image = l1_dssim_loss(out.image, gt, LAMBDA_DSSIM)
        with StageTimer.stage(tm, "blend_bwd"):
            g2 = R.render_backward(d_image, out, splats, binning, WIDTH, HEIGHT, bg)
        prev_order[0] = g2.tile_order
        if sharded is None and os.environ.get("GS_BENCH_UNFUSED") != "1":
            # single GPU: backward_project + stats + Adam fused (no gradient round trip)
            with StageTimer.stage(tm, "preprocess_bwd_adam"):
                adam.backward_step(cloud, cam, splats, g2, DEGREE, iteration[0], config, stats=stats)
        else:
            with StageTimer.stage(tm, "preprocess_bwd"):
                R._backward_project_tensors(params, n, dev, cam, splats, g2, DEGREE, stats, grads, False)
            if sharded is not None:
                with StageTimer.stage(tm, "sharded_adam"):   # reduce-scatter + shard Adam + all-gather
                    sharded.step(cloud, iteration[0], config)
            else:
                with StageTimer.stage(tm, "adam"):
                    adam.step(cloud, grads, iteration[0], config)
        if timed:
            timer.note_instances(binning, out)
        return loss

    binnings = []
    # size the instance buffers once from a synchronous binning of the first view
    R.bin_and_sort(R._project_tensors(cloud.c_params(), n, dev, cam, DEGREE), WIDTH, HEIGHT)
    for _ in range(args.warmup):
        train_step(target, False)
    torch.cuda.synchronize()
    check_binned(binnings)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start.record()
    for _ in range(args.steps):
        train_step(target, True)
    end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    clock_info = clocks.stop()
    check_binned(binnings)   # every timed step binned within capacity (else the step is invalid)
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    if args.profile:
        # profiling mode (ncu): warm-up + timed steps only, one summary line
        if rank == 0:
            print(json.dumps({"profile": True, "ms_per_step": ms_max / args.steps,
                              "stage_ms": timer.mean_ms(), "instances": timer.last_k}), flush=True)
        return

    # end-to-end through the public API: training.train_step, the mirror of the
    # reference's train_step (optimizer.py:222-260) -- render, L1+D-SSIM loss,
    # backward, fused Adam + densify statistics -- on a view whose target image
    # lives in pinned HOST memory and is copied H2D inside every step; the
    # step's result (loss, MSE for the PSNR, instance count) is read D2H.
    from paper_2308_04079_b200.densify import TrainState
    from paper_2308_04079_b200.training import TrainView, train_step
    gt_host = target.cpu().pin_memory()
    e2e_cloud = GaussianCloud(**initial)
    state = TrainState(e2e_cloud, scene_extent=10.0, seed=rank)
    state.active_sh_degree = DEGREE
    e2e_config = TrainConfig(lambda_dssim=LAMBDA_DSSIM, warmup_upsample_iters=(0, 0), sh_band_interval=10**9)
    # one view per rank (each rank trains on its own shard of the view list)
    views = [TrainView(view_for(r), gt_host) for r in range(world)]

    # lookahead (train_step enqueues the next iteration's forward before it
    # waits for this one) is off for the last warm-up and the last timed step,
    # so the timed region holds exactly `steps` forwards, backwards and Adams
    for i in range(args.warmup):
        train_step(state, views, e2e_config, lookahead=i < args.warmup - 1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        report = train_step(state, views, e2e_config, lookahead=i < args.steps - 1)
    e1.record()
    torch.cuda.synchronize()
    e_ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e_ms.item())
    e2e_loss = report.loss
    del state, e2e_cloud, initial

    # inference render FPS (forward only, same scene, same camera): the
    # sync-free render_view_async (K stays on the device; every frame's
    # capacity flags are checked after the loop), and the reference-shaped
    # render_view (one host read of K per frame) for comparison
    # (a TileSchedule carries each frame's per-tile work to the next frame's
    # launch order, heaviest tiles first)
    fps_steps = max(args.steps, 10)
    sched = R.TileSchedule()
    for _ in range(3):
        R.render_view_async(cloud, cam, bg, DEGREE, schedule=sched)[2].check()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kinfos = []
    f0.record()
    for _ in range(fps_steps):
        kinfos.append(R.render_view_async(cloud, cam, bg, DEGREE, schedule=sched)[2].k_info)
    f1.record()
    torch.cuda.synchronize()
    check_binned(kinfos)
    render_ms = f0.elapsed_time(f1) / fps_steps
    for _ in range(3):
        R.render_view(cloud, cam, bg, DEGREE)
    torch.cuda.synchronize()
    f0.record()
    for _ in range(fps_steps):
        R.render_view(cloud, cam, bg, DEGREE)
    f1.record()
    torch.cuda.synchronize()
    render_sync_ms = f0.elapsed_time(f1) / fps_steps

    # evaluated (pixel, splat) pairs E from the forward's own training record, and
    # the FP32 FMA peak of this GPU (the blend kernels' roofline denominator)
    with torch.no_grad():
        out_e, splats_e, binning_e = R.render_view(cloud, cam, bg, DEGREE, training=True)
        e_pairs = evaluated_pairs(out_e, binning_e, WIDTH)
        visible = int((splats_e.radii > 0).sum().item())
    fp32_peak = measure_fp32_peak(dev) / 1e12

    if rank != 0:
        return
    ms_per_step = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)
    e2e_value = world * args.steps / (e2e_ms / 1e3)
    stage_ms = timer.mean_ms()
    pk = dict(peaks())
    pk["fp32_tflops"] = fp32_peak
    traffic_file = ROOT / "profiles" / "traffic_bytes.json"
    if traffic_file.exists():
        pk["traffic_bytes"] = json.loads(traffic_file.read_text()).get("per_launch", {})
    roof = timer.roofline(n, WIDTH, HEIGHT, pk, visible=visible, e_pairs=e_pairs)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 projection geometry)",
        "data": "synthetic (SURVEY §8(d) frustum generator, seed 0; target = seed-1 render)",
        "config": {"workload": "c3: 3M Gaussians SH3, 1920x1080, train step (fwd + L1/D-SSIM loss + bwd + "
                               "fused Adam + densify stats)", "gaussians": n, "width": WIDTH, "height": HEIGHT,
                   "sh_degree": DEGREE, "views_per_step": world,
                   "parallelism": f"dp{world} (view-parallel" + (", ZeRO-1 sharded Adam)" if world > 1 else ")"),
                   "l2": "inputs larger than L2 (708 MB parameters + 2.1 GB Adam state)"},
        "render_fps": round(1e3 / render_ms, 2), "render_ms": round(render_ms, 4),
        "render_fps_sync": round(1e3 / render_sync_ms, 2),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "instances_per_view": timer.last_k, "evaluated_pairs_per_view": e_pairs, "visible_gaussians": visible,
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": WIDTH * HEIGHT * 3 * 4,
                "d2h_bytes_per_step": 8 * 8,   # the guard's report: [loss x4, K, flags, min(K, cap), skip] f64
                "path": "training.train_step (mirror of splatlab optimizer.train_step): target image H2D from "
                        "pinned host memory every step, [loss, L1, SSIM, MSE, K, flags, K, skip] written D2H into "
                        "mapped pinned memory by the step-guard kernel every step; lookahead: the next iteration's forward is enqueued before the host waits",
                "last_loss": round(e2e_loss, 6)},
        "gpu_launches": timer.launches_per_step() * args.steps,
        "roofline": roof["primary"], "roofline_hbm": roof["hbm"], "roofline_stages": roof["stages"],
        "fp32_peak_tflops_measured": round(fp32_peak, 2),
        "clocks": clock_info,
    }
    if args.cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CPU (oracle port) arm

def _cpu_scene(n):
    from paper_2308_04079_b200 import synthetic
    cloud, cam = synthetic.frustum_scene(n, WIDTH, HEIGHT, seed=0)
    return synthetic.round_to_f32(cloud), cam


def cpu_step_timings(cloud, cam, band: int, bands: int, adam_state: dict, it: int) -> dict:
    """One sampled training step of the oracle port: per-Gaussian stages over all
    N; the pixel stages (bin/sort, blend fwd, loss, blend bwd) over one band of
    tile rows (1/bands of the frame).  Returns stage seconds."""
    from oracle import oracle as O
    t = {}
    s = time.perf_counter()
    proj = O.project(cloud, cam, DEGREE)
    t["project"] = time.perf_counter() - s
    ty = (HEIGHT + 15) // 16
    r0, r1 = band * ty // bands, (band + 1) * ty // bands
    proj_b = dict(proj)
    rect = proj["rect"].copy()
    keep = (proj["tiles"] > 0) & (rect[:, 3] >= r0) & (rect[:, 1] < r1)
    rect[:, 1] = np.clip(rect[:, 1], r0, r1 - 1)
    rect[:, 3] = np.clip(rect[:, 3], r0, r1 - 1)
    proj_b["rect"] = rect
    proj_b["tiles"] = np.where(keep, (rect[:, 2] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 1] + 1), 0).astype(
        np.int64)
    s = time.perf_counter()
    bins = O.bin_and_sort(proj_b, WIDTH, HEIGHT)
    t["bin_and_sort"] = time.perf_counter() - s
    s = time.perf_counter()
    fwd = O.render_forward(proj_b, bins, WIDTH, HEIGHT, (0.0, 0.0, 0.0))
    t["blend_fwd"] = time.perf_counter() - s
    s = time.perf_counter()
    d_image = np.sign(fwd["image"] - 0.5) * (1.0 - LAMBDA_DSSIM) / fwd["image"].size  # L1 part only (host)
    t["loss_l1"] = time.perf_counter() - s
    s = time.perf_counter()
    g2 = O.render_backward(d_image, proj_b, bins, fwd, WIDTH, HEIGHT, (0.0, 0.0, 0.0))
    t["blend_bwd"] = time.perf_counter() - s
    s = time.perf_counter()
    grads = O.backward_project(cloud, cam, DEGREE, proj, g2)
    t["preprocess_bwd"] = time.perf_counter() - s
    s = time.perf_counter()
    gmap = {"means": "d_means", "log_scales": "d_log_scales", "rotations": "d_rotations",
            "opacity_logits": "d_opacity_logits", "sh": "d_sh"}
    for k, gk in gmap.items():
        st = adam_state[k]
        O.adam_group(st["p"], grads[gk], st["m"], st["v"], 1e-3, 0.9, 0.999, 1e-15, it,
                     **({"lr_head": 2.5e-3, "period": 48, "head": 3} if k == "sh" else {}))
    t["adam"] = time.perf_counter() - s
    t["K_band"] = int(bins["ids"].shape[0])
    return t


def cpu_full_step_seconds(t: dict, bands: int) -> float:
    pixel = t["bin_and_sort"] + t["blend_fwd"] + t["loss_l1"] + t["blend_bwd"]
    return t["project"] + t["preprocess_bwd"] + t["adam"] + bands * pixel


def cpu_baseline_sample(args) -> dict:
    from oracle import oracle as O
    cloud, cam = _cpu_scene(args.n_gaussians)
    state = {k: {"p": cloud[k].copy(), "m": np.zeros_like(cloud[k]), "v": np.zeros_like(cloud[k])} for k in cloud}
    bands = 8
    t = cpu_step_timings(cloud, cam, 3, bands, state, 1)
    full = cpu_full_step_seconds(t, bands)
    return {"value": round(1.0 / full, 5), "unit": UNIT, "cores": O.num_threads(), "kind": "port",
            "sample": f"one oracle training step: project/backward_project/Adam over all {args.n_gaussians} "
                      f"Gaussians + bin/blend fwd/bwd over 1/{bands} of the tile rows; full-frame step "
                      f"= per-Gaussian stages + {bands} x band stages = {full:.2f} s",
            "stage_s": {k: round(v, 4) if isinstance(v, float) else v for k, v in t.items()}}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    from oracle import oracle as O
    cloud, cam = _cpu_scene(args.n_gaussians)
    state = {k: {"p": cloud[k].copy(), "m": np.zeros_like(cloud[k]), "v": np.zeros_like(cloud[k])} for k in cloud}
    bands = 8
    it = 0
    for _ in range(args.warmup):
        it += 1
        cpu_step_timings(cloud, cam, it % bands, bands, state, it)
    fulls = []
    for _ in range(args.steps):
        it += 1
        fulls.append(cpu_full_step_seconds(cpu_step_timings(cloud, cam, it % bands, bands, state, it), bands))
    total = sum(fulls)
    value = args.steps / total
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator, seed 0)",
        "config": {"workload": "c3: 3M Gaussians SH3, 1920x1080, train step", "gaussians": args.n_gaussians,
                   "width": WIDTH, "height": HEIGHT, "sh_degree": DEGREE},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": O.num_threads(), "kind": "port",
                         "sample": f"float64 C oracle port of splatlab's hot path; each step: per-Gaussian "
                                   f"stages over all N + bin/blend over 1/{bands} of the tile rows (rotating), "
                                   f"full-frame time extrapolated as per-Gaussian + {bands} x band"},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-gaussians", type=int, default=N_GAUSS)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--profile", action="store_true", help="warm-up + timed steps only (for ncu)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks: several ranks on one GPU (GS_DEVICE_OVERRIDE) with gloo
    # (GS_DIST_BACKEND) exercise the multi-rank code path where one GPU is all there is
    if "GS_DEVICE_OVERRIDE" in os.environ:
        local_rank = int(os.environ["GS_DEVICE_OVERRIDE"])
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("GS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
