"""Per-kernel device times (torch.profiler / CUPTI) of one c3 training step's
stages: project, binning, blend forward (+ exact fix-up), loss, blend
backward, fused backward + Adam.

    python tools/kernel_probe.py [--n N] [--w W] [--h H] [--reps R]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200 import synthetic
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.loss import l1_dssim_loss
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--h", type=int, default=1080)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    w, h, bg = args.w, args.h, (0.0, 0.0, 0.0)
    cloud_np, cam = synthetic.frustum_scene(args.n, w, h, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    target = R.render_view(GaussianCloud.from_numpy(**synthetic.frustum_scene(args.n, w, h, seed=1)[0]), cam, bg,
                           3)[0].image
    adam, cfg = DeviceAdam(cloud), TrainConfig()
    stats = R.DensifyStats.zeros(len(cloud), "cuda")

    def step(it):
        out, splats, binning = R.render_view_async(cloud, cam, bg, 3, training=True)
        loss, d_image = l1_dssim_loss(out.image, target, cfg.lambda_dssim)
        g2 = R.render_backward(d_image, out, splats, binning, w, h, bg)
        adam.backward_step(cloud, cam, splats, g2, 3, it, cfg, stats=stats)
        return out

    for it in range(1, 4):
        step(it)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for it in range(4, 4 + args.reps):
            out = step(it)
        torch.cuda.synchronize()
    kern = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            name = ev.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")
            kern[name] = kern.get(name, 0.0) + ev.device_time / args.reps / 1000.0
    res = {"n": args.n, "kernels_ms": {k: round(v, 4) for k, v in sorted(kern.items(), key=lambda x: -x[1])},
           "sum_ms": round(sum(kern.values()), 4)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
