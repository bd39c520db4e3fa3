"""Binning microbenchmark: c3 (3M Gaussians, 1080p) or any frustum config;
times bin_and_sort_async with CUDA events and lists the per-kernel device
time of one call (torch.profiler / CUPTI).

    python tools/bin_probe.py [--n N] [--w W] [--h H]
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

    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200 import synthetic
    from paper_2308_04079_b200.cloud import GaussianCloud

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--h", type=int, default=1080)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--once", action="store_true", help="one binning call after setup (for ncu)")
    args = ap.parse_args()
    cloud_np, cam = synthetic.frustum_scene(args.n, args.w, args.h, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, 3)
    b = R.bin_and_sort(splats, args.w, args.h)
    K = b.num_instances
    cap = int(K * 1.05) + 4096
    if args.once:
        R.bin_and_sort_async(splats, args.w, args.h, capacity=cap)
        torch.cuda.synchronize()
        return
    for _ in range(3):
        R.bin_and_sort_async(splats, args.w, args.h, capacity=cap)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        R.bin_and_sort_async(splats, args.w, args.h, capacity=cap)
    e.record()
    torch.cuda.synchronize()
    res = {"n": args.n, "K": K, "bin_async_ms": s.elapsed_time(e) / args.reps}
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            R.bin_and_sort_async(splats, args.w, args.h, capacity=cap)
        torch.cuda.synchronize()
    kern = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            name = ev.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")
            kern[name] = kern.get(name, 0.0) + ev.device_time / 5 / 1000.0
    res["kernels_ms"] = {k: round(v, 4) for k, v in sorted(kern.items(), key=lambda x: -x[1])}
    res["kernels_sum_ms"] = round(sum(kern.values()), 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
