"""Render loop at c3 (3M Gaussians, 1080p): device ms per frame, host enqueue
ms per frame, and the same frame replayed from a captured CUDA graph.

    python tools/render_probe.py [--n N]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
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
    ap.add_argument("--frames", type=int, default=50)
    args = ap.parse_args()
    cloud_np, cam = synthetic.frustum_scene(args.n, 1920, 1080, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    bg = (0.0, 0.0, 0.0)
    R.render_view(cloud, cam, bg, 3)   # sizes the instance buffers (one host read of K)
    sched = R.TileSchedule()
    for _ in range(3):
        R.render_view_async(cloud, cam, bg, 3, schedule=sched)[2].check()
    torch.cuda.synchronize()

    def loop(fn, k):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        host = (time.perf_counter() - t0) * 1e3 / k
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / k, host

    res = {}
    res["async_device_ms"], res["async_host_ms"] = loop(lambda: R.render_view_async(cloud, cam, bg, 3,
                                                                                    schedule=sched), args.frames)
    # CUDA graph of one frame (the schedule's order buffers are device data)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        R.render_view_async(cloud, cam, bg, 3, schedule=sched)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            out, splats, binning = R.render_view_async(cloud, cam, bg, 3, schedule=sched)
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    binning.check()
    res["graph_device_ms"], res["graph_host_ms"] = loop(g.replay, args.frames)
    binning.check()
    res["fps_async"] = round(1e3 / res["async_device_ms"], 1)
    res["fps_graph"] = round(1e3 / res["graph_device_ms"], 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
