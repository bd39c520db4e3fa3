"""Kernel-variant microbenchmark: times the blend kernels (and the binning)
on the c3 workload (3M Gaussians, 1080p) with CUDA events, for one library
build.  Used to compare compile-time variants:

    GS_B200_LIB=path/to/variant.so python tools/stage_bench.py [--n N]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import numpy as np
    import torch

    from paper_2308_04079_b200 import _lib, synthetic
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.cloud import GaussianCloud

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    lib = _lib.load()
    cloud_np, cam = synthetic.frustum_scene(args.n, 1920, 1080, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    bg = (0.0, 0.0, 0.0)
    out, splats, binning = R.render_view(cloud, cam, bg, 3, training=True)
    d = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (1080, 1920, 3)).astype(np.float32) / 6e6).cuda()

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / args.reps

    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    adam = DeviceAdam(cloud)
    stats = R.DensifyStats.zeros(len(cloud), "cuda")
    g2 = R.render_backward(d, out, splats, binning, 1920, 1080, bg)
    it = [0]

    def bwd_adam():
        it[0] += 1
        adam.backward_step(cloud, cam, splats, g2, 3, it[0], TrainConfig(), stats=stats)

    res = {
        "lib": str(_lib.LIB_PATH),
        "bwd_adam_ms": timeit(bwd_adam),
        "blend_fwd_ms": timeit(lambda: R.render_forward(splats, binning, 1920, 1080, bg, training=True)),
        "blend_bwd_ms": timeit(lambda: R.render_backward(d, out, splats, binning, 1920, 1080, bg)),
        "bin_async_ms": timeit(lambda: R.bin_and_sort_async(splats, 1920, 1080)),
    }
    g_ref = R.render_backward(d, out, splats, binning, 1920, 1080, bg).packed
    res["bwd_checksum"] = float(g_ref.double().abs().sum())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
