"""Active-lane histogram of the backward blend's visited (warp, splat) pairs
at c3 (needs a library built with -DGS_BWD_STATS=1):

    GS_B200_LIB=variants/bwdstats.so python tools/bwd_stats.py
"""
from __future__ import annotations

import ctypes
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
    lib = _lib.load()
    cloud_np, cam = synthetic.frustum_scene(3_000_000, 1920, 1080, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    bg = (0.0, 0.0, 0.0)
    out, splats, binning = R.render_view(cloud, cam, bg, 3, training=True)
    d = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (1080, 1920, 3)).astype(np.float32) / 6e6).cuda()
    h = (ctypes.c_ulonglong * 33)()
    lib.gs_debug_bwd_hist(h, 1)
    R.render_backward(d, out, splats, binning, 1920, 1080, bg)
    torch.cuda.synchronize()
    lib.gs_debug_bwd_hist(h, 1)
    hist = [int(x) for x in h]
    tot = sum(hist)
    cum = np.cumsum(hist) / max(tot, 1)
    print(json.dumps({"visited": tot, "hist": hist, "cum_le": {k: round(float(cum[k]), 4) for k in (0, 1, 2, 4, 8, 16)},
                      "mean_active": sum(i * c for i, c in enumerate(hist)) / max(tot, 1)}))


if __name__ == "__main__":
    main()
