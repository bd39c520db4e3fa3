"""A small scene through every hand-written kernel of the training step and
the deterministic / exact-stop paths, for compute-sanitizer (racecheck,
synccheck, memcheck, initcheck): tests/test_gpu_sanitizer.py runs it."""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import numpy as np
    import torch

    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200 import synthetic
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.loss import l1_dssim_loss
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig

    w, h = 96, 64
    cloud_np, cam = synthetic.frustum_scene(3000, w, h, seed=5)
    cloud_np["opacity_logits"][:] = np.abs(cloud_np["opacity_logits"]) + 2.0   # dense, saturating pixels
    cloud = GaussianCloud.from_numpy(**cloud_np)
    tgt = R.render_view(GaussianCloud.from_numpy(**synthetic.frustum_scene(3000, w, h, seed=6)[0]), cam,
                        (0, 0, 0), 3)[0].image
    adam, cfg = DeviceAdam(cloud), TrainConfig()
    stats = R.DensifyStats.zeros(len(cloud), "cuda")
    for it in (1, 2):
        out, splats, binning = R.render_view(cloud, cam, (0.1, 0.2, 0.3), 3, training=True)
        loss, d_image = l1_dssim_loss(out.image, tgt, 0.2)
        g2 = R.render_backward(d_image, out, splats, binning, w, h, (0.1, 0.2, 0.3))
        R.render_backward(d_image, out, splats, binning, w, h, (0.1, 0.2, 0.3), deterministic=True)
        adam.backward_step(cloud, cam, splats, g2, 3, it, cfg, stats=stats)
    b2 = R.bin_and_sort_async(splats, w, h, with_keys=True)
    b2.check()
    torch.cuda.synchronize()
    print("sanitize scene ok", int(loss[0].isfinite().item()))


if __name__ == "__main__":
    main()
