"""The training loop around the device hot path (the reference's caller).

Mirrors splatlab optimizer.train_step / train (optimizer.py:222-260,
377-400): SH band schedule, epoch-shuffled view sampling from the training
RNG (130-138), resolution warm-up (194-200) with area-average target
downscaling (177-191), L1 + D-SSIM loss with the divergence check
(245-246), backward, densification statistics (252-255), fused Adam
(263-293), densify/prune schedule (389-394) and the progress line format
(395-397).  Every per-pixel / per-Gaussian stage runs in libgs_b200.so.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import rasterizer as R
from .camera import Camera
from .densify import DensifyReport, TrainState, densify_and_prune
from .errors import TrainingDiverged
from .loss import l1_dssim_loss
from .optimizer import TrainConfig


@dataclass
class TrainView:
    camera: Camera
    image: torch.Tensor   # (H,W,3) float32 device, linear RGB in [0,1]
    name: str = ""


@dataclass
class StepReport:
    iteration: int
    loss: float
    psnr: float
    view_index: int
    num_gaussians: int


def warmup_scale(iteration: int, upsample_iters=(250, 500)) -> float:
    """Quarter, half, then full resolution (optimizer.py:194-200)."""
    if iteration < upsample_iters[0]:
        return 0.25
    if iteration < upsample_iters[1]:
        return 0.5
    return 1.0


def downscale_image(image: torch.Tensor, height: int, width: int) -> torch.Tensor:
    """Area-average downscale (optimizer.py:177-191); integer factors on device,
    other factors through Pillow's BOX filter on the host like the reference."""
    h, w = image.shape[:2]
    if (h, w) == (height, width):
        return image
    if h % height == 0 and w % width == 0:
        fy, fx = h // height, w // width
        return image.reshape(height, fy, width, fx, 3).mean(dim=(1, 3))
    from PIL import Image
    host = image.detach().cpu().numpy()
    chans = [np.asarray(Image.fromarray(host[:, :, c].astype(np.float32), mode="F").resize((width, height),
                                                                                        Image.BOX))
             for c in range(3)]
    return torch.from_numpy(np.stack(chans, axis=2).astype(np.float32)).to(image.device)


def next_view(state: TrainState, num_views: int) -> int:
    """Uniform sampling without replacement within each epoch (optimizer.py:130-138)."""
    order = getattr(state, "_epoch_order", None)
    pos = getattr(state, "_epoch_pos", 0)
    if order is None or pos >= len(order) or len(order) != num_views:
        state._epoch_order = state.rng.permutation(num_views)
        state._epoch_pos = 0
    view = int(state._epoch_order[state._epoch_pos])
    state._epoch_pos += 1
    return view


def train_step(state: TrainState, views: Sequence[TrainView], config: TrainConfig) -> StepReport:
    state.iteration += 1
    it = state.iteration
    if it % config.sh_band_interval == 0 and state.active_sh_degree < 3:
        state.active_sh_degree += 1
    view_idx = next_view(state, len(views))
    view = views[view_idx]
    scale = warmup_scale(it, config.warmup_upsample_iters)
    camera = view.camera if scale == 1.0 else view.camera.scaled(scale)
    gt = downscale_image(view.image, camera.height, camera.width)
    bg = config.background
    out, splats, binning = R.render_view(state.cloud, camera, bg, state.active_sh_degree, training=True)
    loss, d_image = l1_dssim_loss(out.image, gt, config.lambda_dssim)
    value = float(loss[0].item())
    if not math.isfinite(value):
        raise TrainingDiverged(f"non-finite loss {value} at iteration {it}")
    g2 = R.render_backward(d_image, out, splats, binning, camera.width, camera.height, bg)
    state.adam.backward_step(state.cloud, camera, splats, g2, state.active_sh_degree, it, config, stats=state.stats)
    mse = float(torch.mean((out.image - gt) ** 2).item())
    psnr = float("inf") if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
    return StepReport(it, value, psnr, view_idx, len(state.cloud))


def train(state: TrainState, views: Sequence[TrainView], config: TrainConfig, *, iterations: int | None = None,
          eval_interval: int = 500, progress: Callable[[str], None] | None = None,
          densify_hook: Callable[[DensifyReport], None] | None = None) -> list[DensifyReport]:
    """Drive training with densification interleaved (optimizer.py:377-400)."""
    iterations = config.total_iters if iterations is None else iterations
    densify_until = config.resolve_densify_until()
    reports = []
    while state.iteration < iterations:
        step = train_step(state, views, config)
        if (config.densify_start < state.iteration <= densify_until
                and state.iteration % config.densify_interval == 0):
            report = densify_and_prune(state, config)
            reports.append(report)
            if densify_hook:
                densify_hook(report)
        if progress and (state.iteration % eval_interval == 0 or state.iteration == iterations):
            progress(f"iter={step.iteration} loss={step.loss:.6f} "
                     f"gaussians={len(state.cloud)} psnr={step.psnr:.2f}")
    return reports


def compute_metrics(render: torch.Tensor, ground_truth: torch.Tensor) -> tuple[float, float]:
    """(PSNR dB, mean SSIM) (optimizer.py:166-174)."""
    mse = float(torch.mean((render - ground_truth) ** 2).item())
    psnr = float("inf") if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
    loss, _ = l1_dssim_loss(render, ground_truth, 0.2)
    return psnr, float(loss[2].item())
