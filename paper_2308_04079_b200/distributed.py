"""View-parallel multi-GPU training plumbing.

Views are independent units of work; parameters and Adam state are
replicated.  Each rank renders its shard of the camera batch, accumulating
its views' gradients into one flat (N x 59) float32 bucket (so a single NCCL
all-reduce covers all five groups), then every rank runs the identical fused
Adam on the reduced gradients.  Densification statistics are per view and
accumulate on each rank before the cross-rank reduction
(optimizer.py:252-254); the reduction sums accum_pos_grad/accum_count and
takes the max of max_radius_frac.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .rasterizer import DensifyStats, GaussianGrads

GROUP_WIDTHS = (("d_means", 3), ("d_rotations", 4), ("d_log_scales", 3), ("d_opacity_logits", 1), ("d_sh", 48))
FLOATS_PER_GAUSSIAN = sum(w for _, w in GROUP_WIDTHS)  # 59


def shard_views(num_views: int, world: int, rank: int) -> list[int]:
    """Contiguous shard of a camera batch: rank r gets views [r*B/G, (r+1)*B/G)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    lo = (num_views * rank) // world
    hi = (num_views * (rank + 1)) // world
    return list(range(lo, hi))


class GradientBucket:
    """One flat float32 buffer with GaussianGrads views into it."""

    def __init__(self, n: int, device, dtype=torch.float32):
        self.n = n
        self.flat = torch.zeros(n * FLOATS_PER_GAUSSIAN, dtype=dtype, device=device)
        parts = torch.split(self.flat, [n * w for _, w in GROUP_WIDTHS])
        shapes = {"d_means": (n, 3), "d_rotations": (n, 4), "d_log_scales": (n, 3), "d_opacity_logits": (n,),
                  "d_sh": (n, 16, 3)}
        views = {name: part.view(shapes[name]) for (name, _), part in zip(GROUP_WIDTHS, parts)}
        self.grads = GaussianGrads(views["d_means"], views["d_rotations"], views["d_log_scales"],
                                   views["d_opacity_logits"], views["d_sh"],
                                   torch.zeros(n, dtype=dtype, device=device))

    def zero_(self) -> None:
        self.flat.zero_()

    def allreduce_(self, group=None) -> None:
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)


def reduce_stats_(stats: DensifyStats, group=None) -> None:
    """Cross-rank densification statistics: sums and max (in place)."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return
    dist.all_reduce(stats.accum_pos_grad, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(stats.accum_count, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(stats.max_radius_frac, op=dist.ReduceOp.MAX, group=group)


def train_step_views(cloud, cameras, targets, adam, config, iteration: int, bucket: GradientBucket,
                     stats: DensifyStats | None = None, background=(0.0, 0.0, 0.0), active_sh_degree: int = 3,
                     group=None) -> torch.Tensor:
    """One multi-view training iteration on this rank's views: per view
    project -> bin -> blend -> loss -> blend bwd -> backward_project
    (accumulated into the bucket), then the all-reduce and the fused Adam.
    Returns the summed loss of this rank's views (device scalar)."""
    from . import rasterizer as R
    from .loss import l1_dssim_loss

    bucket.zero_()
    total = torch.zeros((), dtype=torch.float32, device=cloud.device)
    for cam, gt in zip(cameras, targets):
        out, splats, binning = R.render_view(cloud, cam, background, active_sh_degree, training=True)
        loss, d_image = l1_dssim_loss(out.image, gt, config.lambda_dssim)
        g2 = R.render_backward(d_image, out, splats, binning, cam.width, cam.height, background)
        R.backward_project(cloud, cam, splats, g2, active_sh_degree, stats=stats, out=bucket.grads,
                           accumulate=True)
        total += loss[0]
    bucket.allreduce_(group)
    adam.step(cloud, bucket.grads, iteration, config)
    return total
