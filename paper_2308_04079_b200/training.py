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
from .errors import InvalidPrimitiveError, TrainingDiverged
from .loss import l1_dssim_loss
from .optimizer import TrainConfig, step_guard


@dataclass
class TrainView:
    camera: Camera
    image: torch.Tensor   # (H,W,3) float32, linear RGB in [0,1]; device, or (pinned) host copied per step
    name: str = ""


class _HostScalars:
    """Pinned host landing buffers for the one device->host read per step."""

    def __init__(self):
        self.loss = torch.empty(4, dtype=torch.float32).pin_memory()
        self.k_info = torch.empty(3, dtype=torch.int64).pin_memory()
        # written by the step-guard kernel itself (mapped pinned memory, no copy)
        self.report = torch.zeros(8, dtype=torch.float64).pin_memory()

    def skip_device(self, device) -> torch.Tensor:
        flag = getattr(self, "_skip", None)
        if flag is None or flag.device != torch.device(device):
            flag = self._skip = torch.zeros(1, dtype=torch.int32, device=device)
        return flag

    def read(self, loss: torch.Tensor, k_info: torch.Tensor):
        self.stage(loss, k_info).synchronize()
        return self.values()

    def stage(self, loss: torch.Tensor, k_info: torch.Tensor) -> torch.cuda.Event:
        """Enqueue the D2H copies; the returned event marks their completion."""
        self.loss.copy_(loss, non_blocking=True)
        self.k_info.copy_(k_info, non_blocking=True)
        done = torch.cuda.Event()
        done.record(torch.cuda.current_stream(loss.device))
        return done

    def values(self):
        return self.loss.tolist(), self.k_info.tolist()

    def report_values(self):
        r = self.report.tolist()
        return r[0:4], [int(v) for v in r[4:7]]


_host_scalars: dict = {}


class _ImagePrefetcher:
    """Host-resident view images: the next step's image (known in advance
    from the epoch order) is copied H2D on a side stream while the current
    step computes; two device buffers alternate, each released by an event
    recorded after the loss kernels (its last reader).  A slot holds the view
    object itself (identity-compared, so a recycled id() can never alias a
    stale slot) and the image's pointer and shape."""

    def __init__(self, device):
        self.device = device
        self.stream = torch.cuda.Stream(device)
        self.slots = [None, None]      # (view, (data_ptr, shape), device tensor, ready event, consumed event)
        self.turn = 0

    @staticmethod
    def _tag(view: TrainView):
        return view.image.data_ptr(), tuple(view.image.shape)

    def _issue(self, view: TrainView):
        slot = self.turn
        self.turn ^= 1
        old = self.slots[slot]
        buf = old[2] if old is not None and old[2].shape == view.image.shape else torch.empty(
            view.image.shape, dtype=view.image.dtype, device=self.device)
        ready = torch.cuda.Event()
        with torch.cuda.stream(self.stream):
            if old is not None:
                self.stream.wait_event(old[4])
            buf.copy_(view.image, non_blocking=True)
            ready.record(self.stream)
        self.slots[slot] = (view, self._tag(view), buf, ready, torch.cuda.Event())
        return self.slots[slot]

    def _match(self, s, view: TrainView) -> bool:
        return s is not None and s[0] is view and s[1] == self._tag(view)

    def get(self, view: TrainView, fresh: bool = False):
        """(device image, consumed event) for this step's view.  fresh: copy
        it again even if a slot holds it (its buffer may have been reused)."""
        hit = None if fresh else next((s for s in self.slots if self._match(s, view)), None)
        if hit is None:
            hit = self._issue(view)
        torch.cuda.current_stream(self.device).wait_event(hit[3])
        self.slots = [s if s is not hit else (None, None, s[2], s[3], s[4]) for s in self.slots]
        return hit[2], hit[4]

    def prefetch(self, view: TrainView) -> None:
        if not any(self._match(s, view) for s in self.slots):
            self._issue(view)

    def clear(self) -> None:
        """Drop the view references (end of a training run)."""
        self.slots = [None if s is None else (None, None, s[2], s[3], s[4]) for s in self.slots]


_prefetchers: dict = {}


def _peek_next_view(state: TrainState, num_views: int):
    if num_views == 1:
        return 0
    order = getattr(state, "_epoch_order", None)
    pos = getattr(state, "_epoch_pos", 0)
    if order is None or pos >= len(order) or len(order) != num_views:
        return None   # the next epoch's order is not drawn yet (RNG order must match the reference)
    return int(order[pos])


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


def _world(group) -> tuple[int, int]:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _degree_for(prev_degree: int, it: int, config: TrainConfig) -> int:
    """Active SH degree at iteration `it` given the degree before it (one band
    every sh_band_interval iterations, optimizer.py:232-233)."""
    return prev_degree + 1 if (it % config.sh_band_interval == 0 and prev_degree < 3) else prev_degree


def _cloud_key(state: TrainState) -> tuple:
    c = state.cloud
    return (id(c), len(c), c.means.data_ptr(), c.rotations.data_ptr(), c.sh.data_ptr())


@dataclass
class _Forward:
    """One iteration's sampled view and its enqueued forward + loss."""
    it: int
    view_idx: int
    camera: Camera
    degree: int
    gt: torch.Tensor
    consumed: object
    snapshot: tuple     # view-sampling state before this view was drawn (TrainState.discard_lookahead)
    views: Sequence[TrainView]   # the objects the forward was made for (held: identity compared)
    config: TrainConfig
    cloud_key: tuple
    out: object = None
    splats: object = None
    binning: object = None
    loss: torch.Tensor = None
    d_image: torch.Tensor = None
    prep: object = None   # rasterizer.BackwardPrep (side-stream tile schedule + cleared rows)


def _sample_view(state: TrainState, views: Sequence[TrainView], config: TrainConfig, it: int,
                 degree: int) -> _Forward:
    snapshot = (getattr(state, "_epoch_order", None), getattr(state, "_epoch_pos", 0),
                state.rng.bit_generator.state)
    view_idx = next_view(state, len(views))
    view = views[view_idx]
    scale = warmup_scale(it, config.warmup_upsample_iters)
    camera = view.camera if scale == 1.0 else view.camera.scaled(scale)
    gt, consumed = _ground_truth(state, view, camera)
    device = state.cloud.device
    if view.image.device != device:   # prefetch the next view's image one step ahead
        nxt = _peek_next_view(state, len(views))
        if nxt is not None and views[nxt].image.device != device:
            _prefetchers[str(device)].prefetch(views[nxt])
    return _Forward(it, view_idx, camera, degree, gt, consumed, snapshot, views, config, _cloud_key(state))


def _ground_truth(state: TrainState, view: TrainView, camera: Camera, fresh: bool = False):
    """(target image at the camera's resolution, consumed event or None).
    A host-resident view is copied H2D from pinned memory by the prefetcher;
    fresh: copy it again (the slot's buffer may have been handed on)."""
    device = state.cloud.device
    image, consumed = view.image, None
    if image.device != device:
        pf = _prefetchers.setdefault(str(device), _ImagePrefetcher(device))
        image, consumed = pf.get(view, fresh=fresh)
    return downscale_image(image, camera.height, camera.width), consumed


def _enqueue_forward(state: TrainState, fw: _Forward, config: TrainConfig, splats=None) -> _Forward:
    """splats: the view's projection when the previous step's fused
    backward + Adam already made it (DeviceAdam.backward_step project_next)."""
    # the view's last backward schedule (heavy tiles first) orders this forward's tiles
    orders = getattr(state, "_tile_orders", None)
    order = orders.get((fw.view_idx, fw.camera.width, fw.camera.height)) if orders else None
    fw.out, fw.splats, fw.binning = R.render_view_async(state.cloud, fw.camera, config.background, fw.degree,
                                                        training=True, tile_order=order, splats=splats)
    # the backward's tile schedule and row clearing run on a side stream, beside the loss
    fw.prep = None if config.deterministic else R.prepare_backward(fw.out, fw.splats, fw.binning, fw.camera.width,
                                                                  fw.camera.height)
    fw.loss, fw.d_image = l1_dssim_loss(fw.out.image, fw.gt, config.lambda_dssim)
    if fw.consumed is not None:
        fw.consumed.record()
    return fw


def train_step(state: TrainState, views: Sequence[TrainView], config: TrainConfig, group=None,
               lookahead: bool = False) -> StepReport:
    """One iteration (optimizer.py:222-260), with ONE host synchronisation:
    the loss, the step's MSE (for the PSNR) and the binning's instance count
    and flags are read together at the end of the step.  The backward and
    the fused Adam are enqueued before that read behind a device-side guard
    (`step_guard`: loss not finite, capacity overflow, zero quaternion), so
    the divergence check (optimizer.py:245-246) and a capacity overflow
    (re-render with a larger buffer) still find nothing applied.

    lookahead (opt-in; `train` turns it on): before waiting for this step,
    the NEXT iteration's view is
    drawn and its forward + loss enqueued behind this step's Adam (stream
    order: it sees the updated parameters), so the GPU never idles while the
    host reads the loss; the fused backward + Adam launch also projects the
    updated parameters for that view (gs_preprocess_backward_adam_project).  The next train_step call consumes it when the
    iteration, views, config and cloud still match; otherwise (and in
    densify_and_prune) `TrainState.discard_lookahead` restores the view
    sampling state, so the sampled sequence is exactly the reference's.
    After modifying parameters outside train_step, call
    `state.discard_lookahead()`.

    Under torch.distributed (world > 1) every rank samples a view from its
    contiguous shard of `views`, its gradients go to one flat
    bucket, one NCCL all-reduce sums them and every rank runs the identical
    Adam, so the replicas stay bit-identical (no lookahead)."""
    world, rank = _world(group)
    if world > 1:
        return _train_step_sharded(state, views, config, group, world, rank)
    it = state.iteration + 1
    degree = _degree_for(state.active_sh_degree, it, config)
    fw = getattr(state, "_lookahead", None)
    if fw is not None and (fw.it != it or fw.degree != degree or fw.views is not views or fw.config is not config
                           or fw.cloud_key != _cloud_key(state)):
        state.discard_lookahead()
        fw = None
    state._lookahead = None
    if fw is None:
        fw = _enqueue_forward(state, _sample_view(state, views, config, it, degree), config)
    device = state.cloud.device
    host = _host_scalars.setdefault(str(device), _HostScalars())
    nxt = None
    for attempt in range(3):
        skip = step_guard(fw.loss, fw.binning.k_info, host.skip_device(device), report=host.report)
        # the host waits for this step's forward, loss and guard only: the
        # backward, the guarded Adam and the next forward stay queued behind it
        done = torch.cuda.Event()
        done.record(torch.cuda.current_stream(device))
        g2 = R.render_backward(fw.d_image, fw.out, fw.splats, fw.binning, fw.camera.width, fw.camera.height,
                               config.background, deterministic=config.deterministic, prep=fw.prep)
        if g2.tile_order is not None:
            if not hasattr(state, "_tile_orders"):
                state._tile_orders = {}
            state._tile_orders[(fw.view_idx, fw.camera.width, fw.camera.height)] = g2.tile_order
        # lookahead: the next view is drawn first, so the fused backward + Adam
        # also projects the updated parameters for it (no separate K1 launch)
        nxt = _sample_view(state, views, config, it + 1, _degree_for(degree, it + 1, config)) if lookahead else None
        nsplats = state.adam.backward_step(state.cloud, fw.camera, fw.splats, g2, fw.degree, it, config,
                                           stats=state.stats, skip=skip,
                                           project_next=None if nxt is None else (nxt.camera, nxt.degree))
        if nxt is not None:
            nxt = _enqueue_forward(state, nxt, config, splats=nsplats)
        done.synchronize()
        lvals, kvals = host.report_values()
        try:
            fw.binning.check_host(kvals)
            break
        except R.CapacityError:   # nothing was applied: re-render this view with the larger capacity
            if nxt is not None:
                state._lookahead, nxt = nxt, None
                state.discard_lookahead()
            if attempt == 2:
                raise
            # the lookahead's prefetch may have refilled this view's image buffer: copy it again
            fw.gt, fw.consumed = _ground_truth(state, fw.views[fw.view_idx], fw.camera, fresh=True)
            fw = _enqueue_forward(state, fw, config)
    state.iteration, state.active_sh_degree = it, degree
    value, mse = float(lvals[0]), float(lvals[3])
    if not math.isfinite(value):
        if nxt is not None:
            state._lookahead = nxt
            state.discard_lookahead()
        raise TrainingDiverged(f"non-finite loss {value} at iteration {it}")
    state._lookahead = nxt
    psnr = float("inf") if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
    return StepReport(it, value, psnr, fw.view_idx, len(state.cloud))


def _train_step_sharded(state: TrainState, views: Sequence[TrainView], config: TrainConfig, group, world: int,
                        rank: int) -> StepReport:
    """The view-parallel step: this rank's view of its shard,
    the backward into one flat gradient bucket, one NCCL all-reduce (or, with
    state.shard_optimizer, a reduce-scatter into ZeRO-1 sharded Adam and an
    all-gather), the identical update on every rank.  No host wait before the
    update: every rank's step guard (loss not finite, instance capacity, zero
    quaternion) is MAX-reduced over the ranks on the device, and the
    statistics and Adam apply nothing when any rank vetoed; the host reads the
    reduced verdict once at the end, so every rank raises (or retries a
    capacity overflow) together."""
    from .distributed import GradientBucket, ShardedAdam, max_reduce_, shard_views
    state.discard_lookahead()
    it = state.iteration + 1
    degree = _degree_for(state.active_sh_degree, it, config)
    shard = shard_views(len(views), world, rank)
    view_idx = shard[next_view(state, len(shard))]
    view = views[view_idx]
    scale = warmup_scale(it, config.warmup_upsample_iters)
    camera = view.camera if scale == 1.0 else view.camera.scaled(scale)
    device = state.cloud.device
    gt, consumed = _ground_truth(state, view, camera)
    if view.image.device != device:
        nxt = _peek_next_view(state, len(shard))
        nxt = None if nxt is None else shard[nxt]
        if nxt is not None and views[nxt].image.device != device:
            _prefetchers[str(device)].prefetch(views[nxt])
    bg = config.background
    host = _host_scalars.setdefault(str(device), _HostScalars())
    n = len(state.cloud)
    sharded = None
    if getattr(state, "shard_optimizer", False):
        sharded = getattr(state, "_sharded", None)
        if sharded is None or sharded.n != n:
            sharded = state._sharded = ShardedAdam.from_moments(state.cloud, state.adam.exp_avg,
                                                                 state.adam.exp_avg_sq, group)
        grads = sharded.grads
    else:
        bucket = getattr(state, "_bucket", None)
        if bucket is None or bucket.n != n:
            bucket = state._bucket = GradientBucket(n, device)
        grads = bucket.grads
    for attempt in range(3):
        out, splats, binning = R.render_view_async(state.cloud, camera, bg, degree, training=True)
        loss, d_image = l1_dssim_loss(out.image, gt, config.lambda_dssim)
        if consumed is not None:
            consumed.record()
        step_guard(loss, binning.k_info, host.skip_device(device), report=host.report)
        # every rank's verdict, bit by bit: [zero quaternion, capacity, instance limit, loss not finite]
        fl = binning.k_info[1]
        verdict = torch.stack([(fl & 1) != 0, (fl & 2) != 0, (fl & 4) != 0, ~torch.isfinite(loss[0])]).to(torch.int32)
        max_reduce_(verdict, group)
        skip = verdict.amax().reshape(1).contiguous()
        g2 = R.render_backward(d_image, out, splats, binning, camera.width, camera.height, bg,
                               deterministic=config.deterministic)
        if sharded is not None:
            sharded.zero_()
        else:
            bucket.zero_()
        R.backward_project(state.cloud, camera, splats, g2, degree, stats=state.stats, out=grads, accumulate=True,
                           skip=skip)
        if sharded is not None:
            sharded.step(state.cloud, it, config, skip=skip)
        else:
            bucket.allreduce_(group)
            state.adam.step(state.cloud, grads, it, config, skip=skip)
        zero_q, capacity, limit, nonfinite = (int(v) for v in verdict.tolist())   # the step's one host read
        lvals, kvals = host.report_values()
        # every rank takes the same branch
        if nonfinite:
            raise TrainingDiverged(f"non-finite loss {lvals[0]} at iteration {it}"
                                   + ("" if not math.isfinite(lvals[0]) else " (on another rank)"))
        if zero_q:
            raise InvalidPrimitiveError("zero-norm quaternion cannot be normalized")
        if limit:
            from . import _lib
            _lib.check(_lib.GS_ERR_RESOURCE_LIMIT, "bin_and_sort")
        if not capacity:
            break
        try:   # a rank that overflowed raises its capacity hint; every rank re-renders its view
            binning.check_host(kvals)
        except R.CapacityError:
            pass
        if attempt == 2:
            raise R.CapacityError("bin_and_sort: instance capacity did not converge")
    state.iteration, state.active_sh_degree = it, degree
    value, mse = float(lvals[0]), float(lvals[3])
    psnr = float("inf") if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
    return StepReport(it, value, psnr, view_idx, len(state.cloud))


def train(state: TrainState, views: Sequence[TrainView], config: TrainConfig, *, iterations: int | None = None,
          eval_interval: int = 500, progress: Callable[[str], None] | None = None,
          densify_hook: Callable[[DensifyReport], None] | None = None,
          checkpoint_hook: Callable[[TrainState], None] | None = None,
          checkpoint_iters: Sequence[int] = (7000, 30000), group=None) -> list[DensifyReport]:
    """Drive training with densification interleaved (optimizer.py:377-400),
    including the reference's checkpoint hook (optimizer.py:398-399).

    The lookahead (see train_step) is skipped on iterations followed by a
    densification or a checkpoint, so the hooks see a state with nothing
    pending.  Under torch.distributed the densification statistics are
    reduced over the ranks (sum / max) and every rank densifies with rank 0's
    RNG state, so the replicas clone, split and prune identically."""
    iterations = config.total_iters if iterations is None else iterations
    densify_until = config.resolve_densify_until()
    world, _ = _world(group)
    reports = []
    try:
        while state.iteration < iterations:
            nxt = state.iteration + 1
            densify_next = (config.densify_start < nxt <= densify_until and nxt % config.densify_interval == 0)
            ckpt_next = checkpoint_hook is not None and nxt in checkpoint_iters
            step = train_step(state, views, config, group=group,
                              lookahead=nxt < iterations and not densify_next and not ckpt_next)
            if (config.densify_start < state.iteration <= densify_until
                    and state.iteration % config.densify_interval == 0):
                if world > 1:
                    from .distributed import reduce_stats_, sync_rng_
                    reduce_stats_(state.stats, group)
                    sync_rng_(state, group)
                    sharded = getattr(state, "_sharded", None)
                    if sharded is not None:   # ZeRO-1: realign the full moments, re-shard next step
                        state.adam.exp_avg, state.adam.exp_avg_sq = sharded.full_moments()
                        state._sharded = None
                report = densify_and_prune(state, config)
                reports.append(report)
                if densify_hook:
                    densify_hook(report)
            if progress and (state.iteration % eval_interval == 0 or state.iteration == iterations):
                progress(f"iter={step.iteration} loss={step.loss:.6f} "
                         f"gaussians={len(state.cloud)} psnr={step.psnr:.2f}")
            if checkpoint_hook and state.iteration in checkpoint_iters:
                state.discard_lookahead()
                checkpoint_hook(state)
    finally:
        for pf in _prefetchers.values():
            pf.clear()
    return reports


def views_from_scene(images, pin: bool = True) -> list[TrainView]:
    """TrainViews from colmap.SceneImage entries: the decoded float32 linear
    images stay in (pinned) host memory and are prefetched to the device one
    step ahead by train_step."""
    views = []
    for im in images:
        t = torch.from_numpy(np.ascontiguousarray(im.load_pixels(), dtype=np.float32))
        views.append(TrainView(im.camera, t.pin_memory() if pin and torch.cuda.is_available() else t, im.name))
    return views


def compute_metrics(render: torch.Tensor, ground_truth: torch.Tensor) -> tuple[float, float]:
    """(PSNR dB, mean SSIM) (optimizer.py:166-174)."""
    mse = float(torch.mean((render - ground_truth) ** 2).item())
    psnr = float("inf") if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
    loss, _ = l1_dssim_loss(render, ground_truth, 0.2)
    return psnr, float(loss[2].item())
