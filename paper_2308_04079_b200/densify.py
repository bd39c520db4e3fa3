"""Device adaptive density control.

Mirrors splatlab's TrainState (optimizer.py:88-138) and densify_and_prune
(optimizer.py:304-374) over device tensors: the classification, row
bookkeeping, split sampling transform, pruning and moment realignment run in
libgs_b200.so (gs_densify_classify / gs_densify_apply); only the split
samples z ~ N(0,1) are drawn on the host, from the same numpy Generator the
reference uses (state.rng, optimizer.py:335), so the RNG stream matches.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cloud import PARAM_GROUPS, GaussianCloud
from .optimizer import DeviceAdam, TrainConfig
from .rasterizer import DensifyStats


@dataclass
class DensifyReport:
    cloned: int
    split: int
    pruned: int
    opacity_reset: bool


class TrainState:
    """Gaussians + Adam moments + densification statistics + counters
    (optimizer.py:88-138), device resident.  `rng` is a numpy Generator
    seeded like the reference's (optimizer.py:102)."""

    def __init__(self, cloud: GaussianCloud, scene_extent: float, seed: int = 0):
        if scene_extent <= 0:
            raise ValueError("scene extent must be positive")
        self.cloud = cloud
        self.scene_extent = float(scene_extent)
        self.iteration = 0
        self.active_sh_degree = 0
        self.rng = np.random.default_rng(seed)
        self.adam = DeviceAdam(cloud)
        self.stats = DensifyStats.zeros(len(cloud), cloud.device)

    def discard_lookahead(self) -> None:
        """Drop a speculative next-iteration forward enqueued by train_step
        (lookahead) and restore the view-sampling state it consumed, so the
        next draw (and any other use of `rng`) matches the reference order."""
        la = getattr(self, "_lookahead", None)
        self._lookahead = None
        if la is not None:
            self._epoch_order, self._epoch_pos, rng_state = la.snapshot
            self.rng.bit_generator.state = rng_state

    def reset_stats(self) -> None:
        self.stats = DensifyStats.zeros(len(self.cloud), self.cloud.device)

    def check_alignment(self) -> None:
        n = len(self.cloud)
        for g in PARAM_GROUPS:
            assert self.adam.exp_avg[g].shape == getattr(self.cloud, g).shape
            assert self.adam.exp_avg_sq[g].shape == getattr(self.cloud, g).shape
        for t in (self.stats.accum_pos_grad, self.stats.accum_count, self.stats.max_radius_frac):
            assert t.shape == (n,)


def _state_struct(cloud: GaussianCloud, adam: DeviceAdam, n: int) -> _lib.GsCloudState:
    s = _lib.GsCloudState()
    for i, g in enumerate(PARAM_GROUPS):
        s.param[i] = getattr(cloud, g).data_ptr()
        s.exp_avg[i] = adam.exp_avg[g].data_ptr()
        s.exp_avg_sq[i] = adam.exp_avg_sq[g].data_ptr()
    s.n = n
    return s


def _config_struct(state: TrainState, config: TrainConfig) -> tuple[_lib.GsDensifyConfig, bool]:
    c = _lib.GsDensifyConfig()
    c.grad_threshold = config.densify_grad_threshold
    c.split_scale_threshold = config.resolve_split_threshold(state.scene_extent)
    c.split_log_factor = math.log(config.split_factor)
    c.prune_alpha = config.prune_alpha_threshold
    c.prune_world_scale = config.prune_world_percent * state.scene_extent
    c.prune_screen_fraction = config.prune_screen_fraction
    c.prune_big = int(state.iteration > config.opacity_reset_interval)
    reset = state.iteration > 0 and state.iteration % config.opacity_reset_interval == 0
    c.reset_opacity = int(reset)
    a = config.opacity_reset_alpha
    c.reset_logit = math.log(a / (1.0 - a))
    return c, reset


def densify_and_prune(state: TrainState, config: TrainConfig) -> DensifyReport:
    """Clone small / split large high-gradient Gaussians, prune transparent or
    oversized ones, periodically reset opacity; moments stay aligned and new
    Gaussians start with zero moments; statistics reset (optimizer.py:304-374)."""
    state.discard_lookahead()   # its forward used the pre-densify cloud, and it drew from state.rng
    lib = _lib.load()
    cloud, adam, dev = state.cloud, state.adam, state.cloud.device
    n = len(cloud)
    stream = torch.cuda.current_stream(dev).cuda_stream
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gs_densify_workspace_size(n, ctypes.byref(nbytes)), "densify")
    ws = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=dev)
    src = _state_struct(cloud, adam, n)
    cfg, reset = _config_struct(state, config)
    st = state.stats.c_struct()
    n_clone, n_split = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(lib.gs_densify_classify(ctypes.byref(src), ctypes.byref(st), ctypes.byref(cfg), ws.data_ptr(),
                                       nbytes.value, ctypes.byref(n_clone), ctypes.byref(n_split), stream),
               "densify_classify")
    ns, nc = int(n_split.value), int(n_clone.value)
    z = None
    if ns:  # optimizer.py:335, from the training RNG stream
        z = torch.from_numpy(state.rng.standard_normal((2 * ns, 3)).astype(np.float32)).to(dev)
    cap = n - ns + nc + 2 * ns
    new_cloud = GaussianCloud(*(torch.empty((cap,) + tuple(getattr(cloud, g).shape[1:]), dtype=torch.float32,
                                            device=dev)
                                for g in ("means", "rotations", "log_scales", "opacity_logits", "sh")))
    new_adam = DeviceAdam.__new__(DeviceAdam)
    new_adam.exp_avg = {g: torch.empty_like(getattr(new_cloud, g)) for g in PARAM_GROUPS}
    new_adam.exp_avg_sq = {g: torch.empty_like(getattr(new_cloud, g)) for g in PARAM_GROUPS}
    dst = _state_struct(new_cloud, new_adam, cap)
    n_out = ctypes.c_int64(0)
    _lib.check(lib.gs_densify_apply(ctypes.byref(src), ctypes.byref(st), ctypes.byref(cfg), nc, ns,
                                    z.data_ptr() if z is not None else None, ws.data_ptr(), nbytes.value,
                                    ctypes.byref(dst), ctypes.byref(n_out), stream), "densify_apply")
    m = int(n_out.value)
    state.cloud = GaussianCloud(*(getattr(new_cloud, g)[:m].contiguous()
                                  for g in ("means", "rotations", "log_scales", "opacity_logits", "sh")))
    adam.exp_avg = {g: new_adam.exp_avg[g][:m].contiguous() for g in PARAM_GROUPS}
    adam.exp_avg_sq = {g: new_adam.exp_avg_sq[g][:m].contiguous() for g in PARAM_GROUPS}
    state.reset_stats()
    state.check_alignment()
    return DensifyReport(cloned=nc, split=ns, pruned=cap - m, opacity_reset=reset)
