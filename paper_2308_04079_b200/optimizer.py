"""Fused device Adam and the training-step slice of the hot path.

Mirrors splatlab's optimizer slice: TrainConfig learning rates and the
position-LR decay (optimizer.py:20-75), the dense per-group Adam
(`_adam_step`, optimizer.py:263-293) and the densification statistics
(optimizer.py:252-255).  One gs_adam_step launch updates all five groups.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .cloud import PARAM_GROUPS, GaussianCloud
from .rasterizer import DensifyStats, GaussianGrads


@dataclass
class TrainConfig:
    """The Adam / schedule fields of splatlab TrainConfig (optimizer.py:20-48)."""

    lambda_dssim: float = 0.2
    densify_interval: int = 100
    densify_start: int = 500
    densify_until: int | None = None   # default: half the schedule
    densify_grad_threshold: float = 0.0002
    split_scale_threshold: float | None = None   # world units; default 1% of scene extent
    split_scale_percent: float = 0.01
    split_factor: float = 1.6
    opacity_reset_interval: int = 3000
    opacity_reset_alpha: float = 0.01
    prune_alpha_threshold: float = 0.005
    prune_world_percent: float = 0.10
    prune_screen_fraction: float = 0.5           # of image height
    warmup_upsample_iters: tuple[int, int] = (250, 500)
    total_iters: int = 30000
    lr_means: float = 1.6e-4
    lr_means_final: float = 1.6e-6
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 2.5e-3 / 20.0
    lr_opacity: float = 5e-2
    lr_log_scales: float = 5e-3
    lr_rotations: float = 1e-3
    adam_betas: tuple[float, float] = (0.9, 0.999)
    adam_eps: float = 1e-15
    background: tuple[float, float, float] = (0.0, 0.0, 0.0)
    sh_band_interval: int = 1000
    workers: int = 1                 # the reference's tile threads (kept for API parity; tiles are CTAs)
    deterministic: bool = False      # bit-identical runs: atomic-free backward (the CLI's --deterministic)

    def __post_init__(self):
        if not 0.0 <= self.lambda_dssim <= 1.0:
            raise ValueError("lambda_dssim must be in [0, 1]")
        for name in ("densify_interval", "opacity_reset_interval", "sh_band_interval", "total_iters"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        for name in ("densify_grad_threshold", "split_factor", "prune_alpha_threshold"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    def resolve_split_threshold(self, scene_extent: float) -> float:
        if self.split_scale_threshold is not None:
            return self.split_scale_threshold
        return self.split_scale_percent * scene_extent

    def resolve_densify_until(self) -> int:
        return self.densify_until if self.densify_until is not None else self.total_iters // 2

    def lr_means_at(self, iteration: int) -> float:
        """Exponential position-LR decay (optimizer.py:72-75)."""
        frac = min(iteration, self.total_iters) / self.total_iters
        return self.lr_means * (self.lr_means_final / self.lr_means) ** frac


def _lr_table(t: int, config: "TrainConfig") -> dict:
    return {"means": config.lr_means_at(t), "log_scales": config.lr_log_scales, "rotations": config.lr_rotations,
            "opacity_logits": config.lr_opacity, "sh": config.lr_sh_rest}


def adam_step_tensors(params: dict, grads: dict, exp_avg: dict, exp_avg_sq: dict, iteration: int,
                      config: "TrainConfig", skip: torch.Tensor | None = None) -> None:
    """One gs_adam_step launch over explicit per-group tensors (contiguous
    row ranges of the groups, e.g. one rank's shard; the SH head LR applies to
    the first 3 of every 48 elements, so a range must start on a Gaussian)."""
    t = int(iteration)
    bias1, bias2 = DeviceAdam._bias(t, config)
    lrs = _lr_table(t, config)
    groups = (_lib.GsAdamGroup * len(PARAM_GROUPS))()
    for i, name in enumerate(PARAM_GROUPS):
        p, g, m, v = params[name], grads[name], exp_avg[name], exp_avg_sq[name]
        for x in (p, g, m, v):
            if not x.is_contiguous():
                raise ValueError(f"{name}: Adam tensors must be contiguous")
        G = groups[i]
        G.param, G.grad, G.exp_avg, G.exp_avg_sq = p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr()
        G.numel = p.numel()
        G.lr = lrs[name]
        if name == "sh":  # row 0 (DC) uses lr_sh_dc (optimizer.py:268-269)
            G.lr_head, G.period, G.head = config.lr_sh_dc, 48, 3
        else:
            G.lr_head, G.period, G.head = lrs[name], 0, 0
    beta1, beta2 = config.adam_betas
    _lib.check(_lib.load().gs_adam_step_guarded(groups, len(PARAM_GROUPS), beta1, beta2, config.adam_eps, bias1,
                                                bias2, _lib.ptr(skip), torch.cuda.current_stream().cuda_stream),
               "adam_step")


class DeviceAdam:
    """Adam moments for the five parameter groups, updated in one launch."""

    def __init__(self, cloud: GaussianCloud):
        self.exp_avg = {g: torch.zeros_like(getattr(cloud, g)) for g in PARAM_GROUPS}
        self.exp_avg_sq = {g: torch.zeros_like(getattr(cloud, g)) for g in PARAM_GROUPS}

    def _groups(self, cloud: GaussianCloud, grads: GaussianGrads | None, t: int, config: TrainConfig):
        grad_of = {} if grads is None else {
            "means": grads.d_means, "log_scales": grads.d_log_scales, "rotations": grads.d_rotations,
            "opacity_logits": grads.d_opacity_logits, "sh": grads.d_sh}
        lrs = {"means": config.lr_means_at(t), "log_scales": config.lr_log_scales,
               "rotations": config.lr_rotations, "opacity_logits": config.lr_opacity, "sh": config.lr_sh_rest}
        groups = (_lib.GsAdamGroup * len(PARAM_GROUPS))()
        for i, name in enumerate(PARAM_GROUPS):
            p, g = getattr(cloud, name), grad_of.get(name)
            if not p.is_contiguous() or (g is not None and not g.is_contiguous()):
                raise ValueError(f"{name}: parameters and gradients must be contiguous")
            G = groups[i]
            G.param, G.grad = p.data_ptr(), (g.data_ptr() if g is not None else None)
            G.exp_avg, G.exp_avg_sq = self.exp_avg[name].data_ptr(), self.exp_avg_sq[name].data_ptr()
            G.numel = p.numel()
            G.lr = lrs[name]
            if name == "sh":  # row 0 (DC) uses lr_sh_dc (optimizer.py:268-269)
                G.lr_head, G.period, G.head = config.lr_sh_dc, 48, 3
            else:
                G.lr_head, G.period, G.head = lrs[name], 0, 0
        return groups

    @staticmethod
    def _bias(t: int, config: TrainConfig) -> tuple[float, float]:
        if t < 1:
            raise ValueError("Adam iteration must be >= 1")
        beta1, beta2 = config.adam_betas
        return 1.0 - beta1**t, 1.0 - beta2**t

    def step(self, cloud: GaussianCloud, grads: GaussianGrads, iteration: int, config: TrainConfig,
             skip: torch.Tensor | None = None) -> None:
        """One dense Adam step at `iteration` (= the bias-correction t).
        skip (device int32, e.g. from step_guard): applies nothing when set."""
        t = int(iteration)
        bias1, bias2 = self._bias(t, config)
        groups = self._groups(cloud, grads, t, config)
        beta1, beta2 = config.adam_betas
        _lib.check(_lib.load().gs_adam_step_guarded(groups, len(PARAM_GROUPS), beta1, beta2, config.adam_eps, bias1,
                                                    bias2, _lib.ptr(skip), torch.cuda.current_stream().cuda_stream),
                   "adam_step")

    def backward_step(self, cloud: GaussianCloud, camera, splats, grads2d, active_sh_degree: int, iteration: int,
                      config: TrainConfig, stats=None, grads_out: GaussianGrads | None = None,
                      skip: torch.Tensor | None = None, project_next=None):
        """backward_project + densify statistics + Adam fused in one kernel
        (gs_preprocess_backward_adam): parameters are updated in place, the
        raw gradients never round-trip through HBM unless `grads_out` is given.
        `skip` (device int32 from `step_guard`): when set on the device, the
        launch applies nothing.

        project_next = (camera, active_sh_degree): the same launch also
        projects the updated parameters for the next iteration's view
        (gs_preprocess_backward_adam_project) and returns those splats
        (bit-identical to rasterizer.project after this call; pass them to
        render_view_async(..., splats=...)); otherwise returns None."""
        from .rasterizer import DeviceSplats, _camera
        if not 0 <= active_sh_degree <= 3:
            raise ValueError(f"SH degree must be in 0..3, got {active_sh_degree}")
        t = int(iteration)
        bias1, bias2 = self._bias(t, config)
        groups = self._groups(cloud, None, t, config)
        beta1, beta2 = config.adam_betas
        cs = splats.c_struct()
        cst = stats.c_struct() if stats is not None else None
        cg = grads_out.c_struct() if grads_out is not None else None
        common = (ctypes.byref(cloud.c_params()), ctypes.byref(_camera(camera).to_c()), int(active_sh_degree),
                  ctypes.byref(cs), grads2d.packed.data_ptr(), groups, beta1, beta2, config.adam_eps, bias1, bias2,
                  ctypes.byref(cst) if cst is not None else None, ctypes.byref(cg) if cg is not None else None,
                  skip.data_ptr() if skip is not None else None)
        stream = torch.cuda.current_stream().cuda_stream
        if project_next is None:
            _lib.check(_lib.load().gs_preprocess_backward_adam_guarded(*common, stream), "backward_adam")
            return None
        next_camera, next_degree = project_next
        if not 0 <= next_degree <= 3:
            raise ValueError(f"SH degree must be in 0..3, got {next_degree}")
        nxt = DeviceSplats.empty(len(cloud), cloud.device)
        cn = nxt.c_struct()
        _lib.check(_lib.load().gs_preprocess_backward_adam_project(
            *common, ctypes.byref(_camera(next_camera).to_c()), int(next_degree), ctypes.byref(cn), stream),
            "backward_adam_project")
        return nxt


def step_guard(loss: torch.Tensor, k_info: torch.Tensor, out: torch.Tensor | None = None,
               report: torch.Tensor | None = None) -> torch.Tensor:
    """Device int32 flag: 1 when the step must not update anything (loss not
    finite, or the binning overflowed its capacity), written on the current
    stream without a host synchronisation (gs_step_guard).  report: optional
    float64 (8,) pinned host (or device) tensor that receives [loss[0..3],
    k_info[0..2], skip] from the same kernel."""
    if out is None:
        out = torch.empty(1, dtype=torch.int32, device=loss.device)
    if loss.dtype != torch.float32 or k_info.dtype != torch.int64:
        raise TypeError("step_guard expects float32 loss and int64 k_info")
    if report is not None and (report.dtype != torch.float64 or report.numel() < 8):
        raise TypeError("report must be a float64 tensor of 8 elements")
    _lib.check(_lib.load().gs_step_guard(loss.data_ptr(), k_info.data_ptr(), out.data_ptr(), _lib.ptr(report),
                                         torch.cuda.current_stream(loss.device).cuda_stream), "step_guard")
    return out


__all__ = ["TrainConfig", "DeviceAdam", "DensifyStats", "step_guard"]
