"""Device-resident Gaussian parameters in the reference layout.

Mirrors splatlab `GaussianCloud` (core.py:36-110): raw means (N,3),
quaternions (N,4) (r,i,j,k), log scales (N,3), opacity logits (N,) and SH
coefficients (N,16,3), here as contiguous float32 CUDA tensors.  The
activations (exp, sigmoid, normalisation) happen inside the rasterizer.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

PARAM_GROUPS = ("means", "log_scales", "rotations", "opacity_logits", "sh")  # optimizer.py:85
_SHAPES = {"means": (3,), "rotations": (4,), "log_scales": (3,), "opacity_logits": (), "sh": (16, 3)}


@dataclass
class GaussianCloud:
    means: torch.Tensor
    rotations: torch.Tensor
    log_scales: torch.Tensor
    opacity_logits: torch.Tensor
    sh: torch.Tensor

    def __post_init__(self):
        n = self.means.shape[0]
        for name, shape in _SHAPES.items():
            t = getattr(self, name)
            if tuple(t.shape) != (n, *shape):
                raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {(n, *shape)}")
            if t.dtype != torch.float32:
                raise ValueError(f"{name} must be float32")

    def __len__(self) -> int:
        return self.means.shape[0]

    @property
    def device(self) -> torch.device:
        return self.means.device

    @classmethod
    def from_numpy(cls, means, rotations, log_scales, opacity_logits, sh, device="cuda") -> "GaussianCloud":
        def t(a, shape):
            arr = np.ascontiguousarray(np.asarray(a, dtype=np.float32)).reshape(shape)
            return torch.from_numpy(arr).to(device)
        n = np.asarray(means).reshape(-1, 3).shape[0]
        return cls(t(means, (n, 3)), t(rotations, (n, 4)), t(log_scales, (n, 3)),
                   t(opacity_logits, (n,)), t(sh, (n, 16, 3)))

    @classmethod
    def from_reference(cls, cloud, device="cuda") -> "GaussianCloud":
        """Adopt any object with the reference GaussianCloud's arrays."""
        return cls.from_numpy(cloud.means, cloud.rotations, cloud.log_scales, cloud.opacity_logits,
                              cloud.sh, device=device)

    def numpy(self) -> dict:
        return {k: getattr(self, k).detach().cpu().numpy() for k in PARAM_GROUPS}

    def params(self) -> list[torch.Tensor]:
        return [getattr(self, k) for k in PARAM_GROUPS]

    def c_params(self) -> _lib.GsParams:
        p = _lib.GsParams()
        for name in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
            t = getattr(self, name)
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            setattr(p, name, t.data_ptr())
        p.n = len(self)
        return p


def c_params_from(means, log_scales, rotations, opacity_logits, sh) -> _lib.GsParams:
    p = _lib.GsParams()
    p.means, p.rotations, p.log_scales = means.data_ptr(), rotations.data_ptr(), log_scales.data_ptr()
    p.opacity_logits, p.sh = opacity_logits.data_ptr(), sh.data_ptr()
    p.n = means.shape[0]
    return p
