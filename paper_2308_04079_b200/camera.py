"""Pinhole camera with the reference's conventions and validation.

Mirrors splatlab `Camera` (core.py:113-155): world-to-view rotation and
translation, intrinsics, resolution and near plane; view space is x-right,
y-down, z-forward and pixel centres sit at (col+0.5, row+0.5).  The
constructor raises ValueError for the same invalid inputs (core.py:132-141).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class Camera:
    rotation: np.ndarray       # (3, 3) world-to-view rotation
    translation: np.ndarray    # (3,) world-to-view translation
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.2

    def __post_init__(self):
        R = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        object.__setattr__(self, "rotation", R)
        object.__setattr__(self, "translation", t)
        deviation = float(np.abs(R @ R.T - np.eye(3)).max())
        if deviation > 1e-6:
            raise ValueError(f"camera rotation is not orthonormal (max deviation {deviation:.3g})")
        if min(self.fx, self.fy) <= 0 or min(self.width, self.height) <= 0:
            raise ValueError("camera focal lengths and resolution must be positive")
        if self.near <= 0:
            raise ValueError("camera near plane must be positive")

    @classmethod
    def from_reference(cls, cam) -> "Camera":
        """Adopt any object with the reference Camera's attributes."""
        return cls(cam.rotation, cam.translation, float(cam.fx), float(cam.fy), float(cam.cx),
                   float(cam.cy), int(cam.width), int(cam.height), float(cam.near))

    @property
    def center(self) -> np.ndarray:
        return -(self.rotation.T @ self.translation)

    @property
    def tiles(self) -> tuple[int, int]:
        return (self.width + 15) // 16, (self.height + 15) // 16

    def scaled(self, factor: float) -> "Camera":
        """Same pose at a resolution rescaled by `factor` (core.py:148-155)."""
        return Camera(self.rotation, self.translation, self.fx * factor, self.fy * factor,
                      self.cx * factor, self.cy * factor, max(1, int(round(self.width * factor))),
                      max(1, int(round(self.height * factor))), self.near)

    def to_c(self) -> _lib.GsCamera:
        c = _lib.GsCamera()
        c.rotation[:] = [float(v) for v in self.rotation.reshape(-1)]
        c.translation[:] = [float(v) for v in self.translation]
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.near_plane = float(self.near)
        return c


def look_at(eye, target=(0.0, 0.0, 0.0), *, width: int, height: int, fx: float, fy: float | None = None,
            cx: float | None = None, cy: float | None = None, near: float = 0.2,
            up=(0.0, 0.0, 1.0)) -> Camera:
    """Camera at `eye` looking at `target` with rows (right, down, forward),
    the construction of toydata.orbit_camera (toydata.py:60-68)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    return Camera(R, -R @ eye, fx, fx if fy is None else fy, width / 2.0 if cx is None else cx,
                  height / 2.0 if cy is None else cy, width, height, near)


def orbit_camera(azimuth: float, elevation: float, distance: float, resolution: int = 128,
                 focal: float = 128.0, target=(0.0, 0.0, 0.0), near: float = 0.2) -> Camera:
    """Orbit camera around `target` (toydata.py:50-68)."""
    target = np.asarray(target, dtype=np.float64)
    ce = np.cos(elevation)
    eye = target + distance * np.array([ce * np.cos(azimuth), ce * np.sin(azimuth), np.sin(elevation)])
    return look_at(eye, target, width=resolution, height=resolution, fx=focal, near=near)
