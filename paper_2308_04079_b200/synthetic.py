"""Seeded synthetic scenes for the benchmark configurations.

Host-side numpy generators (float64, the reference's parameter layout);
they produce identical arrays for the reference, the oracle and the device.
  frustum_scene   c2/c3/c5: adapts random_splat_scene (tests/helpers.py:98-114)
  random_splat_scene  the reference test helper's generator (helpers.py:98-114)
  toy_scene       c1: init_random (scene_io.py:339-366) + appearance draws,
                  orbit camera (toydata.py:50-68)
  ball_scene      c4: ball cloud + golden-angle camera band (toydata.py:71-90)
"""
from __future__ import annotations

import numpy as np

from .camera import Camera, orbit_camera


def _cloud(means, rotations, log_scales, opacity_logits, sh) -> dict:
    n = means.shape[0]
    return {"means": np.ascontiguousarray(means, dtype=np.float64).reshape(n, 3),
            "rotations": np.ascontiguousarray(rotations, dtype=np.float64).reshape(n, 4),
            "log_scales": np.ascontiguousarray(log_scales, dtype=np.float64).reshape(n, 3),
            "opacity_logits": np.ascontiguousarray(opacity_logits, dtype=np.float64).reshape(n),
            "sh": np.ascontiguousarray(sh, dtype=np.float64).reshape(n, 16, 3)}


def round_to_f32(cloud: dict) -> dict:
    """The float32-representable copy every implementation is fed."""
    return {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in cloud.items()}


def frustum_scene(n: int, width: int, height: int, seed: int = 0) -> tuple[dict, Camera]:
    """§8(d) frustum generator: one default_rng(seed) stream, draws in order
    x, y, depth, q, scale, opacity, sh; identity camera with fx = fy = W."""
    rng = np.random.default_rng(seed)
    means = np.empty((n, 3))
    means[:, 0] = rng.uniform(-0.45, 0.45, n)
    means[:, 1] = rng.uniform(-0.45, 0.45, n) * (height / width)
    means[:, 2] = 1.0
    depth = rng.uniform(2.0, 20.0, n)
    means *= depth[:, None]
    q = rng.normal(size=(n, 4))
    log_scales = np.log(rng.uniform(0.0005, 0.004, (n, 3)) * depth[:, None])
    opacity = rng.uniform(-2.0, 2.5, n)
    sh = rng.normal(scale=0.35, size=(n, 16, 3))
    cam = Camera(np.eye(3), np.zeros(3), float(width), float(width), width / 2.0, height / 2.0, width, height,
                 near=0.1)
    return _cloud(means, q, log_scales, opacity, sh), cam


def random_splat_scene(rng, count: int, width: int, height: int, depth_range=(2.0, 20.0)) -> tuple[dict, Camera]:
    """Same draws as the reference test helper random_splat_scene."""
    means = np.zeros((count, 3))
    means[:, 0] = rng.uniform(-0.45, 0.45, count)
    means[:, 1] = rng.uniform(-0.45, 0.45, count)
    means[:, 2] = 1.0
    depths = rng.uniform(*depth_range, count)
    means *= depths[:, None]
    q = rng.normal(size=(count, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    log_scales = np.log(rng.uniform(0.02, 0.3, (count, 3)) * depths[:, None] / 10.0)
    opacity_logits = rng.uniform(-2.0, 2.5, count)
    sh = rng.normal(scale=0.35, size=(count, 16, 3))
    cam = Camera(np.eye(3), np.zeros(3), float(width), float(height), width / 2.0, height / 2.0, width, height,
                 near=0.1)
    return _cloud(means, q, log_scales, opacity_logits, sh), cam


def _mean_knn_distance(points: np.ndarray, k: int = 3) -> np.ndarray:
    from scipy.spatial import cKDTree
    dist, _ = cKDTree(points).query(points, k=k + 1)
    return dist[:, 1:].mean(axis=1)


def toy_scene(n: int = 10_000, resolution: int = 256) -> tuple[dict, Camera]:
    """c1: uniform points in (-1.8, 1.8)^3 from default_rng(42), isotropic
    kNN scales (init_random), then SH/rotation/opacity from default_rng(43)."""
    rng = np.random.default_rng(42)
    lo, hi = np.full(3, -1.8), np.full(3, 1.8)
    points = rng.uniform(lo, hi, size=(n, 3))
    dist = np.maximum(_mean_knn_distance(points), 1e-7)
    log_scales = np.repeat(np.log(dist)[:, None], 3, axis=1)
    rng2 = np.random.default_rng(43)
    sh = rng2.normal(scale=0.35, size=(n, 16, 3))
    rotations = rng2.normal(size=(n, 4))
    opacity = rng2.uniform(-2.0, 2.5, n)
    cam = orbit_camera(0.9, 0.25, 4.0, resolution=resolution, focal=float(resolution))
    return _cloud(points, rotations, log_scales, opacity, sh), cam


# --------------------------------------------------------------------------
# the reference's procedural toy problem (toydata.py), used by the
# toy-recovery acceptance run (test_acceptance.py:104-116)

TOY_COLORS = np.array([[0.85, 0.15, 0.10], [0.10, 0.75, 0.20], [0.15, 0.25, 0.90], [0.90, 0.80, 0.10],
                       [0.80, 0.15, 0.80], [0.10, 0.80, 0.80], [0.95, 0.55, 0.15], [0.60, 0.60, 0.60]])
SH_C0 = 0.28209479177387814


def make_toy_cloud(seed: int = 7, count: int = 8) -> dict:
    """Well-separated isotropic coloured blobs on a jittered sphere (toydata.py:26-47)."""
    rng = np.random.default_rng(seed)
    phi = np.linspace(0.0, 2.0 * np.pi, count, endpoint=False)
    zs = np.linspace(-0.7, 0.7, count)
    ring = np.sqrt(1 - zs**2)
    means = np.stack([1.1 * np.cos(phi) * ring, 1.1 * np.sin(phi) * ring, 1.1 * zs], axis=1)
    means = means + rng.normal(scale=0.08, size=means.shape)
    q = np.zeros((count, 4))
    q[:, 0] = 1.0
    sigma = rng.uniform(0.25, 0.35, size=(count, 1))
    alphas = rng.uniform(0.65, 0.9, size=count)
    sh = np.zeros((count, 16, 3))
    sh[:, 0, :] = (TOY_COLORS[:count] - 0.5) / SH_C0
    return _cloud(means, q, np.log(np.repeat(sigma, 3, axis=1)), np.log(alphas / (1 - alphas)), sh)


def make_toy_cameras(n_train: int = 24, n_test: int = 3, distance: float = 4.0, resolution: int = 128,
                     focal: float | None = None) -> tuple[list[Camera], list[Camera]]:
    """Golden-angle training band plus held-out in-betweens (toydata.py:71-90)."""
    if focal is None:
        focal = resolution * distance / 4.0
    golden = np.pi * (3.0 - np.sqrt(5.0))
    train = [orbit_camera(i * golden, np.arcsin(-0.75 + 1.5 * (i + 0.5) / n_train), distance, resolution, focal)
             for i in range(n_train)]
    test = [orbit_camera((i + 0.5) * golden, np.arcsin(-0.5 + 1.0 * (i + 0.5) / max(n_test, 1)), distance,
                         resolution, focal) for i in range(n_test)]
    return train, test


def compute_scene_extent(cameras) -> float:
    """Bounding-sphere radius of the camera centres (scene_io.py:236-248)."""
    if cameras:
        centers = np.stack([c.center for c in cameras])
        extent = float(np.linalg.norm(centers - centers.mean(axis=0), axis=1).max())
        if extent > 0:
            return extent
    return 1.0


def init_random(count: int, bounds, rng) -> dict:
    """Uniform points with isotropic kNN scales, opacity 0.1, zero SH (scene_io.py:339-366)."""
    lo, hi = (np.asarray(b, dtype=np.float64) for b in bounds)
    points = rng.uniform(lo, hi, size=(count, 3))
    dist = (np.maximum(_mean_knn_distance(points), 1e-7) if count >= 4
            else np.full(count, np.linalg.norm(hi - lo) / 10.0))
    q = np.zeros((count, 4))
    q[:, 0] = 1.0
    return _cloud(points, q, np.repeat(np.log(dist)[:, None], 3, axis=1), np.full(count, np.log(0.1 / 0.9)),
                  np.zeros((count, 16, 3)))


def ball_cameras(count: int = 32, width: int = 1920, height: int = 1080, distance: float = 4.0) -> list[Camera]:
    """Golden-angle band of look-at cameras (toydata.py:79-83) at 1080p."""
    from .camera import look_at
    golden = np.pi * (3.0 - np.sqrt(5.0))
    cams = []
    for i in range(count):
        elev = np.arcsin(-0.75 + 1.5 * (i + 0.5) / count)
        az = i * golden
        ce = np.cos(elev)
        eye = distance * np.array([ce * np.cos(az), ce * np.sin(az), np.sin(elev)])
        cams.append(look_at(eye, (0.0, 0.0, 0.0), width=width, height=height, fx=float(width), near=0.2))
    return cams


def ball_scene(n: int, seed: int = 0) -> dict:
    """c4: directions uniform on S^2, radius 1.5 U^(1/3), then q, scales,
    opacity, sh from the same default_rng(seed) stream."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = 1.5 * rng.uniform(0.0, 1.0, n) ** (1.0 / 3.0)
    means = d * r[:, None]
    q = rng.normal(size=(n, 4))
    log_scales = np.log(rng.uniform(0.002, 0.016, (n, 3)))
    opacity = rng.uniform(-2.0, 2.5, n)
    sh = rng.normal(scale=0.35, size=(n, 16, 3))
    return _cloud(means, q, log_scales, opacity, sh)
