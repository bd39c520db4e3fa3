"""Definitions of the golden scenes (shared by tests/golden/make_golden.py and
the parity tests).  Each builder returns the float32-rounded float64 inputs,
the camera, SH degree, background, the d_image seed and the storage mode."""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

from paper_2308_04079_b200 import synthetic
from paper_2308_04079_b200.camera import Camera

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def _scene_a():
    cloud, cam = synthetic.random_splat_scene(np.random.default_rng(7), 120, 64, 64)
    return cloud, cam, 3, (0.1, 0.2, 0.3), 11, False


def _scene_b():
    cloud, cam = synthetic.random_splat_scene(np.random.default_rng(8), 400, 96, 64)
    return cloud, cam, 2, (0.0, 0.0, 0.0), 12, False


def _scene_c():
    # partial edge tiles in both dimensions; culled Gaussians (behind the
    # camera, outside the guard band) mixed in
    cloud, cam = synthetic.random_splat_scene(np.random.default_rng(9), 1500, 200, 136)
    cloud["means"][:40, 2] *= -1.0
    cloud["means"][40:80, 0] *= 4.0
    return cloud, cam, 3, (1.0, 1.0, 1.0), 13, True


def _scene_frustum():
    cloud, cam = synthetic.frustum_scene(3000, 160, 90, seed=0)
    return cloud, cam, 3, (0.0, 0.0, 0.0), 14, True


def _toy_c1():
    cloud, cam = synthetic.toy_scene(10_000, 256)
    return cloud, cam, 3, (0.0, 0.0, 0.0), 1, True


SCENES = {"scene_a": _scene_a, "scene_b": _scene_b, "scene_c": _scene_c, "scene_frustum": _scene_frustum,
          "toy_c1": _toy_c1}


def input_digest(cloud: dict) -> str:
    h = hashlib.sha256()
    for k in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        h.update(np.ascontiguousarray(cloud[k], dtype=np.float32).tobytes())
    return h.hexdigest()


def build(name: str):
    cloud, cam, degree, bg, seed, compact = SCENES[name]()
    return synthetic.round_to_f32(cloud), cam, degree, bg, seed, compact


def d_image_for(seed: int, width: int, height: int) -> np.ndarray:
    """The incoming image gradient of a golden scene (float32 values)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(-1.0, 1.0, (height, width, 3)) / (height * width * 3)
    return d.astype(np.float32).astype(np.float64)


def load(name: str) -> tuple[dict, dict, Camera]:
    """(golden arrays, float64 inputs, camera) for a golden scene."""
    g = dict(np.load(GOLDEN_DIR / f"{name}.npz"))
    cloud, cam, degree, bg, seed, compact = build(name)
    assert str(g["input_sha256"]) == input_digest(cloud), f"{name}: generator drifted from the golden inputs"
    return g, cloud, cam
