"""Host-side logic that needs no GPU: camera validation, config, generators,
argument checking of the stage functions."""
import numpy as np
import pytest

from paper_2308_04079_b200 import synthetic
from paper_2308_04079_b200.camera import Camera, orbit_camera
from paper_2308_04079_b200.optimizer import TrainConfig


def test_camera_validation_matches_reference():
    with pytest.raises(ValueError):
        Camera(np.eye(3) * 1.01, np.zeros(3), 10, 10, 5, 5, 10, 10)
    with pytest.raises(ValueError):
        Camera(np.eye(3), np.zeros(3), -1.0, 10, 5, 5, 10, 10)
    with pytest.raises(ValueError):
        Camera(np.eye(3), np.zeros(3), 10, 10, 5, 5, 10, 10, near=0.0)


def test_camera_center_and_scaled():
    rng = np.random.default_rng(2)
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    r, i, j, k = q
    R = np.array([[1 - 2 * (j * j + k * k), 2 * (i * j - r * k), 2 * (i * k + r * j)],
                  [2 * (i * j + r * k), 1 - 2 * (i * i + k * k), 2 * (j * k - r * i)],
                  [2 * (i * k - r * j), 2 * (j * k + r * i), 1 - 2 * (i * i + j * j)]])
    eye = rng.normal(size=3)
    cam = Camera(R, -R @ eye, 10, 10, 5, 5, 10, 10)
    np.testing.assert_allclose(cam.center, eye, atol=1e-12)
    half = cam.scaled(0.5)
    assert (half.width, half.height, half.fx, half.cx) == (5, 5, 5.0, 2.5)
    c = cam.to_c()
    assert c.width == 10 and abs(c.rotation[1] - R[0, 1]) < 1e-15


def test_orbit_camera_looks_at_origin():
    cam = orbit_camera(0.9, 0.25, 4.0, resolution=256, focal=256.0)
    view = cam.rotation @ np.zeros(3) + cam.translation
    assert abs(view[0]) < 1e-12 and abs(view[1]) < 1e-12 and abs(view[2] - 4.0) < 1e-12


def test_lr_schedule():
    cfg = TrainConfig(total_iters=100)
    assert cfg.lr_means_at(0) == pytest.approx(1.6e-4)
    assert cfg.lr_means_at(100) == pytest.approx(1.6e-6)
    assert cfg.lr_means_at(1000) == pytest.approx(1.6e-6)
    with pytest.raises(ValueError):
        TrainConfig(lambda_dssim=1.5)


def test_frustum_generator_statistics():
    cloud, cam = synthetic.frustum_scene(20000, 1920, 1080, seed=0)
    assert cloud["sh"].shape == (20000, 16, 3)
    z = cloud["means"][:, 2]
    assert z.min() >= 2.0 and z.max() <= 20.0
    u = cam.fx * cloud["means"][:, 0] / z + cam.cx
    assert np.all((u >= 0) & (u <= 1920))


def test_toy_generator_matches_survey_counts():
    from oracle import oracle as O
    cloud, cam = synthetic.toy_scene(10_000, 256)
    proj = O.project(synthetic.round_to_f32(cloud), cam, 3)
    assert int((proj["radius"] > 0).sum()) == 9794      # V = 9,794
    assert int(proj["tiles"].sum()) == 169_420          # K = 169,420


def test_ball_cameras_band():
    cams = synthetic.ball_cameras(32)
    assert len(cams) == 32
    for cam in cams:
        np.testing.assert_allclose(np.linalg.norm(cam.center), 4.0, rtol=1e-12)
