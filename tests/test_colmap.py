"""COLMAP ingestion + initialisation (splatlab scene_io.py:70-366).

Golden data was produced by the reference itself (tests/golden/make_colmap_golden.py):
a COLMAP text dataset written by splatlab's write_toy_dataset, the same
reconstruction in COLMAP binary form, and the reference's load_colmap /
init_from_sfm / mean_knn_distance outputs.
"""
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2308_04079_b200 import colmap as C

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(GOLD / "colmap_golden.npz"))


def check_scene(scene, g, with_pixels):
    assert [im.name for im in scene.images] == list(g["names"])
    for i, im in enumerate(scene.images):
        np.testing.assert_array_equal(im.camera.rotation, g["R"][i])
        np.testing.assert_array_equal(im.camera.translation, g["t"][i])
        c = im.camera
        np.testing.assert_array_equal([c.fx, c.fy, c.cx, c.cy, c.width, c.height], g["intr"][i])
        if with_pixels:
            assert np.abs(im.pixels - g["pixels"][i]).max() < 1e-7   # float32 storage of the float64 decode
    np.testing.assert_array_equal(scene.points, g["points"])
    np.testing.assert_array_equal(scene.point_colors, g["colors"])
    assert scene.scene_extent == float(g["extent"])


def test_load_colmap_text_matches_reference(golden):
    check_scene(C.load_colmap(GOLD / "colmap_toy", load_images=True), golden, True)


def test_load_colmap_binary_matches_reference(golden):
    check_scene(C.load_colmap(GOLD / "colmap_toy_bin", load_images=False), golden, False)


def test_split_every_eighth(golden):
    train, test = C.split_train_test(C.load_colmap(GOLD / "colmap_toy", load_images=False))
    assert [im.name for im in test] == [golden["names"][0], golden["names"][8]]
    assert len(train) == 7


def write_minimal(root, camera_line, points_lines, n_images=2):
    sparse = root / "sparse" / "0"
    sparse.mkdir(parents=True)
    (sparse / "cameras.txt").write_text(camera_line + "\n")
    lines = []
    for i in range(n_images):
        lines += [f"{i + 1} 1 0 0 0 0 0 4 1 img_{i:02d}.png", ""]
    (sparse / "images.txt").write_text("\n".join(lines) + "\n")
    (sparse / "points3D.txt").write_text("\n".join(points_lines) + "\n")


def test_intrinsics_and_errors(tmp_path):
    write_minimal(tmp_path / "a", "1 SIMPLE_PINHOLE 640 480 500 320 240", ["1 0.5 1.0 2.0 255 0 0 0.5"])
    s = C.load_colmap(tmp_path / "a", load_images=False)
    cam = s.images[0].camera
    assert (cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height) == (500, 500, 320, 240, 640, 480)
    np.testing.assert_allclose(s.point_colors, [[1.0, 0.0, 0.0]])
    write_minimal(tmp_path / "b", "1 OPENCV 640 480 500 500 320 240 0 0 0 0", [])
    with pytest.raises(C.SceneLoadError, match="OPENCV"):
        C.load_colmap(tmp_path / "b", load_images=False)
    with pytest.raises(C.SceneLoadError, match="does not exist"):
        C.load_colmap(tmp_path / "nope", load_images=False)
    (tmp_path / "c").mkdir()
    with pytest.raises(C.SceneLoadError, match="no COLMAP cameras"):
        C.load_colmap(tmp_path / "c", load_images=False)
    write_minimal(tmp_path / "d", "2 PINHOLE 64 64 50 50 32 32", [])
    with pytest.raises(C.SceneLoadError, match="unknown camera"):
        C.load_colmap(tmp_path / "d", load_images=False)
    with pytest.raises(C.SceneLoadError, match="image file missing"):
        C.load_colmap(tmp_path / "a", load_images=True)
    sparse = tmp_path / "e" / "sparse" / "0"
    sparse.mkdir(parents=True)
    (sparse / "cameras.bin").write_bytes(struct.pack("<Q", 1) + struct.pack("<iiQ", 1, 1, 64))
    with pytest.raises(C.SceneLoadError, match="unexpected end"):
        C.load_colmap(tmp_path / "e", load_images=False)


def test_srgb_roundtrip():
    x = np.linspace(0, 1, 101)
    np.testing.assert_allclose(C.srgb_to_linear(C.linear_to_srgb(x)), x, atol=1e-12)


@pytest.mark.gpu
def test_device_knn_matches_reference(cuda_device, golden):
    d = C.mean_knn_distance(golden["knn_points"], 3).cpu().numpy()
    ref = golden["knn_dist"]
    assert np.abs(d - ref).max() <= 1e-6 * np.abs(ref).max()
    dup = slice(5000, 5100)   # exact duplicate pairs: the nearest other point is at distance 0
    np.testing.assert_allclose(d[dup], ref[dup], rtol=1e-6, atol=0)


@pytest.mark.gpu
def test_init_from_sfm_matches_reference(cuda_device, golden):
    scene = C.load_colmap(GOLD / "colmap_toy", load_images=False)
    cloud = C.init_from_sfm(scene)
    np.testing.assert_allclose(cloud.log_scales.cpu().numpy(), golden["init_log_scales"], atol=2e-6)
    np.testing.assert_allclose(cloud.sh[:, 0, :].cpu().numpy(), golden["init_sh0"], atol=2e-6)
    np.testing.assert_allclose(cloud.opacity_logits.cpu().numpy(), golden["init_opacity"], atol=1e-6)
    np.testing.assert_array_equal(cloud.rotations.cpu().numpy()[:, 0], 1.0)


@pytest.mark.gpu
def test_device_knn_exact_at_scale(cuda_device):
    import torch
    rng = np.random.default_rng(9)
    # a surface-like cloud (the SfM case) plus uniform clutter, 1M points
    u, v = rng.uniform(0, 2 * np.pi, 800_000), rng.uniform(0, np.pi, 800_000)
    sphere = np.stack([np.cos(u) * np.sin(v), np.sin(u) * np.sin(v), np.cos(v)], 1) * 3.0
    pts = np.concatenate([sphere, rng.uniform(-4, 4, (200_000, 3))])
    d = C.mean_knn_distance(pts, 3)
    q = torch.from_numpy(rng.choice(len(pts), 2000, replace=False)).cuda()
    P = torch.from_numpy(pts).cuda()
    dd = torch.cdist(P[q], P)                                # brute force for 2000 queries (float64)
    dd[torch.arange(2000, device="cuda"), q] = float("inf")  # drop the self match
    ref = dd.topk(3, largest=False).values.mean(1)
    torch.testing.assert_close(d[q].double(), ref, rtol=1e-6, atol=0)


@pytest.mark.gpu
def test_train_from_colmap_dataset(cuda_device):
    """COLMAP dataset -> device init_from_sfm -> train_step on host-resident views."""
    from paper_2308_04079_b200.densify import TrainState
    from paper_2308_04079_b200.optimizer import TrainConfig
    from paper_2308_04079_b200.training import train, views_from_scene
    scene = C.load_colmap(GOLD / "colmap_toy", load_images=True)
    train_imgs, _ = C.split_train_test(scene)
    views = views_from_scene(train_imgs)
    state = TrainState(C.init_from_sfm(scene), scene.scene_extent, seed=0)
    cfg = TrainConfig(total_iters=300, densify_start=100, densify_interval=50)
    losses = []
    train(state, views, cfg, iterations=300, eval_interval=100, progress=losses.append)
    first, last = float(losses[0].split("loss=")[1].split()[0]), float(losses[-1].split("loss=")[1].split()[0])
    assert np.isfinite(last) and last < first
