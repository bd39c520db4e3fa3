"""Golden COLMAP dataset + the REFERENCE's ingestion / initialisation outputs
(splatlab scene_io.load_colmap / init_from_sfm / mean_knn_distance,
scene_io.py:251-336), for the §8(f) row 4 parity tests.

Run in the build container, where /root/reference exists:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_colmap_golden.py
Writes tests/golden/colmap_toy/ (a small COLMAP text dataset written by the
reference's own write_toy_dataset), tests/golden/colmap_toy_bin/ (the same
reconstruction as COLMAP binary files, written here with struct) and
tests/golden/colmap_golden.npz.  Nothing at test time reads /root/reference.
"""
from __future__ import annotations

import shutil
import struct
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from splatlab.scene_io import init_from_sfm, load_colmap, mean_knn_distance  # noqa: E402
from splatlab.toydata import write_toy_dataset  # noqa: E402


def main() -> None:
    text_root = HERE / "colmap_toy"
    if text_root.exists():
        shutil.rmtree(text_root)
    write_toy_dataset(text_root, seed=7, n_images=9, resolution=32)
    scene = load_colmap(text_root, load_images=True)

    # the same reconstruction as COLMAP binary files (no images needed: load_images=False)
    bin_sparse = HERE / "colmap_toy_bin" / "sparse" / "0"
    if bin_sparse.parent.parent.exists():
        shutil.rmtree(bin_sparse.parent.parent)
    bin_sparse.mkdir(parents=True)
    txt = text_root / "sparse" / "0"
    cam_lines = [ln.split() for ln in (txt / "cameras.txt").read_text().splitlines() if ln and ln[0] != "#"]
    with open(bin_sparse / "cameras.bin", "wb") as f:
        f.write(struct.pack("<Q", len(cam_lines)))
        for p in cam_lines:
            f.write(struct.pack("<iiQQ", int(p[0]), 1, int(p[2]), int(p[3])))
            f.write(struct.pack("<dddd", *(float(v) for v in p[4:8])))
    img_lines = [ln.split() for ln in (txt / "images.txt").read_text().splitlines() if ln and ln[0] != "#"]
    with open(bin_sparse / "images.bin", "wb") as f:
        f.write(struct.pack("<Q", len(img_lines)))
        for p in img_lines:
            f.write(struct.pack("<idddddddi", int(p[0]), *(float(v) for v in p[1:8]), int(p[8])))
            f.write(p[9].encode() + b"\x00")
            f.write(struct.pack("<Q", 2))
            f.write(struct.pack("<ddq", 1.0, 2.0, -1) * 2)
    pt_lines = [ln.split() for ln in (txt / "points3D.txt").read_text().splitlines() if ln and ln[0] != "#"]
    with open(bin_sparse / "points3D.bin", "wb") as f:
        f.write(struct.pack("<Q", len(pt_lines)))
        for p in pt_lines:
            f.write(struct.pack("<QdddBBBd", int(p[0]), *(float(v) for v in p[1:4]), *(int(v) for v in p[4:7]),
                                float(p[7])))
            f.write(struct.pack("<Q", 1))
            f.write(struct.pack("<ii", 1, 0))

    cloud = init_from_sfm(scene)
    rng = np.random.default_rng(3)
    knn_pts = np.concatenate([rng.normal(size=(3000, 3)),                    # blob
                              rng.uniform(-5, 5, size=(2000, 3)),             # sparse box
                              np.repeat(rng.normal(size=(50, 3)), 2, axis=0)])  # exact duplicates
    np.savez(HERE / "colmap_golden.npz",
             names=np.array([im.name for im in scene.images]),
             R=np.stack([im.camera.rotation for im in scene.images]),
             t=np.stack([im.camera.translation for im in scene.images]),
             intr=np.array([[im.camera.fx, im.camera.fy, im.camera.cx, im.camera.cy, im.camera.width,
                             im.camera.height] for im in scene.images]),
             pixels=np.stack([im.pixels for im in scene.images]),
             points=scene.points, colors=scene.point_colors, extent=scene.scene_extent,
             init_log_scales=cloud.log_scales, init_sh0=cloud.sh[:, 0, :], init_opacity=cloud.opacity_logits,
             knn_points=knn_pts, knn_dist=mean_knn_distance(knn_pts))
    print("images", len(scene.images), "points", len(scene.points))


if __name__ == "__main__":
    main()
