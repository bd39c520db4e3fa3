"""COLMAP ingestion and scene initialisation into device tensors.

Mirrors splatlab scene_io's dataset side with the same names, conventions
and errors:

  load_colmap          scene_io.py:251-289   cameras / images / points3D, text or
                                             binary, under root or root/sparse[/0]
  split_train_test     scene_io.py:292-301   every 8th image by sorted name held out
  compute_scene_extent scene_io.py:236-248
  mean_knn_distance    scene_io.py:304-311   exact k-NN mean distance -> the device
                                             grid search gs_knn_mean_distance
  init_from_sfm        scene_io.py:314-336   one isotropic Gaussian per SfM point
  init_random          scene_io.py:339-366   (with the device k-NN)
  load_image, srgb_to_linear, linear_to_srgb scene_io.py:70-94

The parsers are host code (they read small text / binary files); images are
decoded on the host and kept as float32 linear RGB, moved to the device on
demand (TrainView accepts host images and prefetches them per step); the
per-point initialisation runs on the device.
"""
from __future__ import annotations

import ctypes
import struct
import warnings
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .camera import Camera
from .cloud import GaussianCloud

SUPPORTED_CAMERA_MODELS = ("SIMPLE_PINHOLE", "PINHOLE")
# COLMAP camera model id -> (name, number of parameters)
CAMERA_MODELS = {0: ("SIMPLE_PINHOLE", 3), 1: ("PINHOLE", 4), 2: ("SIMPLE_RADIAL", 4), 3: ("RADIAL", 5),
                 4: ("OPENCV", 8), 5: ("OPENCV_FISHEYE", 8), 6: ("FULL_OPENCV", 12), 7: ("FOV", 5),
                 8: ("SIMPLE_RADIAL_FISHEYE", 4), 9: ("RADIAL_FISHEYE", 5), 10: ("THIN_PRISM_FISHEYE", 12)}
INIT_OPACITY = 0.1
SH_C0 = 0.28209479177387814


class SceneLoadError(RuntimeError):
    """Raised for missing or malformed datasets (scene_io.py:35-36)."""


@dataclass
class SceneImage:
    name: str
    camera: Camera
    path: Path | None = None
    pixels: np.ndarray | None = None   # (H, W, 3) float32 linear RGB

    def load_pixels(self) -> np.ndarray:
        if self.pixels is None:
            if self.path is None or not self.path.exists():
                raise SceneLoadError(f"image file missing for '{self.name}'")
            self.pixels = load_image(self.path)
        return self.pixels


@dataclass
class SfmScene:
    images: list
    points: np.ndarray         # (P, 3) float64
    point_colors: np.ndarray   # (P, 3) linear [0, 1]
    scene_extent: float

    @property
    def cameras(self) -> list:
        return [im.camera for im in self.images]


# ---------------------------------------------------------------------------
# images

def srgb_to_linear(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return np.where(x <= 0.04045, x / 12.92, np.power((x + 0.055) / 1.055, 2.4))


def linear_to_srgb(x) -> np.ndarray:
    x = np.clip(np.asarray(x, dtype=np.float64), 0.0, 1.0)
    return np.where(x <= 0.0031308, 12.92 * x, 1.055 * np.power(x, 1.0 / 2.4) - 0.055)


def load_image(path) -> np.ndarray:
    """8-bit PNG/JPEG -> float32 linear RGB (scene_io.py:80-84)."""
    from PIL import Image
    with Image.open(path) as im:
        rgb = np.asarray(im.convert("RGB"), dtype=np.float64) / 255.0
    return srgb_to_linear(rgb).astype(np.float32)


# ---------------------------------------------------------------------------
# COLMAP files

def _intrinsics(model: str, width: int, height: int, params) -> dict:
    if model == "SIMPLE_PINHOLE":
        return dict(fx=params[0], fy=params[0], cx=params[1], cy=params[2], width=width, height=height)
    if model == "PINHOLE":
        return dict(fx=params[0], fy=params[1], cx=params[2], cy=params[3], width=width, height=height)
    raise SceneLoadError(f"unsupported COLMAP camera model '{model}'; only {SUPPORTED_CAMERA_MODELS} work "
                         "(undistort images first)")


def _data_lines(path: Path):
    for raw in path.read_text().splitlines():
        line = raw.strip()
        if line and not line.startswith("#"):
            yield line


class _Reader:
    """Little-endian reader over a COLMAP .bin file with the reference's EOF error."""

    def __init__(self, path: Path):
        self.buf = memoryview(path.read_bytes())
        self.pos = 0

    def take(self, fmt: str):
        size = struct.calcsize("<" + fmt)
        if self.pos + size > len(self.buf):
            raise SceneLoadError("unexpected end of COLMAP binary file")
        out = struct.unpack_from("<" + fmt, self.buf, self.pos)
        self.pos += size
        return out

    def skip(self, nbytes: int) -> None:
        self.pos += nbytes

    def cstring(self) -> str:
        end = self.pos
        while end < len(self.buf) and self.buf[end] != 0:
            end += 1
        name = bytes(self.buf[self.pos:end]).decode("utf-8")
        self.pos = min(end + 1, len(self.buf))
        return name


def read_cameras_text(path) -> dict:
    cams = {}
    for line in _data_lines(Path(path)):
        f = line.split()
        cams[int(f[0])] = _intrinsics(f[1], int(f[2]), int(f[3]), [float(v) for v in f[4:]])
    return cams


def read_cameras_binary(path) -> dict:
    r = _Reader(Path(path))
    cams = {}
    for _ in range(r.take("Q")[0]):
        cam_id, model_id, width, height = r.take("iiQQ")
        if model_id not in CAMERA_MODELS:
            raise SceneLoadError(f"unknown COLMAP camera model id {model_id}")
        name, nparams = CAMERA_MODELS[model_id]
        cams[cam_id] = _intrinsics(name, width, height, r.take("d" * nparams))
    return cams


def qvec_to_rotation(qvec) -> np.ndarray:
    """COLMAP (w, x, y, z) world-to-camera quaternion -> rotation matrix."""
    w, x, y, z = (float(v) for v in qvec)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def read_images_text(path) -> list:
    # pose line + (possibly empty) 2D-point line per image: keep blank lines
    # after the header so the pairing survives an image with no points
    lines = [ln.strip() for ln in Path(path).read_text().splitlines()]
    lines = [ln for ln in lines if not ln.startswith("#")]
    while lines and not lines[0]:
        lines.pop(0)
    metas = []
    for pose in lines[0::2]:
        if not pose:
            continue
        f = pose.split()
        metas.append(dict(qvec=[float(v) for v in f[1:5]], tvec=np.array([float(v) for v in f[5:8]]),
                          camera_id=int(f[8]), name=f[9]))
    return metas


def read_images_binary(path) -> list:
    r = _Reader(Path(path))
    metas = []
    for _ in range(r.take("Q")[0]):
        rec = r.take("idddddddi")
        name = r.cstring()
        npts = r.take("Q")[0]
        r.skip(24 * npts)   # (x, y, point3D_id) per observation
        metas.append(dict(qvec=list(rec[1:5]), tvec=np.array(rec[5:8]), camera_id=rec[8], name=name))
    return metas


def read_points3d_text(path):
    xyz, rgb = [], []
    for line in _data_lines(Path(path)):
        f = line.split()
        xyz.append([float(v) for v in f[1:4]])
        rgb.append([int(v) for v in f[4:7]])
    if not xyz:
        return np.zeros((0, 3)), np.zeros((0, 3))
    return np.asarray(xyz, dtype=np.float64), np.asarray(rgb, dtype=np.float64) / 255.0


def read_points3d_binary(path):
    r = _Reader(Path(path))
    xyz, rgb = [], []
    for _ in range(r.take("Q")[0]):
        rec = r.take("QdddBBBd")
        xyz.append(rec[1:4])
        rgb.append(rec[4:7])
        r.skip(8 * r.take("Q")[0])   # track: (image_id, point2D_idx) pairs
    if not xyz:
        return np.zeros((0, 3)), np.zeros((0, 3))
    return np.asarray(xyz, dtype=np.float64), np.asarray(rgb, dtype=np.float64) / 255.0


def _sparse_dir(root: Path) -> Path:
    for cand in (root, root / "sparse" / "0", root / "sparse"):
        if (cand / "cameras.txt").exists() or (cand / "cameras.bin").exists():
            return cand
    raise SceneLoadError(f"no COLMAP cameras file under '{root}'")


def camera_bounds(cameras) -> tuple[np.ndarray, np.ndarray]:
    centers = np.stack([c.center for c in cameras])
    return centers.min(axis=0), centers.max(axis=0)


def compute_scene_extent(cameras, points=None) -> float:
    """Radius of the camera centres' bounding sphere, else of the point cloud, else 1."""
    if cameras:
        c = np.stack([cam.center for cam in cameras])
        ext = float(np.linalg.norm(c - c.mean(axis=0), axis=1).max())
        if ext > 0:
            return ext
    if points is not None and len(points):
        ext = float(np.linalg.norm(points - points.mean(axis=0), axis=1).max())
        if ext > 0:
            return ext
    return 1.0


def load_colmap(path, load_images: bool = True, near: float = 0.2) -> SfmScene:
    root = Path(path)
    if not root.exists():
        raise SceneLoadError(f"dataset directory '{root}' does not exist")
    sparse = _sparse_dir(root)

    def pick(stem, text_reader, binary_reader):
        for suffix, reader in ((".txt", text_reader), (".bin", binary_reader)):
            f = sparse / f"{stem}{suffix}"
            if f.exists():
                return reader(f)
        raise SceneLoadError(f"missing {stem} file in '{sparse}'")

    intrinsics = pick("cameras", read_cameras_text, read_cameras_binary)
    metas = pick("images", read_images_text, read_images_binary)
    points, colors = pick("points3D", read_points3d_text, read_points3d_binary)
    images = []
    for meta in sorted(metas, key=lambda m: m["name"]):
        if meta["camera_id"] not in intrinsics:
            raise SceneLoadError(f"image '{meta['name']}' references unknown camera {meta['camera_id']}")
        cam = Camera(qvec_to_rotation(meta["qvec"]), meta["tvec"], near=near, **intrinsics[meta["camera_id"]])
        img = SceneImage(meta["name"], cam, root / "images" / meta["name"])
        if load_images:
            img.load_pixels()
        images.append(img)
    return SfmScene(images, points, colors, compute_scene_extent([im.camera for im in images], points))


def split_train_test(scene: SfmScene):
    """(train, test): every 8th image by sorted name is held out."""
    ordered = sorted(scene.images, key=lambda im: im.name)
    return ([im for i, im in enumerate(ordered) if i % 8], [im for i, im in enumerate(ordered) if i % 8 == 0])


# ---------------------------------------------------------------------------
# initialisation on the device

def mean_knn_distance(points, k: int = 3, device="cuda") -> torch.Tensor:
    """Mean distance of every point to its k nearest OTHER points (exact), on
    the device: (P,) float32.  Points are taken in float64 like the reference."""
    pts = torch.as_tensor(np.asarray(points, dtype=np.float64) if not torch.is_tensor(points) else points,
                          dtype=torch.float64, device=device).contiguous()
    n = int(pts.shape[0])
    out = torch.empty(n, dtype=torch.float32, device=device)
    if n == 0:
        return out
    max_cells = max(64, 2 * n)
    lib = _lib.load()
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gs_knn_workspace_size(n, max_cells, ctypes.byref(nbytes)), "knn")
    ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=device)
    _lib.check(lib.gs_knn_mean_distance(pts.data_ptr(), n, int(k), max_cells, ws.data_ptr(), nbytes.value,
                                        out.data_ptr(), torch.cuda.current_stream(device).cuda_stream), "knn")
    return out


def _isotropic_cloud(points, dist: torch.Tensor, sh0, device) -> GaussianCloud:
    n = int(points.shape[0])
    means = torch.as_tensor(points, dtype=torch.float32, device=device)
    rot = torch.zeros((n, 4), dtype=torch.float32, device=device)
    rot[:, 0] = 1.0
    log_s = torch.log(torch.clamp(dist.to(torch.float64), min=1e-7)).to(torch.float32)[:, None].repeat(1, 3)
    opac = torch.full((n,), float(np.log(INIT_OPACITY / (1.0 - INIT_OPACITY))), dtype=torch.float32, device=device)
    sh = torch.zeros((n, 16, 3), dtype=torch.float32, device=device)
    if sh0 is not None:
        sh[:, 0, :] = torch.as_tensor(np.asarray(sh0), dtype=torch.float32, device=device)
    return GaussianCloud(means.contiguous(), rot, log_s.contiguous(), opac, sh)


def init_random(count: int, *, bounds=None, scene: SfmScene | None = None, rng=None, device="cuda") -> GaussianCloud:
    """Uniform random Gaussians inside `bounds` or 3x the camera box (scene_io.py:339-366)."""
    rng = np.random.default_rng(0) if rng is None else rng
    if count == 0:
        return _isotropic_cloud(np.zeros((0, 3)), torch.zeros(0, device=device), None, device)
    if bounds is None:
        if scene is None or not scene.images:
            raise ValueError("random init needs bounds or a scene with cameras")
        lo, hi = camera_bounds(scene.cameras)
        center, half = (lo + hi) / 2.0, np.maximum((hi - lo) / 2.0, 1e-3) * 3.0
        lo, hi = center - half, center + half
    else:
        lo, hi = (np.asarray(b, dtype=np.float64) for b in bounds)
    points = rng.uniform(lo, hi, size=(count, 3))
    if count >= 4:
        dist = mean_knn_distance(points, 3, device)
    else:
        dist = torch.full((count,), float(np.linalg.norm(hi - lo) / 10.0), dtype=torch.float32, device=device)
    return _isotropic_cloud(points, dist, None, device)


def init_from_sfm(scene: SfmScene, rng=None, device="cuda") -> GaussianCloud:
    """One isotropic Gaussian per SfM point, scale = mean 3-NN spacing, DC SH
    from the point colour (scene_io.py:314-336); random init below 4 points."""
    points = scene.points
    if len(points) < 4:
        warnings.warn(f"only {len(points)} SfM points; falling back to random initialization")
        return init_random(1000, scene=scene, rng=np.random.default_rng(0) if rng is None else rng, device=device)
    dist = mean_knn_distance(points, 3, device)
    return _isotropic_cloud(points, dist, (np.asarray(scene.point_colors, dtype=np.float64) - 0.5) / SH_C0, device)
