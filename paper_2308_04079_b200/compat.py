"""NumPy-signature mirror of splatlab's stage functions.

splatlab's own stage API takes and returns NumPy arrays in its dataclasses:
`project` (core.py:266-345) -> `ProjectedSplats` (core.py:236-263, the M
visible Gaussians with `source_index`), `bin_and_sort` (rasterizer.py:69-124)
-> `TileBinning` (rasterizer.py:44-52), `render_forward` (rasterizer.py:201-240)
-> `RenderOutput` (rasterizer.py:127-131), `render_backward`
(rasterizer.py:253-316) -> `SplatGrads2D` (rasterizer.py:243-250) and
`backward_project` (gradients.py:192-259) -> `GaussianGrads` (gradients.py:13-27).
This module keeps those signatures, argument meanings and errors and runs
every stage on the device through libgs_b200.so (`rasterizer`), converting
at the boundary only, so splatlab-style stage tests run against the GPU
path (tests/test_gpu_compat.py).  `workers` is accepted and ignored (the
device path is parallel and its results do not depend on it); `dtype` of
render_forward likewise (float32 storage, float64 decisions).

Hand-made ProjectedSplats (tests build them from mean2d / conic / depth /
colour / alpha / radius, test_rasterizer.py:11-36) go to the device through
`DeviceSplats.from_projected`; the device objects are cached on the
returned dataclasses so a pipeline of calls converts each array once.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import rasterizer as R
from .camera import Camera
from .cloud import GaussianCloud
from .errors import InvalidPrimitiveError, ResourceLimitError  # noqa: F401  (re-exported, reference names)

_LOG2E = 1.4426950408889634


@dataclass
class ProjectedSplats:
    """core.py:236-263 (the fields the stage functions read; the backward's
    cached intermediates are recomputed on the device, so they are None)."""

    source_index: np.ndarray
    mean2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    radius: np.ndarray
    color: np.ndarray
    alpha: np.ndarray
    color_active: np.ndarray | None = None
    view_pos: np.ndarray | None = None
    jw: np.ndarray | None = None
    cov3d: np.ndarray | None = None
    cov2d: np.ndarray | None = None
    view_dir: np.ndarray | None = None
    view_dist: np.ndarray | None = None
    basis: np.ndarray | None = None
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def __len__(self) -> int:
        return int(np.asarray(self.source_index).shape[0])


@dataclass
class TileBinning:
    keys: np.ndarray        # (K,) uint64, (tile << 32) | float32 depth bits
    splat_ids: np.ndarray   # (K,) int64 into the ProjectedSplats rows
    ranges: np.ndarray      # (T, 2) [start, end)
    tiles_x: int
    tiles_y: int
    _dev: object = field(default=None, repr=False, compare=False)


@dataclass
class RenderOutput:
    image: np.ndarray
    final_transmittance: np.ndarray | None
    last_contributor: np.ndarray | None
    _dev: object = field(default=None, repr=False, compare=False)


@dataclass
class SplatGrads2D:
    d_color: np.ndarray    # (M, 3)
    d_alpha: np.ndarray    # (M,)
    d_mean2d: np.ndarray   # (M, 2)
    d_conic: np.ndarray    # (M, 3)


@dataclass
class GaussianGrads:
    d_means: np.ndarray
    d_rotations: np.ndarray
    d_log_scales: np.ndarray
    d_opacity_logits: np.ndarray
    d_sh: np.ndarray
    view_pos_grad_norm: np.ndarray


def tile_extent(width: int, height: int) -> tuple[int, int]:
    """rasterizer.py:65-66."""
    return R.tile_extent(width, height)


def make_keys(tile_ids: np.ndarray, depths: np.ndarray) -> np.ndarray:
    """rasterizer.py:55-62: (tile << 32) | float32 bits of the depth (the
    device binning writes the same keys, `bin_and_sort(...).keys`)."""
    t = np.asarray(tile_ids, np.uint64)
    d = np.asarray(depths, np.float64).astype(np.float32).view(np.uint32).astype(np.uint64)
    return (t << np.uint64(32)) | d


def _camera(camera) -> Camera:
    return R._camera(camera)


def _device_cloud(cloud) -> GaussianCloud:
    if isinstance(cloud, GaussianCloud):
        return cloud
    return GaussianCloud.from_numpy(np.asarray(cloud.means), np.asarray(cloud.rotations),
                                    np.asarray(cloud.log_scales), np.asarray(cloud.opacity_logits),
                                    np.asarray(cloud.sh))


def _device_splats(splats: ProjectedSplats, width: int, height: int) -> R.DeviceSplats:
    key = (int(width), int(height))
    dev = splats._dev.get(key)
    if dev is None:
        dev = R.DeviceSplats.from_projected(splats.mean2d, splats.conic, splats.depth, splats.color, splats.alpha,
                                            splats.radius, width, height, color_active=splats.color_active)
        splats._dev[key] = dev
    return dev


def project(cloud, camera, active_sh_degree: int = 3) -> ProjectedSplats:
    """core.py:266-345 on the device; returns the visible rows (radius > 0)
    with `source_index`, in the reference's float64 arrays."""
    dev = _device_cloud(cloud)
    sp = R.project(dev, _camera(camera), active_sh_degree)   # InvalidPrimitiveError like core.py:196
    vis = (sp.radii > 0).nonzero().flatten()
    rec = sp.rec[vis].double().cpu().numpy()
    mask = rec[:, 15].astype(np.int64)
    return ProjectedSplats(
        source_index=vis.cpu().numpy().astype(np.int64),
        mean2d=rec[:, 0:2] + rec[:, 2:4], conic=rec[:, 12:15] + rec[:, 16:19],
        depth=sp.depth[vis].double().cpu().numpy(), radius=sp.radii[vis].cpu().numpy().astype(np.int64),
        color=rec[:, 8:11].copy(), alpha=rec[:, 11] + rec[:, 19],
        color_active=np.stack([(mask >> b) & 1 for b in range(3)], axis=1).astype(bool))


def bin_and_sort(splats: ProjectedSplats, width: int, height: int, workers: int = 1) -> TileBinning:
    """rasterizer.py:69-124 on the device (ResourceLimitError past the tile or
    instance limits, as the reference)."""
    del workers
    dev = _device_splats(splats, width, height)
    b = R.bin_and_sort(dev, width, height, with_keys=True)
    return TileBinning(keys=b.keys.cpu().numpy().astype(np.uint64), splat_ids=b.splat_ids.cpu().numpy().astype(np.int64),
                       ranges=b.ranges.cpu().numpy().astype(np.int64), tiles_x=b.tiles_x, tiles_y=b.tiles_y, _dev=b)


def _device_binning(binning: TileBinning, dev_splats: R.DeviceSplats, width: int, height: int):
    if binning._dev is None:
        binning._dev = R.bin_and_sort(dev_splats, width, height)
    return binning._dev


def render_forward(splats: ProjectedSplats, binning: TileBinning, width: int, height: int, background,
                   training: bool = False, workers: int = 1, dtype=np.float64) -> RenderOutput:
    """rasterizer.py:201-240 on the device: image (H, W, 3); with training,
    final transmittance (H, W) and last contributor (H, W), an index into
    the sorted instances (-1 = none)."""
    del workers, dtype
    dev = _device_splats(splats, width, height)
    b = _device_binning(binning, dev, width, height)
    bg = tuple(float(x) for x in np.asarray(background, np.float64).reshape(3))
    out = R.render_forward(dev, b, width, height, bg, training=training)
    image = out.image.double().cpu().numpy()
    if not training:
        return RenderOutput(image, None, None, _dev=out)
    return RenderOutput(image, out.final_transmittance.double().cpu().numpy(),
                        out.last_contributor.cpu().numpy().astype(np.int64), _dev=out)


def _device_output(output: RenderOutput, width: int, height: int):
    if output._dev is not None:
        return output._dev
    if output.final_transmittance is None or output.last_contributor is None:
        raise ValueError("render_backward needs a training-mode RenderOutput")   # rasterizer.py:263-264
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()  # noqa: E731
    return R.RenderOutput(t(output.image, np.float32), t(output.final_transmittance, np.float32),
                          t(output.last_contributor, np.int32))


def render_backward(d_image, output: RenderOutput, splats: ProjectedSplats, binning: TileBinning, width: int,
                    height: int, background, workers: int = 1) -> SplatGrads2D:
    """rasterizer.py:253-316 + gradients.backward_blend (gradients.py:30-94)
    on the device; float64 arrays aligned with `splats`."""
    del workers
    dev = _device_splats(splats, width, height)
    b = _device_binning(binning, dev, width, height)
    out = _device_output(output, width, height)
    bg = tuple(float(x) for x in np.asarray(background, np.float64).reshape(3))
    d = torch.from_numpy(np.ascontiguousarray(d_image, dtype=np.float32)).cuda()
    g2 = R.render_backward(d, out, dev, b, width, height, bg)
    return SplatGrads2D(d_color=g2.d_color.double().cpu().numpy(), d_alpha=g2.d_alpha.cpu().numpy(),
                        d_mean2d=g2.d_mean2d.cpu().numpy(), d_conic=g2.d_conic.cpu().numpy())


def _moment_rows(grads2d: SplatGrads2D, rec: np.ndarray) -> np.ndarray:
    """Reference-semantics screen gradients -> the device's packed moment rows
    (see SplatGrads2D in rasterizer.py) in the basis K of `rec`:
    S = (2/log2 e)^-1 K^-T d_mean2d, S0 = d_alpha * alpha, M = K Q K^T with
    Q = [[-2 d_a, -d_b], [-d_b, -2 d_c]] from d_conic = (d_a, d_b, d_c)."""
    m = rec.shape[0]
    k = np.asarray(rec[:, 4:8], np.float64)
    alpha = np.asarray(rec[:, 11], np.float64)
    K = np.stack([np.stack([k[:, 0], k[:, 1]], 1), np.stack([k[:, 2], k[:, 3]], 1)], 1)   # rows k1, k2
    dm = np.asarray(grads2d.d_mean2d, np.float64).reshape(m, 2)
    dc = np.asarray(grads2d.d_conic, np.float64).reshape(m, 3)
    det = k[:, 0] * k[:, 3] - k[:, 1] * k[:, 2]
    ok = det != 0
    KT = np.transpose(K, (0, 2, 1))
    S = np.zeros((m, 2))
    S[ok] = np.linalg.solve(KT[ok], dm[ok][..., None])[..., 0] / (2.0 / _LOG2E)
    Q = np.stack([np.stack([-2.0 * dc[:, 0], -dc[:, 1]], 1), np.stack([-dc[:, 1], -2.0 * dc[:, 2]], 1)], 1)
    M = K @ Q @ KT
    rows = np.zeros((m, 12), np.float64)
    rows[:, 0:2] = S
    rows[:, 2] = np.asarray(grads2d.d_alpha, np.float64).reshape(m) * alpha
    rows[:, 4], rows[:, 5], rows[:, 6] = M[:, 0, 0], M[:, 0, 1], M[:, 1, 1]
    rows[:, 8:11] = np.asarray(grads2d.d_color, np.float64).reshape(m, 3)
    return rows.astype(np.float32)


def backward_project(cloud, camera, splats: ProjectedSplats, grads2d: SplatGrads2D,
                     active_sh_degree: int = 3) -> GaussianGrads:
    """gradients.py:192-259 on the device: float64 (N, ...) parameter
    gradients, culled rows exactly zero."""
    dev = _device_cloud(cloud)
    cam = _camera(camera)
    sp = R._project_tensors(dev.c_params(), len(dev), dev.device, cam, active_sh_degree)
    src = torch.from_numpy(np.asarray(splats.source_index, np.int64)).cuda()
    packed = torch.zeros((len(dev), 12), dtype=torch.float32, device=dev.device)
    packed[src] = torch.from_numpy(_moment_rows(grads2d, sp.rec[src].cpu().numpy())).to(dev.device)
    g = R.backward_project(dev, cam, sp, R.SplatGrads2D(packed, None, sp.rec), active_sh_degree)
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    return GaussianGrads(f(g.d_means), f(g.d_rotations), f(g.d_log_scales), f(g.d_opacity_logits), f(g.d_sh),
                         f(g.view_pos_grad_norm))
