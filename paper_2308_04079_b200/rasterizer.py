"""Host side of the B200 rasterizer: the reference's stage functions over
device tensors, and the drop-in torch.autograd.Function.

Stage functions keep the names, argument meaning and error behaviour of the
reference (splatlab):
  project          core.py:266-345        -> gs_preprocess_forward   (K1)
  bin_and_sort     rasterizer.py:69-124   -> gs_bin_and_sort         (K2-K5)
  render_forward   rasterizer.py:201-240  -> gs_blend_forward        (K6)
  render_backward  rasterizer.py:253-316  -> gs_blend_backward_scheduled (K7)
  backward_project gradients.py:192-259   -> gs_preprocess_backward  (K8)
  render_view      optimizer.py:212-219   (composition of the first three)
Everything runs on the current CUDA stream; buffers come from torch's
caching allocator, the library itself never allocates.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .camera import Camera
from .cloud import GaussianCloud, c_params_from
from .errors import InvalidPrimitiveError

TILE_SIZE = 16            # rasterizer.py:13
ALPHA_EPS = 1.0 / 255.0   # rasterizer.py:17
ALPHA_CLAMP = 0.99        # rasterizer.py:18
SATURATION = 0.9999       # rasterizer.py:19
MAX_TILES = 2**32 - 1     # rasterizer.py:24
MAX_INSTANCES = 2**31     # rasterizer.py:25

LOG2E = 1.4426950408889634


def conic_basis(conic: np.ndarray) -> np.ndarray:
    """Host restatement of the device conic_basis (gs_common.cuh): rows
    k = (k1.x, k1.y, k2.x, k2.y) with k_i = sqrt(log2(e) lambda_i / 2) e_i over
    the conic's eigenpairs, so log2(e) * power = -(k1.d)^2 - (k2.d)^2 (record
    word 1; the blend kernels' cancellation-free exponent)."""
    a, b, c = (np.asarray(conic, np.float64).reshape(-1, 3)[:, i] for i in range(3))
    h = 0.5 * (a - c)
    r = np.sqrt(h * h + b * b)
    l1 = 0.5 * (a + c) + r
    det = np.maximum(a * c - b * b, 0.0)
    l2 = np.where(l1 > 0, det / np.where(l1 > 0, l1, 1.0), 0.0)
    ex, ey = np.where(h >= 0, h + r, b), np.where(h >= 0, b, r - h)
    nn = np.sqrt(ex * ex + ey * ey)
    ok = nn > 0
    ex, ey = np.where(ok, ex / np.where(ok, nn, 1.0), 1.0), np.where(ok, ey / np.where(ok, nn, 1.0), 0.0)
    f1, f2 = np.sqrt(0.5 * LOG2E * l1), np.sqrt(0.5 * LOG2E * l2)
    return np.stack([f1 * ex, f1 * ey, -f2 * ey, f2 * ex], axis=1).astype(np.float32)


def resolve_workers(workers: int | None = None, deterministic: bool = False) -> int:
    """The reference's worker resolution (rasterizer.py:32-41), kept for API
    compatibility: CPU tile threads have no GPU counterpart (tiles are CTAs).
    The GPU side of `deterministic` is render_backward(deterministic=True)
    (TrainConfig.deterministic in training): bit-identical runs."""
    if deterministic:
        return 1
    if workers is None:
        workers = __import__("os").cpu_count() or 1
    cap = __import__("os").environ.get("SPLATLAB_THREADS")
    if cap:
        workers = min(workers, max(1, int(cap)))
    return max(1, workers)


def tile_extent(width: int, height: int) -> tuple[int, int]:
    return (width + TILE_SIZE - 1) // TILE_SIZE, (height + TILE_SIZE - 1) // TILE_SIZE


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _camera(camera) -> Camera:
    return camera if isinstance(camera, Camera) else Camera.from_reference(camera)


@dataclass
class DeviceSplats:
    """Per-view projected splats in N-space (see gs_splats_t)."""

    rec: torch.Tensor            # (N,20) float32, see gs_splats_t
    depth: torch.Tensor          # (N,)   float32
    radii: torch.Tensor          # (N,)   int32, 0 = culled
    rect: torch.Tensor           # (N,4)  int32
    tiles_touched: torch.Tensor  # (N,)   int32
    status: torch.Tensor         # (1,)   int32

    @classmethod
    def empty(cls, n: int, device) -> "DeviceSplats":
        f32, i32 = dict(dtype=torch.float32, device=device), dict(dtype=torch.int32, device=device)
        return cls(torch.empty((n, _lib.REC_FLOATS), **f32), torch.empty(n, **f32), torch.empty(n, **i32),
                   torch.empty((n, 4), **i32), torch.empty(n, **i32), torch.empty(1, **i32))

    def __len__(self) -> int:
        return self.radii.shape[0]

    @classmethod
    def from_projected(cls, mean2d, conic, depth, color, alpha, radius, width: int, height: int,
                       color_active=None, device="cuda") -> "DeviceSplats":
        """Adapter from reference-style ProjectedSplats arrays (core.py:236-263)
        to device records, for stage-level tests that bypass project()
        (as test_rasterizer.py:11-36 does).  Tile rectangles follow
        rasterizer.py:86-97 in float64."""
        mean2d = np.asarray(mean2d, np.float64).reshape(-1, 2)
        n = mean2d.shape[0]
        conic = np.asarray(conic, np.float64).reshape(n, 3)
        color = np.asarray(color, np.float64).reshape(n, 3)
        radius = np.asarray(radius, np.int64).reshape(n)
        rec = np.zeros((n, _lib.REC_FLOATS), np.float32)
        hi = mean2d.astype(np.float32)
        rec[:, 0:2] = hi
        rec[:, 2:4] = (mean2d - hi).astype(np.float32)
        rec[:, 4:8] = conic_basis(conic)
        alpha = np.asarray(alpha, np.float64).reshape(n)
        rec[:, 8:11] = color
        rec[:, 11] = alpha
        rec[:, 12:15] = conic
        rec[:, 16:19] = conic - rec[:, 12:15].astype(np.float64)
        rec[:, 19] = alpha - rec[:, 11].astype(np.float64)
        active = np.ones((n, 3), bool) if color_active is None else np.asarray(color_active, bool).reshape(n, 3)
        rec[:, 15] = (active * np.array([1, 2, 4])).sum(axis=1)
        tx, ty = tile_extent(width, height)
        r = radius.astype(np.float64)
        x0, x1 = np.floor((mean2d[:, 0] - r) / TILE_SIZE), np.floor((mean2d[:, 0] + r) / TILE_SIZE)
        y0, y1 = np.floor((mean2d[:, 1] - r) / TILE_SIZE), np.floor((mean2d[:, 1] + r) / TILE_SIZE)
        valid = (x1 >= 0) & (x0 < tx) & (y1 >= 0) & (y0 < ty) & (radius > 0)
        x0, x1 = np.clip(x0, 0, tx - 1), np.clip(x1, 0, tx - 1)
        y0, y1 = np.clip(y0, 0, ty - 1), np.clip(y1, 0, ty - 1)
        rect = np.stack([x0, y0, x1, y1], axis=1).astype(np.int32)
        tiles = np.where(valid, (x1 - x0 + 1) * (y1 - y0 + 1), 0).astype(np.int32)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)  # noqa: E731
        return cls(t(rec, np.float32), t(np.asarray(depth, np.float64).reshape(n), np.float32),
                   t(np.minimum(radius, 2**31 - 1), np.int32), t(rect, np.int32), t(tiles, np.int32),
                   torch.zeros(1, dtype=torch.int32, device=device))

    def c_struct(self) -> _lib.GsSplats:
        s = _lib.GsSplats()
        s.rec, s.depth, s.radii = self.rec.data_ptr(), self.depth.data_ptr(), self.radii.data_ptr()
        s.rect, s.tiles_touched, s.status = self.rect.data_ptr(), self.tiles_touched.data_ptr(), self.status.data_ptr()
        s.n = len(self)
        return s

    # Views in the reference's ProjectedSplats vocabulary (core.py:236-263).
    @property
    def visible(self) -> torch.Tensor:
        return self.radii > 0

    @property
    def mean2d(self) -> torch.Tensor:
        r = self.rec.double()
        return r[:, 0:2] + r[:, 2:4]

    @property
    def conic(self) -> torch.Tensor:
        return self.rec[:, 12:15]

    @property
    def alpha(self) -> torch.Tensor:
        return self.rec[:, 11]

    @property
    def color(self) -> torch.Tensor:
        return self.rec[:, 8:11]

    @property
    def color_active(self) -> torch.Tensor:
        bits = self.rec[:, 15].to(torch.int32)
        return torch.stack([(bits >> c) & 1 for c in range(3)], dim=1).bool()


@dataclass
class TileBinning:
    """Sorted instances (rasterizer.py:44-52): Gaussian id per sorted instance,
    per-tile [start, end) ranges and, when requested (with_keys=True), the
    reference's 64-bit sort keys (tile << 32) | float32 bits of depth
    (make_keys, rasterizer.py:55-62) as int64."""

    splat_ids: torch.Tensor   # (K,) int32 Gaussian index (N-space); (capacity,) when k_info is set
    ranges: torch.Tensor      # (T,2) int32
    tiles_x: int
    tiles_y: int
    k_info: torch.Tensor | None = None   # async binning: device int64 [K, flags, min(K, capacity)]
    n_gaussians: int = 0
    keys: torch.Tensor | None = None     # (K,) int64 (capacity-sized when k_info is set)
    hint: str | None = None              # capacity-hint key (device @ frame size)

    @property
    def num_instances(self) -> int:
        if self.k_info is not None:
            return int(self.k_info[0].item())   # synchronises
        return self.splat_ids.shape[0]

    def check(self) -> None:
        """Raise like the synchronous bin_and_sort would (async binning only;
        synchronises).  A capacity overflow raises CapacityError: the ranges
        were left empty and the frame must be re-binned."""
        if self.k_info is None:
            return
        self.check_host([int(v) for v in self.k_info.tolist()])

    def check_host(self, k_info) -> None:
        """check() on an already-read copy of k_info (no synchronisation)."""
        k, flags = int(k_info[0]), int(k_info[1])
        _capacity.update(self.hint or _capacity.key(self.splat_ids.device, 16 * self.tiles_x, 16 * self.tiles_y),
                         k, self.n_gaussians or None)
        if flags & 1:
            raise InvalidPrimitiveError("zero-norm quaternion cannot be normalized")
        if flags & 4:
            _lib.check(_lib.GS_ERR_RESOURCE_LIMIT, "bin_and_sort")
        if flags & 2:
            raise CapacityError(f"bin_and_sort: {k} instances exceed the capacity {self.splat_ids.shape[0]}")


class CapacityError(RuntimeError):
    """Async binning overflowed its instance capacity (the hint is raised)."""


@dataclass
class RenderOutput:
    image: torch.Tensor                        # (H,W,3) float32
    final_transmittance: torch.Tensor | None   # (H,W) float32, training only
    last_contributor: torch.Tensor | None      # (H,W) int32, -1 = none


@dataclass
class SplatGrads2D:
    """Screen-space gradients (rasterizer.py:243-250) in the packed (N,12) row
    of eigenbasis moments of dp = dL/da a_raw over the offsets v = K (pixel -
    mean) the blends evaluate the exponent from (log2(e) power = -|v|^2;
    K = record words 4:8): [0:2] (S1, S2) = sum dp v, [2] S0 = sum dp,
    [4:7] M = sum dp (v1^2, v1 v2, v2^2), [8:11] d_color.  The properties
    convert them to the reference's quantities: d_mean2d = 2/log2(e) K^T S,
    d_alpha = S0 / alpha, d_conic = -1/2 sum dL/dpower (dx^2, 2 dx dy, dy^2)
    (gradients.py:54-93)."""

    packed: torch.Tensor  # (N,12) float32
    # the longest-first tile schedule the backward ran on (int32 (T,)), a good
    # launch order for the next forward of the same view (render_forward)
    tile_order: torch.Tensor | None = None
    rec: torch.Tensor | None = None   # the splats' records (for d_conic)

    def _need_rec(self, what: str) -> torch.Tensor:
        if self.rec is None:
            raise ValueError(f"{what} needs the splats' records (SplatGrads2D.rec)")
        return self.rec

    @property
    def d_mean2d(self) -> torch.Tensor:
        """(N,2) float64 d_mean2d = 2/log2(e) K^T (S1, S2)."""
        k = self._need_rec("d_mean2d")[:, 4:8].double()
        s1, s2 = self.packed[:, 0].double(), self.packed[:, 1].double()
        c = 2.0 / 1.4426950408889634
        out = torch.stack([c * (k[:, 0] * s1 + k[:, 2] * s2), c * (k[:, 1] * s1 + k[:, 3] * s2)], dim=1)
        # culled rows: S = 0 and the record is undefined (never written)
        ok = (s1 != 0) | (s2 != 0)
        return torch.where(ok[:, None], out, torch.zeros_like(out))

    @property
    def d_alpha(self) -> torch.Tensor:
        """(N,) float64 d_alpha = S0 / alpha (0 where S0 = 0, e.g. culled rows)."""
        alpha = self._need_rec("d_alpha")[:, 11].double()
        s0 = self.packed[:, 2].double()
        ok = s0 != 0
        return torch.where(ok, s0 / torch.where(ok, alpha, torch.ones_like(alpha)), torch.zeros_like(s0))

    @property
    def conic_moments(self) -> torch.Tensor:
        return self.packed[:, 4:7]

    @property
    def d_conic(self) -> torch.Tensor:
        """(N,3) float64 d_conic (a, b, c): Q = K^-1 M K^-T, d_conic =
        (-Q_xx / 2, -Q_xy, -Q_yy / 2)."""
        if self.rec is None:
            raise ValueError("d_conic needs the splats' records (SplatGrads2D.rec)")
        m = self.packed[:, 4:7].double()
        k = self.rec[:, 4:8].double()
        det = k[:, 0] * k[:, 3] - k[:, 1] * k[:, 2]
        ok = (det != 0) & (m != 0).any(dim=1)
        inv = torch.where(ok, 1.0 / torch.where(ok, det, torch.ones_like(det)), torch.zeros_like(det))
        # K^-1 = [[k2y, -k1y], [-k2x, k1x]] / det
        a, b = k[:, 3] * inv, -k[:, 1] * inv
        c, d = -k[:, 2] * inv, k[:, 0] * inv
        m11, m12, m22 = m[:, 0], m[:, 1], m[:, 2]
        qxx = a * (a * m11 + b * m12) + b * (a * m12 + b * m22)
        qxy = a * (c * m11 + d * m12) + b * (c * m12 + d * m22)
        qyy = c * (c * m11 + d * m12) + d * (c * m12 + d * m22)
        out = torch.stack([-0.5 * qxx, -qxy, -0.5 * qyy], dim=1)
        return torch.where(ok[:, None], out, torch.zeros_like(out))   # culled rows: records undefined

    @property
    def d_color(self) -> torch.Tensor:
        return self.packed[:, 8:11]


@dataclass
class GaussianGrads:
    """Parameter gradients (gradients.py:13-27); culled rows are exactly 0."""

    d_means: torch.Tensor
    d_rotations: torch.Tensor
    d_log_scales: torch.Tensor
    d_opacity_logits: torch.Tensor
    d_sh: torch.Tensor
    view_pos_grad_norm: torch.Tensor

    @classmethod
    def zeros(cls, n: int, device) -> "GaussianGrads":
        z = dict(dtype=torch.float32, device=device)
        return cls(torch.zeros((n, 3), **z), torch.zeros((n, 4), **z), torch.zeros((n, 3), **z),
                   torch.zeros(n, **z), torch.zeros((n, 16, 3), **z), torch.zeros(n, **z))

    def c_struct(self) -> _lib.GsGrads:
        g = _lib.GsGrads()
        g.d_means, g.d_rotations = self.d_means.data_ptr(), self.d_rotations.data_ptr()
        g.d_log_scales, g.d_opacity_logits = self.d_log_scales.data_ptr(), self.d_opacity_logits.data_ptr()
        g.d_sh, g.view_pos_grad_norm = self.d_sh.data_ptr(), self.view_pos_grad_norm.data_ptr()
        return g


@dataclass
class DensifyStats:
    """Device densification statistics (TrainState, optimizer.py:106-108)."""

    accum_pos_grad: torch.Tensor   # (N,) float32
    accum_count: torch.Tensor      # (N,) int32
    max_radius_frac: torch.Tensor  # (N,) float32

    @classmethod
    def zeros(cls, n: int, device) -> "DensifyStats":
        return cls(torch.zeros(n, dtype=torch.float32, device=device),
                   torch.zeros(n, dtype=torch.int32, device=device),
                   torch.zeros(n, dtype=torch.float32, device=device))

    def c_struct(self) -> _lib.GsStats:
        s = _lib.GsStats()
        s.accum_pos_grad = self.accum_pos_grad.data_ptr()
        s.accum_count = self.accum_count.data_ptr()
        s.max_radius_frac = self.max_radius_frac.data_ptr()
        return s


# ---------------------------------------------------------------------------
# stage functions

def _project_tensors(params: _lib.GsParams, n: int, device, camera: Camera, active_sh_degree: int) -> DeviceSplats:
    if not 0 <= active_sh_degree <= 3:
        raise ValueError(f"SH degree must be in 0..3, got {active_sh_degree}")  # sh.py:37-38
    lib = _lib.load()
    splats = DeviceSplats.empty(n, device)
    cs = splats.c_struct()
    _lib.check(lib.gs_preprocess_forward(ctypes.byref(params), ctypes.byref(camera.to_c()), int(active_sh_degree),
                                         ctypes.byref(cs), _stream()), "project")
    return splats


def project(cloud: GaussianCloud, camera, active_sh_degree: int = 3) -> DeviceSplats:
    """K1: cull, EWA-project, colour and activate every Gaussian (core.py:266).

    Raises InvalidPrimitiveError for a zero quaternion among the survivors of
    the near/guard-band tests, like the reference (this check synchronises)."""
    camera = _camera(camera)
    splats = _project_tensors(cloud.c_params(), len(cloud), cloud.device, camera, active_sh_degree)
    if len(cloud) and int(splats.status.item()) & 1:
        raise InvalidPrimitiveError("zero-norm quaternion cannot be normalized")
    return splats


class _CapacityHint:
    """Instance-buffer sizing: remembers, per device and frame size, the
    largest K and the largest instances-per-Gaussian ratio seen, so a
    steady-state frame issues exactly one binning call and a cloud that grew
    (densification) gets a proportionally larger buffer.  Never above the
    reference's instance limit (rasterizer.py:25)."""

    def __init__(self):
        self.k = {}
        self.ratio = {}

    HEADROOM = 1.05
    LIMIT = MAX_INSTANCES - 1

    @staticmethod
    def key(device, width: int | None = None, height: int | None = None) -> str:
        d = device if isinstance(device, str) else str(device)
        return d if width is None else f"{d}@{width}x{height}"

    def get(self, key, n: int | None = None) -> int:
        key = self.key(key)
        k = self.k.get(key, 1 << 16)
        if n is not None and key in self.ratio:
            k = max(k, int(self.ratio[key] * n * self.HEADROOM) + 4096)
        return min(k, self.LIMIT)

    def update(self, key, k: int, n: int | None = None) -> None:
        key = self.key(key)
        self.k[key] = min(max(self.k.get(key, 1 << 16), int(k * self.HEADROOM) + 4096), self.LIMIT)
        if n:
            self.ratio[key] = max(self.ratio.get(key, 0.0), k / n)


_capacity = _CapacityHint()


def bin_and_sort(splats: DeviceSplats, width: int, height: int, with_keys: bool = False) -> TileBinning:
    """K2-K5: duplicate, sort by (tile, depth, index), find tile ranges (rasterizer.py:69).
    with_keys: also return the 64-bit sort keys (TileBinning.keys, rasterizer.py:48)."""
    lib = _lib.load()
    tiles_x, tiles_y = tile_extent(width, height)
    device = splats.rec.device
    hint = _capacity.key(device, width, height)
    n = len(splats)
    cs = splats.c_struct()
    stream = _stream()
    cap = _capacity.get(hint, n)
    for _ in range(2):
        ws_bytes = _bin_workspace_bytes(n, width, height, cap)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
        ids = torch.empty(max(cap, 1), dtype=torch.int32, device=device)
        keys = torch.empty(max(cap, 1), dtype=torch.int64, device=device) if with_keys else None
        ranges = torch.empty((tiles_x * tiles_y, 2), dtype=torch.int32, device=device)
        k = ctypes.c_int64(0)
        st = lib.gs_bin_and_sort(ctypes.byref(cs), width, height, ws.data_ptr(), ws_bytes, cap,
                                 ids.data_ptr(), ranges.data_ptr(), _lib.ptr(keys), ctypes.byref(k), stream)
        if st == _lib.GS_ERR_CAPACITY:
            _capacity.update(hint, k.value, n)
            cap = _capacity.get(hint, n)
            continue
        _lib.check(st, "bin_and_sort")
        _capacity.update(hint, k.value, n)
        return TileBinning(ids[:k.value], ranges, tiles_x, tiles_y,
                           keys=keys[:k.value] if keys is not None else None)
    raise RuntimeError("bin_and_sort: instance capacity did not converge")


_ws_sizes: dict = {}


def _bin_workspace_bytes(n: int, width: int, height: int, cap: int) -> int:
    """gs_bin_workspace_size, memoised (a pure function of its arguments)."""
    key = (n, width, height, cap)
    b = _ws_sizes.get(key)
    if b is None:
        nbytes = ctypes.c_size_t(0)
        _lib.check(_lib.load().gs_bin_workspace_size(n, width, height, cap, ctypes.byref(nbytes)), "bin_and_sort")
        b = _ws_sizes[key] = int(nbytes.value)
        if len(_ws_sizes) > 256:
            _ws_sizes.pop(next(iter(_ws_sizes)))
    return b


def bin_and_sort_async(splats: DeviceSplats, width: int, height: int, capacity: int | None = None,
                       with_keys: bool = False) -> TileBinning:
    """bin_and_sort without a host synchronisation: K stays on the device
    (binning.k_info) and the instance buffers are sized by `capacity`
    (default: the largest K seen on this device x 1.15).  Call
    binning.check() later (e.g. after the step) to surface errors."""
    lib = _lib.load()
    tiles_x, tiles_y = tile_extent(width, height)
    device = splats.rec.device
    hint = _capacity.key(device, width, height)
    cap = int(capacity) if capacity is not None else _capacity.get(hint, len(splats))
    ws_bytes = _bin_workspace_bytes(len(splats), width, height, cap)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
    ids = torch.empty(max(cap, 1), dtype=torch.int32, device=device)
    ranges = torch.empty((tiles_x * tiles_y, 2), dtype=torch.int32, device=device)
    keys = torch.empty(max(cap, 1), dtype=torch.int64, device=device) if with_keys else None
    k_info = torch.empty(3, dtype=torch.int64, device=device)
    cs = splats.c_struct()
    _lib.check(lib.gs_bin_and_sort_async(ctypes.byref(cs), width, height, ws.data_ptr(), ws_bytes, cap,
                                         ids.data_ptr(), ranges.data_ptr(), _lib.ptr(keys), k_info.data_ptr(),
                                         _stream()),
               "bin_and_sort")
    return TileBinning(ids, ranges, tiles_x, tiles_y, k_info, len(splats), keys, hint)


def _bg(background) -> ctypes.Array:
    b = np.asarray(background, dtype=np.float64).reshape(3)
    return (ctypes.c_float * 3)(*[float(v) for v in b])


def render_forward(splats: DeviceSplats, binning: TileBinning, width: int, height: int, background,
                   training: bool = False, tile_order: torch.Tensor | None = None,
                   tile_work: torch.Tensor | None = None) -> RenderOutput:
    """K6: per-tile front-to-back blend (rasterizer.py:201).

    tile_order: optional launch order of the tiles (a permutation of
    [0, tiles), e.g. SplatGrads2D.tile_order from the previous backward of the
    same view: heavy tiles first).  tile_work: optional int32 (tiles,) that
    receives each tile's work (see TileSchedule).  The result does not depend
    on either."""
    lib = _lib.load()
    device = splats.rec.device
    image = torch.empty((height, width, 3), dtype=torch.float32, device=device)
    t_final = torch.empty((height, width), dtype=torch.float32, device=device) if training else None
    last = torch.empty((height, width), dtype=torch.int32, device=device) if training else None
    # exact-stop re-blend list (training): count, work counter, pixel indices
    scratch = torch.empty(2 + width * height, dtype=torch.int32, device=device) if training else None
    cs = splats.c_struct()
    tx, ty = tile_extent(width, height)
    if tile_order is not None and (tile_order.numel() != tx * ty or tile_order.device != device):
        tile_order = None
    if tile_work is not None and (tile_work.numel() != tx * ty or tile_work.device != device):
        raise ValueError("tile_work must be a (tiles,) int32 tensor on the splats' device")
    if tile_order is not None or tile_work is not None:
        _lib.check(lib.gs_blend_forward_ordered(ctypes.byref(cs), binning.splat_ids.data_ptr(),
                                                binning.ranges.data_ptr(), width, height, _bg(background),
                                                int(bool(training)), _lib.ptr(tile_order), _lib.ptr(tile_work),
                                                image.data_ptr(), _lib.ptr(t_final), _lib.ptr(last), _lib.ptr(scratch),
                                                _stream()),
                   "render_forward")
    else:
        _lib.check(lib.gs_blend_forward(ctypes.byref(cs), binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
                                        width, height, _bg(background), int(bool(training)), image.data_ptr(),
                                        _lib.ptr(t_final), _lib.ptr(last), _lib.ptr(scratch), _stream()),
                   "render_forward")
    return RenderOutput(image, t_final, last)


@dataclass
class BackwardPrep:
    """The backward's longest-first tile schedule and its cleared gradient rows,
    enqueued on a side stream by prepare_backward (so they overlap the loss)."""

    scratch: torch.Tensor   # int32 (2 T + 2048,): the order in [0, T)
    packed: torch.Tensor    # (N,12) float32, zeroed
    done: torch.cuda.Event
    tiles: int


_side_streams: dict = {}


def prepare_backward(output: RenderOutput, splats: DeviceSplats, binning: TileBinning, width: int,
                     height: int) -> BackwardPrep:
    """Enqueue, on a side stream behind the current stream's work so far (the
    forward), the tile schedule of the coming render_backward and the
    clearing of its gradient rows: they depend only on the forward's
    training record, so they run while the loss is computed.  Pass the
    result to render_backward(prep=...)."""
    if output.last_contributor is None:
        raise ValueError("backward pass needs a training-mode RenderOutput")
    device = splats.rec.device
    tx, ty = tile_extent(width, height)
    scratch = torch.empty(2 * tx * ty + 2048, dtype=torch.int32, device=device)
    packed = torch.empty((len(splats), _lib.GRAD2D_FLOATS), dtype=torch.float32, device=device)
    main = torch.cuda.current_stream(device)
    side = _side_streams.get(str(device))
    if side is None:
        side = _side_streams[str(device)] = torch.cuda.Stream(device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        _lib.check(_lib.load().gs_blend_backward_schedule(binning.ranges.data_ptr(),
                                                          output.last_contributor.data_ptr(), width, height,
                                                          scratch.data_ptr(), side.cuda_stream), "render_backward")
        packed.zero_()
    # the buffers may be dropped unused (a discarded lookahead): keep them out of
    # the allocator's reach until the side stream is done with them
    scratch.record_stream(side)
    packed.record_stream(side)
    done = torch.cuda.Event()
    done.record(side)
    return BackwardPrep(scratch, packed, done, tx * ty)


def render_backward(d_image: torch.Tensor, output: RenderOutput, splats: DeviceSplats, binning: TileBinning,
                    width: int, height: int, background, deterministic: bool = False,
                    stage_timer=None, prep: BackwardPrep | None = None) -> SplatGrads2D:
    """K7: back-to-front blend gradient (rasterizer.py:253).

    deterministic: no float atomics (per-instance partial rows summed per
    splat in a fixed order): bit-identical results run to run, the
    reference's deterministic=True (rasterizer.py:34-35).
    stage_timer (profiling.StageTimer, optional): the tile schedule and the
    clearing of the rows are timed as stage "blend_bwd_setup" and the blend
    kernel alone as "blend_bwd" (the roofline's launch duration).
    prep: the schedule and cleared rows from prepare_backward (then only the
    blend kernel is launched here, after waiting for them)."""
    if output.final_transmittance is None or output.last_contributor is None:
        raise ValueError("backward pass needs a training-mode RenderOutput")  # rasterizer.py:265-266
    lib = _lib.load()
    d_image = d_image.to(dtype=torch.float32).contiguous()
    if tuple(d_image.shape) != (height, width, 3):
        raise ValueError(f"d_image shape {tuple(d_image.shape)} != {(height, width, 3)}")
    cs = splats.c_struct()
    if prep is not None and not deterministic:
        from .profiling import StageTimer
        torch.cuda.current_stream(splats.rec.device).wait_event(prep.done)
        with StageTimer.stage(stage_timer, "blend_bwd"):
            _lib.check(lib.gs_blend_backward_accumulate(
                d_image.data_ptr(), ctypes.byref(cs), binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
                output.final_transmittance.data_ptr(), output.last_contributor.data_ptr(), width, height,
                _bg(background), prep.scratch.data_ptr(), prep.packed.data_ptr(), _stream()), "render_backward")
        return SplatGrads2D(prep.packed, prep.scratch[:prep.tiles], splats.rec)
    packed = torch.empty((len(splats), _lib.GRAD2D_FLOATS), dtype=torch.float32, device=splats.rec.device)
    if deterministic:
        cap = int(binning.splat_ids.shape[0])
        nbytes = ctypes.c_size_t(0)
        _lib.check(lib.gs_blend_backward_det_workspace_size(len(splats), width, height, cap, ctypes.byref(nbytes)),
                   "render_backward")
        ws = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=splats.rec.device)
        _lib.check(lib.gs_blend_backward_deterministic(
            d_image.data_ptr(), ctypes.byref(cs), binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
            output.final_transmittance.data_ptr(), output.last_contributor.data_ptr(), width, height,
            _bg(background), None, ws.data_ptr(), int(nbytes.value), cap, packed.data_ptr(), _stream()),
            "render_backward")
        return SplatGrads2D(packed, None, splats.rec)
    if _BWD_SCHEDULE and stage_timer is not None:
        from .profiling import StageTimer
        tx, ty = tile_extent(width, height)
        scratch = torch.empty(2 * tx * ty + 2048, dtype=torch.int32, device=splats.rec.device)
        with StageTimer.stage(stage_timer, "blend_bwd_setup"):
            _lib.check(lib.gs_blend_backward_schedule(binning.ranges.data_ptr(), output.last_contributor.data_ptr(),
                                                      width, height, scratch.data_ptr(), _stream()), "render_backward")
            packed.zero_()
        with StageTimer.stage(stage_timer, "blend_bwd"):
            _lib.check(lib.gs_blend_backward_accumulate(
                d_image.data_ptr(), ctypes.byref(cs), binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
                output.final_transmittance.data_ptr(), output.last_contributor.data_ptr(), width, height,
                _bg(background), scratch.data_ptr(), packed.data_ptr(), _stream()), "render_backward")
        return SplatGrads2D(packed, scratch[:tx * ty], splats.rec)
    if _BWD_SCHEDULE:
        # longest-first tile order from the forward's training record (scratch: 2 T + 2048 int32)
        tx, ty = tile_extent(width, height)
        scratch = torch.empty(2 * tx * ty + 2048, dtype=torch.int32, device=splats.rec.device)
        _lib.check(lib.gs_blend_backward_scheduled(
            d_image.data_ptr(), ctypes.byref(cs), binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
            output.final_transmittance.data_ptr(), output.last_contributor.data_ptr(), width, height,
            _bg(background), scratch.data_ptr(), packed.data_ptr(), _stream()), "render_backward")
        return SplatGrads2D(packed, scratch[:tx * ty], splats.rec)
    else:
        _lib.check(lib.gs_blend_backward(d_image.data_ptr(), ctypes.byref(cs), binning.splat_ids.data_ptr(),
                                         binning.ranges.data_ptr(), output.final_transmittance.data_ptr(),
                                         output.last_contributor.data_ptr(), width, height, _bg(background),
                                         packed.data_ptr(), _stream()), "render_backward")
    return SplatGrads2D(packed, None, splats.rec)


_BWD_SCHEDULE = __import__("os").environ.get("GS_BWD_SCHEDULE", "1") != "0"


def _backward_project_tensors(params: _lib.GsParams, n: int, device, camera: Camera, splats: DeviceSplats,
                              grads2d: SplatGrads2D, active_sh_degree: int, stats: DensifyStats | None,
                              out: GaussianGrads | None, accumulate: bool,
                              skip: torch.Tensor | None = None) -> GaussianGrads:
    if not 0 <= active_sh_degree <= 3:
        raise ValueError(f"SH degree must be in 0..3, got {active_sh_degree}")
    lib = _lib.load()
    if out is None:
        z = dict(dtype=torch.float32, device=device)
        out = GaussianGrads(torch.empty((n, 3), **z), torch.empty((n, 4), **z), torch.empty((n, 3), **z),
                            torch.empty(n, **z), torch.empty((n, 16, 3), **z), torch.empty(n, **z))
        accumulate = False
    cs = splats.c_struct()
    cg = out.c_struct()
    cst = stats.c_struct() if stats is not None else None
    _lib.check(lib.gs_preprocess_backward_guarded(ctypes.byref(params), ctypes.byref(camera.to_c()),
                                                  int(active_sh_degree), ctypes.byref(cs), grads2d.packed.data_ptr(),
                                                  ctypes.byref(cg), int(bool(accumulate)),
                                                  ctypes.byref(cst) if cst is not None else None, _lib.ptr(skip),
                                                  _stream()), "backward_project")
    return out


def backward_project(cloud: GaussianCloud, camera, splats: DeviceSplats, grads2d: SplatGrads2D,
                     active_sh_degree: int = 3, *, stats: DensifyStats | None = None,
                     out: GaussianGrads | None = None, accumulate: bool = False,
                     skip: torch.Tensor | None = None) -> GaussianGrads:
    """K8: chain screen-space gradients to the raw parameters (gradients.py:192).

    `stats` (optional) receives the densification statistics update of
    optimizer.py:252-255; `out` + `accumulate` sum several views in place;
    `skip` (device int32 from step_guard) leaves the statistics untouched."""
    return _backward_project_tensors(cloud.c_params(), len(cloud), cloud.device, _camera(camera), splats, grads2d,
                                     active_sh_degree, stats, out, accumulate, skip)


def render_view(cloud: GaussianCloud, camera, background, active_sh_degree: int = 3, training: bool = False):
    """project -> bin_and_sort -> render_forward (optimizer.py:212-219)."""
    camera = _camera(camera)
    splats = _project_tensors(cloud.c_params(), len(cloud), cloud.device, camera, active_sh_degree)
    binning = bin_and_sort(splats, camera.width, camera.height)
    out = render_forward(splats, binning, camera.width, camera.height, background, training=training)
    return out, splats, binning


def render_view_async(cloud: GaussianCloud, camera, background, active_sh_degree: int = 3, training: bool = False,
                      capacity: int | None = None, tile_order: torch.Tensor | None = None,
                      schedule: "TileSchedule | None" = None, splats: "DeviceSplats | None" = None):
    """render_view with the sync-free binning: no host synchronisation, so
    the whole forward can be captured in a CUDA graph.  Errors (zero
    quaternion, capacity overflow) surface through binning.check().
    tile_order: see render_forward.  schedule: a TileSchedule for repeated
    renders of one view (its order, when present, overrides tile_order).
    splats: this view's projection when already made (the previous step's
    DeviceAdam.backward_step(..., project_next=(camera, degree))): K1 is
    skipped."""
    camera = _camera(camera)
    if splats is None:
        splats = _project_tensors(cloud.c_params(), len(cloud), cloud.device, camera, active_sh_degree)
    elif len(splats) != len(cloud):
        raise ValueError(f"splats hold {len(splats)} Gaussians, the cloud {len(cloud)}")
    binning = bin_and_sort_async(splats, camera.width, camera.height, capacity)
    work = None
    if schedule is not None:
        order, work = schedule.prepare(camera.width, camera.height, cloud.device)
        tile_order = order if order is not None else tile_order
    out = render_forward(splats, binning, camera.width, camera.height, background, training=training,
                         tile_order=tile_order, tile_work=work)
    if schedule is not None:
        schedule.update()
    return out, splats, binning


class TileSchedule:
    """Launch schedule for repeated renders of one view (a viewer, a render
    benchmark): every forward records each tile's work (splats handed to the
    blend before the tile saturated) and the next frame launches the heaviest
    tiles first (gs_tile_schedule), so light tiles fill the last wave.  The
    images do not depend on it."""

    def __init__(self):
        self.key = None
        self.order = self.work = self.scratch = None
        self.ready = False

    def prepare(self, width: int, height: int, device):
        tx, ty = tile_extent(width, height)
        key = (tx * ty, str(device))
        if key != self.key:
            z = dict(dtype=torch.int32, device=device)
            self.order, self.work = torch.empty(tx * ty, **z), torch.empty(tx * ty, **z)
            self.scratch = torch.empty(tx * ty + 2048, **z)
            self.key, self.ready = key, False
        return (self.order if self.ready else None), self.work

    def update(self) -> None:
        """Rebuild the order from the work just recorded (stream-ordered after
        the forward that read the previous order)."""
        _lib.check(_lib.load().gs_tile_schedule(self.work.data_ptr(), self.work.numel(), self.scratch.data_ptr(),
                                                self.order.data_ptr(), _stream()), "tile_schedule")
        self.ready = True


# ---------------------------------------------------------------------------
# drop-in autograd Function

class _TileOrderCache:
    """Per-camera longest-first tile order from the camera's last backward
    (a few hundred cameras): the next forward of the same view launches its
    heaviest tiles first.  The images do not depend on it."""

    def __init__(self, size: int = 256):
        self.size = size
        self.orders: dict = {}

    @staticmethod
    def key(camera: Camera, device) -> tuple:
        return (str(device), int(camera.width), int(camera.height), float(camera.fx), float(camera.fy),
                float(camera.cx), float(camera.cy), tuple(np.asarray(camera.rotation, np.float64).reshape(-1)),
                tuple(np.asarray(camera.translation, np.float64).reshape(-1)))

    def get(self, key):
        return self.orders.get(key)

    def put(self, key, order) -> None:
        self.orders.pop(key, None)
        self.orders[key] = order
        while len(self.orders) > self.size:
            self.orders.pop(next(iter(self.orders)))


_tile_orders = _TileOrderCache()


class GaussianRasterizer(torch.autograd.Function):
    """Differentiable rasterizer: raw parameters + camera in; image (H,W,3)
    and radii (N,) int32 (0 = culled) out; gradients w.r.t. the raw means,
    log-scales, quaternions, opacity logits and SH coefficients back.

    Forward: one gs_forward call (projection, sync-free binning, blend) on
    the current stream, with the camera's previous longest-first tile order.
    The instance count and flags are copied to pinned host memory behind the
    binning; the backward checks them (by then the loss has consumed the
    image, so the wait is for work already done) and raises like the
    reference — InvalidPrimitiveError for a zero quaternion (core.py:164-165),
    ResourceLimitError past 2^31 instances (rasterizer.py:99-101) — or
    CapacityError when the frame outgrew the instance-buffer hint (the hint is
    raised; re-run the step).  The first frame of a frame size bins
    synchronously to learn its instance count.  The backward's tile schedule
    and gradient-row clearing are enqueued on a side stream at the end of the
    forward (prepare_backward), beside the caller's loss.  Backward: one
    gs_backward_prepared call (scheduled backward blend + backward_project,
    densify statistics when `stats` is given), or the deterministic blend when
    deterministic=True."""

    @staticmethod
    def forward(ctx, means, log_scales, rotations, opacity_logits, sh, camera, background, active_sh_degree=3,
                stats=None, deterministic=False):
        camera = _camera(camera)
        degree = int(active_sh_degree)
        if not 0 <= degree <= 3:
            raise ValueError(f"SH degree must be in 0..3, got {degree}")  # sh.py:37-38
        tensors = [t.detach().contiguous() for t in (means, log_scales, rotations, opacity_logits, sh)]
        params = c_params_from(*tensors)
        n, device = means.shape[0], means.device
        W, H = camera.width, camera.height
        hint = _capacity.key(device, W, H)
        okey = _TileOrderCache.key(camera, device)
        if hint not in _capacity.k:   # first frame of this size: learn K synchronously
            splats = _project_tensors(params, n, device, camera, degree)
            binning = bin_and_sort(splats, W, H)
            out = render_forward(splats, binning, W, H, background, training=True)
            k_report, k_event = None, None
        else:
            lib = _lib.load()
            cap = _capacity.get(hint, n)
            ws_bytes = _bin_workspace_bytes(n, W, H, cap)
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
            tiles_x, tiles_y = tile_extent(W, H)
            splats = DeviceSplats.empty(n, device)
            binning = TileBinning(torch.empty(max(cap, 1), dtype=torch.int32, device=device),
                                  torch.empty((tiles_x * tiles_y, 2), dtype=torch.int32, device=device), tiles_x,
                                  tiles_y, torch.empty(3, dtype=torch.int64, device=device), n, None, hint)
            f32 = dict(dtype=torch.float32, device=device)
            out = RenderOutput(torch.empty((H, W, 3), **f32), torch.empty((H, W), **f32),
                               torch.empty((H, W), dtype=torch.int32, device=device))
            scratch = torch.empty(2 + W * H, dtype=torch.int32, device=device)
            order = _tile_orders.get(okey)
            cs = splats.c_struct()
            _lib.check(lib.gs_forward(ctypes.byref(params), ctypes.byref(camera.to_c()), degree, ctypes.byref(cs),
                                      ws.data_ptr(), ws_bytes, cap, binning.splat_ids.data_ptr(),
                                      binning.ranges.data_ptr(), binning.k_info.data_ptr(), _bg(background), 1,
                                      _lib.ptr(order), out.image.data_ptr(), out.final_transmittance.data_ptr(),
                                      out.last_contributor.data_ptr(), scratch.data_ptr(), _stream()),
                       "render_view")
            k_report = torch.empty(3, dtype=torch.int64).pin_memory()
            k_report.copy_(binning.k_info, non_blocking=True)
            k_event = torch.cuda.Event()
            k_event.record(torch.cuda.current_stream(device))
        # the backward's tile schedule and row clearing on a side stream, beside
        # the caller's loss (gs_backward_prepared consumes them)
        ctx.prep = (prepare_backward(out, splats, binning, W, H)
                    if not deterministic and any(ctx.needs_input_grad[:5]) else None)
        ctx.save_for_backward(*tensors, splats.rec, splats.depth, splats.radii, splats.rect, splats.tiles_touched,
                              splats.status, binning.splat_ids, binning.ranges, out.final_transmittance,
                              out.last_contributor)
        ctx.camera, ctx.background, ctx.degree, ctx.stats = camera, background, degree, stats
        ctx.deterministic, ctx.okey = bool(deterministic), okey
        ctx.tiles, ctx.hint, ctx.k_report, ctx.k_event = (binning.tiles_x, binning.tiles_y), hint, k_report, k_event
        ctx.mark_non_differentiable(splats.radii)
        return out.image, splats.radii

    @staticmethod
    def backward(ctx, d_image, d_radii):
        (means, log_scales, rotations, opacity_logits, sh, rec, depth, radii, rect, tiles_touched, status,
         ids, ranges, t_final, last) = ctx.saved_tensors
        camera = ctx.camera
        if ctx.k_event is not None:   # the forward's deferred binning check
            ctx.k_event.synchronize()
            TileBinning(ids, ranges, *ctx.tiles, ctx.k_report, means.shape[0], None, ctx.hint).check_host(
                [int(v) for v in ctx.k_report.tolist()])
        splats = DeviceSplats(rec, depth, radii, rect, tiles_touched, status)
        n, device = means.shape[0], means.device
        d_image = d_image.to(dtype=torch.float32).contiguous()
        params = c_params_from(means, log_scales, rotations, opacity_logits, sh)
        z = dict(dtype=torch.float32, device=device)
        grads = GaussianGrads(torch.empty((n, 3), **z), torch.empty((n, 4), **z), torch.empty((n, 3), **z),
                              torch.empty(n, **z), torch.empty((n, 16, 3), **z), torch.empty(n, **z))
        if ctx.deterministic:
            g2 = render_backward(d_image, RenderOutput(None, t_final, last), splats, TileBinning(ids, ranges, *ctx.tiles),
                                 camera.width, camera.height, ctx.background, deterministic=True)
            _backward_project_tensors(params, n, device, camera, splats, g2, ctx.degree, ctx.stats, grads, False)
        else:
            tx, ty = ctx.tiles
            prep, ctx.prep = ctx.prep, None
            if prep is None:   # (no parameter required a gradient at forward time)
                prep = prepare_backward(RenderOutput(None, t_final, last), splats, TileBinning(ids, ranges, *ctx.tiles),
                                        camera.width, camera.height)
            cs, cg = splats.c_struct(), grads.c_struct()
            cst = ctx.stats.c_struct() if ctx.stats is not None else None
            torch.cuda.current_stream(device).wait_event(prep.done)
            _lib.check(_lib.load().gs_backward_prepared(
                d_image.data_ptr(), ctypes.byref(params), ctypes.byref(camera.to_c()), ctx.degree, ctypes.byref(cs),
                ids.data_ptr(), ranges.data_ptr(), t_final.data_ptr(), last.data_ptr(), _bg(ctx.background),
                prep.scratch.data_ptr(), prep.packed.data_ptr(), ctypes.byref(cg),
                ctypes.byref(cst) if cst is not None else None, _stream()), "render_backward")
            _tile_orders.put(ctx.okey, prep.scratch[:tx * ty])
        ctx.view_pos_grad_norm = grads.view_pos_grad_norm
        return (grads.d_means, grads.d_log_scales, grads.d_rotations, grads.d_opacity_logits, grads.d_sh,
                None, None, None, None, None)


def rasterize_gaussians(means, log_scales, rotations, opacity_logits, sh, camera, background=(0.0, 0.0, 0.0),
                        active_sh_degree: int = 3, stats: DensifyStats | None = None, deterministic: bool = False):
    """Functional form of GaussianRasterizer.apply -> (image, radii)."""
    return GaussianRasterizer.apply(means, log_scales, rotations, opacity_logits, sh, camera, background,
                                    active_sh_degree, stats, deterministic)
