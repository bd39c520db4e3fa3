"""TEST INFRASTRUCTURE ONLY — numpy front end of the float64 C oracle.

The oracle restates splatlab's hot path on the CPU (see gs_oracle.c for the
file:line of every step).  Only tests/, __graft_entry__.smoke() and the CPU
baseline legs of bench.py may import this module; the product package never
does.

Every function takes/returns float64 numpy arrays in the reference layouts;
per-Gaussian outputs are in N-space (row g = Gaussian g, radius 0 = culled),
instance ids index Gaussians.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int, c_int32, c_int64
from pathlib import Path

import numpy as np

from . import build_oracle

TILE = 16
_lib = None


class OrCamera(ctypes.Structure):
    _fields_ = [("R", c_double * 9), ("t", c_double * 3), ("fx", c_double), ("fy", c_double), ("cx", c_double),
                ("cy", c_double), ("width", c_int32), ("height", c_int32), ("near_plane", c_double)]


def _p(a, ct=c_double):
    return a.ctypes.data_as(POINTER(ct))


def lib():
    global _lib
    if _lib is None:
        path = build_oracle.LIB if build_oracle.LIB.exists() else build_oracle.build()
        _lib = ctypes.CDLL(str(path))
        _lib.or_bin_count.restype = c_int64
        _lib.or_num_threads.restype = c_int
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def num_threads() -> int:
    return int(lib().or_num_threads())


def _cam(camera) -> OrCamera:
    c = OrCamera()
    c.R[:] = [float(v) for v in np.asarray(camera.rotation, dtype=np.float64).reshape(-1)]
    c.t[:] = [float(v) for v in np.asarray(camera.translation, dtype=np.float64).reshape(-1)]
    c.fx, c.fy, c.cx, c.cy = float(camera.fx), float(camera.fy), float(camera.cx), float(camera.cy)
    c.width, c.height, c.near_plane = int(camera.width), int(camera.height), float(camera.near)
    return c


def _f64(a, shape):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(shape))


def params_f64(cloud) -> dict:
    """Raw parameters (any object/dict with the reference's field names) as float64."""
    get = (lambda k: cloud[k]) if isinstance(cloud, dict) else (lambda k: getattr(cloud, k))
    means = get("means")
    if hasattr(means, "detach"):
        get0 = get
        get = lambda k: get0(k).detach().cpu().numpy()  # noqa: E731
    n = np.asarray(get("means")).reshape(-1, 3).shape[0]
    return {"means": _f64(get("means"), (n, 3)), "rotations": _f64(get("rotations"), (n, 4)),
            "log_scales": _f64(get("log_scales"), (n, 3)), "opacity_logits": _f64(get("opacity_logits"), (n,)),
            "sh": _f64(get("sh"), (n, 16, 3))}


def project(params: dict, camera, degree: int = 3) -> dict:
    """core.project (core.py:266-345) + rasterizer tile rectangles, N-space."""
    n = params["means"].shape[0]
    out = {"radius": np.zeros(n, np.int32), "mean2d": np.zeros((n, 2)), "conic": np.zeros((n, 3)),
           "depth": np.zeros(n), "color": np.zeros((n, 3)), "color_mask": np.zeros(n, np.int32),
           "alpha": np.zeros(n), "rect": np.zeros((n, 4), np.int32), "tiles": np.zeros(n, np.int64)}
    cam = _cam(camera)
    err = lib().or_project(c_int64(n), _p(params["means"]), _p(params["rotations"]), _p(params["log_scales"]),
                           _p(params["opacity_logits"]), _p(params["sh"]), ctypes.byref(cam), c_int(degree),
                           _p(out["radius"], c_int32), _p(out["mean2d"]), _p(out["conic"]), _p(out["depth"]),
                           _p(out["color"]), _p(out["color_mask"], c_int32), _p(out["alpha"]),
                           _p(out["rect"], c_int32), _p(out["tiles"], c_int64))
    out["zero_quaternion"] = bool(err & 2)
    return out


def bin_and_sort(proj: dict, width: int, height: int, with_keys: bool = True) -> dict:
    """rasterizer.bin_and_sort (rasterizer.py:69-124); ids are Gaussian indices.
    with_keys=False skips the (K,) uint64 keys (large frames)."""
    n = proj["radius"].shape[0]
    tx, ty = (width + TILE - 1) // TILE, (height + TILE - 1) // TILE
    k = int(lib().or_bin_count(c_int64(n), _p(proj["tiles"], c_int64)))
    keys = np.zeros(max(k, 1), np.uint64) if with_keys else None
    ids = np.zeros(max(k, 1), np.int32)
    ranges = np.zeros((tx * ty, 2), np.int64)
    lib().or_bin_fill(c_int64(n), _p(proj["rect"], c_int32), _p(proj["tiles"], c_int64), _p(proj["depth"]),
                      c_int(tx), c_int64(tx * ty), None if keys is None else _p(keys, ctypes.c_uint64),
                      _p(ids, c_int32), _p(ranges, c_int64))
    return {"keys": None if keys is None else keys[:k], "ids": ids[:k], "ranges": ranges, "tiles_x": tx,
            "tiles_y": ty}


def render_forward(proj: dict, bins: dict, width: int, height: int, background) -> dict:
    """rasterizer.render_forward (rasterizer.py:201-240), training record included."""
    bg = _f64(background, (3,))
    image = np.zeros((height, width, 3))
    t_final = np.zeros((height, width))
    last = np.zeros((height, width), np.int64)
    ids = np.ascontiguousarray(bins["ids"], dtype=np.int32)
    lib().or_render_forward(_p(proj["mean2d"]), _p(proj["conic"]), _p(proj["alpha"]), _p(proj["color"]),
                            _p(ids, c_int32), _p(bins["ranges"], c_int64), c_int(width), c_int(height), _p(bg),
                            _p(image), _p(t_final), _p(last, c_int64))
    return {"image": image, "t_final": t_final, "last": last}


def render_backward(d_image, proj: dict, bins: dict, fwd: dict, width: int, height: int, background) -> np.ndarray:
    """render_backward + backward_blend (rasterizer.py:253-316, gradients.py:30-94).

    Returns (N,9): d_mean2d x,y | d_conic a,b,c | d_alpha | d_color r,g,b."""
    bg = _f64(background, (3,))
    d = _f64(d_image, (height, width, 3))
    n = proj["radius"].shape[0]
    out = np.zeros((n, 9))
    ids = np.ascontiguousarray(bins["ids"], dtype=np.int32)
    lib().or_render_backward(_p(d), _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["alpha"]), _p(proj["color"]),
                             _p(ids, c_int32), _p(bins["ranges"], c_int64), _p(fwd["t_final"]),
                             _p(fwd["last"], c_int64), c_int(width), c_int(height), _p(bg), c_int64(n), _p(out))
    return out


def backward_project(params: dict, camera, degree: int, proj: dict, grads2d: np.ndarray) -> dict:
    """gradients.backward_project (gradients.py:192-259), N-space."""
    n = params["means"].shape[0]
    out = {"d_means": np.zeros((n, 3)), "d_rotations": np.zeros((n, 4)), "d_log_scales": np.zeros((n, 3)),
           "d_opacity_logits": np.zeros(n), "d_sh": np.zeros((n, 16, 3)), "view_pos_grad_norm": np.zeros(n)}
    g2 = _f64(grads2d, (n, 9))
    cam = _cam(camera)
    lib().or_backward_project(c_int64(n), _p(params["means"]), _p(params["rotations"]), _p(params["log_scales"]),
                              _p(params["opacity_logits"]), _p(params["sh"]), ctypes.byref(cam), c_int(degree),
                              _p(proj["radius"], c_int32), _p(proj["color_mask"], c_int32), _p(g2),
                              _p(out["d_means"]), _p(out["d_rotations"]), _p(out["d_log_scales"]),
                              _p(out["d_opacity_logits"]), _p(out["d_sh"]), _p(out["view_pos_grad_norm"]))
    return out


def stats_update(proj: dict, norm: np.ndarray, height: int, stats: dict) -> None:
    """In-place densification statistics (optimizer.py:252-255)."""
    n = proj["radius"].shape[0]
    lib().or_stats_update(c_int64(n), _p(proj["radius"], c_int32), _p(_f64(norm, (n,))), c_int(height),
                          _p(stats["accum_pos_grad"]), _p(stats["accum_count"], c_int64),
                          _p(stats["max_radius_frac"]))


def adam_group(p, grad, m, v, lr, beta1, beta2, eps, t, lr_head=None, period=0, head=0) -> None:
    """In-place dense Adam on one group (optimizer.py:284-293)."""
    for a in (p, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = _f64(grad, p.shape)
    lib().or_adam(c_int64(p.size), _p(p), _p(g), _p(m), _p(v), c_double(lr),
                  c_double(lr if lr_head is None else lr_head), c_int(period), c_int(head), c_double(beta1),
                  c_double(beta2), c_double(eps), c_int64(t))


def render_view(params: dict, camera, background, degree: int = 3) -> tuple[dict, dict, dict]:
    proj = project(params, camera, degree)
    bins = bin_and_sort(proj, int(camera.width), int(camera.height))
    fwd = render_forward(proj, bins, int(camera.width), int(camera.height), background)
    return fwd, proj, bins


def to_reference_order(proj: dict, bins: dict) -> dict:
    """Express N-space binning in the reference's survivor-compacted ids."""
    surv = np.nonzero(proj["radius"] > 0)[0]
    remap = -np.ones(proj["radius"].shape[0], np.int64)
    remap[surv] = np.arange(surv.shape[0])
    return {"keys": bins["keys"], "splat_ids": remap[bins["ids"]], "ranges": bins["ranges"],
            "source_index": surv}


__all__ = ["project", "bin_and_sort", "render_forward", "render_backward", "backward_project", "stats_update",
           "adam_group", "render_view", "params_f64", "to_reference_order", "set_threads", "num_threads"]
_here = Path(__file__).resolve().parent


def l1_dssim_loss(render, ground_truth, lambda_dssim: float = 0.2) -> tuple[np.ndarray, np.ndarray]:
    """optimizer.loss (optimizer.py:141-163): ([loss, mean L1, mean SSIM], d_image)."""
    x = np.ascontiguousarray(np.asarray(render, dtype=np.float64))
    y = np.ascontiguousarray(np.asarray(ground_truth, dtype=np.float64))
    if x.shape != y.shape:
        raise ValueError(f"resolution mismatch: {x.shape} vs {y.shape}")
    h, w = x.shape[0], x.shape[1]
    out = np.zeros(3)
    d = np.zeros_like(x)
    lib().or_l1_dssim(_p(x), _p(y), c_int(h), c_int(w), c_double(lambda_dssim), _p(out), _p(d))
    return out, d
