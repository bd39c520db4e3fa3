"""Generate golden vectors by running the REFERENCE (splatlab) itself.

Run in the build container, where /root/reference exists:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
The outputs (tests/golden/*.npz) are committed; nothing at test or bench
time reads /root/reference.

Every scene is fed to the reference as the float64 image of float32 inputs
(the values the device sees).  For each scene the file holds the inputs,
the reference's project / bin_and_sort / render_forward(training) /
render_backward / backward_project outputs, the densification-statistics
update and two Adam steps (optimizer.py:252-257, 263-293).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

from splatlab.core import Camera as RefCamera, GaussianCloud, project  # noqa: E402
from splatlab.gradients import backward_project  # noqa: E402
from splatlab.optimizer import TrainConfig, TrainState, _adam_step, loss  # noqa: E402
from splatlab.rasterizer import bin_and_sort, render_backward, render_forward  # noqa: E402

sys.path.insert(0, str(REPO / "tests"))
from golden_scenes import SCENES, build, d_image_for, input_digest  # noqa: E402


def ref_camera(cam) -> RefCamera:
    return RefCamera(cam.rotation, cam.translation, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near)


def run_scene(name: str, cloud: dict, cam, degree: int, background, seed: int, compact: bool = False) -> None:
    """compact=True stores float outputs as float32, drops the Adam results,
    the 64-bit keys and the inputs (which the test regenerates from the
    seeded generator and checks against the stored SHA-256)."""
    gc = GaussianCloud(cloud["means"], cloud["rotations"], cloud["log_scales"], cloud["opacity_logits"],
                       cloud["sh"])
    rc = ref_camera(cam)
    W, H = rc.width, rc.height
    bg = np.asarray(background, dtype=np.float64)
    sp = project(gc, rc, degree)
    b = bin_and_sort(sp, W, H)
    out = render_forward(sp, b, W, H, bg, training=True)
    d_image = d_image_for(seed, W, H)
    g2 = render_backward(d_image, out, sp, b, W, H, bg)
    grads = backward_project(gc, rc, sp, g2, degree)

    # densification statistics exactly as train_step applies them
    n = len(gc)
    idx = sp.source_index
    accum = np.zeros(n)
    count = np.zeros(n, np.int64)
    maxr = np.zeros(n)
    accum[idx] += grads.view_pos_grad_norm[idx]
    count[idx] += 1
    np.maximum.at(maxr, idx, sp.radius / H)

    # two Adam steps with the same gradients (iterations 1 and 2)
    state = TrainState(gc.copy(), 1.0)
    config = TrainConfig(total_iters=1000)
    adam = {}
    for it in (1, 2):
        state.iteration = it
        _adam_step(state, grads, config)
        for g in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
            adam[f"adam{it}_{g}"] = getattr(state.cloud, g).copy()

    inputs = {k: cloud[k].astype(np.float32) for k in ("means", "rotations", "log_scales", "opacity_logits", "sh")}
    data = {
        "input_sha256": np.array(input_digest(inputs)),
        "cam_R": rc.rotation, "cam_t": rc.translation,
        "cam_intr": np.array([rc.fx, rc.fy, rc.cx, rc.cy, rc.near]), "cam_size": np.array([W, H]),
        "degree": np.array(degree), "background": bg,
        "source_index": sp.source_index, "radius": sp.radius, "mean2d": sp.mean2d, "conic": sp.conic,
        "depth": sp.depth, "color": sp.color, "alpha": sp.alpha, "color_active": sp.color_active,
        "keys": b.keys, "splat_ids": b.splat_ids.astype(np.int32), "ranges": b.ranges.astype(np.int64),
        "image": out.image, "t_final": out.final_transmittance, "last": out.last_contributor,
        "d_image": d_image.astype(np.float32),
        "g2_d_color": g2.d_color, "g2_d_alpha": g2.d_alpha, "g2_d_mean2d": g2.d_mean2d, "g2_d_conic": g2.d_conic,
        "d_means": grads.d_means, "d_rotations": grads.d_rotations,
        "d_log_scales": grads.d_log_scales, "d_opacity_logits": grads.d_opacity_logits,
        "d_sh": grads.d_sh, "view_pos_grad_norm": grads.view_pos_grad_norm,
        "stat_accum": accum, "stat_count": count, "stat_maxr": maxr,
    }
    if compact:
        data = {k: (v.astype(np.float32) if v.dtype == np.float64 and v.ndim > 0 and v.size > 16 else v)
                for k, v in data.items() if k not in ("keys",)}
    else:
        data.update(inputs)
        data.update(adam)
        # L1 + D-SSIM loss (optimizer.py:141-163) of the float32-rounded render
        # against a seeded float32 target image
        render32 = out.image.astype(np.float32).astype(np.float64)
        target = np.random.default_rng(seed + 100).uniform(0, 1, render32.shape).astype(np.float32)
        value, d_loss = loss(render32, target.astype(np.float64), 0.2)
        data.update({"loss_render": render32.astype(np.float32), "loss_target": target,
                     "loss_value": np.array(value), "loss_d_image": d_loss})
    np.savez_compressed(HERE / f"{name}.npz", **data)
    print(f"{name}: N={n} V={len(sp)} K={len(b.keys)} {W}x{H} deg={degree}")


def run_densify(name: str, iteration: int, extent: float, seed: int) -> None:
    """densify_and_prune (optimizer.py:304-374) on the scene_c cloud with
    seeded float32-representable statistics and moments."""
    from splatlab.optimizer import densify_and_prune
    cloud, cam, *_ = build("scene_c")
    gc = GaussianCloud(cloud["means"], cloud["rotations"], cloud["log_scales"], cloud["opacity_logits"], cloud["sh"])
    n = len(gc)
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    state = TrainState(gc, extent, seed=seed)
    state.iteration = iteration
    state.accum_count = rng.integers(0, 4, n).astype(np.int64)
    state.accum_pos_grad = f32(rng.uniform(0.0, 0.0006, n) * state.accum_count)
    state.max_radius_frac = f32(rng.uniform(0.0, 0.7, n))
    moments = {}
    for g in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
        state.exp_avg[g] = f32(rng.normal(size=getattr(gc, g).shape))
        state.exp_avg_sq[g] = f32(rng.uniform(0, 1, getattr(gc, g).shape))
        moments[f"in_m_{g}"], moments[f"in_v_{g}"] = state.exp_avg[g].copy(), state.exp_avg_sq[g].copy()
    stats_in = {"in_accum": state.accum_pos_grad.copy(), "in_count": state.accum_count.copy(),
                "in_maxr": state.max_radius_frac.copy()}
    rep = densify_and_prune(state, TrainConfig(total_iters=30000))
    out = {"iteration": np.array(iteration), "extent": np.array(extent), "seed": np.array(seed),
           "cloned": np.array(rep.cloned), "split": np.array(rep.split), "pruned": np.array(rep.pruned),
           "opacity_reset": np.array(rep.opacity_reset), **stats_in, **moments}
    for g in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
        out[f"out_{g}"] = getattr(state.cloud, g)
        out[f"out_m_{g}"] = state.exp_avg[g]
        out[f"out_v_{g}"] = state.exp_avg_sq[g]
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: N={n} -> {len(state.cloud)} cloned={rep.cloned} split={rep.split} pruned={rep.pruned} "
          f"reset={rep.opacity_reset}")


def main() -> None:
    for name in SCENES:
        cloud, cam, degree, bg, seed, compact = build(name)
        run_scene(name, cloud, cam, degree, bg, seed, compact=compact)
    run_densify("densify_a", iteration=600, extent=10.0, seed=21)
    run_densify("densify_b", iteration=6000, extent=6.0, seed=22)


if __name__ == "__main__":
    main()
