"""Parity at the benchmark configurations (BASELINE.json configs, SURVEY
§8(d)) against the float64 oracle (pinned to splatlab by
test_oracle_golden.py):

* c3 — 3M SH3 Gaussians, 1920x1080, the benchmarked training step: project,
  bin, blend, L1 + D-SSIM (lambda 0.2), blend backward, projection backward,
  densify statistics and the fused Adam at iteration 1, each stage against the
  oracle run independently on the same float32-representable inputs;
* c2 — 1M Gaussians, 1080p forward render;
* c5 — 6M Gaussians at 4K: radii, tile counts, sorted ids and tile ranges
  (171M instances).

Tolerances are SURVEY §8(c)'s: integers bit-exact, every last contributor
equal (the stop decisions are the reference's), image and final
transmittance <= 1e-4, gradient groups ||d - ref|| / ||ref|| <= 1e-3.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_04079_b200 import rasterizer as R
from paper_2308_04079_b200 import synthetic
from paper_2308_04079_b200.cloud import GaussianCloud
from paper_2308_04079_b200.loss import l1_dssim_loss
from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
from parity_utils import forward_parity

pytestmark = pytest.mark.gpu

GROUPS = (("means", "d_means"), ("log_scales", "d_log_scales"), ("rotations", "d_rotations"),
          ("opacity_logits", "d_opacity_logits"), ("sh", "d_sh"))


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_c3_training_step_vs_oracle(cuda_device):
    w, h, bg = 1920, 1080, (0.0, 0.0, 0.0)
    cloud_np, cam = synthetic.frustum_scene(3_000_000, w, h, seed=0)
    cloud_np = synthetic.round_to_f32(cloud_np)
    tgt_np, _ = synthetic.frustum_scene(3_000_000, w, h, seed=1)
    target = R.render_view(GaussianCloud.from_numpy(**tgt_np), cam, bg, 3)[0].image
    del tgt_np
    cfg = TrainConfig()

    # device: the benchmarked step's stages
    cloud = GaussianCloud.from_numpy(**cloud_np)
    out, splats, binning = R.render_view(cloud, cam, bg, 3, training=True)
    loss, d_image = l1_dssim_loss(out.image, target, cfg.lambda_dssim)
    g2 = R.render_backward(d_image, out, splats, binning, w, h, bg)
    stats = R.DensifyStats.zeros(len(cloud), "cuda")
    grads = R.backward_project(cloud, cam, splats, g2, 3, stats=stats)
    DeviceAdam(cloud).step(cloud, grads, 1, cfg)
    torch.cuda.synchronize()

    # oracle: the same chain in float64
    proj = O.project(cloud_np, cam, 3)
    np.testing.assert_array_equal(splats.radii.cpu().numpy(), proj["radius"])
    np.testing.assert_array_equal(splats.tiles_touched.cpu().numpy(), proj["tiles"])
    bins = O.bin_and_sort(proj, w, h, with_keys=False)
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), bins["ranges"])
    np.testing.assert_array_equal(binning.splat_ids.cpu().numpy(), bins["ids"])
    fwd = O.render_forward(proj, bins, w, h, bg)
    report = forward_parity(out.image.cpu().numpy(), out.final_transmittance.cpu().numpy(),
                            out.last_contributor.cpu().numpy(), fwd["image"], fwd["t_final"], fwd["last"])
    print("c3 forward parity:", report)
    # float32 transmittance error at the stop (what kSatGuard must cover)
    t_dev = out.final_transmittance.cpu().numpy().astype(np.float64)
    stopped = fwd["t_final"] < 2e-4
    print("c3 saturated pixels:", int(stopped.sum()), "max rel T error:",
          float(np.abs(t_dev[stopped] / fwd["t_final"][stopped] - 1).max()))
    tgt = target.cpu().numpy().astype(np.float64)
    oloss, od_image = O.l1_dssim_loss(fwd["image"], tgt, cfg.lambda_dssim)
    lv = loss.cpu().numpy()
    assert abs(lv[0] - oloss[0]) <= 1e-5 * abs(oloss[0]), (lv, oloss)
    assert np.abs(d_image.cpu().numpy() - od_image).max() <= 1e-4 * np.abs(od_image).max()
    og2 = O.render_backward(od_image, proj, bins, fwd, w, h, bg)
    del bins
    p = g2.packed.cpu().numpy()
    assert rel(g2.d_mean2d.cpu().numpy(), og2[:, 0:2]) < 1e-3
    assert rel(g2.d_alpha.cpu().numpy(), og2[:, 5]) < 1e-3        # S0 / alpha
    assert rel(g2.d_conic.cpu().numpy(), og2[:, 2:5]) < 1e-3
    assert rel(p[:, 8:11], og2[:, 6:9]) < 1e-3
    ograds = O.backward_project(cloud_np, cam, 3, proj, og2)
    surv = proj["radius"] > 0
    np.testing.assert_array_equal(stats.accum_count.cpu().numpy(), surv.astype(np.int32))
    assert rel(stats.accum_pos_grad.cpu().numpy(), ograds["view_pos_grad_norm"]) < 1e-3
    for name, key in GROUPS:
        assert rel(getattr(grads, key).cpu().numpy(), ograds[key]) < 1e-3, key
    # Adam at t = 1 moves every element by lr * g / (|g| + eps), i.e. by the
    # gradient's sign: compared where the reference gradient is determined
    # (|g| above the SURVEY §8(c) elementwise floor of 1e-3 max|g|)
    for name, key in GROUPS:
        p0 = cloud_np[name].astype(np.float64)
        pr = p0.copy()
        m, v = np.zeros_like(pr), np.zeros_like(pr)
        if name == "means":
            O.adam_group(pr, ograds[key], m, v, cfg.lr_means_at(1), *cfg.adam_betas, cfg.adam_eps, 1)
        elif name == "sh":
            O.adam_group(pr, ograds[key], m, v, cfg.lr_sh_rest, *cfg.adam_betas, cfg.adam_eps, 1,
                         lr_head=cfg.lr_sh_dc, period=48, head=3)
        else:
            lr = {"log_scales": cfg.lr_log_scales, "rotations": cfg.lr_rotations, "opacity_logits": cfg.lr_opacity}
            O.adam_group(pr, ograds[key], m, v, lr[name], *cfg.adam_betas, cfg.adam_eps, 1)
        got = getattr(cloud, name).cpu().numpy().astype(np.float64)
        g_ref = np.asarray(ograds[key], np.float64).reshape(pr.shape)
        sure = np.abs(g_ref) > 1e-3 * np.abs(g_ref).max()
        assert sure.sum() > 1000, name
        err = np.abs(got - pr)[sure]
        assert err.max() <= 2e-6 * max(1.0, np.abs(pr).max()), (name, float(err.max()))


def test_c2_forward_vs_oracle(cuda_device):
    w, h, bg = 1920, 1080, (0.1, 0.2, 0.3)
    cloud_np, cam = synthetic.frustum_scene(1_000_000, w, h, seed=0)
    cloud_np = synthetic.round_to_f32(cloud_np)
    out, splats, binning = R.render_view(GaussianCloud.from_numpy(**cloud_np), cam, bg, 3, training=True)
    proj = O.project(cloud_np, cam, 3)
    np.testing.assert_array_equal(splats.radii.cpu().numpy(), proj["radius"])
    bins = O.bin_and_sort(proj, w, h, with_keys=False)
    np.testing.assert_array_equal(binning.splat_ids.cpu().numpy(), bins["ids"])
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), bins["ranges"])
    fwd = O.render_forward(proj, bins, w, h, bg)
    report = forward_parity(out.image.cpu().numpy(), out.final_transmittance.cpu().numpy(),
                            out.last_contributor.cpu().numpy(), fwd["image"], fwd["t_final"], fwd["last"])
    print("c2 forward parity:", report)
    # the inference render (no training record) agrees too
    inf = R.render_view(GaussianCloud.from_numpy(**cloud_np), cam, bg, 3)[0].image.cpu().numpy()
    assert np.abs(inf - fwd["image"]).max() <= 2e-4


def test_c5_binning_vs_oracle(cuda_device):
    w, h = 3840, 2160
    cloud_np, cam = synthetic.frustum_scene(6_000_000, w, h, seed=0)
    cloud_np = synthetic.round_to_f32(cloud_np)
    splats = R.project(GaussianCloud.from_numpy(**cloud_np), cam, 3)
    binning = R.bin_and_sort(splats, w, h)
    proj = O.project(cloud_np, cam, 3)
    del cloud_np
    np.testing.assert_array_equal(splats.radii.cpu().numpy(), proj["radius"])
    np.testing.assert_array_equal(splats.tiles_touched.cpu().numpy(), proj["tiles"])
    bins = O.bin_and_sort(proj, w, h, with_keys=False)
    assert binning.num_instances == bins["ids"].shape[0] > 150_000_000
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), bins["ranges"])
    np.testing.assert_array_equal(binning.splat_ids.cpu().numpy(), bins["ids"])
