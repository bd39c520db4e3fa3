"""GPU parity: the CUDA path through the C ABI against the float64 oracle
(pinned to the reference by test_oracle_golden.py) and the golden vectors.

Tolerances (north_star / SURVEY §8(c)):
  radii, culled set, depth keys, sorted ids, tile ranges, last contributor: bit-exact
  image / final transmittance: max-abs <= 1e-4
  screen-space and parameter gradients: ||d - ref|| / ||ref|| <= 1e-3 per group
"""
import numpy as np
import pytest
import torch

import golden_scenes
from parity_utils import forward_parity
from oracle import oracle as O
from paper_2308_04079_b200 import rasterizer as R
from paper_2308_04079_b200.cloud import GaussianCloud
from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-3


def rel(a, b, floor=1e-30):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor))


def device_pipeline(cloud_np, cam, degree, bg, d_image):
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, degree)
    binning = R.bin_and_sort(splats, cam.width, cam.height)
    out = R.render_forward(splats, binning, cam.width, cam.height, bg, training=True)
    g2 = R.render_backward(torch.from_numpy(np.asarray(d_image, np.float32)).cuda(), out, splats, binning,
                           cam.width, cam.height, bg)
    stats = R.DensifyStats.zeros(len(cloud), "cuda")
    grads = R.backward_project(cloud, cam, splats, g2, degree, stats=stats)
    torch.cuda.synchronize()
    return cloud, splats, binning, out, g2, grads, stats


def oracle_pipeline(cloud_np, cam, degree, bg, d_image):
    proj = O.project(cloud_np, cam, degree)
    bins = O.bin_and_sort(proj, cam.width, cam.height)
    fwd = O.render_forward(proj, bins, cam.width, cam.height, bg)
    g2 = O.render_backward(d_image, proj, bins, fwd, cam.width, cam.height, bg)
    grads = O.backward_project(cloud_np, cam, degree, proj, g2)
    return proj, bins, fwd, g2, grads


def check_against_oracle(dev, orc, floor_scale=1e-9, grad_tol=None):
    cloud, splats, binning, out, g2, grads, stats = dev
    proj, bins, fwd, og2, ograds = orc
    radii = splats.radii.cpu().numpy()
    np.testing.assert_array_equal(radii, proj["radius"])
    surv = radii > 0
    np.testing.assert_array_equal(splats.depth.cpu().numpy()[surv], proj["depth"][surv].astype(np.float32))
    np.testing.assert_array_equal(splats.tiles_touched.cpu().numpy(), proj["tiles"])
    # float projections (float32 storage)
    m2 = splats.mean2d.cpu().numpy()[surv]
    assert np.abs(m2 - proj["mean2d"][surv]).max() <= 1e-9 * max(1.0, np.abs(proj["mean2d"]).max())
    assert rel(splats.conic.cpu().numpy()[surv], proj["conic"][surv]) < 1e-6
    assert rel(splats.color.cpu().numpy()[surv], proj["color"][surv]) < 1e-5
    assert rel(splats.alpha.cpu().numpy()[surv], proj["alpha"][surv]) < 1e-6
    # binning: bit-exact
    np.testing.assert_array_equal(binning.splat_ids.cpu().numpy(), bins["ids"])
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), bins["ranges"])
    # forward: every stop decision the reference's (see parity_utils)
    forward_parity(out.image.cpu().numpy(), out.final_transmittance.cpu().numpy(),
                   out.last_contributor.cpu().numpy(), fwd["image"], fwd["t_final"], fwd["last"],
                   color_max=float(proj["color"].max(initial=1.0)))
    # backward blend: packed rows vs oracle's (N,9)
    p = g2.packed.cpu().numpy()
    assert rel(g2.d_mean2d.cpu().numpy(), og2[:, 0:2]) < GRAD_TOL
    assert rel(g2.d_alpha.cpu().numpy(), og2[:, 5]) < GRAD_TOL        # S0 / alpha
    assert rel(g2.d_conic.cpu().numpy(), og2[:, 2:5]) < GRAD_TOL   # from the eigenbasis moments
    assert rel(p[:, 8:11], og2[:, 6:9]) < GRAD_TOL
    # parameter gradients
    floor = floor_scale * max(np.linalg.norm(ograds[k]) for k in ("d_means", "d_log_scales", "d_sh"))
    for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh", "view_pos_grad_norm"):
        got = getattr(grads, key).cpu().numpy()
        tol = (grad_tol or {}).get(key, GRAD_TOL)
        assert rel(got, ograds[key], floor) < tol, (key, rel(got, ograds[key], floor))
        assert np.all(got[~surv] == 0.0), f"{key}: culled rows must be exactly zero"
    # densification statistics
    np.testing.assert_array_equal(stats.accum_count.cpu().numpy(), surv.astype(np.int32))
    assert rel(stats.accum_pos_grad.cpu().numpy(), ograds["view_pos_grad_norm"], floor) < GRAD_TOL
    expect_frac = np.where(surv, proj["radius"] / out.image.shape[0], 0.0)
    np.testing.assert_allclose(stats.max_radius_frac.cpu().numpy(), expect_frac, rtol=1e-6)


@pytest.mark.parametrize("name", list(golden_scenes.SCENES))
def test_golden_scene_vs_oracle(cuda_device, name):
    g, cloud_np, cam = golden_scenes.load(name)
    degree, bg = int(g["degree"]), g["background"]
    d_image = golden_scenes.d_image_for(golden_scenes.SCENES[name]()[4], cam.width, cam.height)
    dev = device_pipeline(cloud_np, cam, degree, bg, d_image)
    orc = oracle_pipeline(cloud_np, cam, degree, bg, d_image)
    check_against_oracle(dev, orc)
    # and directly against the reference's own outputs
    cloud, splats, binning, out, *_ = dev
    surv = splats.radii.cpu().numpy() > 0
    np.testing.assert_array_equal(np.nonzero(surv)[0], g["source_index"])
    np.testing.assert_array_equal(splats.radii.cpu().numpy()[surv], g["radius"])
    forward_parity(out.image.cpu().numpy(), out.final_transmittance.cpu().numpy(),
                   out.last_contributor.cpu().numpy(), g["image"], g["t_final"], g["last"],
                   color_max=float(np.max(g["color"], initial=1.0)))
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), g["ranges"])
    ref_ids = O.to_reference_order({"radius": splats.radii.cpu().numpy()},
                                   {"keys": None, "ids": binning.splat_ids.cpu().numpy(),
                                    "ranges": None})["splat_ids"]
    np.testing.assert_array_equal(ref_ids, g["splat_ids"])


@pytest.mark.parametrize("seed,n,w,h,deg", [(100, 1, 16, 16, 0), (101, 7, 33, 17, 1), (102, 257, 64, 64, 2),
                                            (103, 2000, 128, 72, 3), (104, 5000, 250, 130, 3)])
def test_random_scenes_vs_oracle(cuda_device, seed, n, w, h, deg):
    from paper_2308_04079_b200 import synthetic
    cloud_np, cam = synthetic.random_splat_scene(np.random.default_rng(seed), n, w, h)
    cloud_np = synthetic.round_to_f32(cloud_np)
    bg = np.random.default_rng(seed).uniform(0, 1, 3)
    d_image = golden_scenes.d_image_for(seed, w, h)
    check_against_oracle(device_pipeline(cloud_np, cam, deg, bg, d_image),
                         oracle_pipeline(cloud_np, cam, deg, bg, d_image))


def test_adam_matches_oracle(cuda_device):
    g, cloud_np, cam = golden_scenes.load("scene_b")
    cloud = GaussianCloud.from_numpy(**cloud_np)
    grads = R.GaussianGrads.zeros(len(cloud), "cuda")
    for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        getattr(grads, key).copy_(torch.from_numpy(g[key].astype(np.float32)))
    opt = DeviceAdam(cloud)
    cfg = TrainConfig(total_iters=1000)
    for it in (1, 2):
        opt.step(cloud, grads, it, cfg)
        torch.cuda.synchronize()
        for k in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
            got = getattr(cloud, k).cpu().numpy().astype(np.float64)
            ref = g[f"adam{it}_{k}"]
            # one Adam step moves each value by at most lr; f32 storage of the value dominates
            assert np.abs(got - ref).max() <= 2e-6 * max(1.0, np.abs(ref).max()), k


def test_empty_cloud(cuda_device):
    from paper_2308_04079_b200.camera import Camera
    cam = Camera(np.eye(3), np.zeros(3), 32.0, 32.0, 16.0, 12.0, 32, 24)
    cloud = GaussianCloud.from_numpy(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                                     np.zeros((0, 16, 3)))
    out, splats, binning = R.render_view(cloud, cam, (0.2, 0.3, 0.4), training=True)
    img = out.image.cpu().numpy()
    np.testing.assert_allclose(img, np.broadcast_to(np.float32([0.2, 0.3, 0.4]), img.shape))
    assert np.all(out.final_transmittance.cpu().numpy() == 1.0)
    assert np.all(out.last_contributor.cpu().numpy() == -1)
    assert binning.num_instances == 0


def test_zero_quaternion_raises(cuda_device):
    from paper_2308_04079_b200.errors import InvalidPrimitiveError
    from paper_2308_04079_b200.camera import Camera
    cam = Camera(np.eye(3), np.zeros(3), 100.0, 100.0, 16.0, 16.0, 32, 32, near=0.1)
    sh = np.zeros((1, 16, 3))
    cloud = GaussianCloud.from_numpy([[0.0, 0.0, 10.0]], [[0.0, 0, 0, 0]], [[0.0, 0, 0]], [2.0], sh)
    with pytest.raises(InvalidPrimitiveError):
        R.project(cloud, cam)
    with pytest.raises(InvalidPrimitiveError):
        R.render_view(cloud, cam, (0, 0, 0))
    # behind the camera it is culled before normalisation: no error (core.py:281-295)
    behind = GaussianCloud.from_numpy([[0.0, 0.0, -10.0]], [[0.0, 0, 0, 0]], [[0.0, 0, 0]], [2.0], sh)
    R.render_view(behind, cam, (0, 0, 0))


def test_on_axis_projection_kat(cuda_device):
    # test_core.py:100-108: unit covariance at depth 10, f=100 -> conic 1/100.3, radius ceil(3 sqrt(100.3))
    from paper_2308_04079_b200.camera import Camera
    cam = Camera(np.eye(3), np.zeros(3), 100.0, 100.0, 16.0, 16.0, 32, 32, near=0.1)
    cloud = GaussianCloud.from_numpy([[0.0, 0.0, 10.0]], [[1.0, 0, 0, 0]], [[0.0, 0, 0]], [2.0],
                                     np.zeros((1, 16, 3)))
    sp = R.project(cloud, cam)
    np.testing.assert_allclose(sp.conic.cpu().numpy()[0], [1 / 100.3, 0.0, 1 / 100.3], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(sp.mean2d.cpu().numpy()[0], [16.0, 16.0])
    assert int(sp.radii[0]) == int(np.ceil(3 * np.sqrt(100.3)))
    np.testing.assert_allclose(float(sp.alpha[0]), 1 / (1 + np.exp(-2.0)), rtol=1e-6)
    np.testing.assert_allclose(sp.color.cpu().numpy()[0], [0.5, 0.5, 0.5])


def test_guard_band_and_near_cull(cuda_device):
    # test_core.py:118-129
    from paper_2308_04079_b200.camera import Camera
    cam = Camera(np.eye(3), np.zeros(3), 100.0, 100.0, 16.0, 16.0, 32, 32, near=0.1)
    z = 10.0
    xs = [1.2 * 16 * z / 100.0, 1.4 * 16 * z / 100.0]
    cloud = GaussianCloud.from_numpy([[xs[0], 0, z], [xs[1], 0, z], [0, 0, 0.05]], [[1.0, 0, 0, 0]] * 3,
                                     np.zeros((3, 3)), np.zeros(3), np.zeros((3, 16, 3)))
    r = R.project(cloud, cam).radii.cpu().numpy()
    assert r[0] > 0 and r[1] == 0 and r[2] == 0


def wide(depth, color, alpha, w=32, h=32):
    return dict(mean2d=[w / 2.0, h / 2.0], conic=[1e-8, 0.0, 1e-8], depth=depth, color=color, alpha=alpha,
                radius=10 * max(w, h))


def stack(specs, w, h):
    return R.DeviceSplats.from_projected([s["mean2d"] for s in specs], [s["conic"] for s in specs],
                                         [s["depth"] for s in specs], [s["color"] for s in specs],
                                         [s["alpha"] for s in specs], [s["radius"] for s in specs], w, h)


def test_two_coincident_splats_blend(cuda_device):
    # test_rasterizer.py:122-128: 0.5 red over 0.5 green on black -> (0.5, 0.25, 0)
    sp = stack([wide(1.0, [1, 0, 0], 0.5), wide(2.0, [0, 1, 0], 0.5)], 32, 32)
    b = R.bin_and_sort(sp, 32, 32)
    out = R.render_forward(sp, b, 32, 32, (0, 0, 0))
    np.testing.assert_allclose(out.image.cpu().numpy()[16, 16], [0.5, 0.25, 0.0], atol=1e-6)
    out = R.render_forward(sp, b, 32, 32, (1, 1, 1))
    np.testing.assert_allclose(out.image.cpu().numpy()[16, 16], [0.5 + 0.25, 0.25 + 0.25, 0.25], atol=1e-6)


def test_saturation_stop(cuda_device):
    # test_rasterizer.py:174-187: 64 near-opaque layers
    sp = stack([wide(float(i + 1), [1, 1, 1], 0.97) for i in range(64)], 32, 32)
    b = R.bin_and_sort(sp, 32, 32)
    out = R.render_forward(sp, b, 32, 32, (0, 0, 0), training=True)
    tf = out.final_transmittance.cpu().numpy()
    assert np.all(np.isfinite(out.image.cpu().numpy()))
    assert np.all(1.0 - tf <= 0.9999 + 1e-6)
    last = out.last_contributor.cpu().numpy()
    ranges = b.ranges.cpu().numpy()
    for tile in range(4):
        start = ranges[tile, 0]
        ty, tx = divmod(tile, 2)
        block = last[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        assert np.all(block >= start) and np.all(block - start < 10)


def test_saturated_back_splat_gets_no_grad(cuda_device):
    # test_gradients.py:114-127
    specs = [wide(1.0, [1, 0, 0], 0.97) for _ in range(8)] + [wide(9.0, [0, 1, 0], 0.9)]
    sp = stack(specs, 32, 32)
    b = R.bin_and_sort(sp, 32, 32)
    out = R.render_forward(sp, b, 32, 32, (0, 0, 0), training=True)
    g2 = R.render_backward(torch.ones((32, 32, 3), device="cuda"), out, sp, b, 32, 32, (0, 0, 0))
    p = g2.packed.cpu().numpy()
    assert np.all(p[8] == 0.0)
    assert np.any(p[0, 8:11] != 0.0)


def test_adversarial_alphas_finite(cuda_device):
    # criterion 6 (test_acceptance.py:198-236)
    alphas = [0.0, 1.0 / 255.0 - 1e-7, 0.99, 1.0]
    specs = [wide(float(i + 1), [1.0, 0.5, 0.25], alphas[i % 4]) for i in range(16)]
    sp = stack(specs, 32, 32)
    b = R.bin_and_sort(sp, 32, 32)
    out = R.render_forward(sp, b, 32, 32, (0, 0, 0), training=True)
    g2 = R.render_backward(torch.ones((32, 32, 3), device="cuda"), out, sp, b, 32, 32, (0, 0, 0))
    assert torch.isfinite(out.image).all() and torch.isfinite(out.final_transmittance).all()
    assert torch.isfinite(g2.packed).all()


def test_tile_limit_raises(cuda_device):
    from paper_2308_04079_b200.errors import ResourceLimitError
    sp = stack([dict(mean2d=[8.0, 8.0], conic=[1.0, 0, 1.0], depth=5.0, color=[1, 0, 0], alpha=0.5,
                     radius=1)], 32, 32)
    with pytest.raises(ResourceLimitError):
        R.bin_and_sort(sp, 2**21 * 16, 2**12 * 16)


def test_autograd_function_matches_stages(cuda_device):
    g, cloud_np, cam = golden_scenes.load("scene_c")
    degree, bg = int(g["degree"]), g["background"]
    d_image = golden_scenes.d_image_for(13, cam.width, cam.height)
    cloud, splats, binning, out, g2, grads, _ = device_pipeline(cloud_np, cam, degree, bg, d_image)
    leaves = [t.clone().requires_grad_(True) for t in (cloud.means, cloud.log_scales, cloud.rotations,
                                                        cloud.opacity_logits, cloud.sh)]
    image, radii = R.rasterize_gaussians(*leaves, cam, bg, degree)
    torch.testing.assert_close(image, out.image, rtol=0, atol=0)
    torch.testing.assert_close(radii, splats.radii)
    image.backward(torch.from_numpy(d_image.astype(np.float32)).cuda())
    for leaf, ref in zip(leaves, (grads.d_means, grads.d_log_scales, grads.d_rotations, grads.d_opacity_logits,
                                  grads.d_sh)):
        # same kernels; float atomics make the backward order-nondeterministic (SPEC: <= 1e-5 relative)
        assert rel(leaf.grad.cpu().numpy(), ref.cpu().numpy(), 1e-30) < 1e-5


def test_backward_run_to_run_within_contract(cuda_device):
    # atomic accumulation differs by <= 1e-5 relative across runs
    g, cloud_np, cam = golden_scenes.load("toy_c1")
    d_image = golden_scenes.d_image_for(1, cam.width, cam.height)
    a = device_pipeline(cloud_np, cam, 3, (0, 0, 0), d_image)[5]
    b = device_pipeline(cloud_np, cam, 3, (0, 0, 0), d_image)[5]
    for key in ("d_means", "d_log_scales", "d_opacity_logits", "d_sh"):
        assert rel(getattr(a, key).cpu().numpy(), getattr(b, key).cpu().numpy()) < 1e-5


def test_fused_backward_adam_matches_unfused(cuda_device):
    """gs_preprocess_backward_adam == gs_preprocess_backward + gs_adam_step up to
    float32 contraction differences (same formulas, two inlining contexts)."""
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    g, cloud_np, cam = golden_scenes.load("scene_c")
    degree, bg = int(g["degree"]), g["background"]
    d_image = torch.from_numpy(golden_scenes.d_image_for(13, cam.width, cam.height).astype(np.float32)).cuda()
    cfg = TrainConfig(total_iters=1000)
    a = GaussianCloud.from_numpy(**cloud_np)
    b = GaussianCloud.from_numpy(**cloud_np)
    opt_a, opt_b = DeviceAdam(a), DeviceAdam(b)
    st_a, st_b = R.DensifyStats.zeros(len(a), "cuda"), R.DensifyStats.zeros(len(b), "cuda")
    for it in (1, 2, 3):
        out, splats, binning = R.render_view(a, cam, bg, degree, training=True)
        g2 = R.render_backward(d_image, out, splats, binning, cam.width, cam.height, bg)
        grads = R.backward_project(a, cam, splats, g2, degree, stats=st_a)
        opt_a.step(a, grads, it, cfg)
        grads_b = R.GaussianGrads.zeros(len(b), "cuda")
        opt_b.backward_step(b, cam, splats, g2, degree, it, cfg, stats=st_b, grads_out=grads_b)
        torch.cuda.synchronize()
        for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
            assert rel(getattr(grads_b, key).cpu().numpy(), getattr(grads, key).cpu().numpy()) < 1e-6, key
        for k in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
            torch.testing.assert_close(getattr(b, k), getattr(a, k), rtol=1e-6, atol=1e-7)
            torch.testing.assert_close(opt_b.exp_avg[k], opt_a.exp_avg[k], rtol=1e-5, atol=1e-12)
        # continue both from the unfused state so differences cannot compound
        for k in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
            getattr(b, k).copy_(getattr(a, k))
            opt_b.exp_avg[k].copy_(opt_a.exp_avg[k])
            opt_b.exp_avg_sq[k].copy_(opt_a.exp_avg_sq[k])
    assert torch.equal(st_a.accum_count, st_b.accum_count)
    torch.testing.assert_close(st_b.accum_pos_grad, st_a.accum_pos_grad, rtol=1e-6, atol=0)


@pytest.mark.parametrize("skipped", [False, True])
def test_fused_next_view_projection_bit_identical(cuda_device, skipped):
    """gs_preprocess_backward_adam_project == the guarded backward + Adam
    followed by gs_preprocess_forward for the next view: parameters, moments
    and the next view's splats bit for bit (next view: another pose and
    resolution, with culled and guard-band Gaussians); with the step guard
    set, nothing is updated and the next view is projected from the
    unchanged parameters."""
    from paper_2308_04079_b200.camera import look_at
    g, cloud_np, cam = golden_scenes.load("scene_c")
    degree, bg = int(g["degree"]), g["background"]
    d_image = torch.from_numpy(golden_scenes.d_image_for(17, cam.width, cam.height).astype(np.float32)).cuda()
    centre = cloud_np["means"].mean(axis=0)
    # from inside the cloud: Gaussians behind the near plane and outside the guard band are culled
    nxt_cam = look_at(centre, centre + np.array([1.0, 0.3, 0.2]), width=97, height=61, fx=60.0, near=0.05)
    cfg = TrainConfig(total_iters=1000)
    a, b = GaussianCloud.from_numpy(**cloud_np), GaussianCloud.from_numpy(**cloud_np)
    opt_a, opt_b = DeviceAdam(a), DeviceAdam(b)
    st_a, st_b = R.DensifyStats.zeros(len(a), "cuda"), R.DensifyStats.zeros(len(b), "cuda")
    skip = torch.full((1,), int(skipped), dtype=torch.int32, device="cuda")
    before = {k: getattr(a, k).clone() for k in ("means", "log_scales", "rotations", "opacity_logits", "sh")}
    out, splats, binning = R.render_view(a, cam, bg, degree, training=True)
    g2 = R.render_backward(d_image, out, splats, binning, cam.width, cam.height, bg)
    opt_a.backward_step(a, cam, splats, g2, degree, 1, cfg, stats=st_a, skip=skip)
    ref = R.project(a, nxt_cam, 2)
    got = opt_b.backward_step(b, cam, splats, g2, degree, 1, cfg, stats=st_b, skip=skip, project_next=(nxt_cam, 2))
    torch.cuda.synchronize()
    for k in ("means", "log_scales", "rotations", "opacity_logits", "sh"):
        assert torch.equal(getattr(b, k), getattr(a, k)), k
        assert torch.equal(opt_b.exp_avg[k], opt_a.exp_avg[k]), k
        assert torch.equal(opt_b.exp_avg_sq[k], opt_a.exp_avg_sq[k]), k
        if skipped:
            assert torch.equal(getattr(b, k), before[k]), k
    assert torch.equal(st_a.accum_count, st_b.accum_count)
    assert torch.equal(st_a.accum_pos_grad, st_b.accum_pos_grad)
    vis = ref.radii > 0
    assert 0 < int(vis.sum()) < len(a)   # the next view culls some Gaussians
    for f in ("radii", "tiles_touched", "status"):
        assert torch.equal(getattr(got, f), getattr(ref, f)), f
    for f in ("rec", "depth", "rect"):
        assert torch.equal(getattr(got, f)[vis], getattr(ref, f)[vis]), f


def _fuzz_scene(seed: int):
    """Adversarial mixes: random look-at camera, Gaussians behind / at / beyond
    the near plane and the guard band, extreme anisotropy and scales,
    opacities straddling 1/255 and 0.99, zero-alpha and huge splats."""
    from paper_2308_04079_b200.camera import look_at
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(8, 200)), int(rng.integers(8, 120))
    n = int(rng.integers(1, 3000))
    eye = rng.normal(size=3) * 4.0
    cam = look_at(eye, rng.normal(size=3) * 0.3, width=w, height=h, fx=float(rng.uniform(0.3, 2.0) * w),
                  fy=float(rng.uniform(0.3, 2.0) * w), near=float(rng.uniform(0.05, 1.0)))
    means = rng.normal(size=(n, 3)) * rng.uniform(0.2, 3.0)
    log_scales = rng.uniform(-7.0, 0.5, (n, 3))
    log_scales[rng.random(n) < 0.3] += rng.uniform(-3.0, 3.0, (1, 3))       # strong anisotropy
    q = rng.normal(size=(n, 4))
    logit_eps = np.log((1 / 255) / (1 - 1 / 255))
    op = rng.uniform(-6.0, 6.0, n)
    op[rng.random(n) < 0.1] = logit_eps                  # peak alpha exactly 1/255
    op[rng.random(n) < 0.1] = np.log(0.99 / 0.01)        # peak alpha exactly 0.99
    sh = rng.normal(scale=0.5, size=(n, 16, 3))
    from paper_2308_04079_b200 import synthetic
    cloud = synthetic.round_to_f32(dict(means=means, rotations=q, log_scales=log_scales, opacity_logits=op, sh=sh))
    return cloud, cam, int(rng.integers(0, 4)), rng.uniform(0, 1, 3)


@pytest.mark.parametrize("seed", range(200, 216))
def test_fuzz_scenes_vs_oracle(cuda_device, seed):
    cloud_np, cam, deg, bg = _fuzz_scene(seed)
    d_image = golden_scenes.d_image_for(seed, cam.width, cam.height)
    check_against_oracle(device_pipeline(cloud_np, cam, deg, bg, d_image),
                         oracle_pipeline(cloud_np, cam, deg, bg, d_image))


@pytest.mark.parametrize("seed,thin", [(300, -4.0), (301, -6.0), (302, -8.0)])
def test_needle_splats_vs_oracle(cuda_device, seed, thin):
    """Needle-like Gaussians (one axis e^thin of the other two): screen conics
    with condition numbers up to ~1e5, where the expanded float32 quadratic
    form a dx^2 + 2b dx dy + c dy^2 cancels.  The blends evaluate it as a sum
    of squares in the conic's eigenbasis (gs_common.cuh: make_tile_splat), so
    the full pipeline stays within the oracle tolerances."""
    from paper_2308_04079_b200 import synthetic
    from paper_2308_04079_b200.camera import look_at
    rng = np.random.default_rng(seed)
    n, w, h = 400, 320, 192
    cam = look_at(np.array([0.0, -4.0, 0.5]), np.zeros(3), width=w, height=h, fx=float(w), fy=float(w))
    means = rng.normal(size=(n, 3)) * 0.8
    log_scales = np.empty((n, 3))
    log_scales[:, 0] = rng.uniform(-1.0, 1.0, n)           # long axis
    log_scales[:, 1:] = log_scales[:, :1] + thin            # two thin axes
    log_scales = np.take_along_axis(log_scales, rng.permuted(np.tile(np.arange(3), (n, 1)), axis=1), axis=1)
    cloud = synthetic.round_to_f32(dict(means=means, rotations=rng.normal(size=(n, 4)), log_scales=log_scales,
                                        opacity_logits=rng.uniform(-1.0, 5.0, n),
                                        sh=rng.normal(scale=0.5, size=(n, 16, 3))))
    bg = rng.uniform(0, 1, 3)
    d_image = golden_scenes.d_image_for(seed, w, h)
    # The conic gradient is accumulated as eigenbasis moments (blend_bwd.cu),
    # so the chain to d(log scale, quaternion) no longer amplifies the x/y
    # sums' rounding by cond(conic): every group at the 1e-3 of SURVEY §8(c).
    check_against_oracle(device_pipeline(cloud, cam, 3, bg, d_image), oracle_pipeline(cloud, cam, 3, bg, d_image))


@pytest.mark.parametrize("n,w,h", [(30_000, 320, 200), (200_000, 3840, 2160)])
def test_tile_orders_do_not_change_results(cuda_device, n, w, h):
    """The forward launched in the previous backward's longest-first order,
    and the scheduled backward, give the plain launches' results (forward
    bit-identical; backward within the float atomics' run-to-run contract)."""
    import ctypes
    from paper_2308_04079_b200 import _lib, synthetic
    cloud_np, cam = synthetic.frustum_scene(n, w, h, seed=51)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    bg = (0.2, 0.1, 0.3)
    out, splats, binning = R.render_view(cloud, cam, bg, 3, training=True)
    d = torch.rand_like(out.image) - 0.5
    g2 = R.render_backward(d, out, splats, binning, cam.width, cam.height, bg)
    assert g2.tile_order is not None
    tx, ty = R.tile_extent(cam.width, cam.height)
    assert torch.equal(torch.sort(g2.tile_order.long()).values, torch.arange(tx * ty, device="cuda"))
    out2 = R.render_forward(splats, binning, cam.width, cam.height, bg, training=True, tile_order=g2.tile_order)
    assert torch.equal(out2.image, out.image) and torch.equal(out2.last_contributor, out.last_contributor)
    assert torch.equal(out2.final_transmittance, out.final_transmittance)
    plain = torch.empty_like(g2.packed)
    _lib.check(_lib.load().gs_blend_backward(d.data_ptr(), ctypes.byref(splats.c_struct()),
                                             binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
                                             out.final_transmittance.data_ptr(), out.last_contributor.data_ptr(),
                                             cam.width, cam.height, R._bg(bg), plain.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream), "plain")
    # same sums, different float-atomic order: per-component norms within the
    # run-to-run contract (1e-5 relative)
    diff = torch.linalg.norm((g2.packed - plain).double(), dim=0)
    ref = torch.linalg.norm(plain.double(), dim=0)
    assert bool((diff <= 1e-5 * ref + 1e-30).all()), (diff / ref.clamp_min(1e-30)).tolist()


def test_tile_schedule_repeated_renders(cuda_device):
    """TileSchedule: the forward records per-tile work and the next frame
    launches heaviest-first; every frame's image equals the plain render."""
    from paper_2308_04079_b200 import synthetic
    cloud_np, cam = synthetic.frustum_scene(30_000, 320, 200, seed=52)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    ref = R.render_view(cloud, cam, (0, 0, 0), 3)[0].image
    sched = R.TileSchedule()
    for _ in range(3):
        out, _, binning = R.render_view_async(cloud, cam, (0, 0, 0), 3, schedule=sched)
        binning.check()
        assert torch.equal(out.image, ref)
    tx, ty = R.tile_extent(cam.width, cam.height)
    assert torch.equal(torch.sort(sched.order.long()).values, torch.arange(tx * ty, device="cuda"))
    assert int(sched.work.min()) >= 0 and int(sched.work.max()) > 0
