"""Pin the float64 C oracle to the reference: every golden vector in
tests/golden/ was produced by splatlab itself (make_golden.py)."""
import numpy as np
import pytest

import golden_scenes
from oracle import oracle as O

SCENES = list(golden_scenes.SCENES)


def run_oracle(name):
    g, cloud, cam = golden_scenes.load(name)
    degree = int(g["degree"])
    bg = g["background"]
    proj = O.project(cloud, cam, degree)
    bins = O.bin_and_sort(proj, cam.width, cam.height)
    fwd = O.render_forward(proj, bins, cam.width, cam.height, bg)
    d_image = golden_scenes.d_image_for(golden_scenes.SCENES[name]()[4], cam.width, cam.height)
    g2 = O.render_backward(d_image, proj, bins, fwd, cam.width, cam.height, bg)
    grads = O.backward_project(cloud, cam, degree, proj, g2)
    return g, cloud, cam, proj, bins, fwd, g2, grads


@pytest.fixture(scope="module", params=SCENES)
def scene(request):
    return request.param, run_oracle(request.param)


def rel_err(a, b, floor=1e-15):
    """||a-b|| / ||b||, with an absolute floor for groups that are zero up to
    round-off (e.g. quaternion gradients of isotropic Gaussians)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor))


def test_project_culling_and_radii_exact(scene):
    name, (g, cloud, cam, proj, *_rest) = scene
    surv = np.nonzero(proj["radius"] > 0)[0]
    np.testing.assert_array_equal(surv, g["source_index"])
    np.testing.assert_array_equal(proj["radius"][surv], g["radius"])
    np.testing.assert_array_equal(proj["depth"][surv].astype(np.float32), g["depth"].astype(np.float32))


def test_project_float_outputs(scene):
    name, (g, cloud, cam, proj, *_rest) = scene
    surv = proj["radius"] > 0
    tol = 1e-12 if g["mean2d"].dtype == np.float64 else 1e-6
    for key in ("mean2d", "conic", "color", "alpha"):
        assert rel_err(proj[key][surv], g[key]) < tol, key
    active = np.stack([(proj["color_mask"][surv] >> c) & 1 for c in range(3)], axis=1).astype(bool)
    np.testing.assert_array_equal(active, g["color_active"])


def test_binning_bit_exact(scene):
    name, (g, cloud, cam, proj, bins, *_rest) = scene
    ref = O.to_reference_order(proj, bins)
    np.testing.assert_array_equal(ref["splat_ids"], g["splat_ids"])
    np.testing.assert_array_equal(bins["ranges"], g["ranges"])
    if "keys" in g:
        np.testing.assert_array_equal(bins["keys"], g["keys"])


def test_forward_image_and_training_record(scene):
    name, (g, cloud, cam, proj, bins, fwd, *_rest) = scene
    tol = 1e-10 if g["image"].dtype == np.float64 else 2e-7
    assert np.abs(fwd["image"] - g["image"]).max() < tol
    assert np.abs(fwd["t_final"] - g["t_final"]).max() < tol
    np.testing.assert_array_equal(fwd["last"], g["last"])


def test_backward_blend(scene):
    name, (g, cloud, cam, proj, bins, fwd, g2, grads) = scene
    surv = proj["radius"] > 0
    tol = 1e-9 if g["g2_d_color"].dtype == np.float64 else 1e-5
    assert rel_err(g2[surv, 6:9], g["g2_d_color"]) < tol
    assert rel_err(g2[surv, 5], g["g2_d_alpha"]) < tol
    assert rel_err(g2[surv, 0:2], g["g2_d_mean2d"]) < tol
    assert rel_err(g2[surv, 2:5], g["g2_d_conic"]) < tol


def test_backward_project(scene):
    name, (g, cloud, cam, proj, bins, fwd, g2, grads) = scene
    tol = 1e-9 if g["d_means"].dtype == np.float64 else 1e-5
    # round-off floor: the chain's largest gradient group scaled by 1e-9
    floor = 1e-9 * max(np.linalg.norm(g[k]) for k in ("d_means", "d_log_scales", "d_sh"))
    for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh", "view_pos_grad_norm"):
        assert rel_err(grads[key], g[key], floor) < tol, key
    culled = proj["radius"] == 0
    assert np.all(grads["d_means"][culled] == 0.0) and np.all(grads["d_sh"][culled] == 0.0)


def test_stats(scene):
    name, (g, cloud, cam, proj, bins, fwd, g2, grads) = scene
    n = proj["radius"].shape[0]
    stats = {"accum_pos_grad": np.zeros(n), "accum_count": np.zeros(n, np.int64), "max_radius_frac": np.zeros(n)}
    O.stats_update(proj, grads["view_pos_grad_norm"], cam.height, stats)
    np.testing.assert_array_equal(stats["accum_count"], g["stat_count"])
    assert rel_err(stats["accum_pos_grad"], g["stat_accum"]) < 1e-5
    np.testing.assert_allclose(stats["max_radius_frac"], g["stat_maxr"], rtol=1e-7)


@pytest.mark.parametrize("name", ["scene_a", "scene_b"])
def test_adam_two_steps(name):
    g, cloud, cam = golden_scenes.load(name)
    grads = {"means": g["d_means"], "log_scales": g["d_log_scales"], "rotations": g["d_rotations"],
             "opacity_logits": g["d_opacity_logits"], "sh": g["d_sh"]}
    lrs = {"log_scales": 5e-3, "rotations": 1e-3, "opacity_logits": 5e-2}
    state = {k: cloud[k].copy() for k in grads}
    m = {k: np.zeros_like(v) for k, v in state.items()}
    v = {k: np.zeros_like(v) for k, v in state.items()}
    for it in (1, 2):
        for k in grads:
            if k == "means":
                lr = 1.6e-4 * (1.6e-6 / 1.6e-4) ** (it / 1000)
                O.adam_group(state[k], grads[k], m[k], v[k], lr, 0.9, 0.999, 1e-15, it)
            elif k == "sh":
                O.adam_group(state[k], grads[k], m[k], v[k], 2.5e-3 / 20, 0.9, 0.999, 1e-15, it,
                             lr_head=2.5e-3, period=48, head=3)
            else:
                O.adam_group(state[k], grads[k], m[k], v[k], lrs[k], 0.9, 0.999, 1e-15, it)
            np.testing.assert_allclose(state[k], g[f"adam{it}_{k}"], rtol=0, atol=1e-12)
