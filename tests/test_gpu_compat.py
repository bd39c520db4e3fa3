"""splatlab-style stage tests on the NumPy-signature mirror (compat), i.e.
on the device path: the cases of the reference's test_rasterizer.py
(TestKeys, TestBinning, TestRenderForward, TestOracleEquivalence) and
test_gradients.py (TestBackwardBlend, TestGradientContracts), restated with
the reference's call signatures.  The reference's float64 equalities become
the device's float32 tolerances; brute-force references are the float64
oracle (oracle/, pinned to splatlab's goldens).  The gradient helpers'
sub-steps (backward_conic_to_cov3d, backward_cov3d_to_scale_rotation) are
fused into gs_preprocess_backward and covered by the end-to-end gradient
parity of test_gpu_parity.py."""
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2308_04079_b200 import compat as C
from paper_2308_04079_b200 import synthetic

pytestmark = pytest.mark.gpu


def make_splats(mean2d, conic, depth, color, alpha, radius):
    m = len(depth)
    return C.ProjectedSplats(source_index=np.arange(m), mean2d=np.asarray(mean2d, np.float64).reshape(m, 2),
                             conic=np.asarray(conic, np.float64).reshape(m, 3), depth=np.asarray(depth, np.float64),
                             radius=np.asarray(radius, np.int64), color=np.asarray(color, np.float64).reshape(m, 3),
                             alpha=np.asarray(alpha, np.float64), color_active=np.ones((m, 3), bool))


def wide_splat(depth, color, alpha, width=32, height=32):
    """A nearly flat splat covering the whole image with ~constant weight."""
    return dict(mean2d=[width / 2.0, height / 2.0], conic=[1e-8, 0.0, 1e-8], depth=depth, color=color, alpha=alpha,
                radius=10 * max(width, height))


def stack_splats(specs):
    return make_splats([s["mean2d"] for s in specs], [s["conic"] for s in specs], [s["depth"] for s in specs],
                       [s["color"] for s in specs], [s["alpha"] for s in specs], [s["radius"] for s in specs])


def scene(seed, count, w, h):
    cloud, cam = synthetic.random_splat_scene(np.random.default_rng(seed), count, w, h)
    return SimpleNamespace(**synthetic.round_to_f32(cloud)), cam


def render_for_test(cloud, cam, background, training=False):
    sp = C.project(cloud, cam)
    b = C.bin_and_sort(sp, cam.width, cam.height)
    return C.render_forward(sp, b, cam.width, cam.height, np.asarray(background, np.float64), training=training), sp, b


def oracle_render(cloud, cam, background):
    from oracle import oracle as O
    params = {k: getattr(cloud, k) for k in ("means", "rotations", "log_scales", "opacity_logits", "sh")}
    proj = O.project(params, cam, 3)
    return O.render_forward(proj, O.bin_and_sort(proj, cam.width, cam.height), cam.width, cam.height, background)


class TestKeys:
    def test_device_keys_are_make_keys(self, cuda_device):
        cloud, cam = scene(1, 200, 64, 64)
        sp = C.project(cloud, cam)
        b = C.bin_and_sort(sp, 64, 64)
        tiles = np.repeat(np.arange(len(b.ranges)), b.ranges[:, 1] - b.ranges[:, 0])
        np.testing.assert_array_equal(b.keys, C.make_keys(tiles, sp.depth[b.splat_ids]))
        assert np.all(np.diff(b.keys.astype(np.float64)) >= 0)   # (tile, depth) order; keys < 2^53


class TestBinning:
    def test_single_small_splat_one_tile(self, cuda_device):
        sp = make_splats([[8.0, 8.0]], [[1.0, 0, 1.0]], [5.0], [[1, 0, 0]], [0.5], [1])
        b = C.bin_and_sort(sp, 32, 32)
        assert b.tiles_x == 2 and b.tiles_y == 2
        assert len(b.keys) == 1
        assert b.ranges.tolist() == [[0, 1], [0, 0], [0, 0], [0, 0]]

    def test_corner_splat_hits_four_tiles(self, cuda_device):
        sp = make_splats([[16.0, 16.0]], [[1.0, 0, 1.0]], [5.0], [[1, 0, 0]], [0.5], [20])
        b = C.bin_and_sort(sp, 32, 32)
        assert len(b.keys) == 4
        assert all(end - start == 1 for start, end in b.ranges)

    def test_offscreen_box_empty(self, cuda_device):
        sp = make_splats([[-50.0, -50.0]], [[1.0, 0, 1.0]], [5.0], [[1, 0, 0]], [0.5], [3])
        assert len(C.bin_and_sort(sp, 32, 32).keys) == 0

    def test_depth_nondecreasing_within_ranges(self, cuda_device):
        cloud, cam = scene(1, 200, 64, 64)
        sp = C.project(cloud, cam)
        b = C.bin_and_sort(sp, 64, 64)
        for start, end in b.ranges:
            assert np.all(np.diff(sp.depth[b.splat_ids[start:end]].astype(np.float32)) >= 0)

    def test_matches_oracle_lists(self, cuda_device):
        from oracle import oracle as O
        cloud, cam = scene(2, 1000, 64, 64)
        sp = C.project(cloud, cam)
        b = C.bin_and_sort(sp, 64, 64)
        params = {k: getattr(cloud, k) for k in ("means", "rotations", "log_scales", "opacity_logits", "sh")}
        ob = O.bin_and_sort(O.project(params, cam, 3), 64, 64)
        np.testing.assert_array_equal(b.ranges, ob["ranges"])
        np.testing.assert_array_equal(sp.source_index[b.splat_ids], ob["ids"])   # M-space -> cloud rows

    def test_ranges_partition_instances(self, cuda_device):
        cloud, cam = scene(3, 300, 48, 48)
        b = C.bin_and_sort(C.project(cloud, cam), 48, 48)
        assert sum(int(e - s) for s, e in b.ranges) == len(b.keys)

    def test_tile_count_guard(self, cuda_device):
        sp = make_splats([[8.0, 8.0]], [[1.0, 0, 1.0]], [5.0], [[1, 0, 0]], [0.5], [1])
        with pytest.raises(C.ResourceLimitError):
            C.bin_and_sort(sp, 2**21 * 16, 2**12 * 16)


class TestRenderForward:
    def test_empty_scene_is_background(self, cuda_device):
        sp = make_splats(np.zeros((0, 2)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0),
                         np.zeros(0, np.int64))
        b = C.bin_and_sort(sp, 32, 24)
        out = C.render_forward(sp, b, 32, 24, np.zeros(3), training=True)
        assert np.all(out.image == 0.0)
        assert np.all(out.final_transmittance == 1.0)
        assert np.all(out.last_contributor == -1)

    def test_two_coincident_splats_blend(self, cuda_device):
        sp = stack_splats([wide_splat(1.0, [1, 0, 0], 0.5), wide_splat(2.0, [0, 1, 0], 0.5)])
        b = C.bin_and_sort(sp, 32, 32)
        out = C.render_forward(sp, b, 32, 32, np.zeros(3))
        np.testing.assert_allclose(out.image[16, 16], [0.5, 0.25, 0.0], atol=1e-6)

    def test_white_background_composites(self, cuda_device):
        sp = stack_splats([wide_splat(1.0, [1, 0, 0], 0.5)])
        b = C.bin_and_sort(sp, 32, 32)
        out = C.render_forward(sp, b, 32, 32, np.ones(3))
        np.testing.assert_allclose(out.image[16, 16], [1.0, 0.5, 0.5], atol=1e-6)

    def test_transparent_splat_changes_nothing(self, cuda_device):
        cloud, cam = scene(4, 40, 64, 64)
        out0, sp0, _ = render_for_test(cloud, cam, np.zeros(3))
        ghost = make_splats([[32.0, 32.0]], [[0.01, 0, 0.01]], [1.0], [[1, 1, 1]], [1e-9], [200])
        merged = C.ProjectedSplats(
            source_index=np.concatenate([sp0.source_index, [len(cloud.means)]]),
            mean2d=np.concatenate([sp0.mean2d, ghost.mean2d]), conic=np.concatenate([sp0.conic, ghost.conic]),
            depth=np.concatenate([sp0.depth, ghost.depth]), radius=np.concatenate([sp0.radius, ghost.radius]),
            color=np.concatenate([sp0.color, ghost.color]), alpha=np.concatenate([sp0.alpha, ghost.alpha]),
            color_active=np.concatenate([sp0.color_active, ghost.color_active]))
        b = C.bin_and_sort(merged, 64, 64)
        out1 = C.render_forward(merged, b, 64, 64, np.zeros(3))
        np.testing.assert_array_equal(out0.image, out1.image)

    def test_invariant_to_input_splat_order(self, cuda_device):
        rng = np.random.default_rng(5)
        cloud, cam = scene(5, 60, 64, 64)
        out0, _, _ = render_for_test(cloud, cam, np.zeros(3))
        perm = rng.permutation(len(cloud.means))
        permuted = SimpleNamespace(**{k: getattr(cloud, k)[perm] for k in vars(cloud)})
        out1, _, _ = render_for_test(permuted, cam, np.zeros(3))
        np.testing.assert_allclose(out0.image, out1.image, atol=1e-6)

    def test_saturation_stop(self, cuda_device):
        sp = stack_splats([wide_splat(float(i + 1), [1, 1, 1], 0.97) for i in range(64)])
        b = C.bin_and_sort(sp, 32, 32)
        out = C.render_forward(sp, b, 32, 32, np.zeros(3), training=True)
        assert np.all(np.isfinite(out.image))
        assert np.all(1.0 - out.final_transmittance <= 0.9999 + 1e-7)
        for tile in range(4):
            start, end = b.ranges[tile]
            ty, tx = divmod(tile, 2)
            block = out.last_contributor[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
            assert np.all(block >= start) and np.all(block - start < 10)

    def test_workers_do_not_change_results(self, cuda_device):
        cloud, cam = scene(6, 120, 96, 64)
        sp = C.project(cloud, cam)
        b = C.bin_and_sort(sp, 96, 64)
        out1 = C.render_forward(sp, b, 96, 64, np.zeros(3), training=True, workers=1)
        out4 = C.render_forward(sp, b, 96, 64, np.zeros(3), training=True, workers=4)
        np.testing.assert_array_equal(out1.image, out4.image)
        np.testing.assert_array_equal(out1.last_contributor, out4.last_contributor)


class TestOracleEquivalence:
    def test_float32_close(self, cuda_device):
        rng = np.random.default_rng(8)
        for i in range(4):
            n = int(rng.integers(16, 257))
            cloud, cam = scene(100 + i, n, 64, 64)
            out, _, _ = render_for_test(cloud, cam, (0.1, 0.2, 0.3))
            ref = oracle_render(cloud, cam, (0.1, 0.2, 0.3))
            assert np.abs(out.image - ref["image"]).max() <= 1e-5


class TestBackwardBlend:
    def test_saturated_pixel_gives_no_grad_to_back_splat(self, cuda_device):
        specs = [wide_splat(1.0, [1, 0, 0], 0.97) for _ in range(8)] + [wide_splat(9.0, [0, 1, 0], 0.9)]
        sp = stack_splats(specs)
        b = C.bin_and_sort(sp, 32, 32)
        out = C.render_forward(sp, b, 32, 32, np.zeros(3), training=True)
        assert np.all(1.0 - out.final_transmittance > 0.999)
        g2d = C.render_backward(np.ones((32, 32, 3)), out, sp, b, 32, 32, np.zeros(3))
        assert np.all(g2d.d_color[8] == 0.0)
        assert np.all(g2d.d_alpha[8] == 0.0)
        assert np.any(g2d.d_color[0] != 0.0)

    def test_zero_d_image_zero_grads(self, cuda_device):
        cloud, cam = scene(4, 5, 16, 16)
        out, sp, b = render_for_test(cloud, cam, (0, 0, 0), training=True)
        g2d = C.render_backward(np.zeros((16, 16, 3)), out, sp, b, 16, 16, np.zeros(3))
        grads = C.backward_project(cloud, cam, sp, g2d, 3)
        for name in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
            assert np.all(getattr(grads, name) == 0.0)


class TestGradientContracts:
    def analytic(self, cloud, cam, weights):
        out, sp, b = render_for_test(cloud, cam, (0, 0, 0), training=True)
        g2d = C.render_backward(weights, out, sp, b, cam.width, cam.height, np.zeros(3))
        return C.backward_project(cloud, cam, sp, g2d, 3), g2d, sp

    def test_additive_over_pixels(self, cuda_device):
        cloud, cam = scene(20, 4, 16, 16)
        w_a = np.zeros((16, 16, 3))
        w_a[3, 5, 1] = 1.0
        w_b = np.zeros((16, 16, 3))
        w_b[9, 12, 2] = -0.7
        ga, gb, gab = (self.analytic(cloud, cam, w)[0] for w in (w_a, w_b, w_a + w_b))
        for name in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
            a, b, ab = getattr(ga, name), getattr(gb, name), getattr(gab, name)
            scale = max(np.abs(ab).max(), 1e-30)
            assert np.abs(ab - (a + b)).max() <= 1e-5 * scale, name

    def test_culled_gaussians_zero_grad(self, cuda_device):
        cloud, cam = scene(21, 3, 16, 16)
        cloud.means[1] = [0.0, 0.0, -5.0]   # behind the camera
        grads, _, _ = self.analytic(cloud, cam, np.ones((16, 16, 3)))
        assert np.all(grads.d_means[1] == 0.0)
        assert np.all(grads.d_sh[1] == 0.0)
        assert grads.view_pos_grad_norm[1] == 0.0

    def test_view_pos_grad_norm_is_mean2d_norm(self, cuda_device):
        cloud, cam = scene(22, 3, 16, 16)
        weights = np.random.default_rng(0).uniform(-1, 1, (16, 16, 3))
        grads, g2d, sp = self.analytic(cloud, cam, weights)
        np.testing.assert_allclose(grads.view_pos_grad_norm[sp.source_index], np.linalg.norm(g2d.d_mean2d, axis=1),
                                   rtol=1e-5, atol=1e-12)

    def test_deep_stack_all_contributors_get_color_grad(self, cuda_device):
        sp = stack_splats([wide_splat(float(i + 1), [0.5, 0.5, 0.5], 0.12) for i in range(64)])
        b = C.bin_and_sort(sp, 16, 16)
        out = C.render_forward(sp, b, 16, 16, np.zeros(3), training=True)
        g2d = C.render_backward(np.ones((16, 16, 3)), out, sp, b, 16, 16, np.zeros(3))
        assert np.all(np.abs(g2d.d_color).sum(axis=1) > 0.0)

    def test_screen_gradients_match_oracle(self, cuda_device):
        """render_backward's reference-semantics outputs (d_mean2d, d_conic,
        d_alpha, d_color) against the float64 oracle, row for row."""
        from oracle import oracle as O
        cloud, cam = scene(23, 80, 64, 64)
        out, sp, b = render_for_test(cloud, cam, (0, 0, 0), training=True)
        d_image = np.random.default_rng(23).uniform(-1, 1, (64, 64, 3))
        g2d = C.render_backward(d_image, out, sp, b, 64, 64, np.zeros(3))
        params = {k: getattr(cloud, k) for k in ("means", "rotations", "log_scales", "opacity_logits", "sh")}
        proj = O.project(params, cam, 3)
        bins = O.bin_and_sort(proj, 64, 64)
        og2 = O.render_backward(d_image, proj, bins, O.render_forward(proj, bins, 64, 64, (0, 0, 0)), 64, 64,
                                (0, 0, 0))[sp.source_index]

        def rel(a, r):
            return np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-30)
        assert rel(g2d.d_mean2d, og2[:, 0:2]) < 1e-3
        assert rel(g2d.d_conic, og2[:, 2:5]) < 1e-3
        assert rel(g2d.d_alpha, og2[:, 5]) < 1e-3
        assert rel(g2d.d_color, og2[:, 6:9]) < 1e-3
