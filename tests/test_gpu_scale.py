"""GPU parity at benchmark scale (SURVEY §8(c) "parity at scale").

* 300K-Gaussian frustum scene at 1920x1080 against the float64 oracle: bit-exact
  radii / ids / ranges, last contributor exact, image within tolerance.
* c2 (1M, 1080p) and c5 (6M, 3840x2160): size-independent invariants of the
  binning (ranges partition the instances; per-tile (depth, id) order; every
  Gaussian appears exactly tiles_touched times, each time in a tile of its
  rectangle), finite outputs, backward runs.
* Multi-view accumulation (c4 path): accumulate=True over views == the sum of
  the per-view gradients.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_04079_b200 import rasterizer as R
from paper_2308_04079_b200 import synthetic
from paper_2308_04079_b200.cloud import GaussianCloud
from parity_utils import forward_parity

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def check_binning_invariants(splats, binning, width, height):
    ids = binning.splat_ids.long()
    ranges = binning.ranges.long()
    K = ids.numel()
    tx = binning.tiles_x
    T = ranges.shape[0]
    counts = ranges[:, 1] - ranges[:, 0]
    assert int(counts.sum()) == K
    nonempty = counts > 0
    # ranges are contiguous and ordered by tile
    starts = ranges[nonempty, 0]
    ends = ranges[nonempty, 1]
    assert int(starts[0]) == 0 and int(ends[-1]) == K
    assert torch.equal(starts[1:], ends[:-1])
    # tile of every sorted position
    tile_of = torch.repeat_interleave(torch.arange(T, device=ids.device), counts)
    # every Gaussian appears tiles_touched times
    bc = torch.bincount(ids, minlength=len(splats))
    assert torch.equal(bc.int(), splats.tiles_touched)
    # each instance lies in its Gaussian's rectangle
    rect = splats.rect.long()[ids]
    tcol, trow = tile_of % tx, tile_of // tx
    assert bool(((tcol >= rect[:, 0]) & (tcol <= rect[:, 2]) & (trow >= rect[:, 1]) & (trow <= rect[:, 3])).all())
    # within a tile: non-decreasing float32 depth, ties by increasing Gaussian index
    d = splats.depth[ids]
    same = tile_of[1:] == tile_of[:-1]
    dd = d[1:] - d[:-1]
    assert bool((dd[same] >= 0).all())
    tie = same & (dd == 0)
    assert bool((ids[1:][tie] > ids[:-1][tie]).all())


def test_full_frame_1080p_vs_oracle(cuda_device):
    cloud_np, cam = synthetic.frustum_scene(300_000, 1920, 1080, seed=3)
    cloud_np = synthetic.round_to_f32(cloud_np)
    bg = (0.05, 0.1, 0.15)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    out, splats, binning = R.render_view(cloud, cam, bg, 3, training=True)
    d_image = np.random.default_rng(3).uniform(-1, 1, (1080, 1920, 3)).astype(np.float32) / (1080 * 1920 * 3)
    g2 = R.render_backward(torch.from_numpy(d_image).cuda(), out, splats, binning, 1920, 1080, bg)
    grads = R.backward_project(cloud, cam, splats, g2, 3)
    torch.cuda.synchronize()
    check_binning_invariants(splats, binning, 1920, 1080)

    proj = O.project(cloud_np, cam, 3)
    bins = O.bin_and_sort(proj, 1920, 1080)
    fwd = O.render_forward(proj, bins, 1920, 1080, bg)
    og2 = O.render_backward(d_image.astype(np.float64), proj, bins, fwd, 1920, 1080, bg)
    ograds = O.backward_project(cloud_np, cam, 3, proj, og2)

    np.testing.assert_array_equal(splats.radii.cpu().numpy(), proj["radius"])
    np.testing.assert_array_equal(binning.splat_ids.cpu().numpy(), bins["ids"])
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), bins["ranges"])
    report = forward_parity(out.image.cpu().numpy(), out.final_transmittance.cpu().numpy(),
                            out.last_contributor.cpu().numpy(), fwd["image"], fwd["t_final"], fwd["last"],
                            color_max=float(proj["color"].max()))
    print("1080p parity:", report)
    for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        assert rel(getattr(grads, key).cpu().numpy(), ograds[key]) < 1e-3, key


@pytest.mark.parametrize("n,w,h", [(1_000_000, 1920, 1080), (6_000_000, 3840, 2160)])
def test_binning_invariants_at_scale(cuda_device, n, w, h):
    cloud_np, cam = synthetic.frustum_scene(n, w, h, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    del cloud_np
    out, splats, binning = R.render_view(cloud, cam, (0.0, 0.0, 0.0), 3, training=True)
    check_binning_invariants(splats, binning, w, h)
    assert torch.isfinite(out.image).all()
    assert bool(((out.final_transmittance >= 0) & (out.final_transmittance <= 1)).all())
    d = torch.full((h, w, 3), 1.0 / (h * w * 3), device="cuda")
    g2 = R.render_backward(d, out, splats, binning, w, h, (0.0, 0.0, 0.0))
    grads = R.backward_project(cloud, cam, splats, g2, 3)
    torch.cuda.synchronize()
    for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        assert torch.isfinite(getattr(grads, key)).all(), key


def test_multiview_accumulate_equals_sum(cuda_device):
    cloud_np = synthetic.round_to_f32(synthetic.ball_scene(50_000, seed=0))
    cams = synthetic.ball_cameras(4, width=480, height=270)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    acc = R.GaussianGrads.zeros(len(cloud), "cuda")
    total = R.GaussianGrads.zeros(len(cloud), "cuda")
    stats = R.DensifyStats.zeros(len(cloud), "cuda")
    for i, cam in enumerate(cams):
        out, splats, binning = R.render_view(cloud, cam, (0, 0, 0), 3, training=True)
        d = torch.from_numpy(np.random.default_rng(i).uniform(-1, 1, (270, 480, 3)).astype(np.float32)).cuda()
        g2 = R.render_backward(d, out, splats, binning, 480, 270, (0, 0, 0))
        R.backward_project(cloud, cam, splats, g2, 3, stats=stats, out=acc, accumulate=True)
        single = R.backward_project(cloud, cam, splats, g2, 3)
        for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
            getattr(total, key).add_(getattr(single, key))
    torch.cuda.synchronize()
    for key in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        torch.testing.assert_close(getattr(acc, key), getattr(total, key), rtol=1e-5, atol=1e-12)
    assert int(stats.accum_count.max()) <= 4 and int(stats.accum_count.sum()) > 0


# ---------------------------------------------------------------------------
# sync-free binning (gs_bin_and_sort_async): K stays on the device

def test_async_binning_matches_sync(cuda_device):
    cloud_np, cam = synthetic.frustum_scene(300_000, 1920, 1080, seed=4)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, 3)
    sync = R.bin_and_sort(splats, 1920, 1080)
    K = sync.num_instances
    asy = R.bin_and_sort_async(splats, 1920, 1080, capacity=K + 12345)
    asy.check()
    assert asy.num_instances == K
    assert torch.equal(asy.splat_ids[:K], sync.splat_ids)
    assert torch.equal(asy.ranges, sync.ranges)


def test_async_binning_capacity_overflow_flagged(cuda_device):
    cloud_np, cam = synthetic.frustum_scene(50_000, 640, 360, seed=5)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, 3)
    K = R.bin_and_sort(splats, 640, 360).num_instances
    asy = R.bin_and_sort_async(splats, 640, 360, capacity=K // 2)
    with pytest.raises(R.CapacityError):
        asy.check()
    assert int(asy.ranges.abs().sum()) == 0   # nothing half-binned is exposed
    exact = R.bin_and_sort_async(splats, 640, 360, capacity=K)
    exact.check()
    assert exact.num_instances == K


@pytest.mark.parametrize("w,h,n", [(7680, 4320, 150_000), (256, 256, 20_000)])
def test_binning_other_pass_counts_vs_oracle(cuda_device, w, h, n):
    # 8K: 129,600 tiles -> 4,080 super-tiles (the largest grid at one tile per lane); 256^2: 8
    cloud_np, cam = synthetic.frustum_scene(n, w, h, seed=6)
    cloud_np = synthetic.round_to_f32(cloud_np)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, 3)
    binning = R.bin_and_sort(splats, w, h)
    check_binning_invariants(splats, binning, w, h)
    proj = O.project(cloud_np, cam, 3)
    bins = O.bin_and_sort(proj, w, h)
    np.testing.assert_array_equal(binning.splat_ids.cpu().numpy(), bins["ids"])
    np.testing.assert_array_equal(binning.ranges.cpu().numpy(), bins["ranges"])


def test_forward_captured_in_cuda_graph(cuda_device):
    # project -> async binning -> blend enqueue no host sync: one CUDA graph
    cloud_np, cam = synthetic.frustum_scene(100_000, 960, 540, seed=7)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    eager, _, _ = R.render_view(cloud, cam, (0.1, 0.2, 0.3), 3)
    cap = R.bin_and_sort(R.project(cloud, cam, 3), 960, 540).num_instances + 1024
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):   # warm the allocator on the capture stream
        R.render_view_async(cloud, cam, (0.1, 0.2, 0.3), 3, capacity=cap)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out, _, binning = R.render_view_async(cloud, cam, (0.1, 0.2, 0.3), 3, capacity=cap)
    g.replay()
    torch.cuda.synchronize()
    binning.check()
    assert torch.equal(out.image, eager.image)
