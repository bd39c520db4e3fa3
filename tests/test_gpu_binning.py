"""GPU binning (K2-K5, rasterizer.py:55-124) through the C ABI: the 64-bit
sort keys (TileBinning.keys, make_keys rasterizer.py:55-62) and the sorted
order, bit-exact.

* keys vs the reference's own golden keys (scene_a / scene_b, written by
  splatlab's bin_and_sort) and vs the oracle;
* criterion 5 of the reference's acceptance suite (test_acceptance.py:177-195)
  on the device path: 10^6 (tile, depth) pairs with 5% exact ties in one tile
  and 2% subnormal depths, through DeviceSplats.from_projected;
* the reference's binning KATs (test_rasterizer.py:39-109): key order, one
  instance, the 4-tile corner, off-screen splats;
* edge cases: no survivors, a single Gaussian covering every tile, frames that
  are not a multiple of the 8 x 4-tile super-tile, large-frame super-tiles
  with 2 x 2 tiles per lane.
"""
import numpy as np
import pytest
import torch

import golden_scenes
from oracle import oracle as O
from paper_2308_04079_b200 import rasterizer as R
from paper_2308_04079_b200 import synthetic
from paper_2308_04079_b200.cloud import GaussianCloud

pytestmark = pytest.mark.gpu


def ref_keys(tiles, depths):
    """make_keys (rasterizer.py:55-62): (tile << 32) | float32 bits of depth."""
    d = np.asarray(depths, np.float64).astype(np.float32).view(np.uint32).astype(np.uint64)
    return ((np.asarray(tiles, np.uint64) << np.uint64(32)) | d).view(np.int64)


def point_splats(tiles, depths, tiles_x, tiles_y):
    """One radius-1 splat at the centre of each given tile (its rectangle is
    exactly that tile, rasterizer.py:86-97)."""
    tiles = np.asarray(tiles, np.int64)
    n = tiles.shape[0]
    mean2d = np.stack([(tiles % tiles_x) * 16 + 8.0, (tiles // tiles_x) * 16 + 8.0], axis=1)
    return R.DeviceSplats.from_projected(mean2d, np.tile([0.5, 0.0, 0.5], (n, 1)), depths, np.full((n, 3), 0.5),
                                         np.full(n, 0.5), np.ones(n, np.int64), tiles_x * 16, tiles_y * 16)


@pytest.mark.parametrize("name", ["scene_a", "scene_b"])
def test_keys_match_reference_golden(cuda_device, name):
    g, cloud_np, cam = golden_scenes.load(name)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, int(g["degree"]))
    for binning in (R.bin_and_sort(splats, cam.width, cam.height, with_keys=True),
                    R.bin_and_sort_async(splats, cam.width, cam.height, with_keys=True)):
        binning.check()
        k = binning.num_instances
        keys = binning.keys[:k].cpu().numpy()
        np.testing.assert_array_equal(keys.view(np.uint64), np.asarray(g["keys"], np.uint64))
        proj = O.project(cloud_np, cam, int(g["degree"]))
        bins = O.bin_and_sort(proj, cam.width, cam.height)
        np.testing.assert_array_equal(keys.view(np.uint64), np.asarray(bins["keys"], np.uint64))
        np.testing.assert_array_equal(binning.splat_ids[:k].cpu().numpy(), bins["ids"])


def test_criterion5_million_pairs_ties_and_subnormals(cuda_device):
    # test_acceptance.py:177-195 on the device: same generator, same injections
    rng = np.random.default_rng(5)
    n = 1_000_000
    tiles = rng.integers(0, 5000, n).astype(np.int64)
    depths = rng.uniform(0, 1e4, n).astype(np.float32)
    depths[: n // 20] = np.float32(7.25)
    tiles[: n // 20] = 42
    sub = (rng.uniform(1, 100, n // 50) * np.finfo(np.float32).smallest_subnormal).astype(np.float32)
    depths[n // 20: n // 20 + len(sub)] = sub
    tx, ty = 100, 50   # 5000 tiles
    splats = point_splats(tiles, depths, tx, ty)
    b = R.bin_and_sort(splats, tx * 16, ty * 16, with_keys=True)
    expected = np.lexsort((np.arange(n), depths, tiles))
    got = b.splat_ids.cpu().numpy().astype(np.int64)
    assert int(np.sum(got != expected)) == 0
    keys = ref_keys(tiles, depths)
    np.testing.assert_array_equal(b.keys.cpu().numpy(), keys[expected])
    counts = np.bincount(tiles, minlength=tx * ty)
    ends = np.cumsum(counts)
    ranges = np.where(counts[:, None] > 0, np.stack([ends - counts, ends], 1), 0)
    np.testing.assert_array_equal(b.ranges.cpu().numpy(), ranges)


def test_key_order_kat(cuda_device):
    # test_rasterizer.py:39-45: tiles (0,0,1,1), depths (2,1,0.5,3) -> order (1,0,2,3)
    splats = point_splats([0, 0, 1, 1], [2.0, 1.0, 0.5, 3.0], 2, 1)
    b = R.bin_and_sort(splats, 32, 16, with_keys=True)
    np.testing.assert_array_equal(b.splat_ids.cpu().numpy(), [1, 0, 2, 3])
    np.testing.assert_array_equal(b.keys.cpu().numpy(), ref_keys([0, 0, 1, 1], [1.0, 2.0, 0.5, 3.0]))


def test_depth_bits_order_with_denormals(cuda_device):
    # test_rasterizer.py:47-56 on one tile
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.uniform(0, 1e3, 2000).astype(np.float32),
        (rng.uniform(1, 10, 100) * np.finfo(np.float32).smallest_subnormal).astype(np.float32),
        np.float32([0.0, np.finfo(np.float32).tiny, 1e-30, 3.4e38]),
    ])
    splats = point_splats(np.zeros(len(vals), np.int64), vals, 1, 1)
    b = R.bin_and_sort(splats, 16, 16)
    order = b.splat_ids.cpu().numpy()
    assert np.all(np.diff(vals[order]) >= 0)
    np.testing.assert_array_equal(order, np.lexsort((np.arange(len(vals)), vals)))


def test_binning_kats(cuda_device):
    # test_rasterizer.py:59-104: one instance; a splat on a 4-tile corner; off-screen splats
    s = R.DeviceSplats.from_projected([[8.0, 8.0]], [[1.0, 0.0, 1.0]], [1.0], [[1, 1, 1]], [0.5], [3], 64, 64)
    b = R.bin_and_sort(s, 64, 64)
    assert b.num_instances == 1 and tuple(b.ranges[0].tolist()) == (0, 1)
    s = R.DeviceSplats.from_projected([[16.0, 16.0]], [[1.0, 0.0, 1.0]], [1.0], [[1, 1, 1]], [0.5], [3], 64, 64)
    b = R.bin_and_sort(s, 64, 64)
    assert b.num_instances == 4
    nz = [t for t in range(16) if b.ranges[t, 1] > b.ranges[t, 0]]
    assert nz == [0, 1, 4, 5]
    s = R.DeviceSplats.from_projected([[-100.0, 8.0], [8.0, 500.0]], [[1, 0, 1]] * 2, [1.0, 2.0], [[1, 1, 1]] * 2,
                                      [0.5, 0.5], [3, 3], 64, 64)
    b = R.bin_and_sort(s, 64, 64)
    assert b.num_instances == 0 and int(b.ranges.abs().sum()) == 0


def test_no_survivors_and_empty_cloud(cuda_device):
    s = R.DeviceSplats.from_projected(np.zeros((5, 2)), np.tile([1, 0, 1], (5, 1)), np.ones(5), np.ones((5, 3)),
                                      np.full(5, 0.5), np.zeros(5, np.int64), 100, 60)
    b = R.bin_and_sort_async(s, 100, 60, with_keys=True)
    b.check()
    assert b.num_instances == 0 and int(b.ranges.abs().sum()) == 0
    e = R.DeviceSplats.empty(0, "cuda")
    e.status.zero_()
    b = R.bin_and_sort(e, 100, 60)
    assert b.num_instances == 0 and int(b.ranges.abs().sum()) == 0


@pytest.mark.parametrize("w,h", [(16, 16), (200, 136), (1000, 72), (17, 1000)])
def test_one_gaussian_covering_every_tile(cuda_device, w, h):
    tx, ty = R.tile_extent(w, h)
    n = 300
    rng = np.random.default_rng(3)
    mean2d = rng.uniform(0, 1, (n, 2)) * [w, h]
    radius = rng.integers(1, 40, n)
    radius[7] = 10 * max(w, h)   # one splat covers the whole frame
    depth = rng.uniform(1, 5, n).astype(np.float32)
    depth[11] = depth[12]          # an exact tie
    s = R.DeviceSplats.from_projected(mean2d, np.tile([1, 0, 1], (n, 1)), depth, np.ones((n, 3)), np.full(n, 0.5),
                                      radius, w, h)
    b = R.bin_and_sort(s, w, h, with_keys=True)
    proj = {"radius": radius, "rect": s.rect.cpu().numpy(), "tiles": s.tiles_touched.cpu().numpy().astype(np.int64),
            "depth": depth.astype(np.float64)}
    bins = O.bin_and_sort(proj, w, h)
    np.testing.assert_array_equal(b.splat_ids.cpu().numpy(), bins["ids"])
    np.testing.assert_array_equal(b.ranges.cpu().numpy(), bins["ranges"])
    np.testing.assert_array_equal(b.keys.cpu().numpy().view(np.uint64), np.asarray(bins["keys"], np.uint64))
    assert b.num_instances >= tx * ty


def test_large_frame_two_tiles_per_lane(cuda_device):
    # 16384 x 8192: 1024 x 512 tiles -> 16,384 super-tiles of 8 x 4 > 4,096, so
    # super-tiles of 16 x 8 tiles with 2 x 2 tiles per lane
    w, h, n = 16384, 8192, 60_000
    cloud_np, cam = synthetic.frustum_scene(n, w, h, seed=9)
    cloud_np = synthetic.round_to_f32(cloud_np)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, 0)
    b = R.bin_and_sort(splats, w, h)
    proj = O.project(cloud_np, cam, 0)
    bins = O.bin_and_sort(proj, w, h)
    np.testing.assert_array_equal(b.splat_ids.cpu().numpy(), bins["ids"])
    np.testing.assert_array_equal(b.ranges.cpu().numpy(), bins["ranges"])


def test_capacity_overflow_leaves_ranges_empty_then_exact_capacity(cuda_device):
    cloud_np, cam = synthetic.frustum_scene(50_000, 640, 360, seed=4)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    splats = R.project(cloud, cam, 3)
    full = R.bin_and_sort(splats, 640, 360)
    K = full.num_instances
    over = R.bin_and_sort_async(splats, 640, 360, capacity=K - 1)
    with pytest.raises(R.CapacityError):
        over.check()
    assert int(over.ranges.abs().sum()) == 0
    exact = R.bin_and_sort_async(splats, 640, 360, capacity=K)
    exact.check()
    assert torch.equal(exact.splat_ids[:K], full.splat_ids) and torch.equal(exact.ranges, full.ranges)
    # run to run: bit-identical
    again = R.bin_and_sort(splats, 640, 360)
    assert torch.equal(again.splat_ids, full.splat_ids) and torch.equal(again.ranges, full.ranges)
