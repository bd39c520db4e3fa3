"""Multi-process (gloo, world sizes 2 and 4, CPU) tests of the view-parallel
plumbing: view sharding, the flat gradient bucket and its all-reduce, the
cross-rank densification statistics, the rank-reduced step verdict and the
shared training RNG."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_04079_b200.distributed import (FLOATS_PER_GAUSSIAN, GradientBucket, any_rank_, max_reduce_,
                                                reduce_stats_, shard_views, sync_rng_)
from paper_2308_04079_b200.rasterizer import DensifyStats


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 5
        bucket = GradientBucket(n, "cpu")
        g = bucket.grads
        # each rank writes a distinct per-view gradient through the group views
        g.d_means.fill_(rank + 1.0)
        g.d_sh[:, 0, 0] = 10.0 * (rank + 1)
        g.d_opacity_logits[2] = -1.0
        bucket.allreduce_()
        stats = DensifyStats(torch.full((n,), float(rank + 1)), torch.full((n,), rank + 1, dtype=torch.int32),
                             torch.tensor([0.1 * (rank + 1)] * n))
        reduce_stats_(stats)
        results[rank] = {
            "means": g.d_means.clone(), "sh00": g.d_sh[:, 0, 0].clone(), "opac": g.d_opacity_logits.clone(),
            "flat_is_view": g.d_means.data_ptr() == bucket.flat.data_ptr(),
            "accum": stats.accum_pos_grad.clone(), "count": stats.accum_count.clone(),
            "maxr": stats.max_radius_frac.clone(),
        }
    finally:
        dist.destroy_process_group()


def test_gradient_bucket_and_stats_allreduce_world2():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
        res = dict(results)
    for rank in range(world):
        r = res[rank]
        assert r["flat_is_view"]
        assert torch.all(r["means"] == 3.0)             # 1 + 2
        assert torch.all(r["sh00"] == 30.0)             # 10 + 20
        assert float(r["opac"][2]) == -2.0 and float(r["opac"][0]) == 0.0
        assert torch.all(r["accum"] == 3.0)
        assert torch.all(r["count"] == 3)
        assert torch.allclose(r["maxr"], torch.full((5,), 0.2))
    # replicas hold bit-identical reduced gradients
    assert torch.equal(res[0]["means"], res[1]["means"])


def test_bucket_layout():
    b = GradientBucket(7, "cpu")
    assert FLOATS_PER_GAUSSIAN == 59 and b.flat.numel() >= 7 * FLOATS_PER_GAUSSIAN
    assert b.grads.d_sh.shape == (7, 16, 3) and b.grads.d_rotations.shape == (7, 4)
    # every group view starts 16-byte aligned whatever N (the kernels use vector accesses)
    for t in (b.grads.d_means, b.grads.d_rotations, b.grads.d_log_scales, b.grads.d_opacity_logits, b.grads.d_sh):
        assert t.data_ptr() % 16 == 0 and t.is_contiguous()
    b.grads.d_sh.fill_(1.0)
    assert float(b.flat.sum()) == 7 * 48


@pytest.mark.parametrize("views,world", [(32, 2), (32, 4), (32, 8), (7, 3), (1, 2)])
def test_shard_views_partition(views, world):
    shards = [shard_views(views, world, r) for r in range(world)]
    flat = [v for s in shards for v in s]
    assert flat == list(range(views))
    assert max(map(len, shards)) - min(map(len, shards)) <= 1


def _worker4(rank, world, port, results):
    """World size 4: every rank holds a different shard of a 32-view batch,
    accumulates one gradient per view into its bucket, and the reduced bucket
    equals the sum over all 32 views; the step verdict is the union of the
    ranks' flags; the shared RNG leaves every rank with rank 0's state."""
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 7
        mine = shard_views(32, world, rank)
        bucket = GradientBucket(n, "cpu")
        for v in mine:   # per-view gradients accumulate before the reduction
            bucket.grads.d_means += float(v + 1)
            bucket.grads.d_sh[:, 3, 1] += 0.5
        bucket.allreduce_()
        stats = DensifyStats(torch.full((n,), 1.0), torch.full((n,), len(mine), dtype=torch.int32),
                             torch.full((n,), 0.01 * (rank + 1)))
        reduce_stats_(stats)
        verdict = torch.tensor([1 if rank == 2 else 0, 0, 1 if rank == 3 else 0, 0], dtype=torch.int32)
        max_reduce_(verdict)

        class _S:
            rng = np.random.default_rng(100 + rank)
        st = _S()
        sync_rng_(st)
        results[rank] = {"views": mine, "means": bucket.grads.d_means.clone(), "sh": bucket.grads.d_sh[:, 3, 1].clone(),
                         "accum": stats.accum_pos_grad.clone(), "count": stats.accum_count.clone(),
                         "maxr": stats.max_radius_frac.clone(), "verdict": verdict.tolist(),
                         "any": any_rank_(rank == 1, "cpu"), "draw": float(st.rng.standard_normal())}
    finally:
        dist.destroy_process_group()


def test_view_parallel_plumbing_world4():
    import numpy as np
    world = 4
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker4, args=(world, port, results), nprocs=world, join=True)
        res = dict(results)
    assert sorted(v for r in range(world) for v in res[r]["views"]) == list(range(32))
    expect = float(sum(range(1, 33)))
    for r in range(world):
        assert torch.all(res[r]["means"] == expect)
        assert torch.all(res[r]["sh"] == 16.0)
        assert torch.all(res[r]["accum"] == 4.0) and torch.all(res[r]["count"] == 32)
        assert torch.allclose(res[r]["maxr"], torch.full((7,), 0.04))
        assert res[r]["verdict"] == [1, 0, 1, 0] and res[r]["any"] is True
        assert res[r]["draw"] == float(np.random.default_rng(100).standard_normal())


def _overlap_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_04079_b200.cloud import GaussianCloud
        from paper_2308_04079_b200.distributed import OverlapShardedAdam
        n = 300
        g = torch.Generator().manual_seed(0)
        cloud = GaussianCloud(torch.randn(n, 3, generator=g), torch.randn(n, 4, generator=g),
                              torch.randn(n, 3, generator=g), torch.randn(n, generator=g),
                              torch.randn(n, 16, 3, generator=g))
        means0 = cloud.means.clone()
        opt = OverlapShardedAdam(cloud)
        # every range's gradient block gets a rank-dependent value, then the
        # per-range reductions run as the last view's backward would issue them
        for r, (a, b) in enumerate(opt.bounds):
            cg = opt.chunk_grads(r)
            cg.d_means.fill_(rank + 1.0)
            cg.d_sh[:, 0, 0] = 10.0 * (rank + 1) + r
        for r in range(world):
            opt._reduce_block(r)
        for w in opt._works:
            w.wait()
        own = opt.chunk_grads(opt.rank)
        results[rank] = {"per": opt.per, "bounds": opt.bounds, "lo": opt.lo, "hi": opt.hi,
                         "own_means": own.d_means.clone(), "own_sh00": own.d_sh[:, 0, 0].clone(),
                         "cloud_is_view": cloud.means.data_ptr() == opt.pbuf["means"].data_ptr(),
                         "params_kept": bool(torch.equal(cloud.means, means0)),
                         "block_aligned": all((opt.chunk[r][grp].data_ptr() % 16) == 0
                                              for r in range(world) for grp in opt.chunk[r]),
                         "blocks_in_flat": all(opt.blocks[r].data_ptr() == opt.flat.data_ptr() + 4 * r * opt.block
                                               for r in range(world))}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_overlap_sharded_layout_and_reduction(world):
    """OverlapShardedAdam: rank-major gradient blocks (one per Gaussian range,
    128-row aligned), the cloud re-homed into padded parameter buffers, and
    the per-range reduction leaving every owner its range's summed gradient."""
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_overlap_worker, args=(world, port, results), nprocs=world, join=True)
        res = dict(results)
    total = sum(range(1, world + 1))
    for rank in range(world):
        r = res[rank]
        assert r["per"] % 128 == 0 and r["per"] * world >= 300
        assert r["bounds"][0][0] == 0 and r["bounds"][-1][1] == 300
        assert all(r["bounds"][i][1] == r["bounds"][i + 1][0] for i in range(world - 1))
        assert r["cloud_is_view"] and r["params_kept"] and r["block_aligned"] and r["blocks_in_flat"]
        k = r["hi"] - r["lo"]
        assert r["own_means"].shape == (k, 3)
        assert torch.all(r["own_means"] == float(total))
        assert torch.all(r["own_sh00"] == 10.0 * total + world * rank)
