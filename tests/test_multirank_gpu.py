"""The multi-rank (view-parallel) training path on real kernels.

The pods expose one GPU, so two ranks share cuda:0 over the gloo backend:
that exercises everything the NCCL run does except the transport (view
sharding, the flat gradient bucket, the all-reduce, replicated Adam, the
bench's max-over-ranks timing and rank-0 reporting)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from paper_2308_04079_b200 import synthetic
    cloud_np, cam = synthetic.frustum_scene(30_000, 320, 192, seed=21)
    tgt_np, _ = synthetic.frustum_scene(30_000, 320, 192, seed=22)
    return cloud_np, tgt_np, cam


def _views(cam, tgt_cloud):
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.camera import Camera
    from paper_2308_04079_b200.training import TrainView
    cams = [Camera(np.eye(3), np.array([0.03 * i, -0.02 * i, 0.0]), cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                   cam.height, cam.near) for i in range(2)]
    return [TrainView(c, R.render_view(tgt_cloud, c, (0, 0, 0), 3)[0].image) for c in cams]


def _rank_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.densify import TrainState
    from paper_2308_04079_b200.optimizer import TrainConfig
    from paper_2308_04079_b200.training import train_step
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud_np, tgt_np, cam = _scene()
        views = _views(cam, GaussianCloud.from_numpy(**tgt_np))
        state = TrainState(GaussianCloud.from_numpy(**cloud_np), 10.0, seed=0)
        state.active_sh_degree = 3
        cfg = TrainConfig(warmup_upsample_iters=(0, 0))
        for _ in range(3):
            train_step(state, views, cfg)
        torch.save({g: getattr(state.cloud, g).cpu() for g in ("means", "sh", "opacity_logits")},
                   os.path.join(out_dir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_two_ranks_train_step_matches_accumulated_views(cuda_device, tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_rank_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    r0, r1 = (torch.load(tmp_path / f"rank{r}.pt") for r in range(2))
    for k in r0:   # replicas stay identical: same reduced gradients, same Adam
        assert torch.equal(r0[k], r1[k]), k
    # single process: both views' gradients accumulated, then the same Adam
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.distributed import GradientBucket
    from paper_2308_04079_b200.loss import l1_dssim_loss
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    cloud_np, tgt_np, cam = _scene()
    views = _views(cam, GaussianCloud.from_numpy(**tgt_np))
    cloud = GaussianCloud.from_numpy(**cloud_np)
    adam, cfg = DeviceAdam(cloud), TrainConfig(warmup_upsample_iters=(0, 0))
    bucket = GradientBucket(len(cloud), "cuda")
    for it in range(1, 4):
        bucket.zero_()
        for v in views:
            out, splats, binning = R.render_view(cloud, v.camera, (0, 0, 0), 3, training=True)
            _, d_image = l1_dssim_loss(out.image, v.image, cfg.lambda_dssim)
            g2 = R.render_backward(d_image, out, splats, binning, v.camera.width, v.camera.height, (0, 0, 0))
            R.backward_project(cloud, v.camera, splats, g2, 3, out=bucket.grads, accumulate=True)
        adam.step(cloud, bucket.grads, it, cfg)
    for k in r0:   # float atomics / summation order: within 1e-5 relative
        torch.testing.assert_close(r0[k], getattr(cloud, k).cpu(), rtol=1e-4, atol=1e-6)


def test_bench_two_ranks_one_gpu(cuda_device):
    env = dict(os.environ, GS_DIST_BACKEND="gloo", GS_DEVICE_OVERRIDE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup",
           "3", "--n-gaussians", "200000", "--no-cpu-baseline"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0


def _sharded_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.distributed import GradientBucket, ShardedAdam
    from paper_2308_04079_b200.loss import l1_dssim_loss
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud_np, tgt_np, cam = _scene()
        views = _views(cam, GaussianCloud.from_numpy(**tgt_np))
        cfg = TrainConfig(warmup_upsample_iters=(0, 0))
        cloud_s = GaussianCloud.from_numpy(**cloud_np)
        cloud_r = GaussianCloud.from_numpy(**cloud_np)
        sharded = ShardedAdam(cloud_s)
        replicated, bucket = DeviceAdam(cloud_r), GradientBucket(len(cloud_r), "cuda")
        v = views[rank]
        for it in range(1, 4):
            # one backward (float atomics are order-dependent); both optimisers get the same gradients
            bucket.zero_()
            out, splats, binning = R.render_view(cloud_r, v.camera, (0, 0, 0), 3, training=True)
            _, d_image = l1_dssim_loss(out.image, v.image, cfg.lambda_dssim)
            g2 = R.render_backward(d_image, out, splats, binning, v.camera.width, v.camera.height, (0, 0, 0))
            R.backward_project(cloud_r, v.camera, splats, g2, 3, out=bucket.grads, accumulate=True)
            sharded.zero_()
            for a, b in ((sharded.grads.d_means, bucket.grads.d_means), (sharded.grads.d_sh, bucket.grads.d_sh),
                         (sharded.grads.d_rotations, bucket.grads.d_rotations),
                         (sharded.grads.d_log_scales, bucket.grads.d_log_scales),
                         (sharded.grads.d_opacity_logits, bucket.grads.d_opacity_logits)):
                a.copy_(b)
            sharded.step(cloud_s, it, cfg)
            bucket.allreduce_()
            replicated.step(cloud_r, bucket.grads, it, cfg)
        torch.save({"s": {g: getattr(cloud_s, g).cpu() for g in ("means", "sh", "rotations")},
                    "r": {g: getattr(cloud_r, g).cpu() for g in ("means", "sh", "rotations")},
                    "shard_rows": sharded.exp_avg["means"].shape[0]}, os.path.join(out_dir, f"sh{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_sharded_adam_matches_replicated(cuda_device, tmp_path):
    """Reduce-scatter + Adam on 1/G of the Gaussians + all-gather == all-reduce + full Adam."""
    import torch.multiprocessing as mp
    mp.start_processes(_sharded_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    res = [torch.load(tmp_path / f"sh{r}.pt") for r in range(2)]
    for r in res:
        assert r["shard_rows"] == 15_000   # each rank holds moments for half of the 30,000 Gaussians
        for k in r["s"]:
            assert torch.equal(r["s"][k], r["r"][k]), k
    for k in res[0]["s"]:
        assert torch.equal(res[0]["s"][k], res[1]["s"][k]), k


def _overlap_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.distributed import GradientBucket, OverlapShardedAdam
    from paper_2308_04079_b200.loss import l1_dssim_loss
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud_np, tgt_np, cam = _scene()
        views = _views(cam, GaussianCloud.from_numpy(**tgt_np))
        cfg = TrainConfig(warmup_upsample_iters=(0, 0))
        cloud_o = GaussianCloud.from_numpy(**cloud_np)
        cloud_r = GaussianCloud.from_numpy(**cloud_np)
        opt = OverlapShardedAdam(cloud_o)
        replicated, bucket = DeviceAdam(cloud_r), GradientBucket(len(cloud_r), "cuda")
        mine = [views[rank], views[1 - rank]]   # two views per rank, the second one reduces
        for it in range(1, 4):
            opt.zero_()
            bucket.zero_()
            for i, v in enumerate(mine):
                # the same screen-space gradients feed both paths (the blend's float atomics are order-dependent)
                out, splats, binning = R.render_view(cloud_r, v.camera, (0, 0, 0), 3, training=True)
                _, d_image = l1_dssim_loss(out.image, v.image, cfg.lambda_dssim)
                g2 = R.render_backward(d_image, out, splats, binning, v.camera.width, v.camera.height, (0, 0, 0))
                R.backward_project(cloud_r, v.camera, splats, g2, 3, out=bucket.grads, accumulate=True)
                splats_o = R._project_tensors(cloud_o.c_params(), len(cloud_o), "cuda", v.camera, 3)
                assert torch.equal(splats_o.rec, splats.rec)
                opt.accumulate(cloud_o, v.camera, splats_o, g2, 3, reduce=(i == len(mine) - 1))
            opt.step(cloud_o, it, cfg)
            bucket.allreduce_()
            replicated.step(cloud_r, bucket.grads, it, cfg)
        torch.save({"o": {g: getattr(cloud_o, g).cpu() for g in ("means", "sh", "rotations", "log_scales",
                                                                  "opacity_logits")},
                    "r": {g: getattr(cloud_r, g).cpu() for g in ("means", "sh", "rotations", "log_scales",
                                                                  "opacity_logits")}},
                   os.path.join(out_dir, f"ov{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_overlap_sharded_adam_matches_replicated(cuda_device, tmp_path):
    """Range-by-range backward with the last view's per-range reductions
    enqueued as the ranges finish, Adam on the rank's range, all-gather ==
    all-reduce + full Adam (bit-identical at two ranks)."""
    import torch.multiprocessing as mp
    mp.start_processes(_overlap_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    res = [torch.load(tmp_path / f"ov{r}.pt") for r in range(2)]
    for r in res:
        for k in r["o"]:
            assert torch.equal(r["o"][k], r["r"][k]), k
    for k in res[0]["o"]:
        assert torch.equal(res[0]["o"][k], res[1]["o"][k]), k


def test_multiview_two_streams_matches_one(cuda_device):
    """train_step_views with views alternating over 2 CUDA streams (per-stream
    buckets and statistics merged) == the single-stream accumulation."""
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200 import synthetic
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.distributed import GradientBucket, train_step_views
    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    cloud_np = synthetic.ball_scene(40_000, seed=3)
    cams = synthetic.ball_cameras(6, width=320, height=180)
    tgt = GaussianCloud.from_numpy(**synthetic.ball_scene(40_000, seed=4))
    targets = [R.render_view(tgt, c, (0, 0, 0), 3)[0].image for c in cams]
    results = []
    for streams in (1, 2):
        cloud = GaussianCloud.from_numpy(**cloud_np)
        adam, bucket = DeviceAdam(cloud), GradientBucket(len(cloud), "cuda")
        stats = R.DensifyStats.zeros(len(cloud), "cuda")
        loss = train_step_views(cloud, cams, targets, adam, TrainConfig(), 1, bucket, stats, streams=streams)
        torch.cuda.synchronize()
        results.append((cloud, stats, float(loss)))
    (c1, s1, l1), (c2, s2, l2) = results
    assert abs(l1 - l2) <= 1e-6 * abs(l1)
    for g in ("means", "sh", "rotations", "log_scales", "opacity_logits"):
        torch.testing.assert_close(getattr(c2, g), getattr(c1, g), rtol=1e-5, atol=1e-7)
    assert torch.equal(s1.accum_count, s2.accum_count)
    assert torch.equal(s1.max_radius_frac, s2.max_radius_frac)
    torch.testing.assert_close(s2.accum_pos_grad, s1.accum_pos_grad, rtol=1e-5, atol=1e-9)


def _densify_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.camera import Camera
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.densify import TrainState
    from paper_2308_04079_b200.optimizer import TrainConfig
    from paper_2308_04079_b200.training import TrainView, train
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud_np, tgt_np, cam = _scene()
        tgt = GaussianCloud.from_numpy(**tgt_np)
        # three views over two ranks: uneven shards (1 and 2 views), so the ranks'
        # view-sampling RNG streams diverge before the densify step
        cams = [Camera(np.eye(3), np.array([0.03 * i, -0.02 * i, 0.0]), cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                       cam.height, cam.near) for i in range(3)]
        views = [TrainView(c, R.render_view(tgt, c, (0, 0, 0), 3)[0].image) for c in cams]
        state = TrainState(GaussianCloud.from_numpy(**cloud_np), 2.0, seed=rank)   # different RNG seeds too
        cfg = TrainConfig(warmup_upsample_iters=(0, 0), densify_start=0, densify_interval=3,
                          densify_grad_threshold=2e-6)
        ckpts = []
        reports = train(state, views, cfg, iterations=7, checkpoint_hook=lambda s: ckpts.append(
            (s.iteration, len(s.cloud), getattr(s, "_lookahead", None) is None)), checkpoint_iters=(4, 7))
        torch.save({"params": {g: getattr(state.cloud, g).cpu() for g in ("means", "sh", "opacity_logits")},
                    "n": len(state.cloud), "reports": [(r.cloned, r.split, r.pruned) for r in reports],
                    "ckpts": ckpts}, os.path.join(out_dir, f"dn{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_two_ranks_train_across_densify_stay_identical(cuda_device, tmp_path):
    """train() under torch.distributed crossing two densify intervals: the
    statistics are reduced over the ranks and rank 0's RNG is shared, so both
    replicas clone / split / prune identically and stay bit-identical; the
    checkpoint hook fires at its iterations with no lookahead pending."""
    import torch.multiprocessing as mp
    mp.start_processes(_densify_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    r0, r1 = (torch.load(tmp_path / f"dn{r}.pt") for r in range(2))
    assert r0["reports"] == r1["reports"] and len(r0["reports"]) == 2
    assert sum(c + s for c, s, _ in r0["reports"]) > 0   # the densification really cloned / split
    assert r0["n"] == r1["n"]
    for k in r0["params"]:
        assert torch.equal(r0["params"][k], r1["params"][k]), k
    assert [c[0] for c in r0["ckpts"]] == [4, 7] and all(c[2] for c in r0["ckpts"])


def _zero1_worker(rank, world, port, out_dir, sharded, nan_rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.camera import Camera
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.densify import TrainState
    from paper_2308_04079_b200.errors import TrainingDiverged
    from paper_2308_04079_b200.optimizer import TrainConfig
    from paper_2308_04079_b200.training import TrainView, train, train_step
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud_np, tgt_np, cam = _scene()
        tgt = GaussianCloud.from_numpy(**tgt_np)
        cams = [Camera(np.eye(3), np.array([0.03 * i, -0.02 * i, 0.0]), cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                       cam.height, cam.near) for i in range(4)]
        views = [TrainView(c, R.render_view(tgt, c, (0, 0, 0), 3)[0].image) for c in cams]
        state = TrainState(GaussianCloud.from_numpy(**cloud_np), 2.0, seed=0)
        state.shard_optimizer = sharded
        # deterministic backward: the two runs (separate processes) must not
        # differ by float-atomic order
        cfg = TrainConfig(warmup_upsample_iters=(0, 0), densify_start=0, densify_interval=3,
                          densify_grad_threshold=2e-6, deterministic=True)
        if nan_rank is not None:   # one rank's view diverges: every rank must raise, none may hang
            train_step(state, views, cfg)
            bad = [TrainView(v.camera, v.image.clone()) for v in views]
            if rank == nan_rank:
                for v in bad:
                    v.image[0, 0, 0] = float("nan")
            try:
                train_step(state, bad, cfg)
                raised = False
            except TrainingDiverged:
                raised = True
            torch.save({"raised": raised}, os.path.join(out_dir, f"nan{rank}.pt"))
            return
        reports = train(state, views, cfg, iterations=7)
        torch.save({"params": {g: getattr(state.cloud, g).cpu() for g in ("means", "sh", "opacity_logits")},
                    "n": len(state.cloud), "reports": [(r.cloned, r.split, r.pruned) for r in reports]},
                   os.path.join(out_dir, f"z{int(sharded)}_{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_zero1_training_across_densify_matches_replicated(cuda_device, tmp_path):
    """state.shard_optimizer: reduce-scatter + Adam on 1/G of the Gaussians +
    all-gather, re-sharded after every densification (moments gathered,
    realigned, re-sharded): bit-identical to the replicated all-reduce path."""
    import torch.multiprocessing as mp
    for sharded in (False, True):
        mp.start_processes(_zero1_worker, args=(2, _free_port(), str(tmp_path), sharded, None), nprocs=2,
                           start_method="spawn")
    res = {(s, r): torch.load(tmp_path / f"z{s}_{r}.pt") for s in (0, 1) for r in (0, 1)}
    assert res[(1, 0)]["reports"] == res[(0, 0)]["reports"] and sum(c + s for c, s, _ in res[(1, 0)]["reports"]) > 0
    for r in (0, 1):
        assert res[(1, r)]["n"] == res[(0, r)]["n"]
        for k in res[(0, 0)]["params"]:
            assert torch.equal(res[(1, r)]["params"][k], res[(0, 0)]["params"][k]), (r, k)


def test_one_rank_diverging_raises_on_every_rank(cuda_device, tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_zero1_worker, args=(2, _free_port(), str(tmp_path), False, 1), nprocs=2,
                       start_method="spawn")
    assert all(torch.load(tmp_path / f"nan{r}.pt")["raised"] for r in (0, 1))
