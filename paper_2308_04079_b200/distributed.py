"""View-parallel multi-GPU training plumbing.

Views are independent units of work; parameters and Adam state are
replicated.  Each rank renders its shard of the camera batch, accumulating
its views' gradients into one flat (N x 59) float32 bucket (so a single NCCL
all-reduce covers all five groups), then every rank runs the identical fused
Adam on the reduced gradients.  Densification statistics are per view and
accumulate on each rank before the cross-rank reduction
(optimizer.py:252-254); the reduction sums accum_pos_grad/accum_count and
takes the max of max_radius_frac.

ShardedAdam is the reduce-scatter alternative: the same wire bytes, but each
rank stores and updates the Adam moments of 1/G of the Gaussians only.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from .cloud import PARAM_GROUPS
from .rasterizer import DensifyStats, GaussianGrads

GROUP_WIDTHS = (("d_means", 3), ("d_rotations", 4), ("d_log_scales", 3), ("d_opacity_logits", 1), ("d_sh", 48))
_ROW_SHAPE = {"means": (3,), "rotations": (4,), "log_scales": (3,), "opacity_logits": (), "sh": (16, 3)}
FLOATS_PER_GAUSSIAN = sum(w for _, w in GROUP_WIDTHS)  # 59


def shard_views(num_views: int, world: int, rank: int) -> list[int]:
    """Contiguous shard of a camera batch: rank r gets views [r*B/G, (r+1)*B/G)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    lo = (num_views * rank) // world
    hi = (num_views * (rank + 1)) // world
    return list(range(lo, hi))


def _seg(numel: int) -> int:
    """Segment length padded to 64 floats (256 B), so every group of a flat
    bucket starts 16-byte aligned for the kernels' vector accesses whatever
    the Gaussian count."""
    return -(-numel // 64) * 64


class GradientBucket:
    """One flat float32 buffer with GaussianGrads views into it (one padded,
    aligned segment per parameter group)."""

    def __init__(self, n: int, device, dtype=torch.float32):
        self.n = n
        segs = [_seg(n * w) for _, w in GROUP_WIDTHS]
        self.flat = torch.zeros(sum(segs), dtype=dtype, device=device)
        parts = torch.split(self.flat, segs)
        shapes = {"d_means": (n, 3), "d_rotations": (n, 4), "d_log_scales": (n, 3), "d_opacity_logits": (n,),
                  "d_sh": (n, 16, 3)}
        views = {name: part[:n * w].view(shapes[name]) for (name, w), part in zip(GROUP_WIDTHS, parts)}
        self.grads = GaussianGrads(views["d_means"], views["d_rotations"], views["d_log_scales"],
                                   views["d_opacity_logits"], views["d_sh"],
                                   torch.zeros(n, dtype=dtype, device=device))

    def zero_(self) -> None:
        self.flat.zero_()

    def allreduce_(self, group=None) -> None:
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)


def reduce_stats_(stats: DensifyStats, group=None) -> None:
    """Cross-rank densification statistics: sums and max (in place)."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return
    dist.all_reduce(stats.accum_pos_grad, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(stats.accum_count, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(stats.max_radius_frac, op=dist.ReduceOp.MAX, group=group)


def max_reduce_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place MAX all-reduce of a small device tensor (no host round trip
    on NCCL; gloo stages it through the host)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
            t.copy_(h)
    return t


def any_rank_(flag: bool, device, group=None) -> bool:
    """True on every rank when `flag` is true on any rank (MAX all-reduce)."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return bool(flag)
    dev = device if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return bool(t.item())


def sync_rng_(state, group=None) -> None:
    """Give every rank rank 0's training-RNG state (TrainState.rng), so the
    split samples drawn by densify_and_prune (optimizer.py:335) are identical
    on all replicas."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return
    obj = [state.rng.bit_generator.state]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    state.rng.bit_generator.state = obj[0]


def train_step_views(cloud, cameras, targets, adam, config, iteration: int, bucket: GradientBucket,
                     stats: DensifyStats | None = None, background=(0.0, 0.0, 0.0), active_sh_degree: int = 3,
                     group=None, streams: int = 1) -> torch.Tensor:
    """One multi-view training iteration on this rank's views: per view
    project -> bin -> blend -> loss -> blend bwd -> backward_project
    (accumulated into the bucket), then the all-reduce and the Adam step.
    Returns the summed loss of this rank's views (device scalar).

    streams > 1 runs consecutive views on that many CUDA streams, each with
    its own gradient bucket and statistics (summed / max-reduced before the
    all-reduce), so the latency-bound binning of one view overlaps the
    compute-bound blending of another.  The binning is the sync-free variant
    (instance count and flags checked once, after the batch)."""
    from . import rasterizer as R
    from .loss import l1_dssim_loss

    main = torch.cuda.current_stream(cloud.device)
    lanes = [(main, bucket, stats)]
    if streams > 1:
        aux = getattr(bucket, "_aux_lanes", None)
        if aux is None or len(aux) != streams - 1:
            aux = [(torch.cuda.Stream(cloud.device), GradientBucket(bucket.n, cloud.device),
                    DensifyStats.zeros(bucket.n, cloud.device) if stats is not None else None)
                   for _ in range(streams - 1)]
            bucket._aux_lanes = aux
        lanes += aux
    bucket.zero_()
    for s, b, st in lanes[1:]:
        s.wait_stream(main)
        with torch.cuda.stream(s):
            b.zero_()
            if st is not None:
                st.accum_pos_grad.zero_()
                st.accum_count.zero_()
                st.max_radius_frac.zero_()
    totals, k_infos = [], []
    # per view: the previous batch's longest-first backward schedule orders this forward's tiles
    orders = bucket.__dict__.setdefault("_tile_orders", {})
    for i, (cam, gt) in enumerate(zip(cameras, targets)):
        s, b, st = lanes[i % len(lanes)]
        key = (i, cam.width, cam.height)
        with torch.cuda.stream(s):
            if streams > 1:
                out, splats, binning = R.render_view_async(cloud, cam, background, active_sh_degree, training=True,
                                                           tile_order=orders.get(key))
                k_infos.append(binning.k_info)
            else:
                out, splats, binning = R.render_view(cloud, cam, background, active_sh_degree, training=True)
            prep = R.prepare_backward(out, splats, binning, cam.width, cam.height)   # beside the loss
            loss, d_image = l1_dssim_loss(out.image, gt, config.lambda_dssim)
            g2 = R.render_backward(d_image, out, splats, binning, cam.width, cam.height, background, prep=prep)
            if g2.tile_order is not None:
                orders[key] = g2.tile_order
            R.backward_project(cloud, cam, splats, g2, active_sh_degree, stats=st, out=b.grads, accumulate=True)
            totals.append(loss[0:1])
    for s, b, st in lanes[1:]:
        main.wait_stream(s)
        bucket.flat.add_(b.flat)
        if st is not None:
            stats.accum_pos_grad.add_(st.accum_pos_grad)
            stats.accum_count.add_(st.accum_count)
            torch.maximum(stats.max_radius_frac, st.max_radius_frac, out=stats.max_radius_frac)
    if k_infos and bool((torch.stack(k_infos)[:, 1] != 0).any()):
        raise R.CapacityError("multi-view batch: a view overflowed its instance capacity; re-run the batch")
    bucket.allreduce_(group)
    adam.step(cloud, bucket.grads, iteration, config)
    return torch.cat(totals).sum()


def _world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


class ShardedAdam:
    """View-parallel training with the optimizer sharded over the ranks
    (the reduce-scatter alternative): the summed gradients are
    reduce-scattered by Gaussian range, every rank runs Adam on its shard
    only (its moments are the only ones it stores: 1/G of the Adam state and
    of the Adam HBM traffic), and the updated parameter shards are
    all-gathered.  Same wire bytes as an all-reduce of the gradients.

    The cloud's parameter tensors are re-homed into buffers padded to a
    multiple of the world size (the cloud keeps contiguous views of their
    first N rows).  The Gaussian count is fixed for the lifetime of the
    object: densify / prune gathers the moments (full_moments), realigns them
    with the cloud (densify_and_prune on replicated moments) and re-shards
    (from_moments)."""

    def __init__(self, cloud, group=None):
        self.group = group
        self.world, self.rank = _world(group)
        self.n = n = len(cloud)
        self.per = per = max(1, -(-n // self.world))
        npad = per * self.world
        dev = cloud.device
        self.lo, self.hi = min(n, self.rank * per), min(n, (self.rank + 1) * per)
        z = dict(dtype=torch.float32, device=dev)
        self.pbuf = {}
        for g in PARAM_GROUPS:
            buf = torch.zeros((npad,) + _ROW_SHAPE[g], **z)
            buf[:n].copy_(getattr(cloud, g))
            setattr(cloud, g, buf[:n])
            self.pbuf[g] = buf
        # gradient bucket: one padded segment per group, contiguous in one flat buffer
        widths = [math.prod(_ROW_SHAPE[g]) for g in PARAM_GROUPS]
        segs = [_seg(npad * w) for w in widths]
        self.flat = torch.zeros(sum(segs), **z)
        parts = torch.split(self.flat, segs)
        self.gbuf = {g: part[:npad * w].view((npad,) + _ROW_SHAPE[g]) for g, w, part in zip(PARAM_GROUPS, widths,
                                                                                             parts)}
        self.grads = GaussianGrads(*(self.gbuf[g][:n] for g in ("means", "rotations", "log_scales",
                                                                   "opacity_logits", "sh")),
                                   torch.zeros(n, **z))
        self.shard_grad = {g: torch.zeros((per,) + _ROW_SHAPE[g], **z) for g in PARAM_GROUPS}
        self.exp_avg = {g: torch.zeros((per,) + _ROW_SHAPE[g], **z) for g in PARAM_GROUPS}
        self.exp_avg_sq = {g: torch.zeros((per,) + _ROW_SHAPE[g], **z) for g in PARAM_GROUPS}

    def zero_(self) -> None:
        self.flat.zero_()

    def _reduce_scatter(self, out: torch.Tensor, full: torch.Tensor) -> None:
        if self.world == 1:
            out.copy_(full)
        elif dist.get_backend(self.group) == "nccl":
            dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.SUM, group=self.group)
        else:   # gloo has no reduce-scatter: all-reduce, keep this rank's rows
            dist.all_reduce(full, op=dist.ReduceOp.SUM, group=self.group)
            out.copy_(full[self.rank * self.per:(self.rank + 1) * self.per])

    def _all_gather(self, full: torch.Tensor) -> None:
        shard = full[self.rank * self.per:(self.rank + 1) * self.per]
        if self.world == 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(full, shard, group=self.group)   # in place: the shard is full's slice
        else:
            parts = list(torch.split(full, self.per))
            dist.all_gather(parts, shard.clone(), group=self.group)

    def step(self, cloud, iteration: int, config, skip: torch.Tensor | None = None) -> None:
        """Reduce-scatter the bucket, Adam on this rank's shard, all-gather.
        skip (device int32, the same on every rank): applies nothing."""
        from .optimizer import adam_step_tensors
        for g in PARAM_GROUPS:
            self._reduce_scatter(self.shard_grad[g], self.gbuf[g])
        k = self.hi - self.lo
        if k > 0:
            adam_step_tensors({g: self.pbuf[g][self.lo:self.hi] for g in PARAM_GROUPS},
                              {g: self.shard_grad[g][:k] for g in PARAM_GROUPS},
                              {g: self.exp_avg[g][:k] for g in PARAM_GROUPS},
                              {g: self.exp_avg_sq[g][:k] for g in PARAM_GROUPS}, iteration, config, skip=skip)
        for g in PARAM_GROUPS:
            self._all_gather(self.pbuf[g])

    def full_moments(self) -> tuple[dict, dict]:
        """Every rank's moment shards gathered into full (N, ...) tensors."""
        out = []
        for src in (self.exp_avg, self.exp_avg_sq):
            full = {}
            for g in PARAM_GROUPS:
                buf = torch.zeros((self.per * self.world,) + _ROW_SHAPE[g], dtype=torch.float32,
                                  device=src[g].device)
                buf[self.rank * self.per:(self.rank + 1) * self.per].copy_(src[g])
                self._all_gather(buf)
                full[g] = buf[:self.n].contiguous()
            out.append(full)
        return out[0], out[1]

    @classmethod
    def from_moments(cls, cloud, exp_avg: dict, exp_avg_sq: dict, group=None) -> "ShardedAdam":
        """A ShardedAdam for `cloud` whose shards start from full moments."""
        sa = cls(cloud, group)
        k = sa.hi - sa.lo
        for g in PARAM_GROUPS:
            if k > 0:
                sa.exp_avg[g][:k].copy_(exp_avg[g][sa.lo:sa.hi])
                sa.exp_avg_sq[g][:k].copy_(exp_avg_sq[g][sa.lo:sa.hi])
        return sa


class OverlapShardedAdam:
    """ZeRO-1 view-parallel training whose gradient reduction overlaps the
    per-Gaussian backward.

    The gradient bucket is rank-major: block r holds the five groups' rows of
    rank r's Gaussian range [r P, (r + 1) P) (P = ceil(N / G) rounded up to a
    multiple of 128, so every group's block starts 16-byte aligned).  Each
    view's projection backward runs in G launches, one per range
    (`accumulate`: the kernels see a range as a cloud of its own through
    row-offset tensor views).  For the batch's last view (`reduce=True`) the
    reduction of block r to its owner is enqueued (NCCL `reduce`, async) right
    after range r's backward, so it runs on NCCL's stream while the ranges
    after it are still being computed; `step` waits for the reductions, runs
    Adam on the rank's own block (its moments are the only ones stored) and
    all-gathers the updated parameters.  Same wire bytes as a reduce-scatter;
    with two ranks the result is bit-identical to the all-reduce + replicated
    Adam path (a sum of two terms does not depend on the order)."""

    ALIGN = 128

    def __init__(self, cloud, group=None):
        self.group = group
        self.world, self.rank = _world(group)
        self.n = n = len(cloud)
        per = max(1, -(-n // self.world))
        self.per = per = -(-per // self.ALIGN) * self.ALIGN
        npad = per * self.world
        dev = cloud.device
        z = dict(dtype=torch.float32, device=dev)
        self.bounds = [(min(n, r * per), min(n, (r + 1) * per)) for r in range(self.world)]
        self.lo, self.hi = self.bounds[self.rank]
        self.pbuf = {}
        for g in PARAM_GROUPS:
            buf = torch.zeros((npad,) + _ROW_SHAPE[g], **z)
            buf[:n].copy_(getattr(cloud, g))
            setattr(cloud, g, buf[:n])
            self.pbuf[g] = buf
        widths = [math.prod(_ROW_SHAPE[g]) for g in PARAM_GROUPS]
        segs = [_seg(per * w) for w in widths]
        self.block = sum(segs)
        self.flat = torch.zeros(self.world * self.block, **z)
        self.blocks = list(torch.split(self.flat, self.block))
        self.chunk = []   # per range: {group: (per, ...) view}
        for blk in self.blocks:
            parts = torch.split(blk, segs)
            self.chunk.append({g: part[:per * w].view((per,) + _ROW_SHAPE[g])
                               for g, w, part in zip(PARAM_GROUPS, widths, parts)})
        self._norm = torch.zeros(per, **z)   # view_pos_grad_norm scratch (the statistics take their own)
        self.exp_avg = {g: torch.zeros((per,) + _ROW_SHAPE[g], **z) for g in PARAM_GROUPS}
        self.exp_avg_sq = {g: torch.zeros((per,) + _ROW_SHAPE[g], **z) for g in PARAM_GROUPS}
        self._works = []

    def zero_(self) -> None:
        self.flat.zero_()

    def chunk_grads(self, r: int) -> GaussianGrads:
        a, b = self.bounds[r]
        c = self.chunk[r]
        k = b - a
        return GaussianGrads(c["means"][:k], c["rotations"][:k], c["log_scales"][:k], c["opacity_logits"][:k],
                             c["sh"][:k], self._norm[:k])

    def _reduce_block(self, r: int) -> None:
        if self.world == 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dst = dist.get_global_rank(self.group, r) if self.group is not None else r
            self._works.append(dist.reduce(self.blocks[r], dst=dst, op=dist.ReduceOp.SUM, group=self.group,
                                           async_op=True))
        else:   # gloo: CUDA tensors are reduced with all_reduce (the owner keeps its block)
            self._works.append(dist.all_reduce(self.blocks[r], op=dist.ReduceOp.SUM, group=self.group,
                                               async_op=True))

    def accumulate(self, cloud, camera, splats, grads2d, active_sh_degree: int = 3, stats=None,
                   reduce: bool = False) -> None:
        """Add one view's parameter gradients (range by range); with `reduce`
        (the batch's last view) each range's reduction to its owner is
        enqueued as soon as the range is done."""
        from . import rasterizer as R
        from .cloud import GaussianCloud
        for r, (a, b) in enumerate(self.bounds):
            if b > a:
                sub = GaussianCloud(*(getattr(cloud, g)[a:b] for g in ("means", "rotations", "log_scales",
                                                                      "opacity_logits", "sh")))
                sp = R.DeviceSplats(splats.rec[a:b], splats.depth[a:b], splats.radii[a:b], splats.rect[a:b],
                                    splats.tiles_touched[a:b], splats.status)
                g2 = R.SplatGrads2D(grads2d.packed[a:b], None, grads2d.rec[a:b] if grads2d.rec is not None else None)
                st = (R.DensifyStats(stats.accum_pos_grad[a:b], stats.accum_count[a:b], stats.max_radius_frac[a:b])
                      if stats is not None else None)
                R.backward_project(sub, camera, sp, g2, active_sh_degree, stats=st, out=self.chunk_grads(r),
                                   accumulate=True)
            if reduce:
                self._reduce_block(r)

    def step(self, cloud, iteration: int, config, skip: torch.Tensor | None = None) -> None:
        """Wait for the reductions, Adam on this rank's range, all-gather."""
        from .optimizer import adam_step_tensors
        for w in self._works:
            w.wait()
        self._works = []
        k = self.hi - self.lo
        if k > 0:
            own = self.chunk[self.rank]
            adam_step_tensors({g: self.pbuf[g][self.lo:self.hi] for g in PARAM_GROUPS},
                              {g: own[g][:k] for g in PARAM_GROUPS},
                              {g: self.exp_avg[g][:k] for g in PARAM_GROUPS},
                              {g: self.exp_avg_sq[g][:k] for g in PARAM_GROUPS}, iteration, config, skip=skip)
        if self.world > 1:
            for g in PARAM_GROUPS:
                full = self.pbuf[g]
                shard = full[self.rank * self.per:(self.rank + 1) * self.per]
                if dist.get_backend(self.group) == "nccl":
                    dist.all_gather_into_tensor(full, shard, group=self.group)
                else:
                    parts = list(torch.split(full, self.per))
                    dist.all_gather(parts, shard.clone(), group=self.group)
