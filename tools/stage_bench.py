"""Kernel-variant microbenchmark: times the blend kernels (and the binning)
on the c3 workload (3M Gaussians, 1080p) with CUDA events, for one library
build.  Used to compare compile-time variants:

    GS_B200_LIB=path/to/variant.so python tools/stage_bench.py [--n N]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import numpy as np
    import torch

    from paper_2308_04079_b200 import _lib, synthetic
    from paper_2308_04079_b200 import rasterizer as R
    from paper_2308_04079_b200.cloud import GaussianCloud

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--order", action="store_true", help="also time the backward with heavy tiles first")
    args = ap.parse_args()
    lib = _lib.load()
    W, H = args.width, args.height
    cloud_np, cam = synthetic.frustum_scene(args.n, W, H, seed=0)
    cloud = GaussianCloud.from_numpy(**cloud_np)
    bg = (0.0, 0.0, 0.0)
    out, splats, binning = R.render_view(cloud, cam, bg, 3, training=True)
    d = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (H, W, 3)).astype(np.float32) / 6e6).cuda()

    from paper_2308_04079_b200.loss import l1_dssim_loss
    tgt = torch.rand_like(out.image)

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / args.reps

    from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
    adam = DeviceAdam(cloud)
    stats = R.DensifyStats.zeros(len(cloud), "cuda")
    g2 = R.render_backward(d, out, splats, binning, W, H, bg)
    it = [0]

    def bwd_adam():
        it[0] += 1
        adam.backward_step(cloud, cam, splats, g2, 3, it[0], TrainConfig(), stats=stats)

    def bwd_adam_project():
        it[0] += 1
        adam.backward_step(cloud, cam, splats, g2, 3, it[0], TrainConfig(), stats=stats, project_next=(cam, 3))

    def bwd_adam_then_project():
        bwd_adam()
        R._project_tensors(cloud.c_params(), len(cloud), "cuda", cam, 3)

    res = {
        "lib": str(_lib.LIB_PATH), "n": args.n, "width": W, "height": H,
        "instances": binning.num_instances,
        "bwd_adam_ms": timeit(bwd_adam),
        "bwd_adam_project_ms": timeit(bwd_adam_project),
        "bwd_adam_then_project_ms": timeit(bwd_adam_then_project),
        "blend_fwd_ms": timeit(lambda: R.render_forward(splats, binning, W, H, bg, training=True)),
        "blend_bwd_ms": timeit(lambda: R.render_backward(d, out, splats, binning, W, H, bg)),
        "bin_async_ms": timeit(lambda: R.bin_and_sort_async(splats, W, H)),
        "preprocess_fwd_ms": timeit(lambda: R._project_tensors(cloud.c_params(), len(cloud), "cuda", cam, 3)),
        "loss_ms": timeit(lambda: l1_dssim_loss(out.image, tgt, 0.2)),
    }
    if "--order" in sys.argv:
        import ctypes
        lib, cs, bgc = _lib.load(), splats.c_struct(), R._bg(bg)
        rg = binning.ranges.view(-1, 2)
        lens = (rg[:, 1] - rg[:, 0]).to(torch.int64)
        tx, ty = (1920 + 15) // 16, (1080 + 15) // 16
        last = out.last_contributor.view(1080, 1920)
        pad = torch.full((ty * 16, tx * 16), -1, dtype=last.dtype, device=last.device)
        pad[:1080, :1920] = last
        tl = pad.view(ty, 16, tx, 16).amax(dim=(1, 3)).reshape(-1).to(torch.int64)
        need = torch.where(tl >= rg[:, 0].to(torch.int64), tl - rg[:, 0].to(torch.int64) + 1, torch.zeros_like(tl))
        g2o = torch.zeros((len(splats), 12), device="cuda")
        # super-tile variants: groups of g x g tiles ordered by their summed need,
        # the group's tiles launched consecutively (L2 reuse of shared splats)
        def grouped(g):
            tyy, txx = -(-ty // g), -(-tx // g)
            nd = torch.zeros(tyy * g, txx * g, dtype=torch.int64, device="cuda")
            nd[:ty, :tx] = need.view(ty, tx)
            gs_ = nd.view(tyy, g, txx, g).sum(dim=(1, 3)).reshape(-1)
            gorder = torch.argsort(gs_, descending=True, stable=True)
            gy, gx = gorder // txx, gorder % txx
            oy = torch.arange(g, device="cuda").view(1, g, 1)
            ox = torch.arange(g, device="cuda").view(1, 1, g)
            yy = (gy.view(-1, 1, 1) * g + oy).expand(-1, g, g).reshape(-1)
            xx = (gx.view(-1, 1, 1) * g + ox).expand(-1, g, g).reshape(-1)
            ok = (yy < ty) & (xx < tx)
            return (yy[ok] * tx + xx[ok]).to(torch.int32)
        variants = [("len", lens), ("need", need)]
        for name, key in variants + [("need2x2", None), ("need4x4", None)]:
            if key is None:
                order = grouped(2 if name == "need2x2" else 4)
            else:
                order = torch.argsort(key, descending=True, stable=True).to(torch.int32)
            def run():
                lib.gs_blend_backward_ordered(d.data_ptr(), ctypes.byref(cs), binning.splat_ids.data_ptr(),
                                              binning.ranges.data_ptr(), out.final_transmittance.data_ptr(),
                                              out.last_contributor.data_ptr(), W, H, bgc, order.data_ptr(),
                                              g2o.data_ptr(), torch.cuda.current_stream().cuda_stream)
            res[f"blend_bwd_order_{name}_ms"] = timeit(run)
            res[f"order_{name}_checksum"] = float(g2o.abs().sum().item())
            img = torch.empty_like(out.image)
            tf = torch.empty_like(out.final_transmittance)
            ls = torch.empty_like(out.last_contributor)
            fx = torch.empty(2 + 1920 * 1080, dtype=torch.int32, device="cuda")
            def runf():
                lib.gs_blend_forward_ordered(ctypes.byref(cs), binning.splat_ids.data_ptr(), binning.ranges.data_ptr(),
                                             W, H, bgc, 1, order.data_ptr(), None, img.data_ptr(),
                                             tf.data_ptr(), ls.data_ptr(), fx.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream)
            res[f"blend_fwd_order_{name}_ms"] = timeit(runf)
            res[f"fwd_order_{name}_same"] = bool(torch.equal(img, out.image) and torch.equal(ls, out.last_contributor))
    # the fused projection is bit-identical to projecting after the update
    nxt = adam.backward_step(cloud, cam, splats, g2, 3, it[0] + 1, TrainConfig(), project_next=(cam, 3))
    ref = R._project_tensors(cloud.c_params(), len(cloud), "cuda", cam, 3)
    vis = ref.radii > 0
    res["project_fused_identical"] = (all(torch.equal(getattr(nxt, f), getattr(ref, f))
                                          for f in ("radii", "tiles_touched", "status"))
                                      and all(torch.equal(getattr(nxt, f)[vis], getattr(ref, f)[vis])
                                              for f in ("rec", "depth", "rect")))
    g_ref = R.render_backward(d, out, splats, binning, W, H, bg).packed
    res["bwd_checksum"] = float(g_ref.double().abs().sum())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
