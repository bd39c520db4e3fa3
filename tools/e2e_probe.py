"""Where the end-to-end train_step time goes at c3: host-resident vs
device-resident target, lookahead on/off (CUDA events around K steps)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2308_04079_b200 import rasterizer as R, synthetic
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.densify import TrainState
    from paper_2308_04079_b200.optimizer import TrainConfig
    from paper_2308_04079_b200.training import TrainView, train_step
    cloud_np, cam = synthetic.frustum_scene(3_000_000, 1920, 1080, seed=0)
    tgt_np, _ = synthetic.frustum_scene(3_000_000, 1920, 1080, seed=1)
    with torch.no_grad():
        target = R.render_view(GaussianCloud.from_numpy(**tgt_np), cam, (0, 0, 0), 3)[0].image
    del tgt_np
    cfg = TrainConfig(lambda_dssim=0.2, warmup_upsample_iters=(0, 0), sh_band_interval=10**9)
    host = target.cpu().pin_memory()
    res = {}
    for name, img, look in (("host_lookahead", host, True), ("device_lookahead", target, True),
                            ("host_plain", host, False), ("device_plain", target, False)):
        state = TrainState(GaussianCloud.from_numpy(**cloud_np), 10.0, seed=0)
        state.active_sh_degree = 3
        views = [TrainView(cam, img)]
        for i in range(5):
            train_step(state, views, cfg, lookahead=look and i < 4)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 30
        e0.record()
        for i in range(k):
            train_step(state, views, cfg, lookahead=look and i < k - 1)
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(k * 1e3 / e0.elapsed_time(e1), 2)
        del state
        torch.cuda.empty_cache()
    print(res)


if __name__ == "__main__":
    main()
