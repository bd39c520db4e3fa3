"""Device densify/prune against the reference's own
densify_and_prune outputs (tests/golden/densify_*.npz, make_golden.py)."""
from pathlib import Path

import numpy as np
import pytest
import torch

import golden_scenes

GOLDEN = Path(__file__).resolve().parent / "golden"
GROUPS = ("means", "log_scales", "rotations", "opacity_logits", "sh")


def test_densify_goldens_consistent():
    for name in ("densify_a", "densify_b"):
        g = dict(np.load(GOLDEN / f"{name}.npz"))
        n_out = g["out_means"].shape[0]
        assert n_out == 1500 - int(g["split"]) + int(g["cloned"]) + 2 * int(g["split"]) - int(g["pruned"])
        for grp in GROUPS:
            assert g[f"out_m_{grp}"].shape == g[f"out_{grp}"].shape


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["densify_a", "densify_b"])
def test_device_densify_matches_reference(cuda_device, name):
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.densify import TrainState, densify_and_prune
    from paper_2308_04079_b200.optimizer import TrainConfig

    g = dict(np.load(GOLDEN / f"{name}.npz"))
    _, cloud_np, _ = golden_scenes.load("scene_c")
    cloud = GaussianCloud.from_numpy(**cloud_np)
    state = TrainState(cloud, float(g["extent"]), seed=int(g["seed"]))
    state.iteration = int(g["iteration"])
    for grp in GROUPS:
        state.adam.exp_avg[grp].copy_(torch.from_numpy(g[f"in_m_{grp}"].astype(np.float32)))
        state.adam.exp_avg_sq[grp].copy_(torch.from_numpy(g[f"in_v_{grp}"].astype(np.float32)))
    state.stats.accum_pos_grad.copy_(torch.from_numpy(g["in_accum"].astype(np.float32)))
    state.stats.accum_count.copy_(torch.from_numpy(g["in_count"].astype(np.int32)))
    state.stats.max_radius_frac.copy_(torch.from_numpy(g["in_maxr"].astype(np.float32)))

    rep = densify_and_prune(state, TrainConfig(total_iters=30000))
    torch.cuda.synchronize()
    assert (rep.cloned, rep.split, rep.pruned, rep.opacity_reset) == (
        int(g["cloned"]), int(g["split"]), int(g["pruned"]), bool(g["opacity_reset"]))
    for grp in GROUPS:
        got = getattr(state.cloud, grp).cpu().numpy().astype(np.float64)
        ref = g[f"out_{grp}"]
        assert got.shape == ref.shape, grp
        # float32 parameters vs the reference's float64 (split children: f32 z, f64 transform)
        np.testing.assert_allclose(got, ref, rtol=2e-6, atol=2e-6, err_msg=grp)
        np.testing.assert_array_equal(state.adam.exp_avg[grp].cpu().numpy().astype(np.float64),
                                      g[f"out_m_{grp}"])
        np.testing.assert_array_equal(state.adam.exp_avg_sq[grp].cpu().numpy().astype(np.float64),
                                      g[f"out_v_{grp}"])
    assert int(state.stats.accum_count.sum()) == 0
    state.check_alignment()
