"""L1 + D-SSIM loss (optimizer.py:141-163, ssim.py:50-84).

CPU: the float64 oracle against the reference's own `loss` golden vectors.
GPU: gs_l1_dssim_loss against the oracle and the golden vectors; loss value
relative 1e-6, image gradient ||d - ref|| / ||ref|| <= 1e-4 (float64 moments,
float32 storage of the source maps and of the output)."""
import numpy as np
import pytest

import golden_scenes
from oracle import oracle as O


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["scene_a", "scene_b"])
def test_oracle_loss_matches_reference(name):
    g, _, _ = golden_scenes.load(name)
    out, d = O.l1_dssim_loss(g["loss_render"], g["loss_target"], 0.2)
    assert abs(out[0] - float(g["loss_value"])) <= 1e-12 * max(1.0, abs(float(g["loss_value"])))
    assert rel(d, g["loss_d_image"]) < 1e-10


def test_oracle_loss_edge_cases():
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 1, (20, 33, 3))
    out, d = O.l1_dssim_loss(x, x, 0.2)      # identical images: loss 0, gradient 0 (ssim.py:67-74)
    assert abs(out[0]) < 1e-12 and np.abs(d).max() < 1e-12
    out, d = O.l1_dssim_loss(x, 1 - x, 0.0)  # lambda 0: pure L1
    assert abs(out[0] - np.abs(2 * x - 1).mean()) < 1e-12
    with pytest.raises(ValueError):
        O.l1_dssim_loss(x, x[:, :-1], 0.2)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,lam", [((64, 64, 3), 0.2), ((67, 131, 3), 0.2), ((1080, 1920, 3), 0.2),
                                       ((31, 17, 3), 0.0), ((40, 40, 3), 1.0)])
def test_device_loss_vs_oracle(cuda_device, shape, lam):
    import torch
    from paper_2308_04079_b200.loss import l1_dssim_loss
    rng = np.random.default_rng(shape[0])
    x = rng.uniform(0, 1, shape).astype(np.float32)
    y = np.clip(x + rng.normal(0, 0.1, shape), 0, 1).astype(np.float32)
    loss, d = l1_dssim_loss(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), lam)
    ref, dref = O.l1_dssim_loss(x, y, lam)
    got = loss.cpu().numpy().astype(np.float64)
    assert abs(got[0] - ref[0]) <= 1e-6 * max(abs(ref[0]), 1e-6)
    assert rel(d.cpu().numpy(), dref) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scene_a", "scene_b"])
def test_device_loss_vs_reference_golden(cuda_device, name):
    import torch
    from paper_2308_04079_b200.loss import l1_dssim_loss
    g, _, _ = golden_scenes.load(name)
    loss, d = l1_dssim_loss(torch.from_numpy(g["loss_render"]).cuda(), torch.from_numpy(g["loss_target"]).cuda(),
                            0.2)
    assert abs(float(loss[0]) - float(g["loss_value"])) <= 1e-6 * abs(float(g["loss_value"]))
    assert rel(d.cpu().numpy(), g["loss_d_image"]) < 1e-4
