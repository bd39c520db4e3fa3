"""Programmatic dependent launch changes scheduling, not results: one small
training step (projection, binning, forward + exact re-blend, loss, backward,
fused backward + Adam, next-view projection) run in two processes, with the
launch attribute on (default) and off (GS_PDL_LAUNCH=0), gives bit-identical
binning, images and records, and gradients equal up to the float-RED
ordering of the backward blend."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[2])
from paper_2308_04079_b200 import rasterizer as R, synthetic
from paper_2308_04079_b200.cloud import GaussianCloud
from paper_2308_04079_b200.loss import l1_dssim_loss
from paper_2308_04079_b200.optimizer import DeviceAdam, TrainConfig
cloud_np, cam = synthetic.frustum_scene(30000, 320, 200, seed=5)
cloud = GaussianCloud.from_numpy(**cloud_np)
target = torch.from_numpy(np.random.default_rng(6).uniform(0, 1, (200, 320, 3)).astype(np.float32)).cuda()
R.render_view(cloud, cam, (0, 0, 0), 3)
out, splats, binning = R.render_view_async(cloud, cam, (0, 0, 0), 3, training=True)
prep = R.prepare_backward(out, splats, binning, 320, 200)
loss, d_image = l1_dssim_loss(out.image, target, 0.2)
g2 = R.render_backward(d_image, out, splats, binning, 320, 200, (0, 0, 0), prep=prep)
adam = DeviceAdam(cloud)
grads = R.GaussianGrads.zeros(len(cloud), "cuda")
nxt = adam.backward_step(cloud, cam, splats, g2, 3, 1, TrainConfig(), grads_out=grads, project_next=(cam, 3))
torch.cuda.synchronize()
binning.check()
k = binning.num_instances
np.savez(sys.argv[1], ids=binning.splat_ids[:k].cpu().numpy(), ranges=binning.ranges.cpu().numpy(),
         image=out.image.cpu().numpy(), t_final=out.final_transmittance.cpu().numpy(),
         last=out.last_contributor.cpu().numpy(), loss=loss.cpu().numpy(), d_image=d_image.cpu().numpy(),
         d_means=grads.d_means.cpu().numpy(), d_sh=grads.d_sh.cpu().numpy(), means=cloud.means.cpu().numpy(),
         radii=nxt.radii.cpu().numpy())
"""


def run(tmp_path, pdl: str):
    out = tmp_path / f"pdl{pdl}.npz"
    env = dict(os.environ, GS_PDL_LAUNCH=pdl)
    res = subprocess.run([sys.executable, "-c", SCRIPT, str(out), str(ROOT)], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return np.load(out)


def test_programmatic_launch_does_not_change_results(cuda_device, tmp_path):
    on, off = run(tmp_path, "1"), run(tmp_path, "0")
    for key in ("ids", "ranges", "image", "t_final", "last", "loss", "d_image", "radii"):
        np.testing.assert_array_equal(on[key], off[key], err_msg=key)
    for key in ("d_means", "d_sh", "means"):
        a, b = on[key].astype(np.float64), off[key].astype(np.float64)
        assert np.linalg.norm(a - b) <= 1e-5 * max(np.linalg.norm(b), 1e-30), key
