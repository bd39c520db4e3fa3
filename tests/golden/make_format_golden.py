"""Golden model / PLY / checkpoint files written by the REFERENCE itself
(splatlab scene_io.save_model / export_ply / save_checkpoint,
scene_io.py:394-457), for the format parity tests.

Run in the build container, where /root/reference exists:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_format_golden.py
Writes tests/golden/formats/*; nothing at test time reads /root/reference.
The parameters are float32 values (drawn like test_scene_io.py:226-236) and
the Adam moments float32-representable float64, so a float32 device round
trip is bit-exact.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "formats"
sys.path.insert(0, "/root/reference/pkg/src")

from splatlab.core import GaussianCloud  # noqa: E402
from splatlab.optimizer import PARAM_GROUPS, TrainState  # noqa: E402
from splatlab.scene_io import export_ply, save_checkpoint, save_model  # noqa: E402

N = 23


def cloud(seed: int = 11) -> GaussianCloud:
    rng = np.random.default_rng(seed)
    f = lambda *shape: rng.normal(size=shape).astype(np.float32)  # noqa: E731
    return GaussianCloud(f(N, 3), f(N, 4), f(N, 3), f(N), f(N, 16, 3))


def main() -> None:
    OUT.mkdir(exist_ok=True)
    c = cloud()
    save_model(OUT / "model.splat", c, sh_degree=2)
    save_model(OUT / "empty.splat", GaussianCloud.empty())
    export_ply(OUT / "model.ply", c)
    state = TrainState(c, scene_extent=2.5, seed=1)
    state.iteration = 123
    state.active_sh_degree = 2
    rng = np.random.default_rng(5)
    for g in PARAM_GROUPS:
        state.exp_avg[g][...] = rng.normal(size=state.exp_avg[g].shape).astype(np.float32)
        state.exp_avg_sq[g][...] = rng.uniform(size=state.exp_avg_sq[g].shape).astype(np.float32)
    save_checkpoint(OUT / "state.ckpt", state)
    np.savez(OUT / "params.npz", means=c.means, rotations=c.rotations, log_scales=c.log_scales,
             opacity_logits=c.opacity_logits, sh=c.sh,
             **{f"m_{g}": state.exp_avg[g] for g in PARAM_GROUPS},
             **{f"v_{g}": state.exp_avg_sq[g] for g in PARAM_GROUPS})
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
