"""Host-side checks of the NumPy-signature mirror (paper_2308_04079_b200.compat):
make_keys semantics (rasterizer.py:55-62, test_rasterizer.py:39-56) and the
conversion of reference-semantics screen gradients into the device's moment
rows (the inverse of rasterizer.SplatGrads2D's properties)."""
import numpy as np
import torch

from paper_2308_04079_b200 import compat as C
from paper_2308_04079_b200 import rasterizer as R


def test_make_keys_orders_by_tile_then_depth():
    keys = C.make_keys(np.array([0, 0, 1, 1]), np.array([2.0, 1.0, 0.5, 3.0]))
    np.testing.assert_array_equal(np.argsort(keys, kind="stable"), [1, 0, 2, 3])


def test_make_keys_depth_bits_include_denormals():
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.uniform(0, 1e3, 2000).astype(np.float32),
                           (rng.uniform(1, 10, 100) * np.finfo(np.float32).smallest_subnormal).astype(np.float32),
                           np.float32([0.0, np.finfo(np.float32).tiny, 1e-30, 3.4e38])]).astype(np.float64)
    order = np.argsort(C.make_keys(np.zeros(len(vals), np.int64), vals), kind="stable")
    assert np.all(np.diff(vals[order].astype(np.float32)) >= 0)


def test_moment_rows_invert_the_screen_gradient_properties():
    rng = np.random.default_rng(1)
    m = 64
    rec = np.zeros((m, 20), np.float32)
    rec[:, 4:8] = rng.normal(size=(m, 4)).astype(np.float32)      # eigenbasis rows k1, k2
    rec[:, 11] = rng.uniform(0.05, 0.99, m).astype(np.float32)     # alpha
    packed = np.zeros((m, 12), np.float32)
    packed[:, 0:3] = rng.normal(size=(m, 3))
    packed[:, 4:7] = rng.normal(size=(m, 3))
    packed[:, 8:11] = rng.normal(size=(m, 3))
    g = R.SplatGrads2D(torch.from_numpy(packed), None, torch.from_numpy(rec))
    ref = C.SplatGrads2D(d_color=g.d_color.double().numpy(), d_alpha=g.d_alpha.numpy(),
                         d_mean2d=g.d_mean2d.numpy(), d_conic=g.d_conic.numpy())
    back = C._moment_rows(ref, rec)
    np.testing.assert_allclose(back, packed, rtol=1e-4, atol=1e-5)
