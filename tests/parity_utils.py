"""Shared parity assertions for the GPU tests.

A float32 blend cannot reproduce every float64 stop decision: the running
transmittance carries ~1e-5 relative error, so a pixel whose transmittance
crosses the saturation stop (1 - T > 0.9999, rasterizer.py:179-180) within
that margin may stop one splat earlier or later.  Such pixels are allowed
only when attributed: both transmittances are at the stop (T < 2e-4), their
count is tiny, and the image there differs by at most T * a * c.  Alpha-skip
and clamp decisions (1/255, 0.99) are made in float64 by the kernels'
threshold guard and must match exactly.
"""
import numpy as np

IMG_TOL = 1e-4


def forward_parity(img, tf, last, ref_img, ref_tf, ref_last, color_max=1.0):
    img, tf, last = np.asarray(img), np.asarray(tf), np.asarray(last)
    mism = last != ref_last
    n_mism = int(mism.sum())
    report = {"pixels": int(last.size), "last_mismatch": n_mism}
    if n_mism:
        sat = (tf[mism] < 2e-4) & (ref_tf[mism] < 2e-4)
        assert np.all(sat), f"unattributed last-contributor mismatches: {int((~sat).sum())} of {n_mism}"
        assert n_mism <= 2 + 1e-4 * last.size, f"too many saturation flips: {n_mism}"
    diff = np.abs(img - ref_img).max(axis=-1)
    ok = ~mism
    report["max_abs"] = float(diff.max()) if diff.size else 0.0
    report["max_abs_unflipped"] = float(diff[ok].max()) if ok.any() else 0.0
    assert report["max_abs_unflipped"] <= IMG_TOL, report
    if n_mism:
        assert diff[mism].max() <= 2e-4 * max(1.0, color_max), report
    tdiff = np.abs(tf - ref_tf)
    assert tdiff[ok].max(initial=0.0) <= IMG_TOL, "final transmittance"
    return report
