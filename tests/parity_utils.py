"""Shared parity assertions for the GPU tests.

Every stop decision must be the reference's: alpha skip and clamp
(1/255, 0.99) are decided in float64 by the kernels' threshold guard, and a
pixel whose float32 transmittance is too close to the saturation stop
(1 - T > 0.9999, rasterizer.py:179-180) to decide is re-blended in float64 by
the forward's fix-up kernel.  So the last contributor must match exactly on
every pixel, and image and final transmittance within IMG_TOL everywhere.
"""
import numpy as np

IMG_TOL = 1e-4


def forward_parity(img, tf, last, ref_img, ref_tf, ref_last, color_max=1.0):
    img, tf, last = np.asarray(img), np.asarray(tf), np.asarray(last)
    mism = last != ref_last
    report = {"pixels": int(last.size), "last_mismatch": int(mism.sum())}
    diff = np.abs(img - ref_img).max(axis=-1) if img.size else np.zeros(0)
    report["max_abs"] = float(diff.max()) if diff.size else 0.0
    report["max_abs_t_final"] = float(np.abs(tf - ref_tf).max()) if tf.size else 0.0
    # float32 transmittance error relative to the reference at saturated pixels
    # (the margin the forward's kSatGuard must cover)
    sat = ref_tf < 2e-4
    report["max_rel_t_saturated"] = float(np.abs(tf[sat] / ref_tf[sat] - 1.0).max()) if sat.any() else 0.0
    print("forward_parity", report)
    assert report["last_mismatch"] == 0, f"last-contributor mismatches (stop-decision flips): {report}"
    assert report["max_abs"] <= IMG_TOL, report
    assert report["max_abs_t_final"] <= IMG_TOL, report
    return report
