"""Per-stage CUDA-event timing and roofline arithmetic for bench.py.

Algorithmic bytes / flops per stage follow SURVEY.md §8(d):
  K1 preprocess_fwd  44 N + 192 V read + 48 V write
  K2-K5 bin_and_sort 8 V + (20 V + 12 K) + (8 K + 24 D K) + (8 K + 8 T), D = radix passes of the
                     reference's 64-bit key sort (the algorithmic formula, not this implementation's)
  K6 blend_fwd       40 K + 20 P bytes (training); 25 FP32 ops + 1 ex2 per evaluated (pixel, splat) pair
  K7 blend_bwd       40 K + 20 P + 36 V bytes; 60 FP32 ops + 1 ex2 + 1 rcp per evaluated pair
  K8 preprocess_bwd  276 V + 240 N + 20 N bytes
  K9 adam            1652 N bytes (59 floats x 28 B)
E (evaluated pairs) = sum over pixels of (last_contributor - tile_start + 1), from the forward's
own training record.
"""
from __future__ import annotations

import contextlib
from collections import defaultdict

import torch

# our own __global__ kernels launched per training step (CUB's radix-sort and scan
# kernels, compiled into the same library, are counted separately in DESIGN.md)
KERNELS_PER_STEP = {"preprocess_fwd": 1, "bin_and_sort": 5, "blend_fwd": 1, "loss": 3, "blend_bwd": 1,
                    "preprocess_bwd": 1, "adam": 1}


class StageTimer:
    def __init__(self, enabled: bool = True):
        self.enabled = enabled
        self.events = defaultdict(list)
        self.last_k = None
        self.last_e = None
        self.samples = []

    @staticmethod
    @contextlib.contextmanager
    def stage(timer, name: str):
        if timer is None or not timer.enabled:
            yield
            return
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            timer.events[name].append((s, e))

    def note_instances(self, k: int, out) -> None:
        self.last_k = int(k)
        self._pending_out = out

    def evaluated_pairs(self, out, ranges_start_of_pixel) -> int:
        last = out.last_contributor
        e = torch.where(last >= 0, last - ranges_start_of_pixel + 1, torch.zeros_like(last))
        return int(e.sum().item())

    def mean_ms(self) -> dict:
        torch.cuda.synchronize()
        return {k: sum(s.elapsed_time(e) for s, e in v) / len(v) for k, v in self.events.items() if v}

    def launches_per_step(self) -> int:
        return sum(KERNELS_PER_STEP.get(k, 0) for k in self.events)

    def roofline(self, n: int, width: int, height: int, peaks: dict, visible: int | None = None,
                 e_pairs: int | None = None) -> dict:
        ms = self.mean_ms()
        V = n if visible is None else visible
        K = self.last_k or 0
        P = width * height
        T = ((width + 15) // 16) * ((height + 15) // 16)
        b = max(1, (T - 1).bit_length())
        D = -(-(32 + b) // 8)
        bytes_ = {
            "preprocess_fwd": 44 * n + 192 * V + 48 * V,
            "bin_and_sort": 8 * V + 20 * V + 12 * K + 8 * K + 24 * D * K + 8 * K + 8 * T,
            "blend_fwd": 40 * K + 20 * P,
            "blend_bwd": 40 * K + 20 * P + 36 * V,
            "preprocess_bwd": 276 * V + 240 * n + 20 * n,
            "adam": 1652 * n,
            "loss": 132 * P,
        }
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        stages = {}
        for k, t in ms.items():
            if k in bytes_ and t > 0:
                gbs = bytes_[k] / (t * 1e-3) / 1e9
                stages[k] = {"ms": round(t, 4), "algorithmic_bytes": bytes_[k], "achieved_gbs": round(gbs, 1),
                             "frac_hbm": round(gbs / hbm, 4)}
        dom = max(ms, key=lambda k: ms[k]) if ms else None
        primary = None
        if dom in stages:
            st = stages[dom]
            primary = {"kernel": dom, "bound": "hbm", "achieved": st["achieved_gbs"], "peak": hbm, "unit": "GB/s",
                       "frac": st["frac_hbm"], "traffic": None,
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650"}
        return {"primary": primary, "stages": stages}
