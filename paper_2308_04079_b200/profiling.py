"""Per-stage CUDA-event timing and roofline arithmetic for bench.py.

Algorithmic bytes / flops per stage follow SURVEY.md §8(d), except for the
binning, which is charged the bytes the implemented algorithm must move
(binning.cu; SURVEY's formula assumes the reference's 64-bit sort over K):
  K1 preprocess_fwd  44 N + 192 V read + 48 V write
  K2-K5 bin_and_sort 140 N + 24 E + 4 K + 12 T: depth histogram 8 N, four onesweep passes over the
                     depth keys 16 + 16 + 16 + 12 N (the last writes only the order), bucket count
                     36 N (order, rectangle gather, depth-ordered rectangles), bucket scatter 36 N + 8 E,
                     window count 8 E, instance write 8 E + 4 K, tile ranges 12 T;
                     E = (Gaussian, super-tile) bucket entries
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

# our own __global__ kernels launched per training step (every one hand-written;
# the buffers a stage must clear first are zeroed by a programmatically
# launched kernel, counted with the stage;
# blend_fwd: the blend + the exact re-blend of undecidable stops; blend_bwd:
# the blend (its three tile-schedule kernels: blend_bwd_setup); bin_and_sort: depth histogram,
# sort setup, 4 onesweep passes, bucket count, scan, window setup, bucket
# scatter, window count, window prefix, tile ranges, instance write)
KERNELS_PER_STEP = {"preprocess_fwd": 2, "bin_and_sort": 15, "blend_fwd": 3, "loss": 3, "blend_bwd": 1,
                    "blend_bwd_setup": 3,
                    "preprocess_bwd": 1, "adam": 1, "preprocess_bwd_adam": 1, "preprocess_bwd_adam_project": 2,
                    "sharded_adam": 1}


class StageTimer:
    def __init__(self, enabled: bool = True):
        self.enabled = enabled
        self.events = defaultdict(list)
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

    def note_instances(self, k, out) -> None:
        """k: an instance count, or a TileBinning whose (device-resident) K is
        read only when the roofline is computed, after the timed region."""
        self._k_src = k
        self._pending_out = out

    @property
    def last_k(self):
        src = getattr(self, "_k_src", None)
        if src is None:
            return None
        return int(src) if isinstance(src, int) else int(src.num_instances)

    def evaluated_pairs(self, out, ranges_start_of_pixel) -> int:
        last = out.last_contributor
        e = torch.where(last >= 0, last - ranges_start_of_pixel + 1, torch.zeros_like(last))
        return int(e.sum().item())

    def mean_ms(self) -> dict:
        torch.cuda.synchronize()
        return {k: sum(s.elapsed_time(e) for s, e in v) / len(v) for k, v in self.events.items() if v}

    def spread_ms(self) -> dict:
        """Per stage (min, median, max) over the timed steps."""
        torch.cuda.synchronize()
        out = {}
        for k, v in self.events.items():
            if v:
                t = sorted(s.elapsed_time(e) for s, e in v)
                out[k] = [round(t[0], 4), round(t[len(t) // 2], 4), round(t[-1], 4)]
        return out

    def launches_per_step(self) -> int:
        return sum(KERNELS_PER_STEP.get(k, 0) for k in self.events)

    def roofline(self, n: int, width: int, height: int, peaks: dict, visible: int | None = None,
                 e_pairs: int | None = None, bucket_entries: int | None = None) -> dict:
        ms = self.mean_ms()
        V = n if visible is None else visible
        K = self.last_k or 0
        P = width * height
        T = ((width + 15) // 16) * ((height + 15) // 16)
        E = bucket_entries or 0
        bytes_ = {
            "preprocess_fwd": 44 * n + 192 * V + 48 * V,
            "bin_and_sort": 140 * n + 24 * E + 4 * K + 12 * T,
            "blend_fwd": 40 * K + 20 * P,
            "blend_bwd": 40 * K + 20 * P + 36 * V,
            "preprocess_bwd": 276 * V + 240 * n + 20 * n,
            "adam": 1652 * n,
            # fused K8+K9: the 236 B/Gaussian gradient write and re-read are gone
            "preprocess_bwd_adam": 276 * V + 260 * n + 1652 * n - 472 * n,
            # ... plus K1 for the next view on the updated parameters: only its record write is new
            "preprocess_bwd_adam_project": 276 * V + 260 * n + 1652 * n - 472 * n + 48 * V,
            "loss": 132 * P,
        }
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        # the FP32 roofline's denominator: the larger of the in-run FMA probe
        # and the nominal SMs x 128 x 2 x max clock (a probe run at a dipped
        # clock must not inflate the fraction)
        fp32 = max(peaks.get("fp32_tflops") or 0.0, peaks.get("fp32_nominal_tflops") or 0.0) or None
        flops = {}
        if e_pairs:
            flops = {"blend_fwd": 25.0 * e_pairs, "blend_bwd": 60.0 * e_pairs}
        traffic = peaks.get("traffic_bytes", {})
        stages = {}
        for k, t in ms.items():
            if k in bytes_ and t > 0:
                gbs = bytes_[k] / (t * 1e-3) / 1e9
                st = {"ms": round(t, 4), "algorithmic_bytes": bytes_[k], "achieved_gbs": round(gbs, 1),
                      "frac_hbm": round(gbs / hbm, 4)}
                if k in flops and fp32:
                    tf = flops[k] / (t * 1e-3) / 1e12
                    st.update({"algorithmic_flops": flops[k], "achieved_tflops": round(tf, 2),
                               "frac_fp32": round(tf / fp32, 4)})
                stages[k] = st
        def fp32_entry(k):
            st = stages[k]
            return {"kernel": k, "bound": "fp32", "achieved": st["achieved_tflops"], "peak": round(fp32, 2),
                    "unit": "TFLOP/s", "frac": st["frac_fp32"], "traffic": traffic.get(k),
                    "peak_source": "max(in-run FP32 FMA probe gs_fp32_fma_probe, nominal SMs x 128 x 2 x "
                                   "sm_max_mhz); MEASURED_PEAKS.json has no FP32 figure and this kernel is "
                                   "FP32-issue-bound, not HBM/tensor",
                    "algorithmic": f"{st['algorithmic_flops']:.4g} FLOP per launch "
                                   f"(25|60 FP32 ops x E={e_pairs} evaluated pairs)"}

        def hbm_entry(k):
            st = stages[k]
            return {"kernel": k, "bound": "hbm", "achieved": st["achieved_gbs"], "peak": hbm,
                    "unit": "GB/s", "frac": st["frac_hbm"], "traffic": traffic.get(k),
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650"}

        timed = [k for k in ms if k in stages]
        dom = max(timed, key=lambda k: ms[k]) if timed else None
        primary = None
        if dom is not None:
            primary = fp32_entry(dom) if "frac_fp32" in stages[dom] else hbm_entry(dom)
        hbm_stages = [k for k in timed if k not in flops]
        fp32_stages = [k for k in timed if "frac_fp32" in stages[k]]
        secondary = hbm_entry(max(hbm_stages, key=lambda k: ms[k])) if hbm_stages else None
        top_fp32 = fp32_entry(max(fp32_stages, key=lambda k: ms[k])) if fp32_stages else None
        return {"primary": primary, "hbm": secondary, "fp32": top_fp32, "stages": stages}


def measure_fp32_peak(device=None, iters: int = 4096, trials: int = 7) -> float:
    """FP32 FMA throughput (FLOP/s, FMA = 2) of this GPU, from gs_fp32_fma_probe:
    ~50 ms of untimed launches to bring the clocks up, then the best of
    `trials` timed groups of 5 launches (CUDA events)."""
    from . import _lib
    lib = _lib.load()
    props = torch.cuda.get_device_properties(device)
    blocks = props.multi_processor_count * 8
    scratch = torch.empty(blocks, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream(device).cuda_stream
    for _ in range(200):
        _lib.check(lib.gs_fp32_fma_probe(scratch.data_ptr(), blocks, iters, stream), "fma_probe")
    reps, best = 5, float("inf")
    for _ in range(trials):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            _lib.check(lib.gs_fp32_fma_probe(scratch.data_ptr(), blocks, iters, stream), "fma_probe")
        e.record()
        torch.cuda.synchronize(device)
        best = min(best, s.elapsed_time(e) / 1e3 / reps)
    return blocks * 256 * iters * 8 * 2 / best


def fp32_nominal_tflops(device=None, sm_max_mhz: float | None = None) -> float:
    """Nominal FP32 FMA peak: SMs x 128 FP32 lanes x 2 FLOP x the maximum SM
    clock (MEASURED_PEAKS.json sm_max_mhz, else the device's)."""
    props = torch.cuda.get_device_properties(device)
    mhz = sm_max_mhz or getattr(props, "clock_rate", 0) / 1e3 or 1965.0
    return props.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12


def bucket_entries(splats, width: int, height: int) -> int:
    """(Gaussian, super-tile) pairs of the binning's bucket stage (binning.cu:
    super-tiles of 8 x 4 tiles, 2 x / 4 x larger for frames past 4096 of them)."""
    tx, ty = (width + 15) // 16, (height + 15) // 16
    lq = 0
    while lq < 2 and -(-tx // (8 << lq)) * -(-ty // (4 << lq)) > 4096:
        lq += 1
    rc = splats.rect.long()
    ok = splats.tiles_touched > 0
    nx = (rc[:, 2] >> (3 + lq)) - (rc[:, 0] >> (3 + lq)) + 1
    ny = (rc[:, 3] >> (2 + lq)) - (rc[:, 1] >> (2 + lq)) + 1
    return int(torch.where(ok, nx * ny, torch.zeros_like(nx)).sum().item())


def evaluated_pairs(out, binning, width: int) -> int:
    """E = sum over pixels of (last_contributor - tile_start + 1)."""
    last = out.last_contributor.long()
    h, w = last.shape
    ty = torch.arange(h, device=last.device) // 16
    tx = torch.arange(w, device=last.device) // 16
    tiles = ty[:, None] * binning.tiles_x + tx[None, :]
    start = binning.ranges[:, 0].long()[tiles]
    return int(torch.where(last >= 0, last - start + 1, torch.zeros_like(last)).sum().item())
