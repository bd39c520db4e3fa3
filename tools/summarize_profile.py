"""Summarise an ncu launch list and an `ncu --set full` report into profiles/.

    python tools/summarize_profile.py TAG LAUNCHES.csv FULL.ncu-rep "description"

Writes profiles/TAG_launches.md (+ the raw CSV), profiles/TAG_ncu_full.md and
updates profiles/traffic_bytes.json (dram read+write bytes per launch, by
bench stage) which bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROFILES = ROOT / "profiles"

STAGE_OF = {"blend_bwd_kernel": "blend_bwd", "blend_fwd_kernel": "blend_fwd",
            "preprocess_bwd_adam_kernel": "preprocess_bwd_adam", "preprocess_bwd_kernel": "preprocess_bwd",
            "preprocess_fwd_kernel": "preprocess_fwd", "adam_kernel": "adam"}
# the binning is several kernels per frame: its traffic is summed per frame
# (frames = launches of the last binning kernel, tile_ranges_kernel)
BIN_KERNELS = ("depth_hist_kernel", "onesweep_kernel", "sort_setup_kernel", "bucket_count_kernel", "scan_kernel",
               "bucket_scatter_kernel", "window_setup_kernel", "window_count_kernel", "window_prefix_kernel",
               "instance_write", "tile_ranges_kernel")
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").strip()
    if "cub::" in base:
        return "cub::" + base.split("cub::")[1].split("<")[0]
    return base.split("::")[-1]


def launches(csv_path: Path, tag: str, desc: str) -> None:
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        k = short(r[ki])
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    total = sum(tot.values())
    out = [f"# {tag} — ncu launch list\n", f"{desc}\n",
           "Per-launch device time (ncu `gpu__time_duration.sum`, `--clock-control none`, cold-cache, "
           f"serialised: compare shares, not absolutes).  Raw CSV: `profiles/{tag}_launches.csv`.\n",
           "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / total:.1f}% |")
    (PROFILES / f"{tag}_launches.md").write_text("\n".join(out) + "\n")
    shutil.copy(csv_path, PROFILES / f"{tag}_launches.csv")


def full(rep: Path, tag: str, desc: str) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    ki = h.index("Kernel Name")
    stall = [w for w in h if w.startswith("smsp__average_warps_issue_stalled") and w.endswith("per_issue_active.ratio")]
    out = [f"# {tag} — `ncu --set full` per-launch summary\n", f"{desc}\n",
           f"| kernel | time {u[h.index('gpu__time_duration.sum')]} | DRAM rd+wr MB | DRAM % | issue % | warps % | regs | FMA % | warp instr | top stalls |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = defaultdict(list)
    bin_bytes, bin_frames = 0.0, 0
    for r in rows[2:]:
        name = short(r[ki])
        val = {m: r[h.index(m)] for m in METRICS if m in h}
        rd = float(val["dram__bytes_read.sum"]) * SCALE[u[h.index("dram__bytes_read.sum")]]
        wr = float(val["dram__bytes_write.sum"]) * SCALE[u[h.index("dram__bytes_write.sum")]]
        top = sorted(((float(r[h.index(w)]), w) for w in stall), reverse=True)[:3]
        tops = ", ".join(f"{w.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                         f" {v:.1f}" for v, w in top)
        out.append(f"| `{name}` | {float(val['gpu__time_duration.sum']):.3f} | {(rd + wr) / 1e6:.1f} | "
                   f"{float(val['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                   f"{float(val['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                   f"{float(val['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                   f"{val['launch__registers_per_thread']} | "
                   f"{float(val['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active']):.1f} | "
                   f"{float(val['smsp__inst_executed.sum']) / 1e6:.1f} M | {tops} |")
        stage = next((s for k, s in STAGE_OF.items() if name.startswith(k)), None)
        if stage:
            traffic[stage].append(rd + wr)
        if name.startswith(BIN_KERNELS):
            bin_bytes += rd + wr
            bin_frames += name.startswith("tile_ranges_kernel")
    (PROFILES / f"{tag}_ncu_full.md").write_text("\n".join(out) + "\n")
    res = {k: sum(v) / len(v) for k, v in traffic.items()}
    if bin_frames:
        res["bin_and_sort"] = bin_bytes / bin_frames
    return res


def main() -> None:
    tag, csv_path, rep, desc = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3]), sys.argv[4]
    PROFILES.mkdir(exist_ok=True)
    launches(csv_path, tag, desc)
    traffic = full(rep, tag, desc)
    tj = PROFILES / "traffic_bytes.json"
    data = json.loads(tj.read_text()) if tj.exists() else {}
    data.setdefault("per_launch", {}).update({k: round(v) for k, v in traffic.items()})
    data["source"] = f"profiles/{tag}_ncu_full.md (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    tj.write_text(json.dumps(data, indent=1) + "\n")
    print(f"wrote profiles/{tag}_*.md, traffic {data['per_launch']}")


if __name__ == "__main__":
    main()
