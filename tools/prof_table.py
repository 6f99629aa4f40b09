"""Summarise ncu raw-page CSVs (tools/profile_all.sh) into one roofline table.

For every kernel: duration, DRAM bytes, achieved DRAM GB/s against the
measured copy peak (MEASURED_PEAKS.json) and the measured incompressible
store ceiling, FP64 pipe and DMMA (fp64 tensor) sub-pipe utilisation, issue
utilisation, registers and occupancy. Usage:
    python tools/prof_table.py gpurun_out/prof > profiles/r01_kernels.md
"""

from __future__ import annotations

import csv
import glob
import json
import os
import sys

try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as _f:
        HBM_COPY = float(json.load(_f)["hbm_gbs"])
except (OSError, KeyError, ValueError):
    HBM_COPY = 6549.8
HBM_STORE = 6924.9  # best incompressible streaming-store kernel (profiles/r01_hbm_write_probe.txt)

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "s": 1.0}

METRICS = {
    "kernel": "Kernel Name",
    "time": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
}


def read(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for key, name in METRICS.items():
        if name not in hdr:
            out[key] = None
            continue
        i = hdr.index(name)
        v = vals[i]
        if key == "kernel":
            out[key] = v
            continue
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            out[key] = None
            continue
        out[key] = x * UNITS.get(units[i], 1.0) if key in ("time", "rd", "wr") else x
    return out


def main(d):
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..",
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = HBM_COPY
    print("| capture | kernel | time | DRAM read+write | DRAM GB/s | of copy peak | of store ceiling "
          "| FP64 pipe | DMMA pipe | issue | warps active | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for path in sorted(glob.glob(os.path.join(d, "*.raw.csv"))):
        r = read(path)
        if not r or r["time"] is None:
            continue
        name = os.path.basename(path).replace(".raw.csv", "")
        byt = (r["rd"] or 0) + (r["wr"] or 0)
        gbs = byt / r["time"] / 1e9
        kern = (r["kernel"] or "")[:60]
        fmt = lambda x: "-" if x is None else f"{x:.1f} %"
        print(f"| {name} | `{kern}` | {r['time'] * 1e3:.3f} ms | {byt / 1e9:.3f} GB | {gbs:.0f} | "
              f"{gbs / peak:.2f} | {gbs / HBM_STORE:.2f} | {fmt(r['fp64'])} | {fmt(r['dmma'])} | "
              f"{fmt(r['issue'])} | {fmt(r['warps'])} | {r['regs']:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof")
