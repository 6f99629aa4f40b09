"""Key metrics + top stall reasons from an ncu raw-page CSV (tools/profile_all.sh)."""
import csv
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"== {path}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w} = {vals[i]} {units[i]}")
        st = [(h, vals[i]) for i, h in enumerate(hdr)
              if "issue_stalled" in h and h.endswith("per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:8]
        print("  stalls/issue: " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
            f"={float(v):.2f}" for h, v in st))
