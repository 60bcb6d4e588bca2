"""Key --set full metrics of one or more ncu reports (first kernel in each)."""
import csv, subprocess, sys
W = [("duration (us)", "gpu__time_duration.sum", 1e-6),
     ("DRAM read (MB)", "dram__bytes_read.sum", 1e6), ("DRAM write (MB)", "dram__bytes_write.sum", 1e6),
     ("DRAM throughput (% peak)", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
     ("tensor (DMMA) pipe (% elapsed)", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
     ("FP64 pipe (% active)", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
     ("issue active (%)", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
     ("achieved occupancy (%)", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
     ("registers / thread", "launch__registers_per_thread", 1),
     ("stall wait / issue", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", 1),
     ("stall short_sb / issue", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1),
     ("stall long_sb / issue", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1),
     ("stall barrier / issue", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", 1)]
cols = []
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, r = rows[0], rows[1], rows[2]
    # to base units (s, byte), then the table's scale: us = s / 1e-6, MB = byte / 1e6
    unit_scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3,
                  "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    vals = []
    for _, m, sc in W:
        try:
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            if units[i] in unit_scale:
                v = v * unit_scale[units[i]] / sc
            else:
                v = v * sc
            vals.append(f"{v:.1f}" if abs(v) < 1e4 else f"{v:.3g}")
        except (ValueError, IndexError):
            vals.append("-")
    cols.append((name, vals))
print("| metric | " + " | ".join(f"`{n}`" for n, _ in cols) + " |")
print("|---|" + "---|" * len(cols))
for i, (label, _, _) in enumerate(W):
    print(f"| {label} | " + " | ".join(v[i] for _, v in cols) + " |")
