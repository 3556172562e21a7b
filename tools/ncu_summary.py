"""Summarise an ncu report: key throughput/occupancy metrics + top stall reasons per kernel."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:70]
    print("==", r[h.index("ID")], name)
    for w in want:
        if w in h:
            print(f"   {w:60s} {r[h.index(w)]}")
    idx = [i for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled")
           and not n.endswith("not_issued")]
    vals = sorted([(float(r[i].replace(",", "") or 0), h[i]) for i in idx], reverse=True)[:6]
    tot = sum(float(r[i].replace(",", "") or 0) for i in idx) or 1
    print("   stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')}="
                                 f"{v / tot:.2f}" for v, n in vals))
