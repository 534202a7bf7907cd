"""Summarise an ncu report: per-kernel time, DRAM bytes, throughputs, occupancy, stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active"]
stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled") or
         h.startswith("smsp__pcsamp_warps_issue_stalled")]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:90])
    for w in want[1:]:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:60s} {r[i]:>14s} {units[i]}")
    st = []
    for h in stall:
        i = hdr.index(h)
        try:
            v = float(r[i])
        except ValueError:
            continue
        if v > 0:
            st.append((v, h))
    st.sort(reverse=True)
    for v, h in st[:8]:
        print(f"   stall {h:70s} {v:10.2f}")
