"""Print an ncu --metrics gpu__time_duration.sum CSV launch list: per launch (id, kernel, µs) for
the last `--last N` launches, plus per-kernel totals.  usage: launch_list.py file.csv [--last N]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
out = [(int(r[ii]), r[ki], float(r[vi].replace(",", "")) / 1e3) for r in rows[1:]]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else len(out)
sel = out[-last:]
for i, k, us in sel:
    print(f"{i:5d} {us:10.2f} us  {k[:100]}")
print(f"total {sum(x[2] for x in sel):.2f} us over {len(sel)} launches")
